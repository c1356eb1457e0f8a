"""Small searches through every kernel path (count variants, modes, ADSampling, traces)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import __graft_entry__ as ge  # noqa: E402
import synth  # noqa: E402

ge.build()
import paper_2603_05180_b200 as crisp  # noqa: E402

for cfg, N, D, M, K, bids in ((1, 20000, 256, 8, 50, None), (2, 18001, 90, 4, 31, 4096), (1, 70001, 64, 4, 16, 32768)):
    w = synth.Workload(cfg, D=D)
    X, Qv = w.base(N).numpy(), w.queries(24).numpy()
    if bids:
        os.environ["CRISP_BLOCK_IDS"] = str(bids)
    ix = crisp.Index.build(X, M, K=K, seed=1, kmeans_iters=4)
    os.environ.pop("CRISP_BLOCK_IDS", None)
    for variant in ({"CRISP_COUNT_KERNEL": "0", "CRISP_ROWS4": "0"}, {"CRISP_COUNT_KERNEL": "1"},
                    {"CRISP_COUNT_KERNEL": "1", "CRISP_HAMMING_FUSED": "1"}):
        os.environ.update(variant)
        for mode, ad in ((0, False), (1, False), (1, True)):
            ix.set_search_params(budget=max(50, N // 40), tau=2, patience_factor=3)
            ix.set_adsampling(ad)
            ids, d = ix.search(Qv, 10, mode)
            ids, d, t = ix.trace(Qv[:4], 10, mode)
        for k_ in variant:
            os.environ.pop(k_)
    ix.free()
print("all paths ok")
