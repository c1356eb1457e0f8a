"""Exact global patience over G point shards (include/crisp.h
crisp_shard_gp_*): the Optimized-Mode patience rule over the global
(h, gid) order of the union of the shards' candidates.  G shard indexes of one
dataset (shared R and codebooks, summed cell sizes) run the protocol on one GPU
(dist.emulate_global_search: the collectives done by concatenation); ids and
distances must equal the single index over all rows and the oracle's search,
for every G, with and without the verification filter, with the exact global
fallback, with many short rounds, and with a0 sharded by query (each
shard transforms its slice of the batch, q' concatenated: N9)."""
import numpy as np
import pytest

import oracle
from test_gpu_parity import build_gpu, make_case

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def crisp():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__ as ge

    ge.build()
    import paper_2603_05180_b200 as c

    return c


@pytest.fixture(scope="module")
def case(crisp):
    X, Qv, ox = make_case(cfg=4, N=24000, D=128, Q=40, M=8, K=16, seed=5, rotation=1)
    single = build_gpu(crisp, X, ox, block_ids=4096)
    return X, Qv, ox, single


def shard_indexes(crisp, X, ox, G):
    from paper_2603_05180_b200 import dist

    N = X.shape[0]
    shards, bases = [], []
    for r in range(G):
        lo, hi = dist.shard_range(N, r, G)
        shards.append(crisp.Index.build(X[lo:hi], ox["M"], R=ox["R"], codebooks=ox["cb"], K=ox["K"], gid_base=lo))
        bases.append(lo)
    sizes = sum(s.local_cell_sizes() for s in shards)
    for s in shards:
        s.set_global_cell_sizes(sizes)
    return shards, bases


@pytest.mark.parametrize("G", [2, 3])
@pytest.mark.parametrize("variant", ["exact", "filter", "short_rounds", "sharded_a0"])
def test_global_patience_equals_single_index(crisp, case, monkeypatch, G, variant):
    import torch

    from paper_2603_05180_b200 import dist

    X, Qv, ox, single = case
    if variant == "filter":
        monkeypatch.setenv("CRISP_FILTER_ROUNDS", "2")
        monkeypatch.setenv("CRISP_LB_FIRST", "64")
    if variant == "short_rounds":
        monkeypatch.setenv("CRISP_GP_MIN", "32")
        monkeypatch.setenv("CRISP_GP_MAX", "64")
        monkeypatch.setenv("CRISP_PATIENCE_FIRST", "32")
    shards, bases = shard_indexes(crisp, X, ox, G)
    for s in shards + [single]:
        s.set_verify_filter(variant == "filter")
    dev = torch.device("cuda", 0)
    q_dev = torch.from_numpy(Qv).to(dev)
    # (k, B, tau, P): ordinary, long patience, forced global fallback (tau high, B small)
    for k, B, tau, P in ((10, 2500, 2, 30), (20, 6000, 1, 10), (5, 300, 6, 40)):
        for s in shards + [single]:
            s.set_search_params(budget=B, tau=tau, patience_factor=P)
        ids_s, d_s = single.search(Qv, k, 1)
        engines = []
        for s in shards:
            e = dist.CudaEngine(crisp, dev)
            e.index = s
            engines.append(e)
        st = {}
        ids_g, d_g = dist.emulate_global_search(engines, bases, q_dev, k, 1, stats=st,
                                                sharded_a0=variant == "sharded_a0")
        if variant == "short_rounds" and k == 10:  # |C_q| ~ 8k, stops up to ~1100: many 64-position windows
            assert st["rounds"] >= 10, st
        torch.cuda.synchronize()
        assert np.array_equal(ids_g.cpu().numpy(), ids_s), f"G={G} {variant} k={k}"
        assert np.array_equal(d_g.cpu().numpy(), d_s), f"G={G} {variant} k={k}"
        r_ids, _, _ = oracle.search(ox, Qv, k, 1, B, tau, patience_factor=P)
        assert np.array_equal(ids_s, r_ids)
    for s in shards:
        s.free()
    single.set_verify_filter(True)


@pytest.mark.parametrize("rotation", [0, 1])
def test_transform_queries_is_the_searchs_a0(crisp, rotation):
    """crisp_transform_queries_async writes the q' a search computes (the
    oracle's fl32(q R), zero-padded to the row pitch; the padded queries when
    the index is not rotated), for a slice too (the sharded a0 of N9), and Q = 0
    is a no-op."""
    import torch

    from paper_2603_05180_b200 import dist

    X, Qv, ox = make_case(cfg=2, N=6000, D=90, Q=37, M=4, K=12, rotation=rotation, seed=7)
    ix = build_gpu(crisp, X, ox)
    pitch = ix.info()["pitch"]
    ix.set_search_params(budget=500, tau=2, patience_factor=3)
    _, _, t = ix.trace(Qv, 5, 1)
    e = dist.CudaEngine(crisp, torch.device("cuda", 0))
    e.index = ix
    q_dev = torch.from_numpy(Qv).cuda()
    full = e.transform(q_dev)
    part = e.transform(q_dev[10:29])
    torch.cuda.synchronize()
    assert full.shape == (37, pitch) and np.array_equal(full.cpu().numpy()[:, : ox["Dp"]], t["qrot"])
    assert np.array_equal(full.cpu().numpy()[:, : ox["Dp"]], oracle.search(ox, Qv, 5, 1, 500, 2, trace=True,
                                                                          patience_factor=3)[2]["qrot"])
    assert np.array_equal(part.cpu().numpy(), full.cpu().numpy()[10:29])
    assert e.transform(q_dev[:0]).shape == (0, pitch)
    ix.free()
