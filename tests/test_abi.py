"""Host-side checks of the C ABI (no GPU needed): the library loads, exports
every symbol include/crisp.h declares, the binding lists the same set, and the
oracle and the CUDA path share no code."""
import os
import re
import subprocess

import numpy as np

import __graft_entry__ as ge

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "crisp.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return set(re.findall(r"\b(crisp_[a-z0-9_]+)\s*\(", src))


def test_library_builds_and_loads():
    ge.build()
    import paper_2603_05180_b200 as crisp

    assert crisp.lib().crisp_version().startswith(b"crisp-b200")


def test_exports_every_declared_symbol():
    ge.build()
    import paper_2603_05180_b200 as crisp

    declared = header_functions()
    assert declared == set(crisp.ABI_SYMBOLS)
    out = subprocess.check_output(["nm", "-D", "--defined-only", crisp.LIB_PATH]).decode()
    exported = set(re.findall(r" T (crisp_[a-z0-9_]+)$", out, flags=re.M))
    assert declared <= exported, declared - exported


def test_default_params_no_gpu():
    ge.build()
    import paper_2603_05180_b200 as crisp

    p = crisp.default_params(M=8)
    assert (p.M, p.K, round(p.tau_cev, 6), p.kmeans_iters, p.patience_factor) == (8, 50, 0.85, 20, 40)


def test_exact_parameters_c_abi():
    """B and tau are derived inside the C library (crisp_exact_ceil, the rule
    crisp_set_search_params applies), and agree with the oracle's decimal rule
    (O1) on the cases binary floating point gets wrong and over a grid."""
    ge.build()
    import oracle
    import paper_2603_05180_b200 as crisp

    assert crisp.lib().crisp_exact_ceil(0.035, 20000) == 700
    assert crisp.lib().crisp_exact_ceil(0.07, 100) == 7
    assert crisp.lib().crisp_exact_ceil(0.0, 10) == 0
    for a100 in range(1, 101):
        alpha = a100 / 100
        for M in range(1, 128):
            assert crisp.exact_ceil(alpha, M) == oracle.tau_int(alpha, M), (alpha, M)
    for beta in (0.001, 0.002, 0.005, 0.01, 0.02, 0.035, 0.04, 0.06, 0.1, 0.2, 0.4, 1.0, 1e-7, 0.123456789):
        for N in (1, 7, 20000, 1_000_000, 2_000_000, 1_281_167, 2 ** 31 - 1):
            assert crisp.exact_ceil(beta, N) == oracle.budget_ids(beta, N), (beta, N)


def test_sm100a_cubin_present():
    ge.build()
    import paper_2603_05180_b200 as crisp

    out = subprocess.check_output(["/usr/local/cuda/bin/cuobjdump", "--list-elf", crisp.LIB_PATH]).decode()
    assert "sm_100a" in out


def test_oracle_and_cuda_path_share_no_code():
    pkg = os.path.join(ROOT, "paper_2603_05180_b200")
    for dp, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                s = open(os.path.join(dp, f)).read()
                assert "oracle" not in re.findall(r"(?:import|include)\s+[\"<]?([a-z_./]+)", s), f
                assert "liboracle" not in s and "crisp_oracle" not in s, f
    osrc = open(os.path.join(ROOT, "oracle", "crisp_oracle.c")).read()
    opy = open(os.path.join(ROOT, "oracle", "__init__.py")).read()
    assert not re.search(r"^\s*#\s*include\s*[\"<][^\">]*(crisp|paper_2603)", osrc, flags=re.M)
    assert not re.search(r"^\s*(import|from)\s+paper_2603_05180_b200", opy, flags=re.M)


def test_product_fails_loudly_without_library(tmp_path, monkeypatch):
    import paper_2603_05180_b200 as crisp

    monkeypatch.setattr(crisp, "LIB_PATH", str(tmp_path / "missing.so"))
    monkeypatch.setattr(crisp, "_lib", None)
    try:
        crisp.lib()
        raised = False
    except crisp.CrispError:
        raised = True
    assert raised
