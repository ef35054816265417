"""The C-ABI library loads on a CPU-only host and exports every symbol include/gse.h
declares; host-only entry points behave as documented (no GPU compute here)."""
import ctypes as C
import json
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "gse.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(gse_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    import paper_2411_04686_b200 as g
    names = header_functions()
    assert len(names) >= 18
    lib = C.CDLL(g.LIB_PATH)
    for n in names:
        assert hasattr(lib, n), n
    assert set(g.ABI_SYMBOLS) == set(names)


def test_binding_names_match_abi():
    import paper_2411_04686_b200 as g
    for n in header_functions():
        if n in ("gse_status_string", "gse_last_error_detail",
                 "gse_nccl_unique_id", "gse_dist_create", "gse_encode_dist", "gse_dist_free"):
            continue
        assert callable(getattr(g, n)), n


def test_status_strings_and_defaults():
    import paper_2411_04686_b200 as g
    lib = g.lib()
    assert lib.gse_status_string(0) == b"ok"
    assert b"non-finite" in lib.gse_status_string(12)
    gold = json.load(open(os.path.join(ROOT, "tests", "golden", "spec_examples.json")))["defaults"]
    for solver in ("cg", "gmres"):
        s = g.gse_default_schedule(solver)
        for k, v in gold[solver].items():
            assert getattr(s, k) == v, (solver, k)
        assert s.enabled == 1 and s.verify_at_full == 1 and s.start_level == 1


def test_invalid_args_fail_without_touching_the_gpu():
    import paper_2411_04686_b200 as g
    lib = g.lib()
    assert lib.gse_spmv(None, None, None, 1, None) == g.GSE_ERR_INVALID_ARG
    assert lib.gse_solve_cg(None, None, None, 1e-6, 10, None, None, None) == g.GSE_ERR_INVALID_ARG
    A = g.CsrF64(2, 2, 2, None, 0, None, None)
    opts = g.EncodeOpts(3, 0, 0, 0, 0)  # k_max not a power of two
    out = C.c_void_p()
    assert lib.gse_encode(C.byref(A), C.byref(opts), C.byref(out), None) == g.GSE_ERR_INVALID_ARG
    assert b"k_max" in lib.gse_last_error_detail()


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2411_04686_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "gse_oracle" not in txt, f
