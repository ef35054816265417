"""debug: window-kernel SpMV vs the oracle on the parity-test matrices; prints failing rows"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import gse_inputs as gi, oracle as O, paper_2411_04686_b200 as g
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from test_gpu_parity import MATS, spmv_bound, window_edge_matrix
names = sys.argv[1:] or ["long_rows", "random_classes", "random_mixed", "powerlaw_30k"]
for name in names:
    A = MATS[name]() if name in MATS else window_edge_matrix(name)
    M = g.gse_encode(A.row_ptr, A.col, A.val, A.rows, A.cols)
    R = O.encode_csr(A.rows, A.cols, A.row_ptr, A.col, A.val)
    x = gi.uniform_vec(A.cols, seed=5)
    lens = np.diff(A.row_ptr)
    print(name, "rows", A.rows, "nnz", A.nnz, "mode", M.info["spmv_mode"], "empty", int((lens == 0).sum()))
    for L in (1, 3):
        yg = g.gse_spmv(M, x, segments=L)
        yo = O.spmv_gse(R, x, L)
        bad = np.nonzero(np.abs(yg - yo) > spmv_bound(R, x, L, 1e-12))[0]
        print(f"  L{L} bad rows {bad.size}")
        for r in bad[:12]:
            print(f"    row {r} len {lens[r]} start {A.row_ptr[r]} gpu {yg[r]:.6g} orc {yo[r]:.6g}")
