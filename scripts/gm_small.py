import sys; sys.path.insert(0, '/root/repo')
import numpy as np, gse_inputs as gi, paper_2411_04686_b200 as g
A = gi.convdiff3d(16); b = gi.ones_rhs(A)
M = g.gse_fp64_matrix(A.row_ptr, A.col, A.val, A.rows, A.cols)
x, r = g.gse_solve_gmres(M, b, tol=1e-10)
print(r)
