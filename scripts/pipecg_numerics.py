"""Host check (numpy/scipy) that pipelined CG (Ghysels-Vanroose: the SpMV of
w overlaps the one all-reduce per iteration) keeps the reference iteration
count and accuracy on the FEM-shaped 30880 matrix: the precondition for a
pipelined cluster engine (DESIGN known gaps).  Not product code."""
import numpy as np, sys
sys.path.insert(0,'.')
from paper_1010_4639_b200.genprob import fem_mesh, rhs_for
from oracle import oracle as O
import scipy.sparse as sp
F = fem_mesh()
A = sp.csr_matrix((F.values, F.col_idx, F.row_start), shape=(F.n, F.n))
b, xg = rhs_for(F, seed=1)
ref = O.cg_solve("csr", F.row_start, F.col_idx, F.values, b, max_iter=F.n)
print("ref iters", ref.iterations)
bn = np.linalg.norm(b)
def cgcg(maxit=2000, tol=1e-10):
    # Chronopoulos-Gear (engine 3/5 recurrences)
    x = np.zeros_like(b); r = b.copy(); w = A@r
    g = r@r; d = w@r
    p = np.zeros_like(b); s = np.zeros_like(b); a_old=None; g_old=None
    for k in range(maxit):
        if k == 0: beta = 0.0; alpha = g/d
        else:
            beta = g/g_old; alpha = g/(d - beta*g/a_old)
        p = r + beta*p; s = w + beta*s
        x = x + alpha*p; r = r - alpha*s
        w = A@r
        g_old, a_old = g, alpha
        g = r@r; d = w@r
        if np.sqrt(g) <= tol*bn: return x, k+1
    return x, maxit
def pipecg(maxit=2000, tol=1e-10):
    # Ghysels-Vanroose pipelined CG
    x = np.zeros_like(b); r = b.copy(); w = A@r
    z = np.zeros_like(b); s = np.zeros_like(b); p = np.zeros_like(b)
    g_old=a_old=None
    for k in range(maxit):
        g = r@r; d = w@r
        if np.sqrt(g) <= tol*bn: return x, k
        q = A@w
        if k == 0: beta = 0.0; alpha = g/d
        else:
            beta = g/g_old; alpha = g/(d - beta*g/a_old)
        z = q + beta*z; s = w + beta*s; p = r + beta*p
        x = x + alpha*p; r = r - alpha*s; w = w - alpha*z
        g_old, a_old = g, alpha
    return x, maxit
for name, f in [("cgcg", cgcg), ("pipecg", pipecg)]:
    x, it = f()
    tr = np.linalg.norm(b - A@x)/bn
    print(name, it, "true rel", tr, "x err vs ref", np.linalg.norm(x-ref.x)/np.linalg.norm(ref.x))
