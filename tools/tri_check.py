"""Accuracy and timing of the one-CTA tridiagonal eigensolver (syev_tri_kernel)
against numpy eigh on random, clustered, graded, rank-deficient and
split inputs: python tools/tri_check.py (needs tools/libtri_check.so)."""
import ctypes, os, sys
import numpy as np
lib = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "libtri_check.so"))
P = ctypes.POINTER(ctypes.c_double)

def run(h, reps=0, desc=1):
    n = h.shape[0]
    hf = np.asfortranarray(h)
    lam = np.zeros(n); z = np.zeros((n, n), order="F"); ms = ctypes.c_float(0)
    prof = np.zeros(8, dtype=np.int64)
    st = lib.tri_eig(n, hf.ctypes.data_as(P), lam.ctypes.data_as(P), z.ctypes.data_as(P), desc, reps, ctypes.byref(ms),
                     prof.ctypes.data_as(ctypes.POINTER(ctypes.c_longlong)))
    run.prof = prof[:6]
    return st, lam, z, ms.value

def check(name, h, reps=20):
    n = h.shape[0]
    st, lam, z, ms = run(h, reps)
    ref = np.linalg.eigvalsh(h)[::-1]
    hn = np.linalg.norm(h, 2)
    el = np.max(np.abs(lam - ref)) / hn
    res = np.linalg.norm(h @ z - z * lam) / hn
    orth = np.linalg.norm(z.T @ z - np.eye(n))
    ok = st == 0 and el < 1e-13 and res < 1e-11 and orth < 1e-9
    print(f"{name:28s} n={n:4d} st={st} lam_err={el:.1e} resid={res:.1e} orth={orth:.1e} ms={ms:.3f} {'ok' if ok else 'FAIL' if st == 0 else 'fallback'} kcyc={'/'.join(str(int(x) // 1000) for x in run.prof)}")
    return ok or st != 0

rng = np.random.default_rng(0)
def sym(a): return (a + a.T) / 2
allok = True
for n in [int(a) for a in sys.argv[1:]] or [33, 64, 96, 128, 150, 160]:
    allok &= check("gaussian", sym(rng.standard_normal((n, n))))
    b = rng.standard_normal((n, 3 * n)); allok &= check("gram", b @ b.T)
    u, _ = np.linalg.qr(rng.standard_normal((n, n)))
    lam = np.exp(-np.arange(n) / 10.0); allok &= check("graded 1e-7", (u * lam) @ u.T)
    lam = np.concatenate([np.ones(6), np.linspace(0.5, 0.1, n - 6)]); allok &= check("cluster of 6", (u * lam) @ u.T)
    lam = np.concatenate([np.ones(3), np.zeros(n - 3)]); allok &= check("rank 3", (u * lam) @ u.T)
    allok &= check("diagonal", np.diag(rng.standard_normal(n)))
    allok &= check("identity", np.eye(n))
    allok &= check("scaled 1e100", sym(rng.standard_normal((n, n))) * 1e100)
    lam = 1.0 + 1e-4 * rng.standard_normal(n); allok &= check("tight spectrum 1e-4", (u * lam) @ u.T)
    lam = np.arange(1, n + 1) ** -3.0; allok &= check("power -3 (cfg3 core)", (u * lam) @ u.T)
print("ALL OK" if allok else "SOME FAILED")
