"""One syev_tri_kernel launch on a random symmetric n x n (ncu target): python tools/tri_one.py N"""
import ctypes, os, sys
import numpy as np
lib = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "libtri_check.so"))
P = ctypes.POINTER(ctypes.c_double)
n = int(sys.argv[1])
a = np.random.default_rng(1).standard_normal((n, n)); h = np.asfortranarray((a + a.T) / 2)
lam = np.zeros(n); z = np.zeros((n, n), order="F"); ms = ctypes.c_float(0); prof = np.zeros(8, dtype=np.int64)
st = lib.tri_eig(n, h.ctypes.data_as(P), lam.ctypes.data_as(P), z.ctypes.data_as(P), 1, 0, ctypes.byref(ms),
                 prof.ctypes.data_as(ctypes.POINTER(ctypes.c_longlong)))
print("status", st, "kcyc", prof[:6] // 1000)
