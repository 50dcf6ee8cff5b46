import ctypes as C, sys
sys.path.insert(0,'.')
from paper_2205_09707_b200 import _native
lib=_native.load()
lib.plaid_measure_read_gbs.argtypes=[C.c_int,C.c_uint64,C.c_int,C.POINTER(C.c_double)]
for mb in (64,128,256,512,1024,2048,4096):
    g=C.c_double()
    lib.plaid_measure_read_gbs(0, mb<<20, 5, C.byref(g))
    print(f"read {mb} MiB: {g.value:.0f} GB/s")
