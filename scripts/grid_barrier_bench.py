import sys, ctypes as C; sys.path.insert(0, '.')
import torch; torch.cuda.init()
from paper_2507_01021_b200 import _native
lib = _native.load(); us = C.c_float()
for it in (100, 1000):
    _native.check(lib.dm_bench_grid_barrier(it, C.byref(us))); print("grid barrier us", it, us.value)
