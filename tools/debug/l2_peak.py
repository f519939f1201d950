import ctypes, sys
sys.path.insert(0, '.')
from paper_1509_04681_b200 import Context
c = Context(0)
for s in (0.5, 1.0):
    g, ms = ctypes.c_double(), ctypes.c_double()
    c._check(c.lib.cggm_test_l2_peak(c.h, s, ctypes.byref(g), ctypes.byref(ms)))
    print("l2 GB/s", g.value, ms.value)
