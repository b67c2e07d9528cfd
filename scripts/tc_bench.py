import ctypes as C, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2110_07029_b200 import _lib as L
lib = L.load()
for mode in [int(m) for m in sys.argv[1:]] or range(0, 11):
    for iters in (100, 1000):
        c = C.c_int64()
        L.check(lib.as_tc_bench(mode, iters, C.byref(c)))
        n = 256 if mode == 3 else 128
        print("mode", mode, "iters", iters, "cycles/group %.1f" % (c.value / iters),
              "flop/clk %.0f" % (2 * 128 * n * 128 * iters / c.value))
