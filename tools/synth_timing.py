import sys, time
sys.path.insert(0, ".")
from paper_1809_05018_b200 import engine as E
c = E.Context(0)
for size in (2560, 16384):
    for args in ((0.25, 0.0, 0.0, False), (0.25, 0.05, 100.0, True)):
        c.make_phantom(size, size, *args, 42, copy_out=False)
        t0 = time.perf_counter(); _, _, ties = c.make_phantom(size, size, *args, 42, copy_out=False); t1 = time.perf_counter()
        print(size, args, "%.2f ms" % ((t1 - t0) * 1e3), "ties", ties)
