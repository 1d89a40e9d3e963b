"""Dev check: heat n=2^30 on one GPU (1M tiles, 8 GiB state), swept == classic bitwise.
    PYTHONPATH=. python tools/big_check.py"""
import numpy as np, paper_1811_08282_b200 as s1d, time
n=1<<30
def run(scheme, T):
    c=s1d.LaunchConfig(equation=s1d.Equation.Heat, scheme=scheme, grid_size=n, block_width=1024, ranks=1, steps=T, mode=s1d.Mode.WallClock)
    t=time.time(); r=s1d.run(c); return r.state, r.timing.loop_seconds, time.time()-t
a,ta,wa=run(s1d.Scheme.Swept, 1024)
b,tb,wb=run(s1d.Scheme.Classic, 1024)
print("n=2^30 T=1024 swept==classic:", np.array_equal(a.view(np.uint64), b.view(np.uint64)), "swept %.3f s (%.1f Gpt/s) classic %.3f s" % (ta, n*1024/ta/1e9, tb), "wall", round(wa,1), round(wb,1))
