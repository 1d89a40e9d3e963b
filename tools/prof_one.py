"""Run one configuration twice (warm-up + measured) for ncu / sanitizer runs."""
import argparse

import paper_1811_08282_b200 as s1d

ap = argparse.ArgumentParser()
ap.add_argument("--eq", default="heat")
ap.add_argument("--method", default="lengthening")
ap.add_argument("--scheme", default="swept")
ap.add_argument("--n", type=int, default=24)
ap.add_argument("--w", type=int, default=1024)
ap.add_argument("--steps", type=int, default=1024)
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()
c = s1d.LaunchConfig(equation=s1d.Equation.Heat if a.eq == "heat" else s1d.Equation.Euler,
                     method=s1d.Method.Lengthening if a.method == "lengthening" else s1d.Method.Flattening,
                     scheme=s1d.Scheme.Swept if a.scheme == "swept" else s1d.Scheme.Classic,
                     grid_size=1 << a.n, block_width=a.w, ranks=1, steps=a.steps)
with s1d.Solver(c) as sv:
    for _ in range(a.reps):
        st, tm = sv.advance()
        n = c.grid_size
        print(f"{a.eq} {a.scheme} n=2^{a.n} w={a.w} T={a.steps}: {tm.loop_seconds*1e6/a.steps:.2f} us/step "
              f"{n*a.steps/tm.loop_seconds/1e9:.1f} Gpt/s launches={st.kernel_launches}", flush=True)
