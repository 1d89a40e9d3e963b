"""Quick device-timed sweep (development aid, not the bench contract)."""
import sys
import time

import paper_1811_08282_b200 as s1d


def main():
    ns = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "24").split(",")]
    ws = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "64,256,1024").split(",")]
    steps = int(sys.argv[3]) if len(sys.argv) > 3 else 1024
    eq = sys.argv[4] if len(sys.argv) > 4 else "heat"
    for lg in ns:
        n = 1 << lg
        for scheme in (s1d.Scheme.Classic, s1d.Scheme.Swept):
            for w in ws if scheme == s1d.Scheme.Swept else ws[:1]:
                n = (1 << lg) // w * w  # a whole number of tiles
                c = s1d.LaunchConfig(equation=s1d.Equation.Heat if eq == "heat" else s1d.Equation.Euler,
                                     scheme=scheme, grid_size=n, block_width=w, ranks=1, steps=steps)
                with s1d.Solver(c) as sv:
                    sv.advance()
                    best = 1e9
                    for _ in range(3):
                        st, tm = sv.advance()
                        best = min(best, tm.loop_seconds)
                    rate = n * steps / best
                    print(f"{eq} n=2^{lg} {s1d.to_string(scheme):7s} w={w:5d} T={steps}: "
                          f"{best*1e6/steps:9.2f} us/step  {rate/1e9:8.2f} Gpt/s  launches={st.kernel_launches}",
                          flush=True)


if __name__ == "__main__":
    main()
