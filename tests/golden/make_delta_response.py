"""Writes tests/golden/delta_response_c1.txt: the exact (rational) response of the 3D-model
update to a unit delta, computed by brute force in exact rational arithmetic.

Definition followed (§2 — 10th order in space, 2nd order in time, five cells
each direction per dimension; BASELINE.json configs[0] — coefficients c0..c5 as exact
rationals, u_prev = 0 initially, C = nu^2 = (v dt / dx)^2 = (2000 * 0.001 / 10)^2 = 1/25):

    u^{n+1}(p) = 2 u^n(p) - u^{n-1}(p) + C * sum_axis sum_{o=-5..5} c_|o| u^n(p + o e_axis)

The support stays >= 16 cells from any boundary of a 64^3 grid centred at 32 for n <= 3, so
the zero halo plays no role.  This script uses neither oracle/ nor the CUDA path; it is an
independent brute-force pin.  Run: python tests/golden/make_delta_response.py
"""
from __future__ import annotations

from fractions import Fraction as Fr
from pathlib import Path

COEFFS = (Fr(-5269, 1800), Fr(5, 3), Fr(-5, 21), Fr(5, 126), Fr(-5, 1008), Fr(1, 3150))
C = Fr(1, 25)
STEPS = 3
OFFSETS = [(0, 0, 0), (1, 0, 0), (0, 1, 0), (0, 0, 1), (2, 0, 0), (5, 0, 0), (6, 0, 0),
           (-3, 0, 0), (1, 1, 0), (0, 1, -1), (1, 1, 1), (2, -1, 3), (5, 5, 5), (10, 0, 0),
           (15, 0, 0), (7, 4, 0)]


def apply_L(u: dict) -> dict:
    out: dict = {}
    for (z, y, x), val in u.items():
        for axis in range(3):
            for o in range(-5, 6):
                q = [z, y, x]
                q[axis] += o
                q = tuple(q)
                out[q] = out.get(q, Fr(0)) + COEFFS[abs(o)] * val
    return out


def evolve(steps: int):
    u = {(0, 0, 0): Fr(1)}
    up: dict = {}
    hist = []
    for _ in range(steps):
        Lu = apply_L(u)
        keys = set(u) | set(up) | set(Lu)
        nxt = {}
        for k in keys:
            val = 2 * u.get(k, Fr(0)) - up.get(k, Fr(0)) + C * Lu.get(k, Fr(0))
            if val != 0:
                nxt[k] = val
        up, u = u, nxt
        hist.append(u)
    return hist


def main():
    hist = evolve(STEPS)
    lines = ["# exact delta response, C = 1/25, coefficients of BASELINE.json configs[0]",
             "# columns: n dz dy dx numerator denominator float ; support sizes: "
             + " ".join(str(len(h)) for h in hist)]
    for n, h in enumerate(hist, start=1):
        for (dz, dy, dx) in OFFSETS:
            v = h.get((dz, dy, dx), Fr(0))
            lines.append(f"{n} {dz} {dy} {dx} {v.numerator} {v.denominator} {float(v):.17g}")
    out = Path(__file__).with_name("delta_response_c1.txt")
    out.write_text("\n".join(lines) + "\n")
    print(f"wrote {out}")


if __name__ == "__main__":
    main()
