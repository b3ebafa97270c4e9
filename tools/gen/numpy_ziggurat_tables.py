"""Extract numpy's ziggurat tables for Generator.standard_normal (float64) by driving its PCG64 bit generator.

numpy's `random_standard_normal` (distributions.c) turns one next_uint64 r into idx = r & 0xff, sign = (r >> 8) & 1,
rabs = (r >> 9) & (2^52 - 1), x = rabs * wi[idx], and returns x when rabs < ki[idx].  A PCG64 state can be chosen so
that the next output is any r (output = low word of the post-step state when its high word is 0), so
  wi[idx] = standard_normal() with rabs = 1, and
  ki[idx] = the smallest rabs whose call consumes more than one output (bisection).
fi[idx] (used only to accept/reject in the rare wedge branch) is exp(-x_i^2 / 2) at x_i = wi[idx] * 2^52
(fi[0] = 1), checked against numpy's own wedge decisions: with two controlled outputs (the PCG64 increment is
free), the accept/reject threshold on the uniform must match the tables' for every idx.  Writes paper_2305_15668_b200/csrc/ziggurat_tables.h.
"""
import math
import os

import numpy as np

M = 0x2360ED051FC65DA44385DF649FCCF645  # PCG64 multiplier (numpy pcg64.h PCG_DEFAULT_MULTIPLIER_128)
MASK = (1 << 128) - 1
MINV = pow(M, -1, 1 << 128)


def gen_with_next(r: int, inc: int = 1) -> np.random.Generator:
    """A Generator whose next next_uint64 is r (post-step state = r, high word 0, rotation 0)."""
    pre = ((r - inc) * MINV) & MASK
    bg = np.random.PCG64()
    bg.state = {"bit_generator": "PCG64", "state": {"state": pre, "inc": inc}, "has_uint32": 0, "uinteger": 0}
    return np.random.Generator(bg)


def gen_with_next2(r1: int, r2: int) -> tuple[np.random.Generator, int, int]:
    """A Generator whose next two outputs are r1 and r2 (r2's low bit may be flipped; the increment is chosen)."""
    if ((r2 ^ r1) & 1) == 0:
        r2 ^= 1                                   # inc = r2 - r1 * M must be odd
    inc = (r2 - r1 * M) & MASK
    pre = ((r1 - inc) * MINV) & MASK
    bg = np.random.PCG64()
    bg.state = {"bit_generator": "PCG64", "state": {"state": pre, "inc": inc}, "has_uint32": 0, "uinteger": 0}
    return np.random.Generator(bg), pre, inc


def wedge_threshold(accepts) -> int:
    """Smallest 53-bit m (u = m / 2^53) the wedge test rejects; accepts(m) is monotone (True below it)."""
    lo, hi = 0, 1 << 53
    while lo < hi:
        mid = (lo + hi) // 2
        if accepts(mid):
            lo = mid + 1
        else:
            hi = mid
    return lo


def _numpy_threshold(idx: int, rabs: int) -> int:
    r1 = (rabs << 9) | idx

    def accepts(m):
        g, pre, inc = gen_with_next2(r1, m << 11)
        g.standard_normal()
        return draws_used(g, pre, inc) == 2
    return wedge_threshold(accepts)


def _table_threshold(top: float, f: float, x: float) -> int:
    e = math.exp(-0.5 * x * x)
    return wedge_threshold(lambda m: (top - f) * ((m * 1.0) / 9007199254740992.0) + f < e)


def solve_fi(wi: np.ndarray, ki: np.ndarray, fi: np.ndarray, probes: int = 8) -> None:
    """Replace fi[1..255] by the doubles numpy's own wedge decisions imply.

    With two controlled outputs (the PCG64 increment is free) the uniform at which numpy's wedge test flips from
    accept to reject is measured at `probes` points x of each wedge; given fi[idx-1], the threshold is monotone
    (non-increasing) in fi[idx], so the doubles near exp(-x_i^2 / 2) that reproduce every measured threshold form
    an interval, found by bisection over ulp offsets.  Both sides use the same libm exp.
    """
    moved = ambiguous = 0
    for idx in range(1, 256):
        lo_r = max(int(ki[idx]), 1)
        xs = [lo_r + ((1 << 52) - 1 - lo_r) * j // (probes - 1) for j in range(probes)]
        xs = sorted(set(xs))
        top, est = float(fi[idx - 1]), float(fi[idx])

        def cand(k):
            return _ulp_step(est, k)
        lo, hi = -4096, 4096
        for rabs in xs:
            x = float(rabs) * float(wi[idx])
            want = _numpy_threshold(idx, rabs)
            # first offset whose threshold <= want, and first whose threshold < want
            def first(pred):
                a, b = lo, hi + 1
                while a < b:
                    m = (a + b) // 2
                    if pred(_table_threshold(top, cand(m), x)):
                        b = m
                    else:
                        a = m + 1
                return a
            a = first(lambda t: t <= want)
            b = first(lambda t: t < want) - 1
            lo, hi = max(lo, a), min(hi, b)
            if lo > hi:
                raise SystemExit(f"fi[{idx}]: no double reproduces numpy's wedge decisions")
        fi[idx] = cand((lo + hi) // 2)
        moved += (lo + hi) // 2 != 0
        ambiguous += hi > lo
    print(f"fi: {moved} entries off exp(-x^2/2) by >= 1 ulp, {ambiguous} not pinned to a single double")
    # cross-check at points the solve did not use
    rng = np.random.default_rng(5)
    for idx in range(1, 256):
        for rabs in rng.integers(max(int(ki[idx]), 1), 1 << 52, size=3):
            x = float(int(rabs)) * float(wi[idx])
            if _numpy_threshold(idx, int(rabs)) != _table_threshold(float(fi[idx - 1]), float(fi[idx]), x):
                raise SystemExit(f"fi[{idx}] disagrees with numpy at rabs {int(rabs)}")


def _ulp_step(v: float, k: int) -> float:
    b = np.array([v]).view(np.int64)[0] + k
    return float(np.array([b], dtype=np.int64).view(np.float64)[0])


NOR_R = 3.6541528853610087963519472518      # ziggurat_nor_r, as normal.cu uses it
NOR_INV_R = 0.27366123732975827203338247596  # ziggurat_nor_inv_r


def check_tail(ki: np.ndarray) -> None:
    """The tail constants: an idx-0 slow-path attempt whose first tail pair is accepted returns
    +-(r + xx), xx = -inv_r * log1p(-u1); compare numpy's value bit for bit at controlled u1."""
    checked = 0
    for m in range(1, 1 << 53, (1 << 53) // 997):
        rabs = (1 << 52) - 1 - m % 1000               # >= ki[0]: the tail branch
        assert rabs >= int(ki[0])
        g, pre, inc = gen_with_next2(rabs << 9, m << 11)
        v = g.standard_normal()
        if draws_used(g, pre, inc) != 3:
            continue                                  # first pair rejected (u2 is not controlled)
        u = m * (1.0 / 9007199254740992.0)            # next_double of the second output
        xx = -NOR_INV_R * math.log1p(-u)
        want = -(NOR_R + xx) if (rabs >> 8) & 1 else NOR_R + xx
        if v != want:
            raise SystemExit(f"tail constants disagree with numpy: {v!r} vs {want!r}")
        checked += 1
    print(f"tail: {checked} accepted tail draws match numpy bit for bit")


def draws_used(g: np.random.Generator, start_state: int, inc: int) -> int:
    s = g.bit_generator.state["state"]["state"]
    k, t = 0, start_state
    while t != s and k < 64:
        t = (t * M + inc) & MASK
        k += 1
    return k


def main():
    wi = np.zeros(256)
    ki = np.zeros(256, dtype=np.uint64)
    for idx in range(256):
        r = (1 << 9) | idx
        wi[idx] = gen_with_next(r).standard_normal()
        lo, hi = 0, (1 << 52)  # smallest rabs with a slow path
        while lo < hi:
            mid = (lo + hi) // 2
            g = gen_with_next((mid << 9) | idx)
            pre = g.bit_generator.state["state"]["state"]
            g.standard_normal()
            if draws_used(g, pre, 1) == 1:
                lo = mid + 1
            else:
                hi = mid
        ki[idx] = lo
    # x_i and the wedge tops: fi[i] = exp(-x_i^2 / 2) for i >= 1.  wi[0] is the base strip's (tail) width,
    # not a boundary; fi[0] is the density at 0 (= 1), the top of the wedge test for idx = 1 (whose ki is 0,
    # so every idx-1 attempt goes through it)
    fi = np.exp(-0.5 * (wi * 2.0 ** 52) ** 2)
    fi[0] = 1.0
    solve_fi(wi, ki, fi)
    check_tail(ki)
    # numpy's tail constants: r = x_255 boundary... recover r from the base strip: ki[0] = 2^52 r f(r) / v
    here = os.path.dirname(os.path.abspath(__file__))
    out = os.path.join(here, "..", "..", "paper_2305_15668_b200", "csrc", "ziggurat_tables.h")
    with open(out, "w") as fh:
        fh.write("// numpy Generator.standard_normal (float64) ziggurat tables, extracted from numpy %s by\n"
                 "// tools/gen/numpy_ziggurat_tables.py (wi, ki by driving its PCG64; fi solved from its wedge decisions).\n"
                 "#pragma once\n#include <stdint.h>\n\nnamespace fedhc {\nnamespace zig {\n" % np.__version__)
        fh.write("__device__ __constant__ const uint64_t ki[256] = {\n")
        for i in range(0, 256, 4):
            fh.write("    " + ", ".join("0x%016XULL" % int(v) for v in ki[i:i + 4]) + ",\n")
        fh.write("};\n__device__ __constant__ const double wi[256] = {\n")
        for i in range(0, 256, 4):
            fh.write("    " + ", ".join(float(v).hex() for v in wi[i:i + 4]) + ",\n")
        fh.write("};\n__device__ __constant__ const double fi[256] = {\n")
        for i in range(0, 256, 4):
            fh.write("    " + ", ".join(float(v).hex() for v in fi[i:i + 4]) + ",\n")
        fh.write("};\n}  // namespace zig\n}  // namespace fedhc\n")
    print("wrote", out, "wi[1..3]", wi[1:4], "ki[0..3]", ki[:4])


if __name__ == "__main__":
    main()
