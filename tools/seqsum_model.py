#!/usr/bin/env python
"""Host model of seq_sum_warp (csrc/chunked.cuh): the exact emulation of a sequential fp64
sum  s = RN(s + t[k]), k = 0..m-1, by a warp that commits whole runs of terms at once while
the running sum stays inside one binade.  Checked bit for bit against the plain sequential
loop on adversarial inputs (ties, cancellation through zero, binade crossings, huge and
tiny magnitudes, non-finite values).  Run: python tools/seqsum_model.py [cases]"""
import math
import struct
import sys

import numpy as np

LANES = 32
TWO52, TWO53 = 1 << 52, 1 << 53


def bits(x):
    return struct.unpack("<q", struct.pack("<d", x))[0]


def from_bits(b):
    return struct.unpack("<d", struct.pack("<q", b))[0]


def serial(s, t):
    for v in t:
        s = s + v
    return s


def model(s, t, per):
    m = len(t)
    pos = 0
    while pos < m:
        if m - pos <= 16:
            return serial(s, t[pos:])
        sb = bits(s)
        ex = (sb >> 52) & 0x7FF
        if ex < 54 or ex > 2046:
            s = s + t[pos]
            pos += 1
            continue
        inv_u = from_bits((2098 - ex) << 52)
        u = from_bits((ex - 52) << 52)
        mant = (sb & ((1 << 52) - 1)) | (1 << 52)
        S = -mant if sb < 0 else mant
        # per-lane conversion + local prefix
        lane_P, lane_ok, lane_tot = [], [], []
        for lane in range(LANES):
            acc, P, ok = 0, [], []
            for j in range(per):
                k = pos + lane * per + j
                Q, good = 0, False
                if k < m:
                    q = t[k] * inv_u
                    aq = abs(q)
                    if aq < 9007199254740992.0:  # also false for inf / nan
                        if aq - math.floor(aq) != 0.5:
                            good = True
                            Q = int(np.rint(q))
                acc += Q
                P.append(acc)
                ok.append(good)
            lane_P.append(P)
            lane_ok.append(ok)
            lane_tot.append(acc)
        excl = np.concatenate([[0], np.cumsum(lane_tot)[:-1]]).tolist()
        first_bad = None
        Sprev = None
        for lane in range(LANES):
            for j in range(per):
                Sj = S + excl[lane] + lane_P[lane][j]
                a = abs(Sj)
                inr = lane_ok[lane][j] and TWO52 < a < TWO53 and ((Sj < 0) == (S < 0))
                if not inr:
                    first_bad = lane * per + j
                    Sprev = S + excl[lane] + (lane_P[lane][j - 1] if j > 0 else 0)
                    break
            if first_bad is not None:
                break
        if first_bad is None:
            f = LANES * per
            Sprev = S + excl[-1] + lane_tot[-1]
        else:
            f = first_bad
        if f > 0:
            s = float(Sprev) * u
            pos += f
        if pos < m and f < LANES * per:
            s = s + t[pos]
            pos += 1
        if f < 4:
            e = min(m, pos + 16)
            while pos < e:
                s = s + t[pos]
                pos += 1
    return s


def cases(rng, n):
    for _ in range(n):
        kind = rng.integers(0, 9)
        m = int(rng.integers(1, 1500))
        if kind == 0:
            t = rng.uniform(0, 1, m)  # positive: binade doublings
        elif kind == 1:
            t = rng.uniform(-1, 1, m)  # crosses zero
        elif kind == 2:
            t = rng.integers(-4, 5, m).astype(float) * 0.5  # ties everywhere
        elif kind == 3:
            t = rng.normal(0, 1, m) * np.exp2(rng.integers(-60, 60, m))  # wide range
        elif kind == 4:
            t = np.ones(m)  # integers
        elif kind == 5:
            t = rng.uniform(0, 1, m) * 1e-310  # subnormal terms
        elif kind == 6:
            t = rng.uniform(-1, 1, m)
            t[rng.integers(0, m)] = np.inf if rng.random() < 0.5 else np.nan
        elif kind == 7:
            base = rng.uniform(1, 2)
            t = np.concatenate([[base * 2.0 ** 50], rng.uniform(-3, 3, m - 1)])  # ulp ~ 0.25
        else:
            t = rng.uniform(-1, 1, m) * np.exp2(rng.integers(-1070, -1000))  # tiny sums
        s0 = float(rng.choice([0.0, -0.0, rng.normal(), 1e300, -5e-324]))
        yield s0, t.tolist()


def main(n=300):
    rng = np.random.default_rng(1)
    bad = 0
    for per in (1, 8, 12):
        for s0, t in cases(rng, n):
            a, b = serial(s0, t), model(s0, t, per)
            if not (bits(a) == bits(b) or (math.isnan(a) and math.isnan(b))):
                bad += 1
                print("MISMATCH", per, s0, len(t), a, b)
    print(f"{3 * n} cases, {bad} mismatches")
    return bad


if __name__ == "__main__":
    sys.exit(1 if main(int(sys.argv[1]) if len(sys.argv) > 1 else 300) else 0)
