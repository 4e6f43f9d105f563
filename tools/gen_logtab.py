"""Table for the FP64 log of the particle kernels (fm::log_u in
paper_1808_10580_b200/csrc/fastmath.cuh): 128 entries indexed by the top 7
mantissa bits of x.  Entry i covers m in [1 + i/128, 1 + (i+1)/128):
  inv   = 1/c rounded to double, c the bin centre  (r = fma(m, inv, -1), |r| < 2^-7)
  adj   = 1 for bins at or above sqrt(2) (m is treated as m/2, exponent + 1, so
          x near 1 from below has exponent 0 and no cancellation against ln 2)
  t_hi + t_lo = -log(inv * 2^adj) in 106-bit precision (mpmath, 60 digits)
so log(x) = (e + adj) ln2 + t + log1p(r).

    python tools/gen_logtab.py > /tmp/logtab.txt   (pasted into fastmath.cuh)
"""
import mpmath as mp

mp.mp.dps = 60
rows = []
split = None
for i in range(128):
    c = 1 + (mp.mpf(i) + mp.mpf(1) / 2) / 128
    inv = float(1 / c)
    lo = 1 + mp.mpf(i) / 128
    adj = 1 if lo >= mp.mpf(181) / 128 else 0  # bins from 1.4140625 (the one holding sqrt 2) up
    # the two bins containing 1 (after halving) use c = 1 exactly: r = m - 1 is
    # then exact (Sterbenz) and log1p(r) is the whole result, so x -> 1 keeps
    # full relative accuracy (no cancellation between t and log1p(r))
    if i == 0:
        inv = 1.0
    if i == 127:
        inv = 0.5
    if adj and split is None:
        split = i
    t = -mp.log(mp.mpf(inv) * 2 ** adj)
    t_hi = float(t)
    t_lo = float(t - mp.mpf(t_hi))
    rows.append((inv, float(adj), t_hi, t_lo))
print(f"// first halved bin: {split}")
print("#define SMC_FM_LOGTAB \\")
print(", \\\n".join(f"    {r[0]!r}, {r[1]!r}, {r[2]!r}, {r[3]!r}" for r in rows))
