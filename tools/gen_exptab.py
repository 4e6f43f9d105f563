"""Table and reduction constants for the Gaussian-bump exponential of the
Dirichlet walkers (fm::exp_bump in paper_1808_10580_b200/csrc/fastmath.cuh):
T[j] = 2^(j/256) correctly rounded (mpmath, 60 digits), j = 0..255, and the
hi/lo split of ln2/256.

    python tools/gen_exptab.py > /tmp/exptab.txt   (pasted into fastmath.cuh)
"""
import mpmath as mp

mp.mp.dps = 60
vals = [float(mp.mpf(2) ** (mp.mpf(j) / 256)) for j in range(256)]
c = mp.log(2) / 256
c_hi = float(c)
c_lo = float(c - mp.mpf(c_hi))
inv = float(256 / mp.log(2))
print(f"#define SMC_FM_EXPB {inv!r}, {c_hi!r}, {c_lo!r}")
print("#define SMC_FM_EXPTAB \\")
rows = [", ".join(repr(v) for v in vals[i:i + 4]) for i in range(0, 256, 4)]
print(", \\\n".join(f"    {r}" for r in rows))
