"""Table for the table-driven FP64 exp of the Dirichlet walkers' forcing bumps
(fm::exp_tab in paper_1808_10580_b200/csrc/fastmath.cuh): 2^(j/64) for
j = 0..63 as hi + lo (hi the double nearest, lo the double nearest the
remainder; 60-digit mpmath), and the reduction constants 64/ln2 and
ln2/64 split Cody-Waite style (hi with its low 32 bits zero, so n * hi is
exact for |n| < 2^21).

    python tools/gen_exptab.py > /tmp/exptab.txt   (pasted into fastmath.cuh)
"""
import struct

import mpmath as mp

mp.mp.dps = 60
rows = []
for j in range(64):
    v = mp.power(2, mp.mpf(j) / 64)
    hi = float(v)
    lo = float(v - mp.mpf(hi))
    rows.append((hi, lo))
c = mp.log(2) / 64
hi = float(c)
b = struct.unpack("<Q", struct.pack("<d", hi))[0] & ~((1 << 32) - 1)
hi = struct.unpack("<d", struct.pack("<Q", b))[0]
lo = float(c - mp.mpf(hi))
print(f"#define SMC_FM_EXPTK {float(64 / mp.log(2))!r}, {hi!r}, {lo!r}")
print("#define SMC_FM_EXPTAB \\")
print(", \\\n".join(f"    {h!r}, {l!r}" for h, l in rows))
