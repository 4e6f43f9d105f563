"""Near-minimax polynomial coefficients for the device math in
paper_1808_10580_b200/csrc/fastmath.cuh (Chebyshev-node least squares in
60-digit mpmath arithmetic; the fitted polynomials are then printed as C
double literals).

    python tools/gen_minimax.py > /tmp/coef.txt
"""
import mpmath as mp

mp.mp.dps = 60


def fit(f, deg, a, b, n=400, weight=None):
    """Least squares on Chebyshev nodes of [a, b] for sum_k c_k t^k, t in [a,b]."""
    nodes = [mp.mpf(a + b) / 2 + mp.mpf(b - a) / 2 * mp.cos(mp.pi * (2 * i + 1) / (2 * n)) for i in range(n)]
    A = mp.matrix(n, deg + 1)
    y = mp.matrix(n, 1)
    for i, t in enumerate(nodes):
        w = weight(t) if weight else 1
        for k in range(deg + 1):
            A[i, k] = t ** k * w
        y[i] = f(t) * w
    c = mp.lu_solve(A.T * A, A.T * y)
    err = max(abs(sum(c[k] * t ** k for k in range(deg + 1)) - f(t)) * (weight(t) if weight else 1) for t in nodes)
    return [c[k] for k in range(deg + 1)], err


# sin(pi r) = r * S(r^2),  cos(pi r) = C(r^2),  r in [-1/4, 1/4]  ->  z = r^2 in [0, 1/16]
S, es = fit(lambda z: mp.sin(mp.pi * mp.sqrt(z)) / mp.sqrt(z) if z > 0 else mp.pi, 7, mp.mpf(0), mp.mpf(1) / 16,
            weight=lambda z: 1 / mp.pi)
C, ec = fit(lambda z: mp.cos(mp.pi * mp.sqrt(z)), 7, mp.mpf(0), mp.mpf(1) / 16)
# log1p via s = f / (2 + f): log(1+f) = 2 s + s^3 R(s^2), s in [-0.1716, 0.1716] -> w = s^2 in [0, 0.02944]
smax = (mp.sqrt(2) - 1) / (mp.sqrt(2) + 1)
R, el = fit(lambda w: (2 * mp.atanh(mp.sqrt(w)) - 2 * mp.sqrt(w)) / (w * mp.sqrt(w)) if w > 0 else mp.mpf(2) / 3, 7,
            mp.mpf(0), smax ** 2)
for name, c, e in (("SINPI", S, es), ("COSPI", C, ec), ("LOG_R", R, el)):
    print(f"// {name}: max abs err {mp.nstr(e, 3)}")
    print(", ".join(repr(float(x)) for x in c))

if __name__ == "__main__":
    import sys
    for deg in (5, 6, 7):
        _, e1 = fit(lambda z: mp.sin(mp.pi * mp.sqrt(z)) / mp.sqrt(z) if z > 0 else mp.pi, deg, mp.mpf(0), mp.mpf(1) / 16,
                    weight=lambda z: 1 / mp.pi)
        _, e2 = fit(lambda z: mp.cos(mp.pi * mp.sqrt(z)), deg, mp.mpf(0), mp.mpf(1) / 16)
        _, e3 = fit(lambda w: (2 * mp.atanh(mp.sqrt(w)) - 2 * mp.sqrt(w)) / (w * mp.sqrt(w)) if w > 0 else mp.mpf(2) / 3,
                    deg, mp.mpf(0), smax ** 2)
        print(deg, mp.nstr(e1, 3), mp.nstr(e2, 3), mp.nstr(e3, 3), file=sys.stderr)
