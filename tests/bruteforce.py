"""Independent exact-rational implementation of Alg. 1 for
tiny shapes, written from the definitions with Python ``fractions.Fraction``.
Shares no code with oracle/ or the CUDA path; used only to pin the oracle."""
from fractions import Fraction


def exact_infer(X, B, C):
    N, F = len(X), len(X[0])
    D = len(B[0])
    K = len(C)
    Xq = [[Fraction(float(v)) for v in row] for row in X]
    Bq = [[Fraction(float(v)) for v in row] for row in B]
    Cq = [[Fraction(float(v)) for v in row] for row in C]
    V, H, S, y = [], [], [], []
    for n in range(N):
        v = [sum((Xq[n][f] * Bq[f][d] for f in range(F)), Fraction(0)) for d in range(D)]
        h = [1 if vd >= 0 else -1 for vd in v]            # eq. hardsign
        s = [sum((h[d] * Cq[k][d] for d in range(D)), Fraction(0)) for k in range(K)]
        best = 0
        for k in range(1, K):                              # lowest index wins ties
            if s[k] > s[best]:
                best = k
        V.append(v)
        H.append(h)
        S.append(s)
        y.append(best)
    return V, H, S, y
