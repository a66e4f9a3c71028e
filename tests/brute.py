"""Pure-Python brute force written directly from Eq.1 for tiny inputs -- independent of oracle/.

L_I = -(1/b) sum_i log( e^{x_ii} / sum_j e^{x_ij} ),  L_T the same with rows and columns swapped,
L = (L_I + L_T)/2 (reading Q4).  Sums use math.fsum, exponentials are max-shifted per row (Eq.5's
stabilisation, which does not change the value).  Gradients by central finite differences of this loss.
"""
import math


def dot(u, v):
    return math.fsum(a * b for a, b in zip(u, v))


def loss(I, T, s):
    b = len(I)
    x = [[s * dot(I[i], T[j]) for j in range(b)] for i in range(b)]

    def nll(row, k):
        m = max(row)
        return -(row[k] - (m + math.log(math.fsum(math.exp(v - m) for v in row))))

    L_I = math.fsum(nll(x[i], i) for i in range(b)) / b
    L_T = math.fsum(nll([x[i][j] for i in range(b)], j) for j in range(b)) / b
    return 0.5 * (L_I + L_T)


def fd_grads(I, T, s, h=1e-6):
    I = [list(map(float, r)) for r in I]
    T = [list(map(float, r)) for r in T]
    dI = [[0.0] * len(I[0]) for _ in I]
    dT = [[0.0] * len(T[0]) for _ in T]
    for M, D in ((I, dI), (T, dT)):
        for i in range(len(M)):
            for k in range(len(M[0])):
                v = M[i][k]
                M[i][k] = v + h
                lp = loss(I, T, s)
                M[i][k] = v - h
                lm = loss(I, T, s)
                M[i][k] = v
                D[i][k] = (lp - lm) / (2 * h)
    return dI, dT


def ntxent_loss(A, B, s):
    """NT-Xent written from its definition (SimCLR; oracle/ntxent.py readings N1-N3) with Python loops: views
    z = A + B (2b), each view's positive is the other view of its example, its own similarity is excluded."""
    z = [list(r) for r in A] + [list(r) for r in B]
    n = len(z)
    b = n // 2
    tot = []
    for k in range(n):
        row = [s * dot(z[k], z[j]) for j in range(n) if j != k]
        m = max(row)
        lse = m + math.log(math.fsum(math.exp(v - m) for v in row))
        tot.append(lse - s * dot(z[k], z[(k + b) % n]))
    return math.fsum(tot) / n


def ntxent_fd_grads(A, B, s, h=1e-6):
    A = [list(map(float, r)) for r in A]
    B = [list(map(float, r)) for r in B]
    out = []
    for M in (A, B):
        D = [[0.0] * len(M[0]) for _ in M]
        for i in range(len(M)):
            for k in range(len(M[0])):
                v = M[i][k]
                M[i][k] = v + h
                lp = ntxent_loss(A, B, s)
                M[i][k] = v - h
                lm = ntxent_loss(A, B, s)
                M[i][k] = v
                D[i][k] = (lp - lm) / (2 * h)
        out.append(D)
    return out
