"""Pure-Python big-integer references used to PIN the oracle (not the oracle
itself, and not the product).  Everything here is the textbook definition
written out with Python integers, for tiny N only."""
from __future__ import annotations


def is_prime(n: int) -> bool:
    if n < 2:
        return False
    small = [2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37, 41, 43, 47]
    for p in small:
        if n % p == 0:
            return n == p
    d, s = n - 1, 0
    while d % 2 == 0:
        d //= 2
        s += 1
    for a in small:  # 15 bases: deterministic far beyond 2^64
        x = pow(a, d, n)
        if x in (1, n - 1):
            continue
        for _ in range(s - 1):
            x = x * x % n
            if x == n - 1:
                break
        else:
            return False
    return True


def brv(x: int, bits: int) -> int:
    return int(format(x, f"0{bits}b")[::-1], 2) if bits else 0


def ntt_def(a, q, psi, log_n):
    """C3: ntt(a)_i = sum_j a_j psi^((2 brv(i) + 1) j) mod q."""
    n = 1 << log_n
    return [sum(a[j] * pow(psi, (2 * brv(i, log_n) + 1) * j, q) for j in range(n)) % q for i in range(n)]


def intt_def(ah, q, psi, log_n):
    n = 1 << log_n
    ipsi = pow(psi, -1, q)
    ninv = pow(n, -1, q)
    # a_j = N^{-1} sum_i ah_i psi^{-(2 brv(i)+1) j}
    return [ninv * sum(ah[i] * pow(ipsi, (2 * brv(i, log_n) + 1) * j, q) for i in range(n)) % q for j in range(n)]


def negacyclic_mul(a, b, mod=None):
    n = len(a)
    c = [0] * n
    for i in range(n):
        for j in range(n):
            k = i + j
            if k < n:
                c[k] += a[i] * b[j]
            else:
                c[k - n] -= a[i] * b[j]
    if mod is not None:
        c = [x % mod for x in c]
    return c


def crt(residues, primes):
    """integer in [0, prod) with the given residues"""
    Q = 1
    for p in primes:
        Q *= p
    x = 0
    for r, p in zip(residues, primes):
        Qi = Q // p
        x += int(r) * Qi * pow(Qi % p, -1, p)
    return x % Q, Q


def centred(x, Q):
    return x - Q if x > Q // 2 else x
