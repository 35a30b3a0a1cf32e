"""Shared test helpers (random packed rows, brute-force set oracle)."""
import numpy as np


def pack_bits(bits_bool: np.ndarray) -> np.ndarray:
    """bool [n, L] -> int64 [n, K] in the reference layout (bitpack.cpp:25-26)."""
    n, L = bits_bool.shape
    k = (L + 63) // 64
    out = np.zeros((n, k), np.uint64)
    for j in range(L):
        out[:, j // 64] |= bits_bool[:, j].astype(np.uint64) << np.uint64(j % 64)
    return out.view(np.int64)


def random_rows(rng, n, L, density):
    return pack_bits(rng.random((n, L)) < density)


def to_sets(words: np.ndarray):
    out = []
    for row in words.view(np.uint64):
        s = []
        for w, x in enumerate(row.tolist()):
            while x:
                b = (x & -x).bit_length() - 1
                s.append(w * 64 + b)
                x &= x - 1
        out.append(frozenset(s))
    return out


def brute_force_fit(Xa_sets, Xn_sets):
    """SPEC.md:636 naive set-based oracle: B^c, f, S, P^c."""
    res = []
    for own, opp in ((Xa_sets, Xn_sets), (Xn_sets, Xa_sets)):
        B = set(x for x in own if x)
        for i in range(len(own)):
            for j in range(i + 1, len(own)):
                b = own[i] & own[j]
                if b:
                    B.add(b)
        sup = {b: sum(1 for x in own if b <= x) for b in B}
        sc = {b: sup[b] * len(b) ** 2 for b in B}
        pure = {b for b in B if not any(b <= x for x in opp)}
        res.append((B, sup, sc, pure))
    return res


def sets_to_sorted_words(sets, L):
    """Canonical words::less order (bitpack.hpp:59-68) of a collection of sets."""
    k = (L + 63) // 64
    rows = np.zeros((len(sets), k), np.uint64)
    for i, s in enumerate(sets):
        for b in s:
            rows[i, b // 64] |= np.uint64(1) << np.uint64(b % 64)
    if len(sets) == 0:
        return rows.view(np.int64)
    order = np.lexsort(rows.T[::-1])
    return rows[order].view(np.int64)
