#!/usr/bin/env python3
"""Shared-memory bank-conflict model for phase A's element arrays (index i + R j + P k):
counts wavefronts of the r-pencil vector accesses and the s/t-pencil scalar accesses of one
element group and searches the row pitch R, plane pitch P and t-pencil mapping (TT) that
minimise them.  python tools/smem_layout.py"""
import itertools


def vecw(sT, N):
    if sT == 4:
        return 4 if N % 4 == 0 else (2 if N % 2 == 0 else 1)
    return 2 if N % 2 == 0 else 1


def wavefronts(accs):
    """accs: list of (thread, byte_addr, nbytes) of one warp instruction -> wavefronts."""
    if not accs:
        return 0
    size = accs[0][2]
    per_phase = max(1, 128 // size)
    accs = sorted(accs)
    total = 0
    for p0 in range(0, 32, per_phase):
        banks = {}
        for t, addr, nb in accs:
            if p0 <= t < p0 + per_phase:
                for w in range(addr // 4, (addr + nb) // 4):
                    banks.setdefault(w % 32, set()).add(w)
        if banks:
            total += max(len(v) for v in banks.values())
    return total


def cost(sT, N, R, P, TT, EPB):
    V = vecw(sT, N)
    ESZ = P * N
    N2 = N * N
    nt = ((EPB * N2 + 31) // 32) * 32
    c_r = c_s = c_t = 0
    for w in range(nt // 32):
        th = [q for q in range(32 * w, 32 * w + 32) if q < EPB * N2]
        def geo(q):
            el, qq = divmod(q, N2)
            return el * 3 * ESZ, qq % N, qq // N
        # r-pencil: N/V vector instructions
        for c in range(N // V):
            acc = []
            for q in th:
                base, a, b = geo(q)
                acc.append((q - 32 * w, (base + R * a + P * b + c * V) * sT, V * sT))
            c_r += wavefronts(acc)
        for j in range(N):
            acc = []
            for q in th:
                base, a, b = geo(q)
                acc.append((q - 32 * w, (base + a + R * j + P * b) * sT, sT))
            c_s += wavefronts(acc)
        for k in range(N):
            acc = []
            for q in th:
                base, a, b = geo(q)
                i, jj = (b, a) if TT else (a, b)
                acc.append((q - 32 * w, (base + i + R * jj + P * k) * sT, sT))
            c_t += wavefronts(acc)
    # per element group: 9 r-pencil passes (all chunks), 4 s-pencil and 4 t-pencil passes
    return 9 * c_r + 4 * c_s + 4 * c_t, (c_r, c_s, c_t)


def current(sT, N):
    banks = 32 if sT == 4 else 16
    N2 = N * N
    return N, N2 + ((N - N2) % banks + banks) % banks, False


if __name__ == "__main__":
    for sT in (4, 8):
        for N in (8, 10, 12):
            EPB = 1 if N * N >= 256 else 256 // (N * N)
            V = vecw(sT, N)
            R0, P0, T0 = current(sT, N)
            base = cost(sT, N, R0, P0, T0, EPB)
            best = (base[0], R0, P0, T0, base[1])
            for R in range(N, N + 17):
                if R % V:
                    continue
                for P in range(R * N, R * N + 65):
                    if P % V:
                        continue
                    for TT in (False, True):
                        cst, parts = cost(sT, N, R, P, TT, EPB)
                        if cst < best[0]:
                            best = (cst, R, P, TT, parts)
            print(f"sT={sT} N={N:2d} EPB={EPB}: current R={R0} P={P0} cost={base[0]} {base[1]}  ->  "
                  f"best R={best[1]} P={best[2]} TT={best[3]} cost={best[0]} {best[4]}")
