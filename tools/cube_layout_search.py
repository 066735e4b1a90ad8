"""Offline search of the shared-cube strides of the order-generic kernel (ax_fastn.cu).

For each n1 with EPB elements per CTA, count the shared-memory wavefronts of the
three fibre access patterns (k-fibre, i-row, j-column) over every warp of the
CTA -- 64-bit accesses, served per half-warp, one wavefront per distinct
address in the busiest bank pair -- for the padded strides PJ (j), PK (k) and
the element-to-element cube stride CS, and report the best.

    python tools/cube_layout_search.py [--n1 2,3,4,5,6,7]
"""
import argparse
import itertools

import numpy as np

EPB = {2: 16, 3: 7, 4: 4, 5: 5, 6: 3, 7: 5}
CUR_PJ = {6: 9, 8: 9, 10: 17, 12: 13, 14: 17, 16: 17}
CUR_PK = {2: 5, 3: 18, 4: 19, 6: 54, 7: 52, 8: 72, 10: 170, 12: 156, 14: 238, 16: 272}
CUR_CS = {2: 12, 3: 57, 5: 137, 6: 324, 7: 369}


def cost(n1, epb, pj, pk, cs):
    T = n1 * n1
    nt = T * epb
    tid = np.arange(((nt + 31) // 32) * 32)
    active = tid < nt
    le = np.minimum(tid // T, epb - 1)
    t = tid - le * T
    fi, fj = t % n1, t // n1
    base = le * cs
    kp = fj * pj + fi
    rb = fj * pk + fi * pj
    cb = fj * pk + fi
    total = 0
    # per element the kernel issues 7 n1 k-fibre, 4 n1 i-row and 4 n1 j-column accesses
    for n in range(n1):
        for addr, w in ((base + n * pk + kp, 7), (base + rb + n, 4), (base + cb + n * pj, 4)):
            a = np.where(active, addr, -1)
            for h in range(0, len(a), 16):
                seg = a[h:h + 16]
                seg = np.unique(seg[seg >= 0])
                if len(seg) == 0:
                    continue
                total += w * np.bincount(seg % 16, minlength=16).max()
    return total


def ideal(n1, epb):
    T = n1 * n1
    nt = T * epb
    halves = 0
    for h in range(0, ((nt + 31) // 32) * 32, 16):
        if h < nt:
            halves += 1
    return halves * 15 * n1


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n1", default="2,3,4,5,6,7")
    args = ap.parse_args()
    for n1 in (int(v) for v in args.n1.split(",")):
        epb = EPB[n1]
        pj0 = CUR_PJ.get(n1, n1)
        pk0 = CUR_PK.get(n1, n1 * n1)
        cube0 = max(CUR_CS.get(n1, 0), (n1 - 1) * pk0 + (n1 - 1) * pj0 + n1)
        cur = cost(n1, epb, pj0, pk0, cube0)
        best = None
        for pj in range(n1, n1 + 17):
            for pk in range(n1 * pj, n1 * pj + 33):
                cube = (n1 - 1) * pk + (n1 - 1) * pj + n1
                for cs in range(cube, cube + 33):
                    c = cost(n1, epb, pj, pk, cs)
                    if best is None or c < best[0] or (c == best[0] and cs * 3 < best[3] * 3):
                        best = (c, pj, pk, cs)
        print(f"n1={n1} EPB={epb}: current PJ={pj0} PK={pk0} CS={cube0} -> {cur} wavefronts; "
              f"best PJ={best[1]} PK={best[2]} CS={best[3]} -> {best[0]} (ideal {ideal(n1, epb)})", flush=True)


if __name__ == "__main__":
    main()
