"""Offline search of shared-cube layouts with free row / column roles (ax_fastn.cu).

The order-generic kernel moves each element cube between three fibre
ownerships through shared memory: k-fibres (thread (fi, fj) of element le, the
node stage and the global loads / stores), i-rows and j-columns.  Only the
k-fibre role is tied to the thread (global coalescing, the factors); an i-row or
j-column task of ANY element of the CTA can run on any thread, because the row
and column phases only read and write shared memory between barriers.  A row
access is base + n and a column access base + n PJ (n the compile-time fibre
index), so a half-warp is conflict-free iff the 16 bases are distinct modulo 16
(64-bit accesses, 16 bank pairs, served per half-warp).  For strides (PJ, PK,
CS) this tool

  * counts the k-fibre wavefronts of the natural thread order, and
  * assigns row and column tasks to threads by a max-flow (residue class ->
    half-warp, one task per (class, half-warp)); a full flow means every row /
    column access is one wavefront per half-warp,

and reports, per n1, the cheapest layout and the tables the kernel loads
(packed 16-bit row base | column base << 16 per thread).

    python tools/role_search.py [--n1 2,3,4,5,6,7] [--emit]
"""
import argparse

import numpy as np
from scipy.sparse import csr_matrix
from scipy.sparse.csgraph import maximum_flow

# elements per CTA (ax_fastn.cu epb_of; 1 above), except n1 = 3: 10 (90 threads in 3
# warps) has a conflict-free layout, 7 does not.  n1 = 7 keeps 5 (245 threads, 8 warps)
# with a greedy dealing (5 extra wavefronts per row + column pair over 16 half-warps),
# measured better than the conflict-free 4-element packing (196 threads in 7 warps)
EPB = {2: 16, 3: 10, 4: 4, 5: 5, 6: 3, 7: 5}


def half_warps(nt):
    return [(h, min(h + 16, nt)) for h in range(0, nt, 16)]


def kfibre_cost(n1, epb, pj, pk, cs):
    """wavefronts of one k-fibre access instruction summed over the CTA's half-warps"""
    nt = n1 * n1 * epb
    tid = np.arange(nt)
    le, t = tid // (n1 * n1), tid % (n1 * n1)
    base = le * cs + (t // n1) * pj + (t % n1)
    return sum(np.bincount(np.unique(base[a:b]) % 16, minlength=16).max() for a, b in half_warps(nt))


def assign(bases, nt):
    """tasks (their bases) -> threads with distinct residues per half-warp; None if impossible.

    The CTA is launched with whole warps (nt rounded up to 32): lanes past the
    k-fibre threads exist anyway and take row / column tasks, and any lane may
    stay idle (-1) in a phase."""
    hws = half_warps(nt)
    nh = len(hws)
    res = bases % 16
    # nodes: 0 source, 1..16 classes, 17..16+nh half-warps, 17+nh sink
    src, sink = 0, 17 + nh
    rows, cols, caps = [], [], []
    for c in range(16):
        m = int((res == c).sum())
        if m:
            rows.append(src); cols.append(1 + c); caps.append(m)
            for h in range(nh):
                rows.append(1 + c); cols.append(17 + h); caps.append(1)
    for h, (a, b) in enumerate(hws):
        rows.append(17 + h); cols.append(sink); caps.append(16)
    g = csr_matrix((np.array(caps, dtype=np.int32), (rows, cols)), shape=(sink + 1, sink + 1))
    f = maximum_flow(g, src, sink)
    if f.flow_value != len(bases):
        return None
    flow = f.flow.toarray()
    pools = {c: list(np.flatnonzero(res == c)) for c in range(16)}
    out = np.full(nt, -1, dtype=np.int64)
    for h, (a, b) in enumerate(hws):
        slot = a
        for c in range(16):
            if flow[1 + c, 17 + h] > 0:
                out[slot] = bases[pools[c].pop()]
                slot += 1
        assert slot <= b
    return out


def assign_greedy(bases, nt):
    """fallback when no conflict-free dealing exists: tasks (most frequent residue class
    first) to the half-warp holding the fewest of their class; returns (wavefronts per
    access instruction summed over half-warps, bases per thread)"""
    hws = half_warps(nt)
    nh = len(hws)
    res = bases % 16
    cnt = np.zeros((nh, 16), dtype=np.int64)
    slots = [[] for _ in range(nh)]
    for q in np.argsort(-np.bincount(res, minlength=16)[res], kind="stable"):
        h = min((cnt[h, res[q]], len(slots[h]), h) for h in range(nh) if len(slots[h]) < 16)[2]
        cnt[h, res[q]] += 1
        slots[h].append(q)
    out = np.full(nt, -1, dtype=np.int64)
    for h, (a, b) in enumerate(hws):
        for i, q in enumerate(slots[h]):
            out[a + i] = bases[q]
    return int(cnt.max(axis=1).sum()), out


def layout(n1, epb, pj, pk, cs):
    nt = n1 * n1 * epb
    le = np.repeat(np.arange(epb), n1 * n1)
    a = np.tile(np.arange(n1 * n1), epb)
    lo, hi = a % n1, a // n1
    rows = le * cs + hi * pk + lo * pj          # row task (le, j=lo, k=hi): base of (0, j, k)
    cols = le * cs + hi * pk + lo               # column task (le, i=lo, k=hi): base of (i, 0, k)
    return nt, rows, cols


def padded(n1, epb):
    return (n1 * n1 * epb + 31) // 32 * 32


def search(n1, epb):
    """cheapest (PJ, PK, CS): conflict-free if a flow exists, else the fewest wavefronts
    with greedily dealt rows / columns; ties to the smaller cubes"""
    best = None
    nhk = len(half_warps(n1 * n1 * epb))
    nh = padded(n1, epb) // 16
    for pj in range(n1, n1 + 17):
        for pk in range(n1 * pj, n1 * pj + 33):
            cube = (n1 - 1) * pk + (n1 - 1) * pj + n1
            for cs in (range(cube, cube + 33) if epb > 1 else (cube,)):
                if kfibre_cost(n1, epb, pj, pk, cs) != nhk:
                    continue
                nt, rows, cols = layout(n1, epb, pj, pk, cs)
                nt = padded(n1, epb)
                r = c = None
                if max(np.bincount(rows % 16).max(), np.bincount(cols % 16).max()) <= nh:
                    r, c = assign(rows, nt), assign(cols, nt)
                cr, cc = nhk, nhk
                if r is None:
                    cr, r = assign_greedy(rows, nt)
                if c is None:
                    cc, c = assign_greedy(cols, nt)
                key = (cr + cc, 3 * epb * cs)
                if best is None or key < best[0]:
                    best = (key, pj, pk, cs, r, c)
        if best is not None and best[0][0] == 2 * nhk:
            break
    if best is None:
        return None
    (cost, size), pj, pk, cs, r, c = best
    return size, pj, pk, cs, r, c, cost - 2 * nhk


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n1", default="2,3,4,5,6,7")
    ap.add_argument("--emit", action="store_true", help="print the C tables")
    ap.add_argument("--header", help="write the tables as a CUDA header (csrc/fastn_roles.cuh)")
    args = ap.parse_args()
    blocks = []
    for n1 in (int(v) for v in args.n1.split(",")):
        epb = EPB.get(n1, 1)
        best = search(n1, epb)
        if best is None:
            print(f"n1={n1} EPB={epb}: no conflict-free layout in the search range")
            continue
        size, pj, pk, cs, r, c, extra = best
        print(f"n1={n1} EPB={epb}: PJ={pj} PK={pk} CS={cs} ({size * 8} B of cubes) "
              + ("conflict-free" if extra == 0 else f"{extra} extra wavefront(s) per row+column access pair"),
              flush=True)
        assert max(r.max(), c.max()) < 0xffff
        packed = [(int(a) & 0xffff) | ((int(b) & 0xffff) << 16) for a, b in zip(r, c)]  # 0xffff: no task
        if args.emit:
            print(f"  // n1={n1}: row base | column base << 16 per thread")
            print("  " + ", ".join(str(v) for v in packed))
        body = ",\n".join("    " + ", ".join(str(v) for v in packed[q:q + 8]) for q in range(0, len(packed), 8))
        blocks.append(f"#elif HX_N1 == {n1}\n"
                      f"#define HX_ROLES 1\n"
                      f"constexpr int kRolePJ = {pj}, kRolePK = {pk}, kRoleCS = {cs}, kRoleEPB = {epb};\n"
                      f"static __device__ const unsigned c_roles[{len(packed)}] = {{\n{body}}};\n")
    if args.header:
        with open(args.header, "w") as f:
            f.write("// Generated by tools/role_search.py -- do not edit.\n"
                    "// Conflict-free shared-cube layouts of the order-generic kernel with free\n"
                    "// i-row / j-column roles: per thread, the absolute base of its row task\n"
                    "// (low 16 bits) and column task (high 16 bits) in the CTA's cube arrays.\n"
                    "#pragma once\n"
                    "#if defined(HX_NO_ROLES)  // A/B builds (tools/build_variant.sh)\n"
                    "#define HX_ROLES 0\n"
                    "constexpr int kRolePJ = 0, kRolePK = 0, kRoleCS = 0, kRoleEPB = 0;\n")
            f.write("".join(blocks))
            f.write("#else\n#define HX_ROLES 0\n"
                    "constexpr int kRolePJ = 0, kRolePK = 0, kRoleCS = 0, kRoleEPB = 0;\n#endif\n")


if __name__ == "__main__":
    main()
