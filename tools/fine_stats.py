"""Work census of the fine column-refinement stage (lcsg_tile.cu
column_refine_fine_kernel), emulated in numpy on oracle tables.

    python tools/fine_stats.py [n] [sigma]

For every wide combine of an n x n instance the final reach / trace tables
(C oracle) stand in for the rows the kernel reads as bounds; per fine cell
(rows not on the 8-row grid) this classifies the path the kernel takes and
the candidate-range length it evaluates.  Development tool (not a test).
"""

import os
import sys
from collections import Counter

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]

import oracle as O  # noqa: E402


def census(node, U, L, inf, S=8):
    R, T = node.reach, node.trace
    n1, w1 = R.shape
    Ur, Uk = U.reach, U.kmax
    wl = L.reach.shape[1] - 1
    out = Counter()
    lens = Counter()
    nblk = (n1 - 1 + S - 1) // S
    j = np.arange(w1)
    for blk in range(nblk):
        i0 = blk * S
        rb = min(S, n1 - 1 - i0)
        if rb < 2:
            continue
        top = R[i0]
        # warps of 32 columns whose top row is INF exit
        warp_inf = np.repeat([(top[w:w + 32] >= inf).all() for w in range(0, w1, 32)], 32)[:w1]
        out["cells_warp_exit"] += int(warp_inf.sum()) * (rb - 1)
        live = ~warp_inf
        for r in range(1, rb):
            dl = r & -r
            a, b = r - dl, min(r + dl, rb)
            c = i0 + r
            Ra, Rb = R[i0 + a], R[i0 + b]
            Ta, Tb = T[i0 + a], T[i0 + b]
            kmc = Uk[c]
            m_live = live
            out["cells_live"] += int(m_live.sum())
            fa = m_live & (Ra < inf)
            out["a_inf"] += int((m_live & ~fa).sum())
            fb = fa & (Rb < inf)
            tail = fa & ~fb
            out["tail"] += int(tail.sum())
            # tail range [kl, min(j, kmc)]
            Xa = Ur[i0 + a, np.minimum(Ta, Ur.shape[1] - 1)]
            hi = np.minimum(Ta, kmc)
            lo = np.minimum(np.maximum(0, Ta - dl), hi)
            # first k in [lo, hi] with U[c,k] >= Xa
            Uc = Ur[c]
            kl = lo.copy()
            for t in range(dl):
                k1 = lo + t
                kk = np.minimum(k1, Ur.shape[1] - 1)
                kl += ((k1 < hi) & (Uc[kk] < Xa)).astype(kl.dtype)
            kl = np.maximum(kl, j - wl)
            tl = np.maximum(0, np.minimum(j, kmc) - kl + 1)
            out["tail_cands"] += int(tl[tail].sum())
            Xb = Ur[i0 + b, np.minimum(Tb, Ur.shape[1] - 1)]
            lo2, hi2 = np.minimum(Tb, kmc), np.minimum(Tb + dl, kmc)
            kh = lo2.copy()
            for t in range(dl):
                k2 = lo2 + 1 + t
                kk = np.minimum(k2, Ur.shape[1] - 1)
                kh += ((k2 <= hi2) & (Uc[kk] <= Xb)).astype(kh.dtype)
            kh = np.minimum(kh, j)
            ln = kh - kl + 1
            sel = fb
            longr = sel & (ln - 1 >= 12)
            pinned = sel & (ln == 1) & (Xa == Xb)
            inl = sel & ~longr & ~pinned
            out["long"] += int(longr.sum())
            out["long_cands"] += int(ln[longr].sum())
            out["pinned"] += int(pinned.sum())
            out["pin_eqT"] += int((fb & (Xa == Xb) & (Ta == Tb)).sum())
            out["pin_Tdiff1"] += int((fb & (Xa == Xb) & (Ta == Tb + 1)).sum())
            out["xa_eq_xb"] += int((fb & (Xa == Xb)).sum())
            out["inline"] += int(inl.sum())
            out["inline_cands"] += int(ln[inl].sum())
            out[f"dl{dl}_fin"] += int(fb.sum())
            for v, cnt in zip(*np.unique(np.clip(ln[inl], 0, 13), return_counts=True)):
                lens[int(v)] += int(cnt)
    return out, lens


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
    sigma = int(sys.argv[2]) if len(sys.argv) > 2 else 26
    rng = np.random.default_rng(0)
    a = (rng.integers(0, sigma, n) + 97).astype(np.uint8).tobytes()
    b = (rng.integers(0, sigma, n) + 97).astype(np.uint8).tobytes()
    t = O.OracleTree(a, b, threads=8)
    inf = n + 2
    by_level = {}
    for idx in range(len(t)):
        nd = t.node(idx)
        if nd.upper < 0 or nd.reach.shape[1] <= 65:
            continue
        s = nd.bottom_row - nd.top_row
        out, lens = census(nd, t.node(nd.upper), t.node(nd.lower), inf)
        lv = by_level.setdefault(s, [Counter(), Counter()])
        lv[0].update(out)
        lv[1].update(lens)
    for s in sorted(by_level):
        out, lens = by_level[s]
        tot = out["cells_warp_exit"] + out["cells_live"]
        print(f"s={s}: cells {tot}  warp-exit {out['cells_warp_exit'] / tot:.2f}  "
              f"a-INF {out['a_inf'] / tot:.2f}  tail {out['tail'] / tot:.3f} "
              f"(cands/cell {out['tail_cands'] / max(1, out['tail']):.1f})  "
              f"long {out['long'] / tot:.3f} (cands {out['long_cands'] / max(1, out['long']):.1f})  "
              f"pinned {out['pinned'] / tot:.2f} (Xa=Xb {out['xa_eq_xb'] / tot:.3f}, T equal "
              f"{out['pin_eqT'] / tot:.3f}, T diff 1 {out['pin_Tdiff1'] / tot:.3f})  "
              f"inline {out['inline'] / tot:.2f} "
              f"(cands {out['inline_cands'] / max(1, out['inline']):.2f})")
        print("   inline range lengths:", dict(sorted(lens.items())))


if __name__ == "__main__":
    main()
