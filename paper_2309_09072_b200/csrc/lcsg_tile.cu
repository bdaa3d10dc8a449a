// lcsg_tile.cu -- column-parallel refinement of the wide combines (the fast path).
//
// After the skeleton rows i = 0, S, 2S, ..., n of a combine are known (exact
// Alg. 1, lcsg_refine.cu), every interior row is derived by refinement:
// X(c,j) = U[c, k*(c,j)] is monotone in the start row c (Monge argmin), so
// k*(c,j) lies between bounds read off rows c-delta and c+delta AT THE SAME
// COLUMN j.  Column tiles are therefore independent: one CTA owns a block of
// S+1 consecutive rows (two skeleton rows bracketing S-1 interior rows) times
// TJ columns, keeps the block's (reach, trace) in shared memory, stages the
// window of U rows the block can touch once, and runs all log2(S) refinement
// passes with only the L gathers going to L2/HBM.  Finite cells are written
// once, coalesced; the per-row finalize kernel then writes the INF suffix
// (replaying Alg. 1 for the reference's INF-cell traces) and kmax / wstar.
//
// Cells finite in row a but INF in row b (at most 2*delta per row and pass)
// have no upper bound; they are queued and scanned warp-cooperatively over
// [lower bound, min(j, kmax_c)].
#include <climits>

#include "lcsg_internal.cuh"

namespace lcsg {

#define LCSG_LAUNCH_CHECK()                         \
    do {                                            \
        cudaError_t e__ = cudaGetLastError();       \
        if (e__ != cudaSuccess) return (int)e__;    \
    } while (0)

constexpr int BT_THREADS = 256;
constexpr int BT_MAXS = 64;
constexpr int BT_TAILCAP = 512;
constexpr int FN_SEGS = 40;
constexpr int FN_WARPS = 8;

template <typename Key>
__device__ __forceinline__ Key tpack(int32_t v, int32_t k, int shift) {
    return ((Key)(uint32_t)v << shift) | (Key)(uint32_t)k;
}
template <typename Key>
__device__ __forceinline__ int32_t tval(Key key, int shift) { return (int32_t)(key >> shift); }
template <typename Key>
__device__ __forceinline__ int32_t tk(Key key, int shift) {
    return (int32_t)(key & (((Key)1 << shift) - 1));
}
__device__ __forceinline__ uint32_t twarp_min(uint32_t v) { return __reduce_min_sync(0xffffffffu, v); }
__device__ __forceinline__ uint64_t twarp_min(uint64_t v) {
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
        uint64_t o = __shfl_xor_sync(0xffffffffu, v, d);
        v = o < v ? o : v;
    }
    return v;
}

// cell_value (_kernel.pyx:14-25) with x = U[i,k] already loaded.
__device__ __forceinline__ int32_t tcell(const TabAcc &L, int32_t x, int32_t k, int32_t j,
                                         int32_t inf, int32_t wl) {
    if (k > j || x >= inf || j - k > wl) return inf;
    return tab_get(L, (int64_t)x - 1, j - k);
}

// One lane = one column j of one row block [i0, i0+S]: the block's two
// skeleton cells of column j are loaded, then the S-1 interior cells are
// derived in divide-and-conquer order (delta = S/2 ... 1), all in registers
// (the unrolled passes index R[] / T[] statically).  Neighbouring lanes hold
// neighbouring columns, so U and L reads of a warp hit few lines and the
// final writes are coalesced.  A short last block (rb < S rows) treats the
// local rows >= rb as copies of its bottom skeleton row; the interleave
// search window then over-covers, which keeps the bound valid.
template <typename Key, int S>
__global__ void __launch_bounds__(256)
    column_refine_kernel(const CombineDesc *__restrict__ descs, int32_t ndesc, Ctx c, int shift,
                         int32_t nblk, int32_t w1max, int64_t spd) {
    const int lane = threadIdx.x & 31;
    const int64_t gt = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t di = gt / spd;  // warp-uniform: spd % 32 == 0
    if (di >= ndesc) return;
    const int64_t slot = gt - di * spd;
    const int32_t blk = (int32_t)(slot / w1max);
    const int32_t j = (int32_t)(slot - (int64_t)blk * w1max);
    const CombineDesc &d = descs[di];
    const int64_t n1 = (int64_t)c.n + 1;
    const int32_t inf = c.inf;
    const bool active = blk < nblk && j < d.w1;
    const int64_t i0 = (int64_t)blk * S;
    const int32_t rb = active ? (int32_t)min((int64_t)S, n1 - 1 - i0) : 0;
    const TabAcc U = resolve(d.U, c), L = resolve(d.L, c);
    const int32_t wl = L.w1 - 1;
    const int32_t w1 = d.w1;

    int32_t R[S + 1], T[S + 1];
#pragma unroll
    for (int r = 0; r <= S; ++r) {
        R[r] = inf;
        T[r] = 0;
    }
    if (active && rb >= 2) {
        R[0] = __ldg(d.out_reach + i0 * w1 + j);
        T[0] = __ldg(d.out_trace + i0 * w1 + j);
        const int32_t rbv = __ldg(d.out_reach + (i0 + rb) * w1 + j);
        const int32_t rbt = __ldg(d.out_trace + (i0 + rb) * w1 + j);
#pragma unroll
        for (int r = 1; r <= S; ++r)
            if (r >= rb) {
                R[r] = rbv;
                T[r] = rbt;
            }
    }
#pragma unroll
    for (int dl = S / 2; dl >= 1; dl >>= 1) {
#pragma unroll
        for (int r = dl; r < S; r += 2 * dl) {
            const int a = r - dl, b = r + dl;  // b <= S; rows >= rb mirror the bottom row
            const bool real = active && r < rb;
            const int64_t ci = i0 + r;
            const int32_t kmc = real ? tab_kmax(U, ci, inf) : -1;
            bool tail = false;
            int32_t kl = 0;
            if (real && R[a] < inf) {
                const int32_t Ta = T[a];
                const int32_t Xa = tab_get(U, i0 + a, Ta);
                int32_t hi = min(Ta, kmc);
                int32_t lo = min(max(0, Ta - dl), hi);
                while (lo < hi) {  // first k with U[c,k] >= X(a,j)
                    const int32_t md = (lo + hi) >> 1;
                    if (tab_get(U, ci, md) >= Xa) hi = md; else lo = md + 1;
                }
                kl = max(lo, j - wl);
                if (R[b] < inf) {
                    const int32_t Tb = T[b];
                    const int32_t Xb = tab_get(U, min(i0 + b, i0 + rb), Tb);
                    lo = min(Tb, kmc);
                    hi = min(Tb + dl, kmc);
                    while (lo < hi) {  // last k with U[c,k] <= X(b,j)
                        const int32_t md = (lo + hi + 1) >> 1;
                        if (tab_get(U, ci, md) <= Xb) lo = md; else hi = md - 1;
                    }
                    int32_t kh = min(lo, j);
                    if (kl > kh) {  // safety net: never taken when the bounds hold
                        kl = max(0, j - wl);
                        kh = min(j, kmc);
                    }
                    Key best = ~(Key)0;
                    for (int32_t k = kl; k <= kh; ++k) {
                        const Key key = tpack<Key>(tcell(L, tab_get(U, ci, k), k, j, inf, wl), k, shift);
                        best = key < best ? key : best;
                    }
                    R[r] = tval<Key>(best, shift);
                    T[r] = tk<Key>(best, shift);
                } else {
                    tail = true;
                }
            } else {
                R[r] = inf;
            }
            // tail cells (finite above, INF below: no upper bound): the whole
            // warp scans each one's range [kl, min(j, kmax_c)] in turn
            unsigned mask = __ballot_sync(0xffffffffu, tail);
            while (mask) {
                const int src = __ffs(mask) - 1;
                mask &= mask - 1;
                const int32_t tj = __shfl_sync(0xffffffffu, j, src);
                const int32_t tkl = __shfl_sync(0xffffffffu, kl, src);
                const int32_t tkh = min(tj, __shfl_sync(0xffffffffu, kmc, src));
                const int64_t trow = __shfl_sync(0xffffffffu, ci, src);
                Key best = ~(Key)0;
                for (int32_t k = tkl + lane; k <= tkh; k += 32) {
                    const Key key = tpack<Key>(tcell(L, tab_get(U, trow, k), k, tj, inf, wl), k, shift);
                    best = key < best ? key : best;
                }
                best = twarp_min(best);
                if (lane == src) {
                    R[r] = tval<Key>(best, shift);
                    T[r] = tk<Key>(best, shift);
                }
            }
        }
    }
    // write the finite interior cells; report the finite frontier of each row
#pragma unroll
    for (int r = 1; r < S; ++r) {
        const bool fin = active && r < rb && R[r] < inf;
        if (fin) {
            const int64_t off = (i0 + r) * w1 + j;
            d.out_reach[off] = R[r];
            d.out_trace[off] = T[r];
        }
        // frontier: finite here and the next lane's cell (same row) is not
        const int64_t row = i0 + r;
        const bool nfin = __shfl_down_sync(0xffffffffu, fin, 1);
        const int64_t nrow = __shfl_down_sync(0xffffffffu, row, 1);
        if (fin && (lane == 31 || !nfin || nrow != row)) atomicMax(d.out_kmax + row, j);
    }
}

// Per interior row: kmax is final (max over tiles); write the INF suffix
// (K, w] -- reach INF, trace = `top` of the Alg. 1 node covering the column
// (replay of the reference bisection, _kernel.pyx:53-60) or 0 beyond colhi
// (_kernel.pyx:79-82) -- and fold kmax into wstar.
__global__ void __launch_bounds__(32 * FN_WARPS)
    finalize_rows_kernel(const CombineDesc *__restrict__ descs, int32_t ndesc, Ctx c, int32_t S) {
    __shared__ int4 seg_all[FN_WARPS][FN_SEGS];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int64_t n1 = (int64_t)c.n + 1;
    const int64_t gw = blockIdx.x * (int64_t)FN_WARPS + wid;
    const int64_t di = gw / n1;
    if (di >= ndesc) return;
    const int64_t i = gw - di * n1;
    if (i % S == 0 || i == n1 - 1) return;  // skeleton rows are complete
    int4 *seg = seg_all[wid];
    const CombineDesc &d = descs[di];
    const int32_t inf = c.inf;
    const TabAcc U = resolve(d.U, c);
    const int32_t w = d.w1 - 1;
    const int32_t colhi = min(w, tab_kmax(U, i, inf) + *d.L.wstar);
    const int32_t K = d.out_kmax[i];
    int32_t *reach = d.out_reach + i * d.w1;
    int32_t *trace = d.out_trace + i * d.w1;
    int ns = 0;
    if (lane == 0) {
        int32_t left = 0, right = colhi, fm = -1;
        while (right >= left) {
            const int32_t mid = (left + right + 1) >> 1;
            if (mid <= K) {
                fm = mid;
                left = mid + 1;
            } else {
                if (ns < FN_SEGS) seg[ns++] = make_int4(mid, right, fm, 0);
                right = mid - 1;
            }
        }
    }
    ns = __shfl_sync(0xffffffffu, ns, 0);
    __syncwarp();
    for (int s = lane; s < ns; s += 32) {
        const int32_t fm = seg[s].z;
        seg[s].w = fm >= 0 ? trace[fm] : 0;
    }
    __syncwarp();
    for (int32_t q = K + 1 + lane; q <= w; q += 32) {
        int32_t tv = 0;
        if (q <= colhi)
            for (int s = 0; s < ns; ++s) {
                const int4 sg = seg[s];
                if (q >= sg.x && q <= sg.y) { tv = sg.w; break; }
            }
        reach[q] = inf;
        trace[q] = tv;
    }
    if (lane == 0) atomicMax(d.out_wstar, K);
}

int launch_block_refine(const CombineDesc *descs, int32_t ndesc, Ctx c, int shift, bool key64,
                        int32_t S, int32_t TJ, int32_t WK, int32_t maxw1, cudaStream_t s) {
    (void)TJ;
    (void)WK;
    if (ndesc <= 0) return 0;
    const int64_t n1 = (int64_t)c.n + 1;
    const int32_t nblk = (int32_t)((n1 - 1 + S - 1) / S);
    if (nblk <= 0) return 0;
    const int64_t spd = ((int64_t)nblk * maxw1 + 31) / 32 * 32;
    const unsigned blocks = (unsigned)((spd * ndesc + 255) / 256);
#define LCSG_COLREF(SS)                                                                        \
    if (key64)                                                                                 \
        column_refine_kernel<uint64_t, SS><<<blocks, 256, 0, s>>>(descs, ndesc, c, shift, nblk, \
                                                                  maxw1, spd);                 \
    else                                                                                       \
        column_refine_kernel<uint32_t, SS><<<blocks, 256, 0, s>>>(descs, ndesc, c, shift, nblk, \
                                                                  maxw1, spd);
    switch (S) {
        case 2: LCSG_COLREF(2) break;
        case 4: LCSG_COLREF(4) break;
        case 8: LCSG_COLREF(8) break;
        case 16: LCSG_COLREF(16) break;
        case 32: LCSG_COLREF(32) break;
        default: return (int)cudaErrorInvalidValue;
    }
#undef LCSG_COLREF
    LCSG_LAUNCH_CHECK();
    return 0;
}

int launch_finalize_rows(const CombineDesc *descs, int32_t ndesc, Ctx c, int32_t S,
                         cudaStream_t s) {
    if (ndesc <= 0) return 0;
    const int64_t n1 = (int64_t)c.n + 1;
    const int64_t warps = n1 * ndesc;
    const unsigned blocks = (unsigned)((warps + FN_WARPS - 1) / FN_WARPS);
    finalize_rows_kernel<<<blocks, 32 * FN_WARPS, 0, s>>>(descs, ndesc, c, S);
    LCSG_LAUNCH_CHECK();
    return 0;
}

}  // namespace lcsg
