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
#include <algorithm>
#include <climits>
#include <cstdlib>

#include "lcsg_internal.cuh"

namespace lcsg {

#define LCSG_LAUNCH_CHECK()                         \
    do {                                            \
        cudaError_t e__ = cudaGetLastError();       \
        if (e__ != cudaSuccess) return (int)e__;    \
    } while (0)

constexpr int FN_WARPS = 4;

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
// derived in divide-and-conquer order (delta = S/2 ... 1).  The column's
// (reach, trace) values live in a per-thread slice of shared memory (no
// cross-thread sharing, no barriers); the cell body is a single, non-unrolled
// copy of code (a fully unrolled variant thrashed the instruction cache: 76%
// of stall samples were `no_instructions`).  Neighbouring lanes hold
// neighbouring columns, so U and L reads of a warp hit few lines and the
// final writes are coalesced.  A short last block (rb < S rows) treats the
// local rows >= rb as copies of its bottom skeleton row; the interleave
// search window then over-covers, which keeps the bound valid.  U and L are
// always materialised slabs here (never leaves), so plain row pointers are used.
constexpr int CR_THREADS = 64;
#ifndef LCSG_CR_INLINE
#define LCSG_CR_INLINE 12
#endif
constexpr int CR_INLINE = LCSG_CR_INLINE;  // longer candidate ranges go to the warp-cooperative scan

// Interleave-window counts (column kernels): with U[c,.] strictly
// increasing over finite k, the first k in [lo, hi] with U[c,k] >= Xa is
// lo + #{k in [lo, hi) : U[c,k] < Xa}, and the last k in [lo2, hi2] with
// U[c,k] <= Xb is lo2 + #{k in (lo2, hi2] : U[c,k] <= Xb}.
template <int D>
__device__ __forceinline__ void window_counts(const int32_t *Uc, int32_t lo, int32_t hi,
                                              int32_t Xa, bool fb, int32_t lo2, int32_t hi2,
                                              int32_t Xb, int32_t &c1, int32_t &c2) {
    c1 = 0;
    c2 = 0;
#pragma unroll
    for (int t = 0; t < D; ++t) {
        const int32_t k1 = lo + t, k2 = lo2 + 1 + t;
        const int32_t u1 = k1 < hi ? __ldg(Uc + k1) : INT_MAX;
        const int32_t u2 = (fb && k2 <= hi2) ? __ldg(Uc + k2) : INT_MAX;
        c1 += u1 < Xa;
        c2 += u2 <= Xb;
    }
}
__device__ __forceinline__ void window_counts_n(const int32_t *Uc, int32_t D, int32_t lo,
                                                int32_t hi, int32_t Xa, bool fb, int32_t lo2,
                                                int32_t hi2, int32_t Xb, int32_t &c1, int32_t &c2) {
    c1 = 0;
    c2 = 0;
    for (int t = 0; t < D; ++t) {
        const int32_t k1 = lo + t, k2 = lo2 + 1 + t;
        if (k1 < hi) c1 += __ldg(Uc + k1) < Xa;
        if (fb && k2 <= hi2) c2 += __ldg(Uc + k2) <= Xb;
    }
}


// SC: block size as a compile-time constant (0: runtime S)
template <typename Key, int SC = 0>
__global__ void __launch_bounds__(CR_THREADS)
    column_refine_kernel(const CombineDesc *__restrict__ descs, int32_t ndesc, Ctx c, int shift,
                         int32_t S_arg, int32_t rs, int32_t nblk, FastDiv w1div) {
    const int32_t S = SC > 0 ? SC : S_arg;
    // local row r of block blk is the actual row i0 + r*rs (rs = row step of
    // this refinement stage); rows 0 and S of the block are already known
    extern __shared__ int32_t csm[];
    int32_t *sR = csm + threadIdx.x;  // sR[r * CR_THREADS]
    int32_t *sT = csm + (S + 1) * CR_THREADS + threadIdx.x;
    const int lane = threadIdx.x & 31;
    const int32_t di = (int32_t)(blockIdx.z * 65535u + blockIdx.y);  // CTA-uniform
    if (di >= ndesc) return;
    const int32_t slot = (int32_t)(blockIdx.x * CR_THREADS + threadIdx.x);
    const int32_t blk = fdiv(slot, w1div);
    const int32_t j = slot - blk * w1div.d;
    const CombineDesc &d = descs[di];
    const int32_t n1 = c.n + 1;
    const int32_t inf = c.inf;
    const bool active = blk < nblk && j < d.w1;
    // 32-bit element offsets (n1 * w1 < 2^32 for every refined table)
    const int32_t i0 = blk * S * rs;
    const int32_t span = n1 - 1 - i0;  // actual rows from i0 to the last row
    // local rows r < rb are real; r >= rb mirror the bottom row
    const int32_t rb = active ? min(S, (span + rs - 1) / rs) : 0;
    // bottom bounding row: the next block boundary if it exists, else the last row
    const int32_t ibot = span >= S * rs ? i0 + S * rs : n1 - 1;
    const uint32_t uw1u = (uint32_t)d.U.w1, lw1u = (uint32_t)d.L.w1, w1u = (uint32_t)d.w1;
    const int32_t *__restrict__ Ur = d.U.reach;
    const int32_t *__restrict__ Uk = d.U.kmax;
    const int32_t *__restrict__ Lr = d.L.reach;
    const int32_t uw1 = d.U.w1, lw1 = d.L.w1, wl = lw1 - 1;
    const int32_t w1 = d.w1;
    // output pointers in registers: stores through them must not force
    // re-loads of the descriptor (which lives in global memory)
    int32_t *__restrict__ const out_reach = d.out_reach;
    int32_t *__restrict__ const out_trace = d.out_trace;

    {
        int32_t r0v = inf, r0t = 0, rbv = inf, rbt = 0;
        if (active && rb >= 2) {
            const uint32_t o0 = (uint32_t)i0 * w1u + j, ob = (uint32_t)ibot * w1u + j;
            r0v = __ldg(out_reach + o0);
            r0t = __ldg(out_trace + o0);
            rbv = __ldg(out_reach + ob);
            rbt = __ldg(out_trace + ob);
        }
        // top row INF over the whole warp: every interior cell is INF (reach
        // is nondecreasing in the start row); their traces are finalize's
        if (__all_sync(0xffffffffu, r0v >= inf)) {
            if (active)
                for (int r = 1; r < rb; ++r) out_reach[(uint32_t)(i0 + r * rs) * w1u + j] = inf;
            return;
        }
        sR[0] = r0v;
        sT[0] = r0t;
        for (int r = 1; r <= S; ++r) {
            sR[r * CR_THREADS] = r >= rb ? rbv : inf;
            sT[r * CR_THREADS] = r >= rb ? rbt : 0;
        }
    }
#pragma unroll 1
    for (int dl = S >> 1; dl >= 1; dl >>= 1) {
        const int32_t dist = dl * rs;  // actual row distance to both bounding rows
#pragma unroll 1
        for (int r = dl; r < S; r += 2 * dl) {
            const int a = r - dl, b = r + dl;  // b <= S; rows >= rb mirror the bottom row
            const bool real = active && r < rb;
            const uint32_t ci = (uint32_t)(i0 + r * rs);
            const uint32_t ai = (uint32_t)(i0 + a * rs);
            const uint32_t bi = (uint32_t)(b < rb ? i0 + b * rs : ibot);
            const int32_t *Uc = Ur + ci * uw1u;
            const int32_t kmc = real ? __ldg(Uk + ci) : -1;
            const int32_t Ra = sR[a * CR_THREADS], Rb = sR[b * CR_THREADS];
            bool tail = false;
            int32_t kl = 0, outv = inf, outk = 0;
            if (real && Ra < inf) {
                const bool fb = Rb < inf;
                const int32_t Ta = sT[a * CR_THREADS];
                const int32_t Tb = fb ? sT[b * CR_THREADS] : 0;
                const int32_t Xa = __ldg(Ur + (ai * uw1u + Ta));
                const int32_t Xb = fb ? __ldg(Ur + (bi * uw1u + Tb)) : 0;
                const int32_t hi1 = min(Ta, kmc);
                const int32_t lo1 = min(max(0, Ta - dist), hi1);
                const int32_t lo2 = min(Tb, kmc), hi2 = min(Tb + dist, kmc);
                int32_t lo, kh0;
                if (dist <= 8) {  // short windows: independent counting loads
                    int32_t c1, c2;
                    window_counts<8>(Uc, lo1, hi1, Xa, fb, lo2, hi2, Xb, c1, c2);
                    lo = lo1 + c1;
                    kh0 = lo2 + c2;
                } else {
                    lo = lo1;
                    int32_t hi = hi1;
                    while (lo < hi) {  // first k with U[c,k] >= X(a,j)
                        const int32_t md = (lo + hi) >> 1;
                        if (__ldg(Uc + md) >= Xa) hi = md; else lo = md + 1;
                    }
                    kh0 = lo2;
                    if (fb) {
                        int32_t l2 = lo2, h2 = hi2;
                        while (l2 < h2) {  // last k with U[c,k] <= X(b,j)
                            const int32_t md = (l2 + h2 + 1) >> 1;
                            if (__ldg(Uc + md) <= Xb) l2 = md; else h2 = md - 1;
                        }
                        kh0 = l2;
                    }
                }
                kl = max(lo, j - wl);
                if (fb) {
                    int32_t kh = min(kh0, j);
                    if (kl > kh) {  // safety net: never taken when the bounds hold
                        kl = max(0, j - wl);
                        kh = min(j, kmc);
                    }
                    Key best = ~(Key)0;
                    for (int32_t k = kl; k <= kh; ++k) {
                        const int32_t x = __ldg(Uc + k);  // finite: k <= kmax_c
                        const int32_t v = __ldg(Lr + ((uint32_t)(x - 1) * lw1u + (j - k)));
                        const Key key = tpack<Key>(v, k, shift);
                        best = key < best ? key : best;
                    }
                    outv = tval<Key>(best, shift);  // (b,j) finite => non-empty range
                    outk = tk<Key>(best, shift);
                } else {
                    tail = true;
                }
            }
            if (!tail) {
                sR[r * CR_THREADS] = outv;
                sT[r * CR_THREADS] = outk;
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
                const uint32_t trow = __shfl_sync(0xffffffffu, ci, src);
                const int32_t *Ut = Ur + trow * uw1u;
                Key best = ~(Key)0;
                for (int32_t k = tkl + lane; k <= tkh; k += 32) {
                    int32_t v = inf;
                    if (tj - k <= wl) v = __ldg(Lr + ((uint32_t)(__ldg(Ut + k) - 1) * lw1u + (tj - k)));
                    const Key key = tpack<Key>(v, k, shift);
                    best = key < best ? key : best;
                }
                best = twarp_min(best);
                if (lane == src) {  // an empty candidate range means INF
                    sR[r * CR_THREADS] = best == ~(Key)0 ? inf : tval<Key>(best, shift);
                    sT[r * CR_THREADS] = best == ~(Key)0 ? 0 : tk<Key>(best, shift);
                }
            }
        }
    }
    // write every interior cell's reach (INF included: later stages read these
    // rows as bounds, finalize finds each row's finite prefix in them) and the
    // finite cells' traces
#pragma unroll 1
    for (int r = 1; r < S; ++r) {
        const int32_t v = sR[r * CR_THREADS];
        if (active && r < rb) {
            const uint32_t off = (uint32_t)(i0 + r * rs) * w1u + j;
            out_reach[off] = v;
            if (v < inf) out_trace[off] = sT[r * CR_THREADS];
        }
    }
}

// Per-warp scratch of the segmented cooperative scan (fine kernel).
template <typename Key>
struct CoopSlot {
    int32_t start, kl, j, row;
    Key key;
};
__device__ __forceinline__ void key_atomic_min(uint32_t *p, uint32_t v) { atomicMin(p, v); }
__device__ __forceinline__ void key_atomic_min(uint64_t *p, uint64_t v) {
    atomicMin((unsigned long long *)p, (unsigned long long)v);
}
template <typename Key>
__device__ __forceinline__ CoopSlot<Key> *coop_slots() {
    __shared__ CoopSlot<Key> slots[CR_THREADS];
    return slots;
}

// rs == 1 specialisation (the hot one): identical cell logic, fewer registers.
// SC: block size S as a compile-time constant (0: runtime S) -- constant
// shared-memory offsets and unrolled init / write loops
template <typename Key, int SC>
__global__ void __launch_bounds__(CR_THREADS)
    column_refine_fine_kernel(const CombineDesc *__restrict__ descs, int32_t ndesc, Ctx c, int shift,
                         int32_t S_arg, int32_t nblk, FastDiv w1div) {
    const int32_t S = SC > 0 ? SC : S_arg;
    extern __shared__ int32_t csm[];
    int32_t *sR = csm + threadIdx.x;                     // sR[r * CR_THREADS]
    int32_t *sT = csm + (S + 1) * CR_THREADS + threadIdx.x;
    const int lane = threadIdx.x & 31;
    const int32_t di = (int32_t)(blockIdx.z * 65535u + blockIdx.y);  // CTA-uniform
    if (di >= ndesc) return;
    const int32_t slot = (int32_t)(blockIdx.x * CR_THREADS + threadIdx.x);
    const int32_t blk = fdiv(slot, w1div);
    const int32_t j = slot - blk * w1div.d;
    const CombineDesc &d = descs[di];
    const int32_t n1 = c.n + 1;
    const int32_t inf = c.inf;
    const bool active = blk < nblk && j < d.w1;
    // 32-bit element offsets: every refined table has n1 * w1 < 2^32
    // (lcsg_api.cu node kinds), so an address is one IMAD + one IMAD.WIDE
    const uint32_t i0 = (uint32_t)blk * (uint32_t)S;
    const int32_t rb = active ? min(S, n1 - 1 - (int32_t)i0) : 0;
    const int32_t *__restrict__ Ur = d.U.reach;
    const int32_t *__restrict__ Uk = d.U.kmax;
    const int32_t *__restrict__ Lr = d.L.reach;
    const int32_t uw1 = d.U.w1, lw1 = d.L.w1, wl = lw1 - 1;
    const int32_t w1 = d.w1;
    // output pointers in registers: stores through them must not force
    // re-loads of the descriptor (which lives in global memory)
    int32_t *__restrict__ const out_reach = d.out_reach;
    int32_t *__restrict__ const out_trace = d.out_trace;

    {
        int32_t r0v = inf, r0t = 0, rbv = inf, rbt = 0;
        if (active && rb >= 2) {
            const uint32_t o0 = i0 * (uint32_t)w1 + j, ob = (i0 + rb) * (uint32_t)w1 + j;
            r0v = __ldg(out_reach + o0);
            r0t = __ldg(out_trace + o0);
            rbv = __ldg(out_reach + ob);
            rbt = __ldg(out_trace + ob);
        }
        // top row INF over the whole warp: every interior cell is INF
        if (__all_sync(0xffffffffu, r0v >= inf)) {
            if (active) {
                uint32_t o = i0 * (uint32_t)w1 + j;
                for (int r = 1; r < rb; ++r) out_reach[o += w1] = inf;
            }
            return;
        }
        sR[0] = r0v;
        sT[0] = r0t;
#pragma unroll
        for (int r = 1; r <= S; ++r) {
            sR[r * CR_THREADS] = r >= rb ? rbv : inf;
            sT[r * CR_THREADS] = r >= rb ? rbt : 0;
        }
    }
#pragma unroll 1
    for (int dl = S >> 1; dl >= 1; dl >>= 1) {
#pragma unroll 1
        for (int r = dl; r < S; r += 2 * dl) {
            const int a = r - dl, b = r + dl;  // b <= S; rows >= rb mirror the bottom row
            const bool real = active && r < rb;
            const uint32_t ci = i0 + r;
            const int32_t *Uc = Ur + ci * (uint32_t)uw1;
            const int32_t kmc = real ? __ldg(Uk + ci) : -1;
            const int32_t Ra = sR[a * CR_THREADS], Rb = sR[b * CR_THREADS];
            bool tail = false, longr = false;
            int32_t kl = 0, khl = 0, outv = inf, outk = 0;
            if (real && Ra < inf) {
                const bool fb = Rb < inf;
                const int32_t Ta = sT[a * CR_THREADS];
                const int32_t Tb = fb ? sT[b * CR_THREADS] : 0;
                // both interleave windows hold <= dl+1 candidates: count them
                // with independent loads (no dependent binary-search steps)
                const int32_t Xa = __ldg(Ur + ((i0 + a) * (uint32_t)uw1 + Ta));
                const int32_t Xb =
                    fb ? __ldg(Ur + ((i0 + min(b, rb)) * (uint32_t)uw1 + Tb)) : 0;
                const int32_t hi = min(Ta, kmc);
                const int32_t lo = min(max(0, Ta - dl), hi);
                const int32_t lo2 = min(Tb, kmc), hi2 = min(Tb + dl, kmc);
                int32_t c1, c2;
                switch (dl) {
                    case 1: window_counts<1>(Uc, lo, hi, Xa, fb, lo2, hi2, Xb, c1, c2); break;
                    case 2: window_counts<2>(Uc, lo, hi, Xa, fb, lo2, hi2, Xb, c1, c2); break;
                    case 4: window_counts<4>(Uc, lo, hi, Xa, fb, lo2, hi2, Xb, c1, c2); break;
                    default: window_counts_n(Uc, dl, lo, hi, Xa, fb, lo2, hi2, Xb, c1, c2); break;
                }
                kl = max(lo + c1, j - wl);  // first k with U[c,k] >= X(a,j)
                if (fb) {
                    int32_t kh = min(lo2 + c2, j);  // last k with U[c,k] <= X(b,j)
                    if (kl > kh) {  // safety net: never taken when the bounds hold
                        kl = max(0, j - wl);
                        kh = min(j, kmc);
                    }
                    if (kh - kl >= CR_INLINE) {
                        // long candidate range: evaluated by the whole warp below
                        // (a profile showed the per-lane loop at 7.8 active lanes)
                        longr = true;
                        khl = kh;
                    } else if (kl == kh && Xa == Xb) {
                        // pinned crossing: X(c,j) = X(a,j) = X(b,j) = U[c,kl]
                        // is already known -- one gather, no U load
                        outv = __ldg(Lr + ((uint32_t)(Xa - 1) * (uint32_t)lw1 + (j - kl)));
                        outk = kl;
                    } else {
                        Key best = ~(Key)0;
#pragma unroll 2
                        for (int32_t k = kl; k <= kh; ++k) {
                            const int32_t x = __ldg(Uc + k);  // finite: k <= kmax_c
                            const int32_t v = __ldg(Lr + ((uint32_t)(x - 1) * (uint32_t)lw1 + (j - k)));
                            const Key key = tpack<Key>(v, k, shift);
                            best = key < best ? key : best;
                        }
                        outv = tval<Key>(best, shift);  // (b,j) finite => non-empty range
                        outk = tk<Key>(best, shift);
                    }
                } else {
                    tail = true;
                }
            }
            if (!tail && !longr) {
                sR[r * CR_THREADS] = outv;
                sT[r * CR_THREADS] = outk;
            }
            // tail cells (finite above, INF below: no upper bound; range
            // [kl, min(j, kmax_c)]) and long ranges: the candidates of all such
            // cells of the warp are concatenated (prefix sum of the range
            // lengths) and spread over the lanes; keys reduce per cell with a
            // shared-memory atomicMin.  (One cell per warp pass left ~2/3 of
            // the lanes idle and cost ~40% of the kernel's instructions.)
            const bool coop = tail || longr;
            if (__any_sync(0xffffffffu, coop)) {
                const int32_t chi = tail ? min(j, kmc) : khl;
                const int32_t len = coop ? max(0, chi - kl + 1) : 0;
                int32_t incl = len;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int32_t t = __shfl_up_sync(0xffffffffu, incl, o);
                    if (lane >= o) incl += t;
                }
                const int32_t total = __shfl_sync(0xffffffffu, incl, 31);
                CoopSlot<Key> *ws = coop_slots<Key>() + (threadIdx.x >> 5) * 32;
                ws[lane].start = incl - len;
                ws[lane].kl = kl;
                ws[lane].j = j;
                ws[lane].row = (int32_t)ci;
                ws[lane].key = ~(Key)0;
                __syncwarp();
                for (int32_t g = lane; g < total; g += 32) {
                    int o = 0;  // owner: last lane whose range starts at or before g
#pragma unroll
                    for (int step = 16; step > 0; step >>= 1)
                        if (ws[o + step].start <= g) o += step;
                    const int32_t k = ws[o].kl + (g - ws[o].start), tj = ws[o].j;
                    int32_t v = inf;
                    if (tj - k <= wl)
                        v = __ldg(Lr + ((uint32_t)(__ldg(Ur + ((uint32_t)ws[o].row * (uint32_t)uw1 + k)) - 1) *
                                            (uint32_t)lw1 + (tj - k)));
                    key_atomic_min(&ws[o].key, tpack<Key>(v, k, shift));
                }
                __syncwarp();
                if (coop) {
                    const Key best = ws[lane].key;  // empty range (j beyond kmax_c + wl): INF
                    sR[r * CR_THREADS] = len > 0 ? tval<Key>(best, shift) : inf;
                    sT[r * CR_THREADS] = len > 0 ? tk<Key>(best, shift) : 0;
                }
                __syncwarp();
            }
        }
    }
    // write every interior cell's reach (INF included: finalize finds each
    // row's finite prefix in it) and the finite cells' traces
    if (active) {
        const uint32_t o0 = i0 * (uint32_t)w1 + j;
        int32_t *orr = out_reach + o0, *otr = out_trace + o0;
        if (SC > 0) {
#pragma unroll
            for (int r = 1; r < S; ++r) {
                if (r < rb) {
                    const int32_t v = sR[r * CR_THREADS];
                    orr[r * w1] = v;
                    if (v < inf) otr[r * w1] = sT[r * CR_THREADS];
                }
            }
        } else {
#pragma unroll 1
            for (int r = 1; r < rb; ++r) {
                orr += w1;
                otr += w1;
                const int32_t v = sR[r * CR_THREADS];
                *orr = v;
                if (v < inf) *otr = sT[r * CR_THREADS];
            }
        }
    }
}

// Per interior row: kmax is final (max over column blocks); write the INF
// suffix (K, w] -- reach INF, trace = `top` of the Alg. 1 node covering the
// column (replay of the reference bisection, _kernel.pyx:53-60) or 0 beyond
// colhi (_kernel.pyx:79-82) -- and fold kmax into wstar.  A warp owns RPW
// consecutive rows: lane r replays row r's path (no gathers; the INF nodes'
// mids tile (K, colhi] in descending order), then the warp fills the rows
// one after another with coalesced stores.
// FN_MAXSEG: INF nodes on one bisection path over [0, colhi] -- at most one
// per halving step, i.e. <= bit_length(colhi + 1) + 1: 18 covers w < 65536
// (the segment buffers bound the kernel's occupancy, so the wide case is a
// separate instantiation)
template <int FN_MAXSEG>
__global__ void __launch_bounds__(32 * FN_WARPS)
    finalize_rows_kernel(const CombineDesc *__restrict__ descs, int32_t ndesc, Ctx c, int32_t S,
                         int rpw, int pre) {
    // pre != 0 (after the row sweep, lcsg_sweep.cu): kmax of every interior row
    // is already written -- the replay runs on kmax alone (no reach probes)
    __shared__ int2 seg_all[FN_WARPS][32][FN_MAXSEG];
    __shared__ int nseg_all[FN_WARPS][32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int32_t n1 = c.n + 1;
    const int32_t di = (int32_t)(blockIdx.z * 65535u + blockIdx.y);  // CTA-uniform
    if (di >= ndesc) return;
    const int32_t r0 = ((int32_t)blockIdx.x * FN_WARPS + wid) * rpw;
    if (r0 >= n1) return;  // warp-uniform
    const CombineDesc &d = descs[di];
    const int32_t inf = c.inf;
    const TabAcc U = resolve(d.U, c);
    const int32_t w = d.w1 - 1;
    const int32_t wstarL = *d.L.wstar;
    int32_t *__restrict__ const out_reach = d.out_reach;
    int32_t *__restrict__ const out_trace = d.out_trace;
    int32_t *__restrict__ const out_kmax = d.out_kmax;
    const int32_t w1 = d.w1;
    // phase 1: lane = row
    const int32_t i = r0 + lane;
    const bool act = lane < rpw && i < n1 - 1 && (i % S) != 0;  // rows at multiples of S are skeleton rows
    int32_t K = -1, colhi = -1, kmax_warp = -1;
    if (act) {
        colhi = min(w, tab_kmax(U, i, inf) + wstarL);
        // 32-bit element offsets (n1 * w1 < 2^32 for every refined table)
        const int32_t *reach = out_reach + (uint32_t)i * (uint32_t)w1;
        const int32_t *trace = out_trace + (uint32_t)i * (uint32_t)w1;
        // the replay of Alg. 1's bisection over [0, colhi] IS a binary search
        // for the end of the row's finite prefix: finite mids go right, INF
        // mids are the INF nodes (their segments) and go left; K = left - 1
        int32_t left = 0, right = colhi, fm = -1;
        int ns = 0;
        const int32_t Kpre = pre ? out_kmax[i] : -1;
        // common at the lower levels: the whole [0, colhi] is finite, every
        // mid goes right and there is no INF node (fm is then unused)
        if (pre ? Kpre >= colhi : __ldg(reach + colhi) < inf) left = colhi + 1;
        while (right >= left) {
            const int32_t mid = (left + right + 1) >> 1;
            if (pre ? mid <= Kpre : __ldg(reach + mid) < inf) {
                fm = mid;
                left = mid + 1;
            } else {
                if (ns < FN_MAXSEG) seg_all[wid][lane][ns++] = make_int2(mid, fm);
                right = mid - 1;
            }
        }
        K = left - 1;
        if (!pre) out_kmax[i] = K;
        for (int s = 0; s < ns; ++s) {  // resolve tops (independent loads)
            const int32_t f = seg_all[wid][lane][s].y;
            seg_all[wid][lane][s].y = f >= 0 ? __ldg(trace + f) : 0;
        }
        nseg_all[wid][lane] = ns;
        kmax_warp = K;
    }
    kmax_warp = __reduce_max_sync(0xffffffffu, kmax_warp);
    __syncwarp();
    // phase 2: fill the INF suffix traces of each row, coalesced (the reach
    // cells are already written): 0 over (colhi, w], and each INF node's segment
    // [mid_s, hi_s] (hi_0 = colhi, hi_s = mid_{s-1} - 1) with its `top`
    // only the rows with INF cells (K < w) have anything to fill
    unsigned todo = __ballot_sync(0xffffffffu, act && K < w);
    while (todo) {
        const int rr = __ffs(todo) - 1;
        todo &= todo - 1;
        const int32_t Kr = __shfl_sync(0xffffffffu, K, rr);
        const int32_t ch = __shfl_sync(0xffffffffu, colhi, rr);
        const int ns = nseg_all[wid][rr];
        const int2 *sg = seg_all[wid][rr];
        int32_t *trace = out_trace + (uint32_t)(r0 + rr) * (uint32_t)w1;
        for (int32_t q = max(ch, Kr) + 1 + lane; q <= w; q += 32) trace[q] = 0;
        int32_t hi = ch;
        for (int sgi = 0; sgi < ns; ++sgi) {
            const int2 e = sg[sgi];
            for (int32_t q = e.x + lane; q <= hi; q += 32) trace[q] = e.y;
            hi = e.x - 1;
        }
    }
    // wstar = max kmax: most warps bring nothing new (kmax is nonincreasing in the
    // start column), so look before the atomic -- thousands of warps share the word
    if (lane == 0 && kmax_warp >= 0 && kmax_warp > *(volatile int32_t *)d.out_wstar)
        atomicMax(d.out_wstar, kmax_warp);
}

int launch_block_refine(const CombineDesc *descs, int32_t ndesc, Ctx c, int shift, bool key64,
                        int32_t S, int32_t rs, int32_t maxw1, cudaStream_t s) {
    if (ndesc <= 0) return 0;
    if (S < 2 || S > 64 || rs < 1) return (int)cudaErrorInvalidValue;
    const int64_t n1 = (int64_t)c.n + 1;
    const int32_t nblk = (int32_t)((n1 - 1 + (int64_t)S * rs - 1) / ((int64_t)S * rs));
    if (nblk <= 0) return 0;
    // grid: x = column slots of one combine (blocks x maxw1), y/z = combine
    const int64_t slots = (int64_t)nblk * maxw1;
    if (slots >= ((int64_t)1 << 31)) return (int)cudaErrorInvalidValue;
    const dim3 blocks((unsigned)((slots + CR_THREADS - 1) / CR_THREADS),
                      (unsigned)std::min<int32_t>(ndesc, 65535), (unsigned)((ndesc + 65534) / 65535));
    const FastDiv w1div = make_fastdiv(maxw1);
    const size_t smem = (size_t)2 * (S + 1) * CR_THREADS * 4;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(column_refine_kernel<uint32_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, 140 * 1024);
        cudaFuncSetAttribute(column_refine_kernel<uint64_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, 140 * 1024);
        cudaFuncSetAttribute(column_refine_fine_kernel<uint32_t, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 140 * 1024);
        cudaFuncSetAttribute(column_refine_fine_kernel<uint64_t, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 140 * 1024);
        attr = true;
    }
    if (rs == 1) {  // last stage: lean kernel (finite cells only; finalize writes INF)
        // shared-memory carveout (percent; -1 = driver default) of the fine
        // kernels.  Long strings: 72% keeps ~27 resident CTAs per SM and leaves
        // the rest to L1, which holds the U rows the interleave windows re-read
        // (cfg5 28.16 -> 27.69 ms, cfg4 6.78 -> 6.58; 50% and 80% both lose).
        // Short strings (n < 8193) keep the max-occupancy default (cfg2/cfg3
        // lose 5% at 72%).  Set at every launch: the attribute is per function.
        const char *co_env = getenv("LCSG_FINE_CARVEOUT");
        const int carve = co_env ? atoi(co_env) : (n1 > 8193 ? 72 : -1);
#define FINE_LAUNCH(K, SCV)                                                                      \
    do {                                                                                         \
        cudaFuncSetAttribute(column_refine_fine_kernel<K, SCV>,                                  \
                             cudaFuncAttributePreferredSharedMemoryCarveout, carve);             \
        column_refine_fine_kernel<K, SCV><<<blocks, CR_THREADS, smem, s>>>(descs, ndesc, c, shift, \
                                                                          S, nblk, w1div);       \
    } while (0)
        // compile-time S (32 registers) for every width up to LCSG_FINE_SC_MAXW1
        const char *sc_env = getenv("LCSG_FINE_SC_MAXW1");
        const int sc_max = sc_env ? atoi(sc_env) : INT_MAX;
        const int32_t Ssel = maxw1 <= sc_max ? S : 0;
        if (key64) {
            switch (Ssel) {
                case 2: FINE_LAUNCH(uint64_t, 2); break;
                case 4: FINE_LAUNCH(uint64_t, 4); break;
                case 8: FINE_LAUNCH(uint64_t, 8); break;
                default: FINE_LAUNCH(uint64_t, 0); break;
            }
        } else {
            switch (Ssel) {
                case 2: FINE_LAUNCH(uint32_t, 2); break;
                case 4: FINE_LAUNCH(uint32_t, 4); break;
                case 8: FINE_LAUNCH(uint32_t, 8); break;
                case 16: FINE_LAUNCH(uint32_t, 16); break;
                default: FINE_LAUNCH(uint32_t, 0); break;
            }
        }
#undef FINE_LAUNCH
    } else {
        // carveout of the row-step stages (measured: 50% for long strings,
        // 30% below n = 8193; cfg5 -0.03 ms, cfg2 -0.1 ms vs the default)
        const char *co_env = getenv("LCSG_RS_CARVEOUT");
        const int carve = co_env ? atoi(co_env) : (n1 > 8193 ? 50 : 30);
        if (key64) {
            cudaFuncSetAttribute(column_refine_kernel<uint64_t>,
                                 cudaFuncAttributePreferredSharedMemoryCarveout, carve);
            column_refine_kernel<uint64_t><<<blocks, CR_THREADS, smem, s>>>(descs, ndesc, c, shift, S,
                                                                           rs, nblk, w1div);
        } else if (S == 8) {
            cudaFuncSetAttribute(column_refine_kernel<uint32_t, 8>,
                                 cudaFuncAttributePreferredSharedMemoryCarveout, carve);
            column_refine_kernel<uint32_t, 8><<<blocks, CR_THREADS, smem, s>>>(descs, ndesc, c, shift,
                                                                              S, rs, nblk, w1div);
        } else {
            cudaFuncSetAttribute(column_refine_kernel<uint32_t>,
                                 cudaFuncAttributePreferredSharedMemoryCarveout, carve);
            column_refine_kernel<uint32_t><<<blocks, CR_THREADS, smem, s>>>(descs, ndesc, c, shift, S,
                                                                           rs, nblk, w1div);
        }
    }
    LCSG_LAUNCH_CHECK();
    return 0;
}

int launch_finalize_rows(const CombineDesc *descs, int32_t ndesc, Ctx c, int32_t S,
                         cudaStream_t s, int32_t maxw1, bool pre) {
    if (ndesc <= 0) return 0;
    const int64_t n1 = (int64_t)c.n + 1;
    const int rpw = maxw1 <= 512 ? 32 : (maxw1 <= 2048 ? 8 : (maxw1 <= 8192 ? 2 : 1));
    if (S < 2) return (int)cudaErrorInvalidValue;
    const int64_t warps = (n1 + rpw - 1) / rpw;  // per combine
    const dim3 blocks((unsigned)((warps + FN_WARPS - 1) / FN_WARPS),
                      (unsigned)std::min<int32_t>(ndesc, 65535), (unsigned)((ndesc + 65534) / 65535));
    if (maxw1 <= 65536)
    {
        // shared-memory carveout 75%: fewer resident CTAs, L1 for the reach
        // cells the replay probes (cfg5 26.55 -> 26.40 ms vs the default)
        const char *e = getenv("LCSG_FIN_CARVEOUT");
        cudaFuncSetAttribute(finalize_rows_kernel<18>, cudaFuncAttributePreferredSharedMemoryCarveout,
                             e ? atoi(e) : 75);
        finalize_rows_kernel<18><<<blocks, 32 * FN_WARPS, 0, s>>>(descs, ndesc, c, S, rpw, pre ? 1 : 0);
    }
    else
        finalize_rows_kernel<34><<<blocks, 32 * FN_WARPS, 0, s>>>(descs, ndesc, c, S, rpw, pre ? 1 : 0);
    LCSG_LAUNCH_CHECK();
    return 0;
}

}  // namespace lcsg
