// lcsg_narrow.cu -- the narrow combines (tables <= 33 wide: the bottom five
// levels of a power-of-two tree, ~1/4 of a cfg5 solve in the bisection form).
//
// Reference: _combine_tables (solver.py:91-110) -> combine_level / col_mins
// (_kernel.pyx:28-82).  For a finite output cell the reference's Alg. 1 value
// and trace equal the global first-wins argmin over every admissible split
// k (0 <= k <= min(j, kmax_U), j-k <= w_L) -- the same fact the column
// refinement (lcsg_tile.cu) rests on.  For narrow tables that global minimum
// is cheapest computed outright: a CTA stages its block of U rows and the
// window of L rows they reach (x-1 for every finite x = U[i,k]) in shared
// memory, then each thread folds the (w_U+1) x (w_L+1) candidates of its row
// into registers with compile-time indices -- one LDS, one IMAD (pack) and
// one unsigned min per candidate, no stack, no divergence.  INF cells get the
// reference's bisection artefacts: trace = `top` of the Alg. 1 node covering
// the column (replayed from the finite traces, O(log w)), and (INF, 0) beyond
// colhi = min(w, kmax_U + wstar_L) (_kernel.pyx:79-82).  Rows leave through a
// shared-memory transpose as one contiguous, fully coalesced block.
#include "lcsg_internal.cuh"

namespace lcsg {

constexpr int NR_THREADS = 256;

template <int P>
struct NarrowGeom {
    static constexpr int PITCH = (P + 1) | 1;  // odd pitch: per-row reads conflict-free
    // rows per thread: the per-CTA latency chain (descriptor -> U block -> L
    // window -> fold -> store) is amortised over more rows when the fold is short
    static constexpr int RPT = P <= 2 ? 4 : P == 4 ? 2 : 1;
    static constexpr int ROWS = NR_THREADS * RPT;  // output rows per CTA
    // dynamic shared memory: U block + L window (~ROWS + 26 P rows at sigma =
    // 26); after the fold the whole area holds the output staging 2 x ROWS x w1
    static constexpr int BYTES = P == 1 ? 32 * 1024 : P <= 4 ? 40 * 1024 : P == 8 ? 48 * 1024
                                                                                : 72 * 1024;
    static_assert(2 * ROWS * (2 * P + 1) * 4 <= BYTES, "output staging must fit");
    static_assert((ROWS + 64) * PITCH * 4 <= BYTES, "U block + a minimal L window must fit");
};

template <typename Key>
__device__ __forceinline__ Key npack(int32_t v, int32_t k, int shift) {
    return ((Key)(uint32_t)v << shift) | (Key)(uint32_t)k;
}

// rows [row0, row0 + nrows) of a table into shared memory at pitch PT
// (columns >= w1 are INF).  A block of slab rows is one contiguous range of
// the table, copied flat when w1 == PT (every power-of-two tree level).
template <int PT>
__device__ __forceinline__ void stage_rows(int32_t *dst, const TabAcc &t, int64_t row0,
                                           int32_t nrows, int32_t inf) {
    const int tid = threadIdx.x;
    if (t.nx) {  // leaf: (r + 1, NX[sym][r]) (breakout.py:37-55)
        const int32_t *nx = t.nx + row0;
        const bool w2 = t.w1 > 1;
        for (int r = tid; r < nrows; r += NR_THREADS) {
            int32_t *d = dst + r * PT;
            d[0] = (int32_t)(row0 + r + 1);
            if (PT > 1) d[1] = w2 ? __ldg(nx + r) : inf;
#pragma unroll
            for (int k = 2; k < PT; ++k) d[k] = inf;
        }
    } else if (t.w1 == PT) {
        const int32_t *src = t.reach + row0 * PT;
        const int tot = nrows * PT;
        int g = tid;
        for (; g + 3 * NR_THREADS < tot; g += 4 * NR_THREADS) {
            const int32_t a = __ldg(src + g), b = __ldg(src + g + NR_THREADS);
            const int32_t c2 = __ldg(src + g + 2 * NR_THREADS), e = __ldg(src + g + 3 * NR_THREADS);
            dst[g] = a;
            dst[g + NR_THREADS] = b;
            dst[g + 2 * NR_THREADS] = c2;
            dst[g + 3 * NR_THREADS] = e;
        }
        for (; g < tot; g += NR_THREADS) dst[g] = __ldg(src + g);
    } else {
        for (int idx = tid; idx < nrows * PT; idx += NR_THREADS) {
            const int r = idx / PT, k = idx - r * PT;
            dst[idx] = k < t.w1 ? __ldg(t.reach + (row0 + r) * t.w1 + k) : inf;
        }
    }
}

// P: bucket >= every U and L weight (w1 - 1) of the launch
template <int P, typename Key>
__global__ void __launch_bounds__(NR_THREADS)
    narrow_combine_kernel(const CombineDesc *__restrict__ descs, Ctx c, int shift, int32_t bpd,
                          int32_t lcap) {
    using G = NarrowGeom<P>;
    constexpr int PT = G::PITCH, RPT = G::RPT, ROWS = G::ROWS;
    extern __shared__ int32_t nsm[];
    int32_t *sU = nsm;               // ROWS x PT
    int32_t *sL = nsm + ROWS * PT;   // (lcap + 1) x PT; row lcap = all INF
    __shared__ int32_t s_xmax, s_wstar;
    const int32_t di = blockIdx.x / bpd;
    const int64_t i0 = (int64_t)(blockIdx.x - di * bpd) * ROWS;
    const CombineDesc &d = descs[di];
    const int64_t n1 = (int64_t)c.n + 1;
    const int nr = (int)min((int64_t)ROWS, n1 - i0);
    const int32_t inf = c.inf;
    const TabAcc U = resolve(d.U, c), L = resolve(d.L, c);
    const int32_t wl = L.w1 - 1;
    const int tid = threadIdx.x;
    if (tid == 0) {
        s_xmax = 0;
        s_wstar = -1;
    }
    // 1. U rows of the block (columns beyond w_U are INF: no candidate)
    stage_rows<PT>(sU, U, i0, nr, inf);
    for (int idx = tid; idx < PT; idx += NR_THREADS) sL[lcap * PT + idx] = inf;
    __syncthreads();
    // kmax_U of each row (finite prefix of the U row) and the reach of the block
    int32_t ku[RPT];
    int32_t xlast = 0;
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
        const int r = tid + q * NR_THREADS;
        ku[q] = -1;
        if (r < nr) {
#pragma unroll
            for (int k = 0; k <= P; ++k) {
                const int32_t x = sU[r * PT + k];
                if (x < inf) {
                    ku[q] = k;
                    xlast = max(xlast, x);
                }
            }
        }
    }
    xlast = __reduce_max_sync(0xffffffffu, xlast);
    if ((tid & 31) == 0) atomicMax(&s_xmax, xlast);
    __syncthreads();
    // 2. the L rows every finite x of the block lands on: [base, base + nL)
    const int64_t base = (int64_t)sU[0] - 1;  // U[i0, 0] = smallest x of the block
    const int32_t nL = (int32_t)min((int64_t)s_xmax - base, (int64_t)lcap);
    stage_rows<PT>(sL, L, base, nL, inf);
    __syncthreads();
    // 3. first-wins minimum over every candidate of each row, in registers
    Key best[RPT][2 * P + 1];
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
#pragma unroll
        for (int j = 0; j <= 2 * P; ++j) best[q][j] = ~(Key)0;
        const int r = tid + q * NR_THREADS;
        if (r < nr) {
#pragma unroll
            for (int k = 0; k <= P; ++k) {
                const int32_t x = sU[r * PT + k];
                const int64_t lr = x < inf ? (int64_t)x - 1 - base : lcap;
                if (lr < nL || lr == lcap) {
                    const int32_t *row = sL + lr * PT;
#pragma unroll
                    for (int e = 0; e <= P; ++e) {
                        const Key key = npack<Key>(row[e], k, shift);
                        best[q][k + e] = key < best[q][k + e] ? key : best[q][k + e];
                    }
                } else {  // beyond the staged window (sparse matches): read L directly
#pragma unroll
                    for (int e = 0; e <= P; ++e) {
                        const int32_t v = e <= wl ? tab_get(L, (int64_t)x - 1, e) : inf;
                        const Key key = npack<Key>(v, k, shift);
                        best[q][k + e] = key < best[q][k + e] ? key : best[q][k + e];
                    }
                }
            }
        }
    }
    __syncthreads();  // sU and sL are reused as the output staging area below
    const int32_t w1 = d.w1, w = w1 - 1;
    const int32_t wstar_l = *d.L.wstar;
    int32_t *sR = nsm;
    int32_t *sT = nsm + ROWS * w1;
    int32_t wmax = -1;
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
        const int r = tid + q * NR_THREADS;
        if (r >= nr) continue;
        int32_t *rr = sR + r * w1;
        int32_t *tr = sT + r * w1;
        int32_t kfin = -1;
#pragma unroll
        for (int j = 0; j <= 2 * P; ++j) {
            if (j <= w) {
                const int32_t v = (int32_t)(best[q][j] >> shift);
                if (v < inf) kfin = j;
                rr[j] = v < inf ? v : inf;
                tr[j] = (int32_t)(best[q][j] & (((Key)1 << shift) - 1));
            }
        }
        // INF cells: Alg. 1's node `top` (replay of the bisection path over
        // the finite traces), 0 beyond colhi
        const int32_t colhi = min(w, ku[q] + wstar_l);
        for (int32_t qq = kfin + 1; qq <= w; ++qq) {
            int32_t t = 0;
            if (qq <= colhi) {
                int32_t left = 0, right = colhi, top = 0;
                for (;;) {
                    const int32_t mid = (left + right + 1) >> 1;
                    if (mid <= kfin) {  // finite node: qq lies to its right
                        top = tr[mid];
                        left = mid + 1;
                    } else if (qq >= mid) {
                        break;  // INF node: mid..right all get `top`
                    } else {
                        right = mid - 1;
                    }
                }
                t = top;
            }
            tr[qq] = t;
        }
        d.out_kmax[i0 + r] = kfin;
        wmax = max(wmax, kfin);
    }
    wmax = __reduce_max_sync(0xffffffffu, wmax);
    if ((tid & 31) == 0 && wmax >= 0) atomicMax(&s_wstar, wmax);
    __syncthreads();
    // 4. the block's rows are one contiguous range of the output
    int32_t *gr = d.out_reach + i0 * w1;
    const int tot = nr * w1;
    for (int idx = tid; idx < tot; idx += NR_THREADS) gr[idx] = sR[idx];
    if (d.out_trace) {
        int32_t *gt = d.out_trace + i0 * w1;
        for (int idx = tid; idx < tot; idx += NR_THREADS) gt[idx] = sT[idx];
    }
    if (tid == 0 && s_wstar >= 0) atomicMax(d.out_wstar, s_wstar);
}

template <int P, typename Key>
static int launch_narrow_t(const CombineDesc *descs, int32_t ndesc, Ctx c, int shift,
                           cudaStream_t s) {
    constexpr int PT = NarrowGeom<P>::PITCH, BYTES = NarrowGeom<P>::BYTES;
    cudaError_t e = cudaFuncSetAttribute(narrow_combine_kernel<P, Key>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, BYTES);
    if (e != cudaSuccess) return (int)e;
    const int64_t n1 = (int64_t)c.n + 1;
    const int32_t bpd = (int32_t)((n1 + NarrowGeom<P>::ROWS - 1) / NarrowGeom<P>::ROWS);
    // L window rows: whatever the budget leaves after the U block
    const int32_t lcap = (int32_t)(BYTES / 4 - NarrowGeom<P>::ROWS * PT) / PT - 1;
    const int64_t blocks = (int64_t)ndesc * bpd;
    if (blocks == 0) return 0;
    if (blocks >= ((int64_t)1 << 31)) return (int)cudaErrorInvalidConfiguration;
    narrow_combine_kernel<P, Key><<<(unsigned)blocks, NR_THREADS, BYTES, s>>>(
        descs, c, shift, bpd, lcap);
    return (int)cudaGetLastError();
}

int narrow_bucket(int32_t max_weight) {
    int P = 1;
    while (P < max_weight) P *= 2;
    return P <= 16 ? P : -1;
}

int launch_narrow(const CombineDesc *descs, int32_t ndesc, Ctx c, int shift, bool key64,
                  int32_t P, cudaStream_t s) {
#define NARROW_CASE(PP)                                                              \
    case PP:                                                                         \
        return key64 ? launch_narrow_t<PP, uint64_t>(descs, ndesc, c, shift, s)      \
                     : launch_narrow_t<PP, uint32_t>(descs, ndesc, c, shift, s);
    switch (P) {
        NARROW_CASE(1)
        NARROW_CASE(2)
        NARROW_CASE(4)
        NARROW_CASE(8)
        NARROW_CASE(16)
        default:
            return (int)cudaErrorInvalidValue;
    }
#undef NARROW_CASE
}

}  // namespace lcsg
