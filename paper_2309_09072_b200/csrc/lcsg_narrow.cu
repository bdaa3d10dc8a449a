// lcsg_narrow.cu -- the narrow combines (tables <= 65 wide: the bottom six
// levels of a power-of-two tree).
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
// one unsigned min per candidate, no stack, no divergence.  For the widest
// bucket the L window is staged per chunk of split weights k (the window of
// all k would not fit next to the U block).  INF cells get the
// reference's bisection artefacts: trace = `top` of the Alg. 1 node covering
// the column (replayed from the finite traces, O(log w)), and (INF, 0) beyond
// colhi = min(w, kmax_U + wstar_L) (_kernel.pyx:79-82).  Rows leave through a
// shared-memory transpose as one contiguous, fully coalesced block.
#include <cstdlib>
#include <type_traits>

#include "lcsg_internal.cuh"

namespace lcsg {

template <int P>
struct NarrowGeom {
    static constexpr int PITCH = (P + 1) | 1;  // odd pitch: per-row reads conflict-free
    static constexpr int NT = P <= 16 ? 256 : 128;  // threads per CTA
    // rows per thread: the per-CTA latency chain (descriptor -> U block -> L
    // window -> fold -> store) is amortised over more rows when the fold is short
    static constexpr int RPT = P <= 2 ? 4 : P == 4 ? 2 : 1;
    // resident CTAs the register budget is sized for (<= 48 registers for
    // P <= 4: 5 CTAs per SM, as many as their 40 KB of shared memory allows;
    // measured 820 -> 776 us (P = 2), 805 -> 742 us (P = 4) at cfg5)
    static constexpr int MINB = P <= 4 ? 5 : 4;
    static constexpr int ROWS = NT * RPT;  // output rows per CTA
    // split weights k per staged L window
    static constexpr int KC = P <= 16 ? P + 1 : 8;
    static constexpr int NCH = (P + 1 + KC - 1) / KC;
    // dynamic shared memory: U block + L window (~ROWS + 26 KC rows at sigma
    // = 26); after the fold the whole area holds the output staging 2 x ROWS x w1
    static constexpr int BYTES = P == 1 ? 32 * 1024 : P <= 4 ? 40 * 1024 : P == 8 ? 48 * 1024
                                                                                : 72 * 1024;
    static_assert(2 * ROWS * (2 * P + 1) * 4 <= BYTES, "output staging must fit");
    static_assert((ROWS + 64) * PITCH * 4 <= BYTES, "U block + a minimal L window must fit");
};

// packed key (v << shift) | k; `mul` = 1 << shift, so the 32-bit pack is one
// IMAD with the compile-time k as addend
__device__ __forceinline__ uint32_t npack(uint32_t v, int32_t k, int shift, uint32_t mul) {
    return v * mul + (uint32_t)k;
}
__device__ __forceinline__ uint64_t npack(uint64_t v, int32_t k, int shift, uint32_t) {
    return (v << shift) | (uint64_t)(uint32_t)k;
}

__device__ __forceinline__ void cp_async4(int32_t *dst, const int32_t *src) {
    const uint32_t sa = (uint32_t)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(sa), "l"(src));
}
__device__ __forceinline__ void cp_async16(int32_t *dst, const int32_t *src) {
    const uint32_t sa = (uint32_t)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(src));
}
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
}

// ---- TMA bulk copies (cp.async.bulk, sm_90+): the 16-byte-aligned body of a
// contiguous block of table rows moves global -> shared as ONE asynchronous
// bulk transfer issued by a single thread, completing on an mbarrier (the
// Blackwell-native replacement of per-thread cp.async; no register staging,
// no per-thread address arithmetic).  LCSG_TMA_STAGE=0 builds the cp.async path.
#ifndef LCSG_TMA_STAGE
#define LCSG_TMA_STAGE 1
#endif
struct StageBar {
    uint64_t *bar;    // mbarrier in shared memory (initialised by stage_bar_init)
    uint32_t phase;   // parity of the next completion (identical in every thread)
};
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void stage_bar_init(uint64_t *bar) {
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    // order earlier generic-proxy accesses of this shared memory (made visible
    // to this thread by the preceding barrier) before the async-proxy writes
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void stage_bar_wait(StageBar &sb) {
    uint32_t done = 0;
    do {
        asm volatile(
            "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
            "selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(smem_u32(sb.bar)), "r"(sb.phase)
            : "memory");
    } while (!done);
    sb.phase ^= 1u;
}

// Traces of the INF cells (kfin, w] of one output row whose finite prefix
// [0, kfin] (reach and trace) is already in `tr`: Alg. 1 (_kernel.pyx:28-60)
// visits the INF cells as nodes whose mid is INF; such a node fills
// [mid, right] with its `top` (the split bound inherited from the last finite
// mid on its path, else 0) and recurses left.  One replay of that path over
// [0, colhi] therefore tiles (kfin, colhi] into <= log2(w)+1 segments; cells
// beyond colhi get 0 (_kernel.pyx:79-82).
__device__ __forceinline__ void inf_traces(int32_t *tr, int32_t kfin, int32_t colhi, int32_t w) {
    for (int32_t qq = max(kfin, colhi) + 1; qq <= w; ++qq) tr[qq] = 0;
    int32_t left = 0, right = colhi, top = 0;
    while (right > kfin) {  // [left, right] still holds INF cells
        const int32_t mid = (left + right + 1) >> 1;
        if (mid <= kfin) {  // finite node: its trace bounds the right half
            top = tr[mid];
            left = mid + 1;
        } else {  // INF node: mid..right get `top`
            for (int32_t qq = mid; qq <= right; ++qq) tr[qq] = top;
            right = mid - 1;
        }
    }
}

// rows [row0, row0 + nrows) of a table into shared memory at pitch PT
// (columns >= w1 are INF).  A block of slab rows is one contiguous range of
// the table, copied flat when w1 == PT (every power-of-two tree level).
template <int PT, int NT>
__device__ __forceinline__ void stage_rows(int32_t *dst, const TabAcc &t, int64_t row0,
                                           int32_t nrows, int32_t inf, StageBar &sb) {
    const int tid = threadIdx.x;
    if (t.nx2) {  // virtual height-1 node: closed form of its two leaves
        for (int r = tid; r < nrows; r += NT) {
            int32_t *d = dst + r * PT;
            const int64_t row = row0 + r;
            const int32_t xa = __ldg(t.nx + row);
            d[0] = (int32_t)(row + 1);
            d[1] = min(__ldg(t.nx2 + row), xa);
            d[2] = xa < inf ? __ldg(t.nx2 + (xa - 1)) : inf;
#pragma unroll
            for (int k = 3; k < PT; ++k) d[k] = inf;
        }
    } else if (t.nx) {  // leaf: (r + 1, NX[sym][r]) (breakout.py:37-55)
        const int32_t *nx = t.nx + row0;
        const bool w2 = t.w1 > 1;
        for (int r = tid; r < nrows; r += NT) {
            int32_t *d = dst + r * PT;
            d[0] = (int32_t)(row0 + r + 1);
            if (PT > 1) {
                if (w2) cp_async4(d + 1, nx + r);
                else d[1] = inf;
            }
#pragma unroll
            for (int k = 2; k < PT; ++k) d[k] = inf;
        }
        cp_async_wait_all();
    } else if (t.w1 == PT) {
        // contiguous: asynchronous global -> shared copies (LDGSTS), all in
        // flight at once without staging registers; 16-byte copies for the
        // aligned body when source and destination are congruent mod 16
        const int32_t *src = t.reach + row0 * PT;
        const int tot = nrows * PT;
        if ((((uintptr_t)src ^ (uintptr_t)__cvta_generic_to_shared(dst)) & 15) == 0) {
            const int h = min(tot, (int)(((16 - ((uintptr_t)src & 15)) & 15) >> 2));
            const int nb = (tot - h) >> 2;
            if (tid < h) cp_async4(dst + tid, src + tid);
#if LCSG_TMA_STAGE
            if (nb > 0 && tid == 0) bulk_g2s(dst + h, src + h, (uint32_t)nb * 16u, sb.bar);
#else
            for (int c2 = tid; c2 < nb; c2 += NT) cp_async16(dst + h + 4 * c2, src + h + 4 * c2);
#endif
            const int t0 = h + 4 * nb;
            if (t0 + tid < tot) cp_async4(dst + t0 + tid, src + t0 + tid);
            cp_async_wait_all();
#if LCSG_TMA_STAGE
            if (nb > 0) stage_bar_wait(sb);  // CTA-uniform
#endif
            return;
        } else {
            for (int g = tid; g < tot; g += NT) cp_async4(dst + g, src + g);
        }
        cp_async_wait_all();
    } else {
        for (int idx = tid; idx < nrows * PT; idx += NT) {
            const int r = idx / PT, k = idx - r * PT;
            dst[idx] = k < t.w1 ? __ldg(t.reach + (row0 + r) * t.w1 + k) : inf;
        }
    }
}

// shared -> global copy of a contiguous block: 16-byte vectors when the
// destination is 16-byte aligned (the staging area always is)
template <int NT>
__device__ __forceinline__ void copy_out(int32_t *g, const int32_t *sm, int tot) {
    const int tid = threadIdx.x;
    if (((uintptr_t)g & 15) == 0) {
        const int n4 = tot >> 2;
        for (int v = tid; v < n4; v += NT)
            reinterpret_cast<int4 *>(g)[v] = reinterpret_cast<const int4 *>(sm)[v];
        const int t0 = n4 << 2;
        if (t0 + tid < tot) g[t0 + tid] = sm[t0 + tid];
    } else {
        for (int idx = tid; idx < tot; idx += NT) g[idx] = sm[idx];
    }
}

// shared -> global of the block's output rows with TMA bulk stores
// (cp.async.bulk.global.shared::cta): one thread moves the 16-byte body of
// both tables, the other threads write the < 4-int tails.  The caller has
// synchronised the block after filling `sr` / `st`; the issuing thread waits
// for the bulk reads of shared memory before it exits (bulk_store_drain).
template <int NT>
__device__ __forceinline__ void copy_out_rows(int32_t *gr, int32_t *gt, const int32_t *sr,
                                              const int32_t *st, int tot) {
#if LCSG_TMA_STAGE
    const bool al = (((uintptr_t)gr | (gt ? (uintptr_t)gt : 0)) & 15) == 0 &&
                    (((uintptr_t)sr | (uintptr_t)st) & 15) == 0;
    if (al) {
        const int body = tot & ~3;
        if (threadIdx.x == 0 && body > 0) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gr),
                         "r"(smem_u32(sr)), "r"((uint32_t)body * 4u)
                         : "memory");
            if (gt)
                asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gt),
                             "r"(smem_u32(st)), "r"((uint32_t)body * 4u)
                             : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
        const int idx = body + (int)threadIdx.x;
        if (idx < tot) {
            gr[idx] = sr[idx];
            if (gt) gt[idx] = st[idx];
        }
        return;
    }
#endif
    copy_out<NT>(gr, sr, tot);
    if (gt) copy_out<NT>(gt, st, tot);
}
__device__ __forceinline__ void bulk_store_drain() {
#if LCSG_TMA_STAGE
    if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
#endif
}

// out-of-line copy for the chunked (widest) bucket, whose k-chunk loop is
// unrolled: one shared body instead of one inlined copy per chunk
template <int PT, int NT>
__device__ __noinline__ void stage_rows_call(int32_t *dst, const TabAcc &t, int64_t row0,
                                             int32_t nrows, int32_t inf, StageBar &sb) {
    stage_rows<PT, NT>(dst, t, row0, nrows, inf, sb);
}

// P: bucket >= every U and L weight (w1 - 1) of the launch
// FW: every combine of the launch has the full output width 2P+1 (each level
// of a power-of-two tree) -- compile-time row pitch and bounds in the epilogue
template <int P, typename Key, bool FW = false>
__global__ void __launch_bounds__(NarrowGeom<P>::NT, NarrowGeom<P>::MINB)
    narrow_combine_kernel(const CombineDesc *__restrict__ descs, Ctx c, int shift, int32_t bpd,
                          int32_t lcap) {
    using G = NarrowGeom<P>;
    constexpr int PT = G::PITCH, RPT = G::RPT, ROWS = G::ROWS, NT = G::NT, KC = G::KC,
                  NCH = G::NCH;
    extern __shared__ int32_t nsm[];
    int32_t *sU = nsm;               // ROWS x PT
    int32_t *sL = nsm + ROWS * PT;   // lcap x PT
    __shared__ int32_t s_xmax[NCH], s_wstar;
    __shared__ uint64_t s_bar;
    const int32_t di = blockIdx.x / bpd;
    const int64_t i0 = (int64_t)(blockIdx.x - di * bpd) * ROWS;
    const CombineDesc &d = descs[di];
    const int64_t n1 = (int64_t)c.n + 1;
    const int nr = (int)min((int64_t)ROWS, n1 - i0);
    const int32_t inf = c.inf;
    const TabAcc U = resolve(d.U, c), L = resolve(d.L, c);
    const int tid = threadIdx.x;
    const uint32_t mul = 1u << (shift & 31);
    if (tid < NCH) s_xmax[tid] = 0;
    if (tid == 0) s_wstar = -1;
    stage_bar_init(&s_bar);
    __syncthreads();
    StageBar sb{&s_bar, 0u};
    // 1. U rows of the block (columns beyond w_U are INF: no candidate)
    stage_rows<PT, NT>(sU, U, i0, nr, inf, sb);
    __syncthreads();
    // kmax_U of each row (finite prefix of the U row) and, per chunk of split
    // weights, the largest finite x of the block
    int32_t ku[RPT];
    int32_t xlast[NCH];
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch) xlast[ch] = 0;
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
        const int r = tid + q * NT;
        ku[q] = -1;
        if (r < nr) {
#pragma unroll
            for (int k = 0; k <= P; ++k) {
                const int32_t x = sU[r * PT + k];
                if (x < inf) {
                    ku[q] = k;
                    xlast[k / KC] = max(xlast[k / KC], x);
                }
            }
        }
    }
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch) {
        const int32_t m = __reduce_max_sync(0xffffffffu, xlast[ch]);
        if ((tid & 31) == 0 && m > 0) atomicMax(&s_xmax[ch], m);
    }
    // 2./3. per chunk: the L rows its finite x land on, [base, base + nL), then
    // the first-wins minimum over the chunk's candidates, in registers
    Key best[RPT][2 * P + 1];
#pragma unroll
    for (int q = 0; q < RPT; ++q)
#pragma unroll
        for (int j = 0; j <= 2 * P; ++j) best[q][j] = ~(Key)0;
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch) {
        const int k0 = ch * KC;
        __syncthreads();  // U block / xmax ready
        // U[i0, k0] is the smallest x of the chunk (U rows nondecreasing in i);
        // INF there means no finite candidate in this chunk or beyond
        const int32_t x0 = sU[k0];
        if (x0 >= inf) break;  // CTA-uniform
        const int64_t base = (int64_t)x0 - 1;
        const int64_t need = (int64_t)s_xmax[ch] - base;  // L rows of the chunk
        // usually one window; sparse matches can need several (each candidate
        // is folded in the window holding its L row; INF candidates are
        // skipped -- INF cells take their trace from the replay below)
        for (int64_t w0 = 0; w0 < need; w0 += lcap) {
            const int32_t nL = (int32_t)min(need - w0, (int64_t)lcap);
            if (w0 > 0) __syncthreads();  // previous window consumed
            // shift the window by 0..3 ints so that it is congruent mod 16
            // bytes with its source rows (16-byte async copies)
            const int sh = L.nx ? 0 : (int)(((uintptr_t)(L.reach + (base + w0) * PT) >> 2) & 3);
            int32_t *sLw = sL + sh;
            if (NCH > 1)
                stage_rows_call<PT, NT>(sLw, L, base + w0, nL, inf, sb);
            else
                stage_rows<PT, NT>(sLw, L, base + w0, nL, inf, sb);
            __syncthreads();
#pragma unroll
            for (int q = 0; q < RPT; ++q) {
                const int r = tid + q * NT;
                if (r < nr) {
#pragma unroll
                    for (int kk = 0; kk < KC; ++kk) {
                        const int k = ch * KC + kk;
                        if (k > P) break;
                        const int32_t x = sU[r * PT + k];
                        const int64_t lr = (int64_t)x - 1 - base - w0;
                        if (x < inf && lr >= 0 && lr < nL) {
                            const int32_t *row = sLw + lr * PT;
#pragma unroll
                            for (int e = 0; e <= P; ++e) {
                                const Key key = npack((Key)(uint32_t)row[e], k, shift, mul);
                                best[q][k + e] = key < best[q][k + e] ? key : best[q][k + e];
                            }
                        }
                    }
                }
            }
            __syncthreads();  // window consumed (next window / chunk / staging)
        }
    }
    __syncthreads();  // sU and sL are reused as the output staging area below
    const int32_t w1 = FW ? 2 * P + 1 : d.w1, w = w1 - 1;
    const int32_t wstar_l = *d.L.wstar;
    // descriptor fields in registers (stores below must not force re-loads)
    int32_t *__restrict__ const out_kmax = d.out_kmax;
    int32_t *__restrict__ const out_reach = d.out_reach;
    int32_t *__restrict__ const out_trace = d.out_trace;
    int32_t *const out_wstar = d.out_wstar;
    int32_t *sR = nsm;
    int32_t *sT = nsm + ROWS * w1;
    int32_t wmax = -1;
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
        const int r = tid + q * NT;
        if (r >= nr) continue;
        int32_t *rr = sR + r * w1;
        int32_t *tr = sT + r * w1;
        int32_t kfin = -1;
#pragma unroll
        for (int j = 0; j <= 2 * P; ++j) {
            if (j <= w) {
                // compare in the key domain: an untouched slot (~0, no
                // candidate) must read as INF also for 64-bit keys, whose
                // shifted value does not fit an int32
                const Key vk = best[q][j] >> shift;
                const int32_t v = vk < (Key)(uint32_t)inf ? (int32_t)vk : inf;
                if (v < inf) kfin = j;
                rr[j] = v;
                tr[j] = (int32_t)(best[q][j] & (((Key)1 << shift) - 1));
            }
        }
        // INF cells: Alg. 1's node `top`, 0 beyond colhi
        inf_traces(tr, kfin, min(w, ku[q] + wstar_l), w);
        out_kmax[i0 + r] = kfin;
        wmax = max(wmax, kfin);
    }
    wmax = __reduce_max_sync(0xffffffffu, wmax);
    if ((tid & 31) == 0 && wmax >= 0) atomicMax(&s_wstar, wmax);
    __syncthreads();
    // 4. the block's rows are one contiguous range of the output
    const int tot = nr * w1;
    copy_out_rows<NT>(out_reach + i0 * w1, out_trace ? out_trace + i0 * w1 : nullptr, sR, sT, tot);
    if (tid == 0 && s_wstar >= 0) atomicMax(out_wstar, s_wstar);
    bulk_store_drain();
}

// narrow<32> with a ROLLED k-chunk loop (32-bit keys only).  The unrolled
// fold of narrow_combine_kernel<32> is ~107 KB of code -- a fifth of its
// stall samples were instruction-cache misses.  Here one chunk body serves
// every chunk: the thread's keys live in a 40-register window W[t] = output
// column 8c + t; chunk c (splits k = 8c .. 8c+7) folds into W[kk + e] with
// compile-time indices, after which columns 8c .. 8c+7 are final (later
// splits only reach larger columns).  They are parked in the thread's own U
// row -- slots 8c .. 8c+7 were that chunk's split columns, never read again
// (chunk c+1 reads row 0's slot 8(c+1) as its window base, untouched) -- and
// the window shifts by 8.  Split k = 32 (the last chunk) is folded after the
// loop, then the epilogue is the same as narrow_combine_kernel's.  Same
// candidates and first-wins keys, hence the same output.
constexpr int R32_NT = 128, R32_KC = 8, R32_PT = 33, R32_BYTES = 72 * 1024;

template <bool FW>  // FW: every output row is 65 wide (compile-time epilogue pitch)
__global__ void __launch_bounds__(R32_NT)
    narrow32_roll_kernel(const CombineDesc *__restrict__ descs, Ctx c, int shift, int32_t bpd,
                         int32_t lcap) {
    constexpr int P = 32, PT = R32_PT, NT = R32_NT, ROWS = R32_NT, KC = R32_KC;
    constexpr int NCH = 5;  // chunks 0..3 rolled (k < 32), chunk 4 = k 32
    extern __shared__ int32_t nsm[];
    int32_t *sU = nsm;
    int32_t *sL = nsm + ROWS * PT;
    __shared__ int32_t s_xmax[NCH], s_wstar;
    __shared__ uint64_t s_bar;
    const int32_t di = blockIdx.x / bpd;
    const int64_t i0 = (int64_t)(blockIdx.x - di * bpd) * ROWS;
    const CombineDesc &d = descs[di];
    const int64_t n1 = (int64_t)c.n + 1;
    const int nr = (int)min((int64_t)ROWS, n1 - i0);
    const int32_t inf = c.inf;
    const TabAcc U = resolve(d.U, c), L = resolve(d.L, c);
    const int tid = threadIdx.x;
    const int r = tid;
    const uint32_t mul = 1u << (shift & 31);
    if (tid < NCH) s_xmax[tid] = 0;
    if (tid == 0) s_wstar = -1;
    stage_bar_init(&s_bar);
    __syncthreads();
    StageBar sb{&s_bar, 0u};
    stage_rows<PT, NT>(sU, U, i0, nr, inf, sb);
    __syncthreads();
    int32_t ku = -1;
    int32_t xlast[NCH];
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch) xlast[ch] = 0;
    if (r < nr) {
#pragma unroll
        for (int k = 0; k <= P; ++k) {
            const int32_t x = sU[r * PT + k];
            if (x < inf) {
                ku = k;
                xlast[k / KC] = max(xlast[k / KC], x);
            }
        }
    }
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch) {
        const int32_t m = __reduce_max_sync(0xffffffffu, xlast[ch]);
        if ((tid & 31) == 0 && m > 0) atomicMax(&s_xmax[ch], m);
    }
    uint32_t W[40];
#pragma unroll
    for (int t = 0; t < 40; ++t) W[t] = ~0u;
    // chunk body: fold splits k0 + kk (kk < nk) into W[kk + e]
    auto chunk = [&](int ch, int k0, auto nk_c) {
        constexpr int NK = decltype(nk_c)::value;
        __syncthreads();  // previous window consumed / U block and xmax ready
        const int32_t x0 = sU[k0];
        if (x0 >= inf) return false;  // CTA-uniform: no finite split from here on
        const int64_t base = (int64_t)x0 - 1;
        const int64_t need = (int64_t)s_xmax[ch] - base;
        for (int64_t w0 = 0; w0 < need; w0 += lcap) {
            const int32_t nL = (int32_t)min(need - w0, (int64_t)lcap);
            if (w0 > 0) __syncthreads();
            const int sh = L.nx ? 0 : (int)(((uintptr_t)(L.reach + (base + w0) * PT) >> 2) & 3);
            int32_t *sLw = sL + sh;
            stage_rows_call<PT, NT>(sLw, L, base + w0, nL, inf, sb);
            __syncthreads();
            if (r < nr) {
#pragma unroll
                for (int kk = 0; kk < NK; ++kk) {
                    const int32_t k = k0 + kk;
                    const int32_t x = sU[r * PT + k];
                    const int64_t lr = (int64_t)x - 1 - base - w0;
                    if (x < inf && lr >= 0 && lr < nL) {
                        const int32_t *row = sLw + lr * PT;
#pragma unroll
                        for (int e = 0; e <= P; ++e) {
                            const uint32_t key = (uint32_t)row[e] * mul + (uint32_t)k;
                            W[kk + e] = key < W[kk + e] ? key : W[kk + e];
                        }
                    }
                }
            }
            if (w0 + lcap < need) __syncthreads();
        }
        return true;
    };
    // every chunk runs (a chunk without finite splits folds nothing) so that
    // the window always ends aligned to column 32
#pragma unroll 1
    for (int ch = 0; ch < 4; ++ch) {
        chunk(ch, ch * KC, std::integral_constant<int, KC>{});
        // columns 8ch .. 8ch+7 are final: park them in this row's consumed
        // split slots, shift the window (also when the chunk had no split:
        // the parked keys are then the untouched ~0 = INF)
        __syncthreads();  // every thread is done reading row 0's slot 8ch
        if (r < nr) {
#pragma unroll
            for (int t = 0; t < KC; ++t) sU[r * PT + ch * KC + t] = (int32_t)W[t];
        }
#pragma unroll
        for (int t = 0; t < 32; ++t) W[t] = W[t + 8];
#pragma unroll
        for (int t = 32; t < 40; ++t) W[t] = ~0u;
    }
    chunk(4, 32, std::integral_constant<int, 1>{});
    __syncthreads();  // folds done; sU keeps the parked columns 0..31
    const int32_t w1 = FW ? 2 * P + 1 : d.w1, w = w1 - 1;
    const int32_t wstar_l = *d.L.wstar;
    int32_t *__restrict__ const out_kmax = d.out_kmax;
    int32_t *__restrict__ const out_reach = d.out_reach;
    int32_t *__restrict__ const out_trace = d.out_trace;
    int32_t *const out_wstar = d.out_wstar;
    // all 65 keys of the row into registers (the staging area overlaps sU)
    uint32_t best[2 * P + 1];
    if (r < nr) {
#pragma unroll
        for (int j = 0; j < 32; ++j) best[j] = (uint32_t)sU[r * PT + j];
    }
#pragma unroll
    for (int j = 32; j <= 2 * P; ++j) best[j] = W[j - 32];
    __syncthreads();
    int32_t *sR = nsm;
    int32_t *sT = nsm + ROWS * w1;
    int32_t wmax = -1;
    if (r < nr) {
        int32_t *rr = sR + r * w1;
        int32_t *tr = sT + r * w1;
        int32_t kfin = -1;
#pragma unroll
        for (int j = 0; j <= 2 * P; ++j) {
            if (j <= w) {
                const uint32_t vk = best[j] >> shift;
                const int32_t v = vk < (uint32_t)inf ? (int32_t)vk : inf;
                if (v < inf) kfin = j;
                rr[j] = v;
                tr[j] = (int32_t)(best[j] & ((1u << shift) - 1));
            }
        }
        inf_traces(tr, kfin, min(w, ku + wstar_l), w);
        out_kmax[i0 + r] = kfin;
        wmax = kfin;
    }
    wmax = __reduce_max_sync(0xffffffffu, wmax);
    if ((tid & 31) == 0 && wmax >= 0) atomicMax(&s_wstar, wmax);
    __syncthreads();
    const int tot = nr * w1;
    copy_out_rows<NT>(out_reach + i0 * w1, out_trace ? out_trace + i0 * w1 : nullptr, sR, sT, tot);
    if (tid == 0 && s_wstar >= 0) atomicMax(out_wstar, s_wstar);
    bulk_store_drain();
}

template <bool FW>
static int launch_narrow32_roll(const CombineDesc *descs, int32_t ndesc, Ctx c, int shift,
                                cudaStream_t s) {
    cudaError_t e = cudaFuncSetAttribute(narrow32_roll_kernel<FW>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, R32_BYTES);
    if (e != cudaSuccess) return (int)e;
    const int64_t n1 = (int64_t)c.n + 1;
    const int32_t bpd = (int32_t)((n1 + R32_NT - 1) / R32_NT);
    const int32_t lcap = (int32_t)(R32_BYTES / 4 - R32_NT * R32_PT - 3) / R32_PT;
    const int64_t blocks = (int64_t)ndesc * bpd;
    if (blocks == 0) return 0;
    if (blocks >= ((int64_t)1 << 31)) return (int)cudaErrorInvalidConfiguration;
    narrow32_roll_kernel<FW><<<(unsigned)blocks, R32_NT, R32_BYTES, s>>>(descs, c, shift, bpd, lcap);
    return (int)cudaGetLastError();
}

// Height-1 combines (two leaf children, rows of 3 cells): the fold needs only
// NX_a[i], NX_b[i] and NX_b[NX_a[i] - 1] (breakout.py:37-55 leaf rows), all in
// L2 (26 symbols x (n+1) ints), so nothing is staged on the way in; rows
// still leave through the shared-memory transpose.  Same first-wins values,
// traces and INF replay as narrow_combine_kernel<1>.
constexpr int LP_NT = 256, LP_RPT = 4, LP_ROWS = LP_NT * LP_RPT;

// W3: the output width is 3 (n >= 2, every leaf is 2 wide) -- constant
// shared-memory offsets and a closed-form INF replay
template <typename Key, bool W3>
__global__ void __launch_bounds__(LP_NT)
    narrow_leafpair_kernel(const CombineDesc *__restrict__ descs, Ctx c, int shift, int32_t bpd) {
    __shared__ __align__(16) int32_t sR[LP_ROWS * 3];
    __shared__ __align__(16) int32_t sT[LP_ROWS * 3];
    __shared__ int32_t s_wstar;
    const int32_t di = blockIdx.x / bpd;
    const int64_t i0 = (int64_t)(blockIdx.x - di * bpd) * LP_ROWS;
    const CombineDesc &d = descs[di];
    const int64_t n1 = (int64_t)c.n + 1;
    const int nr = (int)min((int64_t)LP_ROWS, n1 - i0);
    const int32_t inf = c.inf;
    const TabAcc U = resolve(d.U, c), L = resolve(d.L, c);  // both leaves
    const int32_t w1 = W3 ? 3 : d.w1, w = w1 - 1;
    const int32_t wstar_l = *d.L.wstar;
    int32_t *__restrict__ const out_kmax = d.out_kmax;
    int32_t *__restrict__ const out_reach = d.out_reach;
    int32_t *__restrict__ const out_trace = d.out_trace;
    const uint32_t mul = 1u << (shift & 31);
    const int tid = threadIdx.x;
    if (tid == 0) s_wstar = -1;
    int32_t wmax = -1;
#pragma unroll
    for (int q = 0; q < LP_RPT; ++q) {
        const int r = tid + q * LP_NT;
        if (r >= nr) continue;
        const int64_t i = i0 + r;
        // U row (i+1, NX_a[i]); L row x-1: (x, NX_b[x-1])
        const int32_t xa = (W3 || U.w1 > 1) ? __ldg(U.nx + i) : inf;
        const int32_t nb = (W3 || L.w1 > 1) ? __ldg(L.nx + i) : inf;
        const int32_t nb2 = (xa < inf && (W3 || L.w1 > 1)) ? __ldg(L.nx + (xa - 1)) : inf;
        // candidates (k, e): j = k + e; first-wins min of packed keys
        Key best[3];
        best[0] = npack((Key)(uint32_t)(i + 1), 0, shift, mul);  // (0,0): L[i][0] = i+1
        const Key k01 = npack((Key)(uint32_t)nb, 0, shift, mul);           // (0,1): L[i][1]
        const Key k10 = npack((Key)(uint32_t)(xa < inf ? xa : inf), 1, shift, mul);  // (1,0)
        best[1] = k01 < k10 ? k01 : k10;
        best[2] = npack((Key)(uint32_t)nb2, 1, shift, mul);              // (1,1)
        const int32_t ku = xa < inf ? 1 : 0;
        int32_t kfin = -1;
        int32_t *rr = sR + r * w1;
        int32_t *tr = sT + r * w1;
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            if (j <= w) {
                const Key vk = best[j] >> shift;
                const int32_t v = vk < (Key)(uint32_t)inf ? (int32_t)vk : inf;
                if (v < inf) kfin = j;
                rr[j] = v;
                tr[j] = (int32_t)(best[j] & (((Key)1 << shift) - 1));
            }
        }
        if (W3) {
            // Alg. 1 over [0, colhi], w = 2: its first mid is 1; finite (kfin
            // >= 1) -> the only INF cell left is 2, in the node with top =
            // trace[1]; INF -> every INF node keeps top = 0; 0 beyond colhi
            const int32_t colhi = min(2, ku + wstar_l);
            const int32_t top = kfin >= 1 ? tr[1] : 0;
#pragma unroll
            for (int j = 0; j < 3; ++j)
                if (j > kfin) tr[j] = j <= colhi ? top : 0;
        } else {
            inf_traces(tr, kfin, min(w, ku + wstar_l), w);  // Alg. 1 replay for INF cells
        }
        out_kmax[i] = kfin;
        wmax = max(wmax, kfin);
    }
    wmax = __reduce_max_sync(0xffffffffu, wmax);
    if ((tid & 31) == 0 && wmax >= 0) atomicMax(&s_wstar, wmax);
    __syncthreads();
    const int tot = nr * w1;
    copy_out_rows<LP_NT>(out_reach + i0 * w1, out_trace ? out_trace + i0 * w1 : nullptr, sR, sT,
                         tot);
    if (tid == 0 && s_wstar >= 0) atomicMax(d.out_wstar, s_wstar);
    bulk_store_drain();
}

int launch_narrow_leafpair(const CombineDesc *descs, int32_t ndesc, Ctx c, int shift, bool key64,
                           cudaStream_t s) {
    const int64_t n1 = (int64_t)c.n + 1;
    const int32_t bpd = (int32_t)((n1 + LP_ROWS - 1) / LP_ROWS);
    const int64_t blocks = (int64_t)ndesc * bpd;
    if (blocks == 0) return 0;
    if (blocks >= ((int64_t)1 << 31)) return (int)cudaErrorInvalidConfiguration;
    const bool w3 = c.n >= 2;  // every height-1 output is 3 wide
    if (key64) {
        if (w3) narrow_leafpair_kernel<uint64_t, true><<<(unsigned)blocks, LP_NT, 0, s>>>(descs, c, shift, bpd);
        else narrow_leafpair_kernel<uint64_t, false><<<(unsigned)blocks, LP_NT, 0, s>>>(descs, c, shift, bpd);
    } else {
        if (w3) narrow_leafpair_kernel<uint32_t, true><<<(unsigned)blocks, LP_NT, 0, s>>>(descs, c, shift, bpd);
        else narrow_leafpair_kernel<uint32_t, false><<<(unsigned)blocks, LP_NT, 0, s>>>(descs, c, shift, bpd);
    }
    return (int)cudaGetLastError();
}

template <int P, typename Key, bool FW = false>
static int launch_narrow_t(const CombineDesc *descs, int32_t ndesc, Ctx c, int shift,
                           cudaStream_t s) {
    using G = NarrowGeom<P>;
    constexpr int PT = G::PITCH, BYTES = G::BYTES;
    cudaError_t e = cudaFuncSetAttribute(narrow_combine_kernel<P, Key, FW>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, BYTES);
    if (e != cudaSuccess) return (int)e;
    const int64_t n1 = (int64_t)c.n + 1;
    const int32_t bpd = (int32_t)((n1 + G::ROWS - 1) / G::ROWS);
    // L window rows: whatever the budget leaves after the U block
    const int32_t lcap = (int32_t)(BYTES / 4 - G::ROWS * PT - 3) / PT;  // 3: window shift
    const int64_t blocks = (int64_t)ndesc * bpd;
    if (blocks == 0) return 0;
    if (blocks >= ((int64_t)1 << 31)) return (int)cudaErrorInvalidConfiguration;
    narrow_combine_kernel<P, Key, FW><<<(unsigned)blocks, G::NT, BYTES, s>>>(descs, c, shift, bpd,
                                                                             lcap);
    return (int)cudaGetLastError();
}

int narrow_bucket(int32_t max_weight) {
    int P = 1;
    while (P < max_weight) P *= 2;
    return P <= 32 ? P : -1;
}

int launch_narrow(const CombineDesc *descs, int32_t ndesc, Ctx c, int shift, bool key64,
                  int32_t P, cudaStream_t s, bool full_width) {
#define NARROW_CASE(PP)                                                              \
    case PP:                                                                         \
        if (full_width && !key64) return launch_narrow_t<PP, uint32_t, true>(descs, ndesc, c, shift, s); \
        return key64 ? launch_narrow_t<PP, uint64_t>(descs, ndesc, c, shift, s)      \
                     : launch_narrow_t<PP, uint32_t>(descs, ndesc, c, shift, s);
    switch (P) {
        NARROW_CASE(1)
        NARROW_CASE(2)
        NARROW_CASE(4)
        NARROW_CASE(8)
        NARROW_CASE(16)
        case 32: {
            const char *e = getenv("LCSG_NARROW32_ROLL");
            if (!key64 && (e == nullptr || atoi(e) != 0))
                return full_width ? launch_narrow32_roll<true>(descs, ndesc, c, shift, s)
                                  : launch_narrow32_roll<false>(descs, ndesc, c, shift, s);
            return key64 ? launch_narrow_t<32, uint64_t>(descs, ndesc, c, shift, s)
                         : launch_narrow_t<32, uint32_t>(descs, ndesc, c, shift, s);
        }
        default:
            return (int)cudaErrorInvalidValue;
    }
#undef NARROW_CASE
}

}  // namespace lcsg
