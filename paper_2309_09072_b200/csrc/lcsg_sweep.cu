// lcsg_sweep.cu -- row-sweep generation of the wide combines' interior rows.
//
// A slab table is the inverse of a unit-Monge LCS score matrix, so consecutive
// rows differ by one event: with S_c = {reach[c][j]} (sorted, S_c[0] = c+1),
//     S_{c+1} = S_c \ {c+1} + {t_c},
// i.e. row c+1 is row c with the prefix [1, j1] shifted left by one and one new
// element t_c inserted at rank j1 (none when t_c = INF).  For the combine
// C = U (x) L (solver.py:91-110, _kernel.pyx:28-82) the first-wins split
// k*(c,j) obeys the same structure (derivation and proof sketch in DESIGN.md 5b;
// checked bit-exact against the reference on every test input):
//   * cells right of the insertion whose split lies right of U's own
//     insertion rank ju1 (trace[c][j] > ju1): value and trace unchanged;
//   * cells left of the insertion: value = C[c][j+1], trace = trace[c][j+1]-1
//     (while that trace is >= 1);
//     (a zero trace stays zero: k = 0 still reaches the value through L's own
//     shift);
//   * only the cells between (j1 <= j <= J, J = last j with trace[c][j] <= ju1)
//     need candidates evaluated, each over a split range bounded by ju1 below
//     and by its right neighbour's split above.
// So a row costs a handful of L gathers plus a streaming rewrite of the row
// instead of a search per cell.  The chain over rows is cut by the skeleton
// rows (exact Alg. 1 every S rows, lcsg_refine.cu): one thread group sweeps
// the S-1 interior rows below a skeleton row.  Two kernels: the
// register-resident one (row state in registers; the fast path, below) and a
// generic one (row state ping-ponged in shared memory, or kept in the output
// rows themselves when the finite prefix does not fit; 64-bit keys) that
// also redoes the blocks the fast path flags.
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

// consistency violations seen by the sweep (a non-zero value means a row
// failed one of the structural invariants; tests read it through
// lcsg_sweep_errors and fail loudly)
__device__ int32_t g_sweep_err = 0;
// path counters (tests assert the fallback paths really run): blocks redone by
// the generic kernel after a register-kernel flag, blocks swept with the row
// state in the output rows (finite prefix beyond the shared-memory capacity)
__device__ unsigned long long g_sweep_paths[2];
#ifdef LCSG_SWEEP_STATS
// per launch-size class (log2 of group threads - 5): row steps, evaluation
// rounds, walk cells, splits per cell
__device__ unsigned long long g_sweep_stat[8][8];
#define SW_STAT(cls, idx, val) atomicAdd(&g_sweep_stat[cls][idx], (unsigned long long)(val))
#else
#define SW_STAT(cls, idx, val) do {} while (0)
#endif

namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr uint64_t KEY_NONE = ~(uint64_t)0;

// Insertion rank of row c+1 against row c of a materialised table: the first
// k in [0, kmax[c+1]] with reach[c+1][k] != reach[c][k+1] (the predicate is
// monotone: equal below the insertion, different from it on), kmax[c+1]+1
// when nothing was inserted.  One thread per row, binary search.
__global__ void __launch_bounds__(256)
    table_events_kernel(const CombineDesc *__restrict__ descs, int32_t ndesc, Ctx c) {
    const int32_t di = blockIdx.y;
    if (di >= ndesc) return;
    const CombineDesc &d = descs[di];
    if (!d.U_ev_make) return;
    const int32_t row = (int32_t)(blockIdx.x * blockDim.x + threadIdx.x);
    if (row >= c.n) return;
    const int32_t w1 = d.U.w1;
    const int32_t *a = d.U.reach + (size_t)row * w1, *b = a + w1;
    const int32_t kb = __ldg(d.U.kmax + row + 1);
    int32_t lo = 0, hi = kb + 1;  // answer in [lo, hi]
    while (lo < hi) {
        const int32_t md = (lo + hi) >> 1;
        if (__ldg(b + md) != __ldg(a + md + 1)) hi = md; else lo = md + 1;
    }
    d.U_ev[row] = lo;
}

// last j in [0, K] with T[j] <= thr; T is nondecreasing on [0, K] and
// T[0] <= thr.  Warp-cooperative 32-ary search (all lanes get the result).
__device__ __forceinline__ int32_t warp_last_le(const int32_t *T, int32_t K, int32_t thr, int lane) {
    int32_t lo = 0, hi = K + 1;
    while (hi - lo > 1) {
        const int32_t step = (hi - lo - 1 + 31) >> 5;
        const int32_t p = lo + (lane + 1) * step;
        const bool ok = p < hi && T[p] <= thr;
        const int cnt = __popc(__ballot_sync(FULL, ok));
        lo += cnt * step;
        hi = min(hi, lo + step);
    }
    return lo;
}

__device__ __forceinline__ uint64_t warp_min64(uint64_t v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const uint64_t t = __shfl_xor_sync(FULL, v, o);
        v = t < v ? t : v;
    }
    return v;
}

constexpr int SW_MAXQ = 64;  // cells evaluated per round
constexpr int SW_SEG = 64;   // prefetched U entries from the insertion rank on

__device__ __forceinline__ void cp_async4(void *smem, const void *gmem) {
    const uint32_t sa = (uint32_t)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
}

// One thread group (the CTA) sweeps the rows (a, a+S) of one combine.  Per
// step (row cr -> cr+1): every warp locates J in the shared row state, all
// threads evaluate the candidate (cell, split) pairs of the cells J, J-1, ...
// at once (one round of dependent L gathers; keys reduce per cell with
// shared-memory atomicMin), every warp reads off the insertion rank j1, and
// all threads rewrite / store the row.  The U-side inputs of the next step
// (insertion rank, kmax, the U entries from the rank on) are fetched a step
// ahead with cp.async.
__global__ void sweep_kernel(const CombineDesc *__restrict__ descs, int32_t ndesc, Ctx c, int32_t S,
                             int32_t nblk, int32_t cap, int flagged_only) {
    extern __shared__ int32_t ssm[];  // R0[cap] T0[cap] R1[cap] T1[cap] evs[S] kms[S]
    __shared__ unsigned long long cellkey[2][SW_MAXQ];
    __shared__ int32_t useg[2][SW_SEG];
    const int32_t di = (int32_t)(blockIdx.z * 65535u + blockIdx.y);
    if (di >= ndesc) return;
    const int32_t blk = blockIdx.x;
    const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31;
    const CombineDesc &d = descs[di];
    const int32_t n = c.n, inf = c.inf;
    const int32_t a = blk * S;
    if (a >= n) return;
    if (flagged_only && !d.blk_flags[blk]) return;  // the register kernel did this block
    const int32_t nsteps = min(S, n - a);  // rows a+1 .. a+nsteps; the last one is a skeleton row
    const int32_t w1 = d.w1, uw1 = d.U.w1, lw1 = d.L.w1, wl = lw1 - 1;
    const int32_t *__restrict__ Ur = d.U.reach;
    const int32_t *__restrict__ Lr = d.L.reach;
    int32_t *const out_reach = d.out_reach;
    int32_t *const out_trace = d.out_trace;
    int32_t *const out_ev = d.out_ev;
    int32_t *const evs = ssm + 4 * (size_t)cap, *const kms = evs + S;

    int32_t K = d.out_kmax[a];  // written by the skeleton kernel
    const bool in_smem = K + 2 <= cap;
    if (tid == 0) {
        if (flagged_only) atomicAdd(&g_sweep_paths[0], 1ull);
        if (!in_smem) atomicAdd(&g_sweep_paths[1], 1ull);
    }
    // row state: old = row c, new = row c+1
    int32_t *oR, *oT, *nR, *nT;
    if (in_smem) {
        oR = ssm;
        oT = ssm + cap;
        nR = ssm + 2 * (size_t)cap;
        nT = ssm + 3 * (size_t)cap;
        const int32_t *gr = out_reach + (size_t)a * w1, *gt = out_trace + (size_t)a * w1;
        for (int32_t j = tid; j <= K; j += nt) {
            oR[j] = gr[j];
            oT[j] = gt[j];
        }
    } else {
        oR = out_reach + (size_t)a * w1;
        oT = out_trace + (size_t)a * w1;
        nR = oR + w1;
        nT = oT + w1;
    }
    for (int32_t t = tid; t < nsteps; t += nt) {
        evs[t] = d.U_ev[a + t];
        kms[t] = d.U.kmax[a + t + 1];
    }
    for (int t = tid; t < 2 * SW_MAXQ; t += nt) cellkey[0][t] = KEY_NONE;
    __syncthreads();
    for (int t = tid; t < SW_SEG; t += nt) {
        const int32_t k = evs[0] + t;
        if (k <= kms[0]) useg[0][t] = Ur[(size_t)(a + 1) * uw1 + k];
    }
    __syncthreads();

    for (int32_t st = 0; st < nsteps; ++st) {
        const int32_t cr = a + st;  // row cr -> row cr + 1
        const bool dowrite = st + 1 < nsteps;
        const int32_t ju1 = evs[st], kmU = kms[st];
        const int32_t *Uc = Ur + (size_t)(cr + 1) * uw1;
        const int32_t *seg = useg[st & 1];
        unsigned long long *ck = cellkey[st & 1];
        if (dowrite)  // the next step's U entries, a step ahead
            for (int t = tid; t < SW_SEG; t += nt) {
                const int32_t k = evs[st + 1] + t;
                if (k <= kms[st + 1]) cp_async4(&useg[(st + 1) & 1][t], Uc + uw1 + k);
            }
        const int32_t J = warp_last_le(oT, K, ju1, lane);
        int32_t jb = J;
        int32_t ubR = J < K ? oT[J + 1] : INT_MAX;
        int32_t j1 = -1, Qc = 0;
        int32_t qcap = 8;  // most walks are short: few speculative cells first
        while (true) {
            const int32_t ub0 = min(kmU, ubR);
            const int32_t lmax = ub0 - ju1 + 1;  // splits per cell (before the j clamps)
            const int32_t ls = max(lmax, 1);
            Qc = min(min(jb + 1, qcap), max(4, 2 * nt / ls));
            qcap = SW_MAXQ;
            const int32_t npair = Qc * ls;
            for (int32_t p = tid; p < npair; p += nt) {
                const int32_t q = p / ls, r = p - q * ls;
                const int32_t j = jb - q, k = ju1 + r;
                if (r < lmax && k <= j && j - k <= wl) {
                    const int32_t x = r < SW_SEG ? seg[r] : Uc[k];  // finite: k <= kmax_U
                    const int32_t v = Lr[(size_t)(x - 1) * lw1 + (j - k)];
                    atomicMin(&ck[q], ((unsigned long long)(uint32_t)v << 32) | (uint32_t)k);
                }
            }
            __syncthreads();
            // every warp reads off the first cell (from the right) whose value changed
            int first = -1;
            for (int32_t q0 = 0; q0 < Qc && first < 0; q0 += 32) {
                const int32_t q = q0 + lane;
                bool chg = false;
                if (q < Qc) {
                    const unsigned long long my = ck[q];
                    chg = !(my != KEY_NONE && (int32_t)(my >> 32) < inf &&
                            (int32_t)(my >> 32) == oR[jb - q]);
                }
                const unsigned nb = __ballot_sync(FULL, chg);
                if (nb) first = q0 + __ffs(nb) - 1;
            }
            if (first >= 0) {
                j1 = jb - first;
                break;
            }
            // all Qc cells kept their value (new splits): store them, go further left
            ubR = (int32_t)(uint32_t)ck[Qc - 1];
            if (dowrite)
                for (int32_t q = tid; q < Qc; q += nt) {  // a round may hold more cells than threads
                    nR[jb - q] = (int32_t)(ck[q] >> 32);
                    nT[jb - q] = (int32_t)(uint32_t)ck[q];
                }
            __syncthreads();
            for (int32_t q = tid; q < Qc; q += nt) ck[q] = KEY_NONE;
            __syncthreads();
            jb -= Qc;
            if (jb < 0) {  // cannot happen: cell 0 always changes (c+1 -> c+2)
                if (tid == 0) atomicAdd(&g_sweep_err, 1);
                j1 = 0;
                jb = 0;
                break;
            }
        }
        // cells j1 .. jb are in ck (q = jb - j), cells (jb, J] already in nR / nT
        const unsigned long long newkey = ck[jb - j1];
        int32_t nv = newkey == KEY_NONE ? inf : (int32_t)(newkey >> 32);
        const int32_t nk = (int32_t)(uint32_t)newkey;
        if (nv >= inf) {
            nv = inf;
            if (j1 != K && tid == 0) atomicAdd(&g_sweep_err, 1);
        }
        const int32_t Knew = nv < inf ? K : K - 1;
        if (tid == 0) out_ev[cr] = j1;
        if (!dowrite) break;
        {
            int32_t *gR = out_reach + (size_t)(cr + 1) * w1, *gT = out_trace + (size_t)(cr + 1) * w1;
            for (int32_t j = tid; j < w1; j += nt) {
                if (j <= Knew) {
                    int32_t v, t;
                    if (j >= j1 && j <= jb) {  // this round's cells
                        const unsigned long long key = ck[jb - j];
                        v = (int32_t)(key >> 32);
                        t = (int32_t)(uint32_t)key;
                    } else if (j > jb && j <= J) {  // cells of earlier rounds
                        if (!in_smem) continue;  // already in the output row
                        v = nR[j];
                        t = nT[j];
                    } else if (j < j1) {
                        v = oR[j + 1];
                        t = max(oT[j + 1] - 1, 0);  // a zero split stays zero (k = 0 still wins)
                    } else {
                        v = oR[j];
                        t = oT[j];
                    }
                    if (in_smem) {
                        nR[j] = v;
                        nT[j] = t;
                    }
                    gR[j] = v;
                    gT[j] = t;
                } else {
                    gR[j] = inf;  // INF suffix: its traces are the finalize kernel's
                }
            }
            if (tid == 0) d.out_kmax[cr + 1] = Knew;
            K = Knew;
        }
        for (int t = tid; t < SW_MAXQ; t += nt) cellkey[(st + 1) & 1][t] = KEY_NONE;
        cp_async_wait_all();
        __syncthreads();
        if (in_smem) {
            int32_t *t0 = oR, *t1 = oT;
            oR = nR;
            oT = nT;
            nR = t0;
            nT = t1;
        } else {
            oR = nR;
            oT = nT;
            nR += w1;
            nT += w1;
        }
    }
}


// ---------------------------------------------------------------------------
// Register-resident sweep (the fast path).  A group of gn threads (one warp,
// four groups per CTA; or a whole CTA) owns a block of rows; thread gt keeps
// CPT cells of the current row in registers -- reach R[i] and split T[i],
// (INF, INT_MAX) beyond the finite prefix.  Per step: J comes from per-thread
// counts (the splits are nondecreasing along a row); all threads evaluate the
// (cell, split) pairs of the walk at once (keys reduce with shared-memory
// atomicMin); the owners of the walk cells compare and the largest changed
// cell is j1; the row is rewritten in registers (neighbour cell by shuffle)
// and stored.  Anything outside the fast path's bounds (finite prefix wider
// than gn * CPT, walks longer than the key array, a broken invariant) flags
// the block; the generic kernel above then redoes flagged blocks.
// ---------------------------------------------------------------------------
constexpr int RG_SEG = 32;   // prefetched U entries from the insertion rank on
constexpr int RG_MAXS = 128;  // rows per block
constexpr uint32_t K32_NONE = 0xffffffffu;

// CKN: evaluated cells per step kept as keys (bounds the walk and the
// zero-split run)
template <int CKN>
struct RegGroupSm {
    uint32_t ck[2][CKN];   // walk cells: key of cell j at [J - j]
    int32_t useg[2][RG_SEG];
    int32_t evs[RG_MAXS], kms[RG_MAXS];
    int32_t cnt[2][4];     // counts (cA | cZ << 16), min split > ju1, min split > 0, j1
    int32_t edgeR[2][32], edgeT[2][32];  // first cell of every warp (its left neighbour's neighbour)
};

template <bool MULTI>
__device__ __forceinline__ void gsync() {
    if (MULTI) __syncthreads(); else __syncwarp();
}

__device__ __forceinline__ int ceil_log2(int32_t x) { return x <= 1 ? 0 : 32 - __clz(x - 1); }

// Cell ownership: warp gw of the group holds the cells [gw*32*CPT, (gw+1)*32*CPT),
// lane-strided: j = gw*32*CPT + lane + 32*i.  The right neighbour of a cell is
// the next lane's (same i), or lane 0's cell i+1 -- shuffles only; the warp's
// very last cell takes the next warp's first cell from shared memory.
// Keys are 32-bit (value << shift | split): the host routes combines whose
// keys need 64 bits to the generic kernel.
//
// A step costs three group barriers: (A) counts -> J and the split bound
// right of it (the splits are nondecreasing along a row, so "last cell with
// split <= x" is a count and "split of the next cell" a minimum); (P) all
// threads evaluate the (cell, split) pairs of the walk left of J (one round of
// dependent L gathers, 32-bit shared-memory atomicMin per cell); (D) the
// owners of the walk cells compare the new value with their old one and the
// largest changed cell is j1.  Longer walks take further rounds (two barriers
// each).
template <int CPT, bool MULTI>
__device__ __forceinline__ void
    sweep_reg_body(const CombineDesc *__restrict__ descs, int32_t ndesc, Ctx c, int32_t S,
                     int32_t nblk, int shift, int64_t ngroups, int flagged_only) {
    constexpr int GPB = MULTI ? 1 : 4;  // groups per CTA
    constexpr int CKN = MULTI ? 512 : 128;
    constexpr int QMAX = MULTI ? 256 : 32;  // cells per round
    using Sm = RegGroupSm<CKN>;
    __shared__ Sm gsm_all[GPB];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int gi = MULTI ? 0 : warp;
    const int gt = MULTI ? (int)threadIdx.x : lane;
    const int gn = MULTI ? (int)blockDim.x : 32;
    const int gw = MULTI ? warp : 0, nw = gn >> 5;
    const int64_t g = (int64_t)blockIdx.x * GPB + gi;
    if (g >= ngroups) return;
    const int32_t di = (int32_t)(g / nblk);
    const int32_t blk = (int32_t)(g - (int64_t)di * nblk);
    Sm &sm = gsm_all[gi];
    const CombineDesc &d = descs[di];
    const int32_t n = c.n, inf = c.inf;
    const int32_t a = blk * S;
    if (a >= n) return;
    const int32_t nsteps = min(S, n - a);
    const int32_t w1 = d.w1, uw1 = d.U.w1, lw1 = d.L.w1, wl = lw1 - 1;
    const int32_t *__restrict__ Ur = d.U.reach;
    const int32_t *__restrict__ Lr = d.L.reach;
    int32_t *const out_reach = d.out_reach;
    int32_t *const out_trace = d.out_trace;
    int32_t *const out_ev = d.out_ev;
    int32_t *const flag = d.blk_flags + blk;
    int32_t *const out_kmax = d.out_kmax;
    const int32_t capc = gn * CPT;        // cells held in registers
    const int32_t wbase = gw * 32 * CPT;  // first cell of this warp
    const int32_t jl = wbase + lane;      // this thread's cell 0
    const uint32_t kmask = (1u << shift) - 1u;

    // second pass of the cascade (wider groups): only the blocks the first flagged
    if (flagged_only) {
        if (!*flag) return;
        gsync<MULTI>();
        if (gt == 0) *flag = 0;
    }
    int32_t K = d.out_kmax[a];  // written by the skeleton kernel
    if (K + 1 > capc) {
        if (gt == 0) *flag = 1;
        return;
    }
    int32_t R[CPT], T[CPT];
    {
        const int32_t *gr = out_reach + (size_t)a * w1, *gtr = out_trace + (size_t)a * w1;
#pragma unroll
        for (int i = 0; i < CPT; ++i) {
            const int32_t j = jl + 32 * i;
            R[i] = j <= K ? gr[j] : inf;
            T[i] = j <= K ? gtr[j] : INT_MAX;
        }
    }
    for (int32_t t = gt; t < nsteps; t += gn) {
        sm.evs[t] = d.U_ev[a + t];
        sm.kms[t] = d.U.kmax[a + t + 1];
    }
    for (int t = gt; t < 2 * CKN; t += gn) sm.ck[0][t] = K32_NONE;
    if (gt < 8) sm.cnt[0][gt] = (gt & 3) == 0 ? 0 : ((gt & 3) == 3 ? -1 : INT_MAX);
    gsync<MULTI>();
    if (gt < RG_SEG) {
        const int32_t k = sm.evs[0] + gt;
        if (k <= sm.kms[0]) sm.useg[0][gt] = Ur[(size_t)(a + 1) * uw1 + k];
    }
    gsync<MULTI>();

#define RG_FALLBACK()                 \
    do {                              \
        if (gt == 0) *flag = 1;       \
        cp_async_wait_all();          \
        return;                       \
    } while (0)

    int32_t dirty_other = 0;  // key slots of the other buffer that are in use
    for (int32_t st = 0; st < nsteps; ++st) {
        const int par = st & 1;
        const int32_t cr = a + st;  // row cr -> row cr + 1
        const bool dowrite = st + 1 < nsteps;
        const int32_t ju1 = sm.evs[st], kmU = sm.kms[st];
        const int32_t *Uc = Ur + (size_t)(cr + 1) * uw1;
        const int32_t *seg = sm.useg[par];
        uint32_t *ck = sm.ck[par];
        // ---- A. J and the split bound right of it ----
        if (MULTI && lane == 0) {
            sm.edgeR[par][gw] = R[0];
            sm.edgeT[par][gw] = T[0];
        }
        int32_t J, ubR;
        {
            int32_t cA = 0, mA = INT_MAX;
#pragma unroll
            for (int i = 0; i < CPT; ++i) {
                const int32_t t = T[i];
                cA += t <= ju1;
                mA = t > ju1 ? min(mA, t) : mA;
            }
            cA = __reduce_add_sync(FULL, cA);
            mA = __reduce_min_sync(FULL, mA);
            if (MULTI) {
                if (lane == 0) {
                    atomicAdd(&sm.cnt[par][0], cA);
                    atomicMin(&sm.cnt[par][1], mA);
                }
                __syncthreads();
                cA = sm.cnt[par][0];
                mA = sm.cnt[par][1];
                if (gt < 4) sm.cnt[par ^ 1][gt] = gt == 0 ? 0 : (gt == 3 ? -1 : INT_MAX);
            }
            J = cA - 1;
            ubR = mA;  // split of cell J + 1 (INT_MAX: none)
        }
        if (dowrite && gt < RG_SEG) {  // the next step's U entries, a step ahead
            const int32_t e1 = sm.evs[st + 1], k1 = sm.kms[st + 1];
            if (e1 + gt <= k1) cp_async4(&sm.useg[par ^ 1][gt], Uc + uw1 + e1 + gt);
        }
        // ---- P / D. the walk left of J: evaluate cells until one changes value ----
        int32_t jb = J, j1 = -1, dirty_this = 0;
        for (int round = 0;; ++round) {
            const int32_t ub0 = min(kmU, ubR);
            const int32_t lmax = ub0 - ju1 + 1;  // splits per cell (before the j clamps)
            const int lgs = ceil_log2(lmax);
            const int32_t qwant =
                round == 0 ? max(4, min(32, (MULTI ? 2 * gn : gn) >> lgs)) : (round == 1 ? 32 : QMAX);
            const int32_t Qc = min(min(jb + 1, qwant), CKN - (J - jb));
            if (Qc <= 0) RG_FALLBACK();
            const int32_t npA = Qc << lgs;
            for (int32_t p = gt; p < npA; p += gn) {
                const int32_t q = p >> lgs, r = p & ((1 << lgs) - 1);
                const int32_t j = jb - q, k = ju1 + r;
                if (r < lmax && k <= j && j - k <= wl) {
                    const int32_t x = r < RG_SEG ? seg[r] : Uc[k];  // finite: k <= kmax_U
                    const int32_t v = Lr[(size_t)(x - 1) * lw1 + (j - k)];
                    atomicMin(&ck[J - j], ((uint32_t)v << shift) | (uint32_t)k);
                }
            }
            gsync<MULTI>();
            // owners: the largest walk cell whose value changed
            const int32_t lo = jb - Qc + 1;
            dirty_this = J - lo + 1;  // key slots [0, J - lo] are in use
            int32_t found = -1;
            if (Qc <= 32) {  // at most one cell per thread
                const int32_t i0 = lo > jl ? (lo - jl + 31) >> 5 : 0;
                const int32_t j0 = jl + 32 * i0;
                if (i0 < CPT && j0 <= jb) {
                    int32_t r = inf;
#pragma unroll
                    for (int i = 0; i < CPT; ++i)
                        if (i == i0) r = R[i];
                    const uint32_t key = ck[J - j0];
                    const int32_t v = (int32_t)(key >> shift);
                    if (!(key != K32_NONE && v < inf && v == r)) found = j0;
                }
            } else {
#pragma unroll
                for (int i = 0; i < CPT; ++i) {
                    const int32_t j = jl + 32 * i;
                    if (j >= lo && j <= jb) {
                        const uint32_t key = ck[J - j];
                        const int32_t v = (int32_t)(key >> shift);
                        if (!(key != K32_NONE && v < inf && v == R[i])) found = max(found, j);
                    }
                }
            }
            found = __reduce_max_sync(FULL, found);
            if (MULTI) {
                if (lane == 0 && found >= 0) atomicMax(&sm.cnt[par][3], found);
                __syncthreads();
                found = sm.cnt[par][3];
            }
#ifdef LCSG_SWEEP_STATS
            if (gt == 0) SW_STAT(31 - __clz(gn) - 5, 1, 1);
#endif
            if (found >= 0) {
                j1 = found;
                break;
            }
            // all Qc cells kept their value (new splits): go further left
            ubR = (int32_t)(ck[J - lo] & kmask);
            jb = lo - 1;
            if (jb < 0) RG_FALLBACK();  // cannot happen: cell 0 always changes
        }
        const uint32_t newkey = ck[J - j1];
        const int32_t nv = newkey == K32_NONE ? inf : min((int32_t)(newkey >> shift), inf);
        const int32_t nk = (int32_t)(newkey & kmask);
        if (nv >= inf && j1 != K) RG_FALLBACK();
#ifdef LCSG_SWEEP_STATS
        if (gt == 0) {
            const int cls = 31 - __clz(gn) - 5;
            SW_STAT(cls, 0, 1);
            SW_STAT(cls, 2, J - j1 + 1);
            SW_STAT(cls, 3, max(0, min(kmU, ubR) - ju1 + 1));
        }
#endif
        const int32_t Knew = nv < inf ? K : K - 1;
        if (gt == 0) out_ev[cr] = j1;
        if (!dowrite) break;
        // ---- rewrite the row in registers and store it ----
        {
            int32_t *gR = out_reach + (size_t)(cr + 1) * w1, *gT = out_trace + (size_t)(cr + 1) * w1;
            // the next warp's first cell: neighbour of this warp's last cell
            const int32_t eR = (MULTI && gw + 1 < nw) ? sm.edgeR[par][gw + 1] : inf;
            const int32_t eT = (MULTI && gw + 1 < nw) ? sm.edgeT[par][gw + 1] : INT_MAX;
#pragma unroll
            for (int i = 0; i < CPT; ++i) {
                const int32_t cb = wbase + 32 * i;  // this warp's cells cb .. cb+31 (warp-uniform)
                const int32_t j = cb + lane;
                if (cb > K) continue;  // already (INF, none): the tail loop stores the INF cells
                if (cb > J && cb + 31 <= Knew) {  // all unchanged
                    if (j < w1) {
                        gR[j] = R[i];
                        gT[j] = T[i];
                    }
                    continue;
                }
                int32_t v = R[i], t = T[i];
                if (cb < j1) {  // some shifted cells: the right neighbour's old cell
                    const int32_t ra = __shfl_down_sync(FULL, R[i], 1), ta = __shfl_down_sync(FULL, T[i], 1);
                    const int32_t rb = __shfl_sync(FULL, i + 1 < CPT ? R[i + 1 < CPT ? i + 1 : i] : eR, 0);
                    const int32_t tb = __shfl_sync(FULL, i + 1 < CPT ? T[i + 1 < CPT ? i + 1 : i] : eT, 0);
                    if (j < j1) {
                        v = lane == 31 ? rb : ra;
                        t = max((lane == 31 ? tb : ta) - 1, 0);  // a zero split stays zero (k = 0 still wins)
                    }
                }
                if (j >= j1 && j <= J) {
                    const uint32_t key = ck[J - j];
                    v = (int32_t)(key >> shift);
                    t = (int32_t)(key & kmask);
                }
                if (j > Knew) {
                    v = inf;
                    t = INT_MAX;
                }
                R[i] = v;
                T[i] = t;
                if (j <= Knew) {
                    gR[j] = v;
                    gT[j] = t;
                }
            }
            // INF suffix (Knew, w1) of the reach row; its traces (the Alg. 1 replay's
            // and the zeros beyond colhi) are written by the finalize kernel from kmax
            if (gt == 0) out_kmax[cr + 1] = Knew;
            if (!MULTI) {
                for (int32_t j = Knew + 1 + gt; j < w1; j += 32) gR[j] = inf;
            } else {  // scalar stores up to a 16-byte boundary, then int4
                const int32_t j0 = Knew + 1;
                const int32_t head = (int32_t)((4 - (((uintptr_t)(gR + j0) >> 2) & 3)) & 3);  // the table base may be a row window
                const int32_t jv = min(j0 + head, w1);  // first aligned cell
                if (gt < jv - j0) gR[j0 + gt] = inf;
                const int32_t nv4 = (w1 - jv) >> 2;
                int4 *g4 = reinterpret_cast<int4 *>(gR + jv);
                const int4 inf4 = make_int4(inf, inf, inf, inf);
                for (int32_t q = gt; q < nv4; q += gn) g4[q] = inf4;
                const int32_t jt = jv + 4 * nv4;
                if (gt < w1 - jt) gR[jt + gt] = inf;
            }
            K = Knew;
        }
        // keys used two steps ago live in the other buffer: clear them for the next step
        if (gt < dirty_other) sm.ck[par ^ 1][gt] = K32_NONE;  // usually a handful of slots
        if (dirty_other > gn)
            for (int t = gt + gn; t < dirty_other; t += gn) sm.ck[par ^ 1][t] = K32_NONE;
        dirty_other = dirty_this;
        cp_async_wait_all();
        if (!MULTI) __syncwarp();
    }
#undef RG_FALLBACK
}

template <int CPT, bool MULTI>
__global__ void __launch_bounds__(MULTI ? 1024 : 128)
    sweep_reg_kernel(const CombineDesc *__restrict__ descs, int32_t ndesc, Ctx c, int32_t S,
                     int32_t nblk, int shift, int64_t ngroups, int flagged_only) {
    sweep_reg_body<CPT, MULTI>(descs, ndesc, c, S, nblk, shift, ngroups, flagged_only);
}

// CTA groups of <= 256 threads: a register cap (48) keeps 40 instead of 32 warps
// resident per SM (cfg5 levels of 1024 / 2048 rows: -3% / -8%)
template <int CPT>
__global__ void __launch_bounds__(256, 5)
    sweep_reg_small_kernel(const CombineDesc *__restrict__ descs, int32_t ndesc, Ctx c, int32_t S,
                           int32_t nblk, int shift, int64_t ngroups, int flagged_only) {
    sweep_reg_body<CPT, true>(descs, ndesc, c, S, nblk, shift, ngroups, flagged_only);
}

}  // namespace

int launch_table_events(const CombineDesc *descs, int32_t ndesc, Ctx c, cudaStream_t s) {
    if (ndesc <= 0 || c.n <= 0) return 0;
    if (ndesc > 65535) return (int)cudaErrorInvalidValue;
    const dim3 blocks((unsigned)((c.n + 255) / 256), (unsigned)ndesc);
    table_events_kernel<<<blocks, 256, 0, s>>>(descs, ndesc, c);
    LCSG_LAUNCH_CHECK();
    return 0;
}

int launch_sweep(const CombineDesc *descs, int32_t ndesc, Ctx c, int shift, bool key64, int32_t S,
                 int32_t maxw1, cudaStream_t s) {
    if (ndesc <= 0 || c.n <= 0) return 0;
    if (S > 1024) return (int)cudaErrorInvalidValue;
    const int32_t nblk = (c.n + S - 1) / S;
    // knobs are read at every launch (tests flip them inside one process)
    auto env_or = [](const char *name, int def) {
        const char *e = getenv(name);
        return e && *e ? atoi(e) : def;
    };
    constexpr int CAP_LIMIT = 12800;  // 16 B per cell: 200 KB of shared memory
    const int cap_max = std::max(4, std::min(CAP_LIMIT, env_or("LCSG_SWEEP_CAP", CAP_LIMIT)));
    const int cpt = std::max(1, env_or("LCSG_SWEEP_CPT", 8));
    const int use_reg = env_or("LCSG_SWEEP_REG", 1);
    const int one_warp_max = env_or("LCSG_SWEEP_ONE_WARP_MAXW1", 544);
    static bool attr_set = false;
    if (!attr_set) {
        cudaFuncSetAttribute(sweep_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             16 * CAP_LIMIT + 8 * 1024);
        attr_set = true;
    }
    // register-resident fast path: one warp per block of rows up to 32 * 17
    // cells, else a CTA of 9 cells per thread (a finite prefix beyond 1024 * 9
    // cells flags the block for the generic kernel)
    const bool reg = use_reg && S <= RG_MAXS && !key64 && shift < 32;
    if (reg) {
        const int64_t ngroups = (int64_t)ndesc * nblk;
        if (maxw1 <= one_warp_max && maxw1 <= 32 * 17) {
            const unsigned nb = (unsigned)((ngroups + 3) / 4);
            if (maxw1 <= 32 * 5)
                sweep_reg_kernel<5, false><<<nb, 128, 0, s>>>(descs, ndesc, c, S, nblk, shift, ngroups, 0);
            else if (maxw1 <= 32 * 9)
                sweep_reg_kernel<9, false><<<nb, 128, 0, s>>>(descs, ndesc, c, S, nblk, shift, ngroups, 0);
            else
                sweep_reg_kernel<17, false><<<nb, 128, 0, s>>>(descs, ndesc, c, S, nblk, shift, ngroups, 0);
        } else {
            int lg_max = 6;
            {
                const int v = env_or("LCSG_SWEEP_GN_MAX", 1024);
                while (lg_max < 10 && (1 << (lg_max + 1)) <= v) ++lg_max;
            }
            int lg = 6;
            while (lg < lg_max && (9 << lg) < maxw1) ++lg;
            // 1024-thread groups leave one CTA per SM: blocks whose finite prefix
            // fits 512 threads' registers go first in half-size groups (two CTAs
            // per SM), the rest (flagged) in a second pass (cfg5, 8192-row level:
            // 1.17 -> 0.77 ms).  Not for tables wider than 1024 * 9 cells (the
            // root of cfg5): there the second pass, run after the first, costs more
            // than the first saves (0.75 -> 1.02 ms)
            const bool cascade = lg >= env_or("LCSG_SWEEP_CASCADE_MINLG", 10) && maxw1 <= (9 << 10) &&
                                 env_or("LCSG_SWEEP_CASCADE", 1) != 0;
            if (cascade) {
                sweep_reg_kernel<9, true><<<(unsigned)ngroups, 1 << (lg - 1), 0, s>>>(
                    descs, ndesc, c, S, nblk, shift, ngroups, 0);
                LCSG_LAUNCH_CHECK();
            }
            if (lg <= 8 && env_or("LCSG_SWEEP_SMALL_CAP", 1))
                sweep_reg_small_kernel<9><<<(unsigned)ngroups, 1 << lg, 0, s>>>(
                    descs, ndesc, c, S, nblk, shift, ngroups, cascade ? 1 : 0);
            else
                sweep_reg_kernel<9, true><<<(unsigned)ngroups, 1 << lg, 0, s>>>(
                    descs, ndesc, c, S, nblk, shift, ngroups, cascade ? 1 : 0);
        }
        LCSG_LAUNCH_CHECK();
    }
    const int32_t cap = std::min(maxw1 + 1, cap_max);
    int nt = 32;
    while (nt < 1024 && nt * cpt < maxw1) nt *= 2;
    const dim3 blocks((unsigned)nblk, (unsigned)std::min<int32_t>(ndesc, 65535),
                      (unsigned)((ndesc + 65534) / 65535));
    sweep_kernel<<<blocks, nt, (size_t)16 * cap + (size_t)8 * S, s>>>(descs, ndesc, c, S, nblk, cap,
                                                                      reg ? 1 : 0);
    LCSG_LAUNCH_CHECK();
    return 0;
}

// Rows per block for one level: CTA groups of >= 512 threads leave one or two
// CTAs per SM, so the blocks run in waves of sm_count (or 2 * sm_count) and the
// last wave is partly empty; pick the block size in [3/4 S, S] with the fewest
// wave-rows (cfg5 root: 256 blocks of 64 rows = 2 waves = 128 row steps; 293
// blocks of 56 rows = 2 waves = 112).  Other levels keep S.
int sweep_pick_block(int32_t S, int32_t maxw1, int32_t count, int32_t n, int shift, bool key64,
                     int sm_count) {
    auto env_or = [](const char *name, int def) {
        const char *e = getenv(name);
        return e && *e ? atoi(e) : def;
    };
    if (S < 16 || sm_count <= 0 || key64 || shift >= 32 || !env_or("LCSG_SWEEP_REG", 1) ||
        !env_or("LCSG_SWEEP_PICK", 1))
        return S;
    if (maxw1 <= env_or("LCSG_SWEEP_ONE_WARP_MAXW1", 544) && maxw1 <= 32 * 17) return S;
    if (env_or("LCSG_SWEEP_GN_MAX", 1024) < 1024) return S;
    int lg = 6;
    while (lg < 10 && (9 << lg) < maxw1) ++lg;
    if (lg < 9) return S;
    const bool cascade = lg == 10 && maxw1 <= (9 << 10) && env_or("LCSG_SWEEP_CASCADE", 1) != 0;
    const int64_t slots = (int64_t)sm_count * ((lg == 9 || cascade) ? 2 : 1);
    int32_t best = S;
    int64_t best_cost = INT64_MAX;
    for (int32_t cand = S; cand >= S - S / 4; cand -= std::max(1, S / 16)) {
        const int64_t blocks = (int64_t)count * ((n + cand - 1) / cand);
        const int64_t cost = (blocks + slots - 1) / slots * cand;
        if (cost < best_cost) {
            best_cost = cost;
            best = cand;
        }
    }
    return best;
}

// kernels one launch_sweep call launches (for the handle's launch counter)
int sweep_launch_count(int shift, bool key64, int32_t S, int32_t maxw1) {
    auto env_or = [](const char *name, int def) {
        const char *e = getenv(name);
        return e && *e ? atoi(e) : def;
    };
    if (!(env_or("LCSG_SWEEP_REG", 1) && S <= RG_MAXS && !key64 && shift < 32)) return 1;
    const bool warp = maxw1 <= env_or("LCSG_SWEEP_ONE_WARP_MAXW1", 544) && maxw1 <= 32 * 17;
    const bool cascade = !warp && (9 << 9) < maxw1 && maxw1 <= (9 << 10) &&
                         env_or("LCSG_SWEEP_GN_MAX", 1024) >= 1024 &&
                         env_or("LCSG_SWEEP_CASCADE", 1) != 0;
    return cascade ? 3 : 2;
}

int sweep_error_count(int32_t *count, bool reset) {
    cudaError_t e = cudaMemcpyFromSymbol(count, g_sweep_err, sizeof(int32_t));
    if (e != cudaSuccess) return (int)e;
    if (reset) {
        const int32_t z = 0;
        e = cudaMemcpyToSymbol(g_sweep_err, &z, sizeof(int32_t));
    }
    return (int)e;
}

}  // namespace lcsg

#ifdef LCSG_SWEEP_STATS
extern "C" int lcsg_sweep_stats(unsigned long long *out) {
    return (int)cudaMemcpyFromSymbol(out, lcsg::g_sweep_stat, sizeof(unsigned long long) * 64);
}
#endif

extern "C" int lcsg_sweep_paths(int device, int64_t *redone_blocks, int64_t *global_state_blocks,
                                int reset) {
    int prev = 0;
    if (cudaGetDevice(&prev) != cudaSuccess) return -2;
    if (cudaSetDevice(device) != cudaSuccess) return -2;
    unsigned long long v[2] = {0, 0};
    cudaError_t e = cudaMemcpyFromSymbol(v, lcsg::g_sweep_paths, sizeof(v));
    if (e == cudaSuccess && reset) {
        const unsigned long long z[2] = {0, 0};
        e = cudaMemcpyToSymbol(lcsg::g_sweep_paths, z, sizeof(z));
    }
    cudaSetDevice(prev);
    if (redone_blocks) *redone_blocks = (int64_t)v[0];
    if (global_state_blocks) *global_state_blocks = (int64_t)v[1];
    return e == cudaSuccess ? 0 : -2;
}

extern "C" int lcsg_sweep_errors(int device, int32_t *count, int reset) {
    if (!count) return -1;
    int prev = 0;
    if (cudaGetDevice(&prev) != cudaSuccess) return -2;
    if (cudaSetDevice(device) != cudaSuccess) return -2;
    const int e = lcsg::sweep_error_count(count, reset != 0);
    cudaSetDevice(prev);
    return e ? -2 : 0;
}
