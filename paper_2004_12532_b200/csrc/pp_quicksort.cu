// pp_quicksort.cu -- in-place quicksort layered on the partition
// (§5 "Example Application: A Full Quicksort").
//
// The paper runs the parallel partition at the top levels of the recursion
// and a serial partition once subproblems are small.
// The GPU analogue is a breadth-first level loop:
//   - big segments (>= qs_big keys): the full multi-CTA partition pipeline of
//     pp_partition.cu, one segment at a time;
//   - mid segments: ONE launch for all of them: the Smoothed Striding group
//     kernel with (segment, group) tasks, then one CTA per segment reduces its
//     groups and cleans its (small) window by the rank-matched walk;
//   - leaves (<= leaf keys): sorted entirely in shared memory (bitonic
//     network), one CTA per leaf, all leaves in one launch at the end.
// Pivot: median of A[lo], A[lo+(len-1)/2], A[hi-1]; split by x < p; when that
// split is empty (p is the segment minimum) the next level splits by x <= p
// and the left part (all == p) is final (reading R14).
#include <algorithm>
#include <vector>

#include "pp_engine.cuh"

namespace pp {

void note_launches(uint64_t k);

struct QSeg {
    uint64_t lo, hi;   // [lo, hi)
    uint64_t pivot;    // effective strict pivot (key < pivot goes left)
    uint64_t gbase;    // first task (CTA) of this segment in the group launch
    uint64_t g;        // groups of this segment
    uint32_t mode;     // 0: pivot = median-of-3 (computed on device); 1: pivot given
    uint32_t pad;
};

template <typename K>
__device__ __forceinline__ K median3(K a, K b, K c) {
    if (a > b) { K t = a; a = b; b = t; }
    if (b > c) b = c;
    return a > b ? a : b;
}

template <typename K>
__global__ void qs_pivot_kernel(const K* __restrict__ keys, QSeg* __restrict__ segs, uint64_t nseg) {
    for (uint64_t s = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; s < nseg; s += (uint64_t)gridDim.x * blockDim.x) {
        QSeg q = segs[s];
        if (q.mode == 0) {
            const uint64_t len = q.hi - q.lo;
            segs[s].pivot = (uint64_t)median3<K>(keys[q.lo], keys[q.lo + (len - 1) / 2], keys[q.hi - 1]);
        }
    }
}

template <typename K>
__device__ __forceinline__ uint64_t seg_head(const K* keys, uint64_t lo, uint64_t len) {
    const uint64_t addr = (uint64_t)(uintptr_t)(keys + lo);
    uint64_t h = ((16 - (addr & 15)) & 15) / sizeof(K);
    return h > len ? len : h;
}

template <typename K>
__global__ void __launch_bounds__(GroupCfg<K>::NT) qs_group_kernel(K* __restrict__ keys,
                                                                   const QSeg* __restrict__ segs, uint64_t nseg,
                                                                   uint64_t seed, GroupOut* __restrict__ gout) {
    extern __shared__ __align__(128) unsigned char smem[];
    using C = GroupCfg<K>;
    const uint64_t task = blockIdx.x;
    // segment of this task: last s with gbase <= task
    uint64_t lo = 0, hi = nseg;
    while (hi - lo > 1) {
        const uint64_t mid = (lo + hi) >> 1;
        if (segs[mid].gbase <= task) lo = mid; else hi = mid;
    }
    const QSeg q = segs[lo];
    const uint64_t len = q.hi - q.lo;
    const uint64_t h = seg_head<K>(keys, q.lo, len);
    const uint64_t n_lines = (len - h) / C::LK;
    ss_group_engine<GroupCfg<K>>(keys + q.lo + h, n_lines, (uint32_t)q.g, (uint32_t)(task - q.gbase), seed, (K)q.pivot,
                       gout + task, smem);
}

// One CTA per mid segment: reduce the segment's group outputs, then clean its
// dirty set with the single-CTA rank-matched walk; writes the split.
template <typename K>
__global__ void __launch_bounds__(SW_NT) qs_cleanup_kernel(K* __restrict__ keys, const QSeg* __restrict__ segs,
                                                            const GroupOut* __restrict__ gout,
                                                            uint64_t* __restrict__ splits) {
    using C = GroupCfg<K>;
    __shared__ StreamBuf<SW_NT, SW_EPT2> sb;
    __shared__ uint64_t red[4][SW_NT / 32];
    const QSeg q = segs[blockIdx.x];
    K* seg = keys + q.lo;
    const uint64_t len = q.hi - q.lo;
    const K pivot = (K)q.pivot;
    const uint64_t h = seg_head<K>(keys, q.lo, len);
    const uint64_t n_lines = (len - h) / C::LK;
    const uint64_t region_end = n_lines * C::LK;
    uint64_t T = 0, vmin = region_end, vmax = 0, ht = 0;
    for (uint64_t i = threadIdx.x; i < q.g; i += SW_NT) {
        const GroupOut o = gout[q.gbase + i];
        T += o.T;
        vmin = o.vlo < vmin ? o.vlo : vmin;
        vmax = o.vhi > vmax ? o.vhi : vmax;
    }
    for (uint64_t x = threadIdx.x; x < h; x += SW_NT) ht += is_pred(seg[x], pivot) ? 1 : 0;
    for (uint64_t x = h + region_end + threadIdx.x; x < len; x += SW_NT) ht += is_pred(seg[x], pivot) ? 1 : 0;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        T += __shfl_xor_sync(0xffffffffu, T, o);
        ht += __shfl_xor_sync(0xffffffffu, ht, o);
        const uint64_t a = __shfl_xor_sync(0xffffffffu, vmin, o);
        const uint64_t b = __shfl_xor_sync(0xffffffffu, vmax, o);
        vmin = a < vmin ? a : vmin;
        vmax = b > vmax ? b : vmax;
    }
    if (lane == 0) {
        red[0][warp] = T;
        red[1][warp] = ht;
        red[2][warp] = vmin;
        red[3][warp] = vmax;
    }
    __syncthreads();
    T = 0; ht = 0; vmin = region_end; vmax = 0;
    for (int w = 0; w < SW_NT / 32; ++w) {
        T += red[0][w];
        ht += red[1][w];
        vmin = red[2][w] < vmin ? red[2][w] : vmin;
        vmax = red[3][w] > vmax ? red[3][w] : vmax;
    }
    const uint64_t Ks = T + ht;
    uint64_t a[3], b[3];
    a[0] = 0; b[0] = h;
    a[1] = (h + vmin) < Ks ? (h + vmin) : Ks;
    b[1] = (h + vmax) > Ks ? (h + vmax) : Ks;
    if (vmin > vmax) { a[1] = b[1] = 0; }
    a[2] = h + region_end; b[2] = len;
    Ctl c;
    finish_ctl(&c, len, Ks, a, b);
    Dirty d;
#pragma unroll
    for (int k = 0; k < 3; ++k) { d.s[k] = c.ds[k]; d.l[k] = c.dl[k]; }
    walk_swap_stream<K, SW_NT, SW_EPT2>(seg, d, pivot, 0, c.Kv, c.Kv, c.W, sb);
    if (threadIdx.x == 0) splits[blockIdx.x] = Ks;
}

// Leaf sort: one CTA sorts one segment of <= LEAF keys with a bitonic
// network (padding with the maximum key, never stored back).  Each thread
// holds E = 8 consecutive keys in registers: compare-exchange stages with
// stride j < 8 run in registers, 8 <= j < 256 through warp shuffles, and only
// j >= 256 through shared memory.
constexpr int LEAF_E = 8;

template <int J, typename K>
__device__ __forceinline__ void leaf_reg_stage(K (&v)[LEAF_E], uint32_t base, uint32_t k) {
#pragma unroll
    for (int r = 0; r < LEAF_E; ++r) {
        if ((r & J) == 0) {
            const bool asc = ((base + r) & k) == 0;
            const K a = v[r], b = v[r + J];
            if ((a > b) == asc) {
                v[r] = b;
                v[r + J] = a;
            }
        }
    }
}

__device__ __forceinline__ void leaf_bar(uint32_t nthr) {
    asm volatile("bar.sync 1, %0;" ::"r"(nthr) : "memory");
}

template <typename K>
__device__ __forceinline__ void cmpx(K& a, K& b) {
    const K lo = a < b ? a : b, hi = a < b ? b : a;
    a = lo;
    b = hi;
}

// Shared-memory index padding for the merge sorts: one spare slot per 8 keys,
// so that a warp whose lanes each own 8 consecutive keys hits distinct banks
// (stride 9 words instead of 8).
__device__ __forceinline__ uint32_t lpad(uint32_t i) { return i + (i >> 3); }

template <typename K>
__device__ __forceinline__ void sort8(K (&v)[8]) {  // Batcher's 19-comparator network
    cmpx(v[0], v[1]); cmpx(v[2], v[3]); cmpx(v[4], v[5]); cmpx(v[6], v[7]);
    cmpx(v[0], v[2]); cmpx(v[1], v[3]); cmpx(v[4], v[6]); cmpx(v[5], v[7]);
    cmpx(v[1], v[2]); cmpx(v[5], v[6]);
    cmpx(v[0], v[4]); cmpx(v[1], v[5]); cmpx(v[2], v[6]); cmpx(v[3], v[7]);
    cmpx(v[2], v[4]); cmpx(v[3], v[5]);
    cmpx(v[1], v[2]); cmpx(v[3], v[4]); cmpx(v[5], v[6]);
}

// One merge step for the 8 outputs starting at `base`: runs of length L in
// src (padded layout) -> dst.  Runs A = [blk, blk+La), B = [blk+La, +Lb)
// (the last pair may be short); the start is found on the merge path by
// binary search (ties: A first).
template <typename K>
__device__ __forceinline__ void merge_chunk(const K* __restrict__ src, K* __restrict__ dst, uint32_t base,
                                            uint32_t L, uint32_t P) {
    const K KMAX = (K)~(K)0;
    const uint32_t blk = base / (2 * L) * (2 * L);
    const uint32_t d = base - blk;
    const uint32_t La = min(L, P - blk);
    const uint32_t Lb = min(L, P - blk - La);
    const uint32_t A0 = blk, B0 = blk + La;
    uint32_t a0 = d > Lb ? d - Lb : 0, a1 = d < La ? d : La;
    while (a0 < a1) {
        const uint32_t mid = (a0 + a1) >> 1;
        if (src[lpad(A0 + mid)] <= src[lpad(B0 + d - 1 - mid)]) a0 = mid + 1; else a1 = mid;
    }
    const uint32_t a = a0, b = d - a0;
    // The 8 outputs are the 8 smallest of A[a, a+8) u B[b, b+8): load all 16
    // at once (independent loads instead of a chain of 8 load->compare
    // steps), keep c[i] = min(A[a+i], B[b+7-i]) (bitonic half-cleaner: the
    // lower half of the bitonic sequence A ++ reverse(B)) and sort that
    // bitonic sequence with 3 compare-exchange stages.
    K c[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const K xa = a + i < La ? src[lpad(A0 + a + i)] : KMAX;
        const K xb = b + 7 - i < Lb ? src[lpad(B0 + b + 7 - i)] : KMAX;
        c[i] = xa < xb ? xa : xb;
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) cmpx(c[i], c[i + 4]);
#pragma unroll
    for (int i = 0; i < 8; i += 4) {
        cmpx(c[i], c[i + 2]);
        cmpx(c[i + 1], c[i + 3]);
    }
#pragma unroll
    for (int i = 0; i < 8; i += 2) cmpx(c[i], c[i + 1]);
#pragma unroll
    for (int i = 0; i < 8; ++i) dst[lpad(base + i)] = c[i];
}

// Leaf sort by merging: every thread sorts its 8 keys in registers (Batcher's
// 19-comparator network), then log2(P/8) rounds merge pairs of sorted runs
// in shared memory; each thread produces 8 outputs of a merge, locating its
// start on the merge path by binary search (ties: left run first -- the sort
// is a plain ascending sort, stability is irrelevant for keys).
template <typename K, int LEAF, int NT>
__global__ void __launch_bounds__(NT) qs_leaf_merge_kernel(K* __restrict__ keys,
                                                           const uint64_t* __restrict__ leaf_lo,
                                                           const uint32_t* __restrict__ leaf_len) {
    static_assert(LEAF == NT * LEAF_E, "one block holds LEAF keys");
    extern __shared__ __align__(16) unsigned char lsm[];
    K* src = reinterpret_cast<K*>(lsm);
    K* dst = src + lpad(LEAF);
    const uint64_t lo = leaf_lo[blockIdx.x];
    const uint32_t len = leaf_len[blockIdx.x];
    // pad to whole warps of 8 keys per thread (not to a power of two)
    const uint32_t P = (len + 32 * LEAF_E - 1) / (32 * LEAF_E) * (32 * LEAF_E);
    const uint32_t nthr = P / LEAF_E;
    const uint32_t tid = threadIdx.x;
    if (tid >= nthr) return;
    const K KMAX = (K)~(K)0;
    for (uint32_t i = tid; i < P; i += nthr) src[lpad(i)] = i < len ? keys[lo + i] : KMAX;
    leaf_bar(nthr);
    const uint32_t base = tid * LEAF_E;
    K v[LEAF_E];
#pragma unroll
    for (int r = 0; r < LEAF_E; ++r) v[r] = src[lpad(base + r)];
    sort8(v);
#pragma unroll
    for (int r = 0; r < LEAF_E; ++r) src[lpad(base + r)] = v[r];
    leaf_bar(nthr);
    for (uint32_t L = LEAF_E; L < P; L <<= 1) {
        merge_chunk<K>(src, dst, base, L, P);
        leaf_bar(nthr);
        K* t = src;
        src = dst;
        dst = t;
    }
    for (uint32_t i = tid; i < len; i += nthr) keys[lo + i] = src[lpad(i)];
}

// ===========================================================================
// CTA-level quicksort of small segments (LEAF < len <= qs_small keys): one
// CTA runs the whole remaining recursion of its segment -- partitions with
// the group engine (g = 1: a plain two-ended line partition) plus the
// streaming cleanup of its head / tail / open lines, depth first with an
// explicit stack (smaller part first), and sorts pieces <= SMALL_LEAF keys in
// shared memory by merging.  This removes the deepest, least efficient
// levels of the breadth-first loop (many tiny CTAs, one launch + sync each).
// ===========================================================================
// V = 0: 256 threads, 8 KiB lines, 4 KiB... 64 KiB sort buffers (2 CTAs/SM);
// V = 1: lean -- 128 threads, 4 KiB lines with 2 in flight per end, 32 KiB
// sort buffers: ~37 KiB of shared memory, 4 CTAs per SM (more independent
// recursions per SM to hide the latency-bound merge rounds).
template <typename K, int V>
struct SmallCfg;
template <typename K>
struct SmallCfg<K, 0> {
    static constexpr int NT = 256, MINB = 2;
    using GC = GroupCfgT<K, 8192, 256, 4, false>;
    static constexpr uint32_t LEAFC = sizeof(K) == 8 ? 4096 : 8192;  // 2 x LEAFC keys <= 64 KiB
    static constexpr size_t SORT = 2 * (LEAFC + LEAFC / 8) * sizeof(K);  // two padded buffers
    static constexpr size_t SMEM = GC::SMEM > SORT ? GC::SMEM : SORT;
};
template <typename K>
struct SmallCfg<K, 1> {
    static constexpr int NT = 128, MINB = 4;
    using GC = GroupCfgT<K, 4096, 128, 2, false>;
    static constexpr uint32_t LEAFC = sizeof(K) == 8 ? 2048 : 4096;
    static constexpr size_t SORT = 2 * (LEAFC + LEAFC / 8) * sizeof(K);
    static constexpr size_t SMEM = GC::SMEM > SORT ? GC::SMEM : SORT;
};

// Merge sort of len <= NT*8*V keys held in global memory at g (in place),
// through two shared-memory buffers A, B; all NT threads participate, each
// handling chunks of 8 keys (thread t: chunks t, t+NT, ...).
template <typename K, int NT>
__device__ void cta_merge_sort(K* __restrict__ g, uint32_t len, K* A, K* B) {
    const K KMAX = (K)~(K)0;
    const uint32_t P = (len + 7) / 8 * 8, nch = P / 8;
    for (uint32_t i = threadIdx.x; i < P; i += NT) A[lpad(i)] = i < len ? g[i] : KMAX;
    __syncthreads();
    for (uint32_t c = threadIdx.x; c < nch; c += NT) {
        K v[8];
#pragma unroll
        for (int r = 0; r < 8; ++r) v[r] = A[lpad(8 * c + r)];
        sort8(v);
#pragma unroll
        for (int r = 0; r < 8; ++r) A[lpad(8 * c + r)] = v[r];
    }
    __syncthreads();
    K* src = A;
    K* dst = B;
    for (uint32_t L = 8; L < P; L <<= 1) {
        for (uint32_t c = threadIdx.x; c < nch; c += NT) merge_chunk<K>(src, dst, 8 * c, L, P);
        __syncthreads();
        K* t = src;
        src = dst;
        dst = t;
    }
    for (uint32_t i = threadIdx.x; i < len; i += NT) g[i] = src[lpad(i)];
    __syncthreads();
}

// In-place partition of seg[0, len) by key < pivot with one CTA; returns K.
template <typename K, int V>
__device__ uint64_t cta_partition(K* __restrict__ seg, uint64_t len, K pivot, uint64_t seed, unsigned char* smem,
                                  GroupOut* scratch, Ctl* sc, uint64_t* red) {
    using S = SmallCfg<K, V>;
    using GC = typename S::GC;
    constexpr int NT = S::NT, NW = NT / 32;
    const uint64_t addr = (uint64_t)(uintptr_t)seg;
    uint64_t h = ((16 - (addr & 15)) & 15) / sizeof(K);
    if (h > len) h = len;
    const uint64_t nl = (len - h) / GC::LK;
    uint64_t T = 0, v = 0;
    // this CTA's earlier generic-proxy stores to the segment must be visible
    // to the engine's bulk-copy (async-proxy) loads
    asm volatile("fence.proxy.async;" ::: "memory");
    __syncthreads();
    if (nl > 0) {
        ss_group_engine<GC>(seg + h, nl, 1, 0, seed, pivot, scratch, smem);
        __syncthreads();
        T = scratch->T;
        v = scratch->vlo;
    }
    const uint64_t region_end = nl * GC::LK;
    uint64_t ht = 0;
    for (uint64_t x = threadIdx.x; x < h; x += NT) ht += is_pred(seg[x], pivot) ? 1 : 0;
    for (uint64_t x = h + region_end + threadIdx.x; x < len; x += NT) ht += is_pred(seg[x], pivot) ? 1 : 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ht += __shfl_xor_sync(0xffffffffu, ht, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ht;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < NW; ++w) ht += red[w];
        const uint64_t Ks = T + ht;
        uint64_t a[3], b[3];
        a[0] = 0; b[0] = h;
        a[1] = (h + v) < Ks ? (h + v) : Ks;
        b[1] = (h + v) > Ks ? (h + v) : Ks;
        if (nl == 0) { a[1] = b[1] = 0; }
        a[2] = h + region_end; b[2] = len;
        finish_ctl(sc, len, Ks, a, b);
    }
    __syncthreads();
    Dirty d;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        d.s[k] = sc->ds[k];
        d.l[k] = sc->dl[k];
    }
    const uint64_t Ks = sc->K, Kv = sc->Kv, W = sc->W;
    walk_swap_stream<K, NT, SW_EPT2>(seg, d, pivot, 0, Kv, Kv, W,
                                     *reinterpret_cast<StreamBuf<NT, SW_EPT2>*>(smem));
    __syncthreads();
    return Ks;
}

template <typename K, int V>
__global__ void __launch_bounds__(SmallCfg<K, V>::NT, SmallCfg<K, V>::MINB)
    qs_small_kernel(K* __restrict__ keys, const uint64_t* __restrict__ seg_lo, const uint32_t* __restrict__ seg_len,
                    uint64_t seed, GroupOut* __restrict__ scratch) {
    using S = SmallCfg<K, V>;
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ Ctl sc;
    __shared__ uint64_t red[S::NT / 32];
    __shared__ uint64_t st_lo[64], st_hi[64], st_p[64];
    __shared__ int st_mode[64];
    __shared__ int sp;
    const K KMAX = (K)~(K)0;
    K* A = reinterpret_cast<K*>(smem);
    K* B = A + lpad(S::LEAFC);
    if (threadIdx.x == 0) {
        st_lo[0] = seg_lo[blockIdx.x];
        st_hi[0] = st_lo[0] + seg_len[blockIdx.x];
        st_mode[0] = 0;
        st_p[0] = 0;
        sp = 1;
    }
    __syncthreads();
    while (sp > 0) {
        const int top = sp - 1;
        const uint64_t lo = st_lo[top], hi = st_hi[top], pm = st_p[top];
        const int mode = st_mode[top];
        __syncthreads();
        if (threadIdx.x == 0) sp = top;
        const uint64_t len = hi - lo;
        if (len <= 1) {
            __syncthreads();
            continue;
        }
        if (len <= S::LEAFC) {
            cta_merge_sort<K, S::NT>(keys + lo, (uint32_t)len, A, B);
            continue;
        }
        K p;
        if (mode == 0) p = median3<K>(keys[lo], keys[lo + (len - 1) / 2], keys[hi - 1]);
        else p = (K)pm;
        const uint64_t k = cta_partition<K, V>(keys + lo, len, p, seed, smem, scratch + blockIdx.x, &sc, red);
        if (threadIdx.x == 0) {
            int s = sp;
            if (mode == 0 && k == 0) {
                if (p != KMAX) {  // p is the minimum: split by x <= p next (reading R14)
                    st_lo[s] = lo; st_hi[s] = hi; st_mode[s] = 1; st_p[s] = (uint64_t)(K)(p + 1); ++s;
                }
            } else if (mode == 1) {
                st_lo[s] = lo + k; st_hi[s] = hi; st_mode[s] = 0; st_p[s] = 0; ++s;  // [lo, lo+k) all == p
            } else {
                // push the larger part first: the smaller is processed next (stack depth <= log2 len)
                const bool left_small = k < len - k;
                const uint64_t a0 = left_small ? lo + k : lo, a1 = left_small ? hi : lo + k;
                const uint64_t b0 = left_small ? lo : lo + k, b1 = left_small ? lo + k : hi;
                st_lo[s] = a0; st_hi[s] = a1; st_mode[s] = 0; st_p[s] = 0; ++s;
                st_lo[s] = b0; st_hi[s] = b1; st_mode[s] = 0; st_p[s] = 0; ++s;
            }
            sp = s;
        }
        __syncthreads();
    }
}

template <typename K, int LEAF, int NT>
__global__ void __launch_bounds__(NT) qs_leaf_kernel(K* __restrict__ keys, const uint64_t* __restrict__ leaf_lo,
                                                     const uint32_t* __restrict__ leaf_len) {
    static_assert(LEAF == NT * LEAF_E, "one block holds LEAF keys");
    extern __shared__ __align__(16) unsigned char lsm_b[];
    K* sk = reinterpret_cast<K*>(lsm_b);  // LEAF keys (dynamic shared memory)
    const uint64_t lo = leaf_lo[blockIdx.x];
    const uint32_t len = leaf_len[blockIdx.x];
    uint32_t P = 32 * LEAF_E;
    while (P < len) P <<= 1;
    const uint32_t nthr = P / LEAF_E;  // whole warps
    const uint32_t tid = threadIdx.x;
    if (tid >= nthr) return;
    const K KMAX = (K)~(K)0;
    for (uint32_t i = tid; i < P; i += nthr) sk[i] = i < len ? keys[lo + i] : KMAX;
    leaf_bar(nthr);
    const uint32_t base = tid * LEAF_E;
    K v[LEAF_E];
#pragma unroll
    for (int r = 0; r < LEAF_E; ++r) v[r] = sk[base + r];
    for (uint32_t k = 2; k <= P; k <<= 1) {
        for (uint32_t j = k >> 1; j > 0; j >>= 1) {
            if (j >= 32 * LEAF_E) {  // partner in another warp: exchange through smem
                leaf_bar(nthr);
#pragma unroll
                for (int r = 0; r < LEAF_E; ++r) sk[base + r] = v[r];
                leaf_bar(nthr);
#pragma unroll
                for (int r = 0; r < LEAF_E; ++r) {
                    const uint32_t i = base + r, p = i ^ j;
                    const K y = sk[p];
                    const bool keep_min = ((i < p) == ((i & k) == 0));
                    v[r] = keep_min ? (v[r] < y ? v[r] : y) : (v[r] > y ? v[r] : y);
                }
            } else if (j >= LEAF_E) {  // partner lane in this warp
                const int lm = (int)(j / LEAF_E);
#pragma unroll
                for (int r = 0; r < LEAF_E; ++r) {
                    const K y = __shfl_xor_sync(0xffffffffu, v[r], lm);
                    const uint32_t i = base + r, p = i ^ j;
                    const bool keep_min = ((i < p) == ((i & k) == 0));
                    v[r] = keep_min ? (v[r] < y ? v[r] : y) : (v[r] > y ? v[r] : y);
                }
            } else if (j == 4) {
                leaf_reg_stage<4>(v, base, k);
            } else if (j == 2) {
                leaf_reg_stage<2>(v, base, k);
            } else {
                leaf_reg_stage<1>(v, base, k);
            }
        }
    }
    leaf_bar(nthr);
#pragma unroll
    for (int r = 0; r < LEAF_E; ++r) sk[base + r] = v[r];
    leaf_bar(nthr);
    for (uint32_t i = tid; i < len; i += nthr) keys[lo + i] = sk[i];
}

template <typename K>
struct LeafCfg {
    static constexpr int LEAF = 8192;
    static constexpr int NT = LEAF / LEAF_E;
};

// quicksort workspace (separate from the partition workspace)
static void* g_qws = nullptr;
static size_t g_qws_bytes = 0;
// With a caller workspace (pp_set_workspace) the quicksort's region starts
// after the partition region of the top-level call: [partition | quicksort].
static size_t g_qs_user_base = 0;
static size_t g_qs_peak = 0;
static inline size_t al256(size_t b) { return (b + 255) & ~size_t(255); }
// leaf / small-segment descriptor lists are uploaded in chunks of this many
// entries, so the quicksort workspace stays o(n) however many leaves there are
static constexpr uint64_t QS_LIST_CHUNK = 1u << 20;

static void* qs_workspace(size_t bytes) {
    g_qs_peak = std::max(g_qs_peak, bytes);
    void* uw = nullptr;
    size_t ub = 0;
    if (user_workspace(&uw, &ub)) {
        if (g_qs_user_base + bytes <= ub) return static_cast<unsigned char*>(uw) + g_qs_user_base;
        set_error("caller workspace too small for quicksort (pp_workspace_bytes(n, key_bytes, 1))");
        return nullptr;
    }
    if (bytes <= g_qws_bytes) return g_qws;
    if (g_qws) {
        cudaDeviceSynchronize();
        cudaFree(g_qws);
    }
    g_qws = nullptr;
    g_qws_bytes = 0;
    size_t want = bytes + (bytes >> 1);
    if (cudaMalloc(&g_qws, want) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    g_qws_bytes = want;
    return g_qws;
}

// Size thresholds of the quicksort driver (current params).
struct QsGeom {
    uint64_t LEAF;      // segments <= LEAF: one smem sort
    uint64_t SMALL;     // segments in (LEAF, SMALL]: per-CTA recursion
    uint64_t BIG;       // segments >= BIG: full multi-CTA partition
    uint64_t G_TARGET;  // CTAs of one batched mid-level group launch
};
template <typename K>
static QsGeom qs_geom() {
    using C = GroupCfg<K>;
    using LC = LeafCfg<K>;
    const Params& P = params();
    QsGeom q;
    // leaf capacity: default LC::LEAF (8192 keys); "leaf" may lower it
    q.LEAF = (P.leaf > 0 && (uint64_t)P.leaf <= (uint64_t)LC::LEAF) ? (uint64_t)P.leaf : (uint64_t)LC::LEAF;
    q.BIG = P.qs_cta_max > 0 ? (uint64_t)P.qs_cta_max : (uint64_t)1 << 25;
    q.SMALL = P.qs_small > 0 ? std::max<uint64_t>((uint64_t)P.qs_small, q.LEAF) : q.LEAF;
    int occ = 1;
    cudaFuncSetAttribute(qs_group_kernel<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, qs_group_kernel<K>, C::NT, C::SMEM);
    q.G_TARGET = (uint64_t)sm_count() * (uint64_t)std::max(occ, 1) * (uint64_t)std::max<int64_t>(P.qs_waves, 1);
    return q;
}

// Upper bound of the quicksort's own workspace for n keys (excluding the
// partition region used by big segments).  Per level: mid segments are
// disjoint and longer than SMALL (<= n/SMALL + 1 of them), each gets
// <= its proportional share of G_TARGET groups + 1 (rounding, the max(1,.)
// floor), big ones number <= n/BIG + 1.  The final lists are chunked.
template <typename K>
uint64_t quicksort_workspace_bound(uint64_t n) {
    const QsGeom q = qs_geom<K>();
    const uint64_t nmid = n / (q.SMALL + 1) + 1, nbig = n / q.BIG + 1;
    const uint64_t gtot = q.G_TARGET + 2 * nmid + 1;
    const size_t level = al256(sizeof(QSeg) * nmid) + al256(sizeof(GroupOut) * gtot) + al256(8 * (nmid + nbig + 1));
    const uint64_t cl = std::min<uint64_t>(n / 2 + 1, QS_LIST_CHUNK);
    const uint64_t cs = std::min<uint64_t>(n / (q.LEAF + 1) + 1, QS_LIST_CHUNK);
    const size_t lists = al256(8 * cl) + al256(4 * cl) + al256(8 * cs) + al256(4 * cs) + al256(sizeof(GroupOut) * cs) + 256;
    return std::max(level, lists);
}
template uint64_t quicksort_workspace_bound<uint64_t>(uint64_t);
template uint64_t quicksort_workspace_bound<uint32_t>(uint64_t);

template <typename K>
pp_status quicksort_device(K* keys, uint64_t n, cudaStream_t st) {
    using C = GroupCfg<K>;
    using LC = LeafCfg<K>;
    const Params& P = params();
    const QsGeom geom = qs_geom<K>();
    const uint64_t LEAF = geom.LEAF, BIG = geom.BIG, G_TARGET = geom.G_TARGET;
    const uint64_t MINL = 16;  // at least this many lines per group for mid segments
    const K KMAX = (K)~(K)0;
    g_qs_user_base = al256(partition_workspace_bound(n));
    g_qs_peak = 0;

    struct HSeg {
        uint64_t lo, hi, pivot;
        uint32_t mode;
    };
    std::vector<HSeg> cur{{0, n, 0, 0}}, next;
    std::vector<uint64_t> leaf_lo, small_lo;
    std::vector<uint32_t> leaf_len, small_len;
    // segments in (LEAF, SMALL] finish in one CTA each (qs_small_kernel)
    const uint64_t SMALL = geom.SMALL;
    auto add_child = [&](uint64_t lo, uint64_t hi) {
        const uint64_t len = hi - lo;
        if (len <= 1) return;
        if (len <= LEAF) {
            leaf_lo.push_back(lo);
            leaf_len.push_back((uint32_t)len);
        } else if (len <= SMALL) {
            small_lo.push_back(lo);
            small_len.push_back((uint32_t)len);
        } else {
            next.push_back({lo, hi, 0, 0});
        }
    };
    if (n <= SMALL) {
        cur.clear();
        add_child(0, n);
    }
    std::vector<QSeg> mids;
    std::vector<uint64_t> splits_h, pivots_h;
    std::vector<size_t> order;  // cur index -> splits index
    cudaError_t e;
    cudaFuncSetAttribute(qs_group_kernel<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
    while (!cur.empty()) {
        // ---- classify ----
        mids.clear();
        std::vector<size_t> big_idx, mid_idx;
        uint64_t gtot = 0;
        // mid segments share one launch: give each a number of groups
        // proportional to its length so that one wave of G_TARGET CTAs
        // carries the level (small windows, balanced CTAs)
        uint64_t mid_keys = 0;
        for (size_t i = 0; i < cur.size(); ++i) {
            const uint64_t len = cur[i].hi - cur[i].lo;
            if (len < BIG) mid_keys += len;
        }
        for (size_t i = 0; i < cur.size(); ++i) {
            const uint64_t len = cur[i].hi - cur[i].lo;
            if (len >= BIG) {
                big_idx.push_back(i);
            } else {
                mid_idx.push_back(i);
                QSeg q;
                q.lo = cur[i].lo;
                q.hi = cur[i].hi;
                q.pivot = cur[i].pivot;
                q.mode = cur[i].mode;
                q.pad = 0;
                // lines of the aligned region (host mirror of seg_head)
                const uint64_t addr = (uint64_t)(uintptr_t)(keys + q.lo);
                uint64_t h = ((16 - (addr & 15)) & 15) / sizeof(K);
                if (h > len) h = len;
                const uint64_t nl = (len - h) / C::LK;
                const uint64_t gp = (uint64_t)((double)len * (double)G_TARGET / (double)mid_keys + 0.5);
                q.g = std::max<uint64_t>(1, std::min<uint64_t>(gp, nl / MINL));
                q.gbase = gtot;
                gtot += q.g;
                mids.push_back(q);
            }
        }
        const uint64_t nmid = mids.size(), nbig = big_idx.size();
        // ---- workspace: [segs][gout][splits] ----
        const size_t segB = ((sizeof(QSeg) * std::max<uint64_t>(nmid, 1)) + 255) & ~size_t(255);
        const size_t goB = ((sizeof(GroupOut) * std::max<uint64_t>(gtot, 1)) + 255) & ~size_t(255);
        const size_t spB = ((8 * (nmid + nbig + 1)) + 255) & ~size_t(255);
        unsigned char* ws = static_cast<unsigned char*>(qs_workspace(segB + goB + spB));
        if (!ws) return PP_E_NOMEM;
        QSeg* d_segs = reinterpret_cast<QSeg*>(ws);
        GroupOut* d_gout = reinterpret_cast<GroupOut*>(ws + segB);
        uint64_t* d_splits = reinterpret_cast<uint64_t*>(ws + segB + goB);

        // ---- big segments: full multi-CTA partition, one at a time ----
        pivots_h.assign(cur.size(), 0);
        for (size_t bi = 0; bi < nbig; ++bi) {
            HSeg& s = cur[big_idx[bi]];
            uint64_t p = s.pivot;
            if (s.mode == 0) {
                K three[3];
                const uint64_t len = s.hi - s.lo;
                e = cudaMemcpyAsync(&three[0], keys + s.lo, sizeof(K), cudaMemcpyDeviceToHost, st);
                if (e == cudaSuccess)
                    e = cudaMemcpyAsync(&three[1], keys + s.lo + (len - 1) / 2, sizeof(K), cudaMemcpyDeviceToHost, st);
                if (e == cudaSuccess)
                    e = cudaMemcpyAsync(&three[2], keys + s.hi - 1, sizeof(K), cudaMemcpyDeviceToHost, st);
                if (e == cudaSuccess) e = cudaStreamSynchronize(st);
                if (e != cudaSuccess) return cuda_fail(e, "quicksort pivot");
                K a = three[0], b = three[1], c = three[2];
                if (a > b) std::swap(a, b);
                if (b > c) b = c;
                p = (uint64_t)(a > b ? a : b);
            }
            pivots_h[big_idx[bi]] = p;
            pp_status ps = partition_device<K>(keys + s.lo, s.hi - s.lo, (K)p, st, d_splits + nmid + bi, nullptr);
            if (ps != PP_OK) return ps;
        }
        // ---- mid segments: one batched pass ----
        if (nmid > 0) {
            e = cudaMemcpyAsync(d_segs, mids.data(), sizeof(QSeg) * nmid, cudaMemcpyHostToDevice, st);
            if (e != cudaSuccess) return cuda_fail(e, "quicksort H2D");
            qs_pivot_kernel<K><<<(unsigned)((nmid + 255) / 256), 256, 0, st>>>(keys, d_segs, nmid);
            qs_group_kernel<K><<<(unsigned)gtot, C::NT, C::SMEM, st>>>(keys, d_segs, nmid, P.seed, d_gout);
            qs_cleanup_kernel<K><<<(unsigned)nmid, SW_NT, 0, st>>>(keys, d_segs, d_gout, d_splits);
            note_launches(3);
            e = cudaGetLastError();
            if (e != cudaSuccess) return cuda_fail(e, "quicksort mid launch");
        }
        // ---- read back splits (and mid pivots) ----
        splits_h.assign(nmid + nbig, 0);
        if (nmid + nbig > 0) {
            e = cudaMemcpyAsync(splits_h.data(), d_splits, 8 * (nmid + nbig), cudaMemcpyDeviceToHost, st);
            if (e != cudaSuccess) return cuda_fail(e, "quicksort D2H");
        }
        if (nmid > 0) {
            e = cudaMemcpyAsync(mids.data(), d_segs, sizeof(QSeg) * nmid, cudaMemcpyDeviceToHost, st);
            if (e != cudaSuccess) return cuda_fail(e, "quicksort D2H");
        }
        e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) return cuda_fail(e, "quicksort level");
        for (size_t mi = 0; mi < nmid; ++mi) pivots_h[mid_idx[mi]] = mids[mi].pivot;
        // ---- next level ----
        next.clear();
        auto visit = [&](const HSeg& s, uint64_t p, uint64_t k) {
            if (s.mode == 0) {
                if (k == 0) {
                    // p is the segment minimum; split by x <= p next (unless all == MAX)
                    if ((K)p != KMAX) next.push_back({s.lo, s.hi, (uint64_t)(K)(p + 1), 1});
                } else {
                    add_child(s.lo, s.lo + k);
                    add_child(s.lo + k, s.hi);
                }
            } else {
                add_child(s.lo + k, s.hi);  // [lo, lo+k) is all equal: final
            }
        };
        for (size_t mi = 0; mi < nmid; ++mi) visit(cur[mid_idx[mi]], pivots_h[mid_idx[mi]], splits_h[mi]);
        for (size_t bi = 0; bi < nbig; ++bi) visit(cur[big_idx[bi]], pivots_h[big_idx[bi]], splits_h[nmid + bi]);
        cur.swap(next);
    }
    // ---- small segments (one CTA each) and leaves: one workspace, lists
    // uploaded in chunks of QS_LIST_CHUNK (stream order makes reuse safe) ----
    const uint64_t nleaf = leaf_lo.size(), nsmall = small_lo.size();
    const uint64_t cl = std::min<uint64_t>(nleaf, QS_LIST_CHUNK), cs = std::min<uint64_t>(nsmall, QS_LIST_CHUNK);
    const size_t loB = al256(8 * cl), lnB = al256(4 * cl), sloB = al256(8 * cs), slnB = al256(4 * cs);
    const size_t scrB = al256(sizeof(GroupOut) * cs);
    unsigned char* qws = static_cast<unsigned char*>(qs_workspace(loB + lnB + sloB + slnB + scrB + 256));
    if (!qws) return PP_E_NOMEM;
    if (nsmall > 0) {
        uint64_t* d_slo = reinterpret_cast<uint64_t*>(qws + loB + lnB);
        uint32_t* d_sln = reinterpret_cast<uint32_t*>(qws + loB + lnB + sloB);
        GroupOut* d_scr = reinterpret_cast<GroupOut*>(qws + loB + lnB + sloB + slnB);
        for (uint64_t b0 = 0; b0 < nsmall; b0 += QS_LIST_CHUNK) {
            const uint64_t cnt = std::min<uint64_t>(nsmall - b0, QS_LIST_CHUNK);
            e = cudaMemcpyAsync(d_slo, small_lo.data() + b0, 8 * cnt, cudaMemcpyHostToDevice, st);
            if (e == cudaSuccess)
                e = cudaMemcpyAsync(d_sln, small_len.data() + b0, 4 * cnt, cudaMemcpyHostToDevice, st);
            if (e != cudaSuccess) return cuda_fail(e, "quicksort small H2D");
            if (P.qs_small_cfg == 0) {
                using S = SmallCfg<K, 0>;
                cudaFuncSetAttribute(qs_small_kernel<K, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S::SMEM);
                qs_small_kernel<K, 0><<<(unsigned)cnt, S::NT, S::SMEM, st>>>(keys, d_slo, d_sln, P.seed, d_scr);
            } else {
                using S = SmallCfg<K, 1>;
                cudaFuncSetAttribute(qs_small_kernel<K, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S::SMEM);
                qs_small_kernel<K, 1><<<(unsigned)cnt, S::NT, S::SMEM, st>>>(keys, d_slo, d_sln, P.seed, d_scr);
            }
            note_launches(1);
            e = cudaGetLastError();
            if (e != cudaSuccess) return cuda_fail(e, "quicksort small launch");
        }
    }
    if (nleaf > 0) {
        uint64_t* d_lo = reinterpret_cast<uint64_t*>(qws);
        uint32_t* d_len = reinterpret_cast<uint32_t*>(qws + loB);
        for (uint64_t b0 = 0; b0 < nleaf; b0 += QS_LIST_CHUNK) {
            const uint64_t cnt = std::min<uint64_t>(nleaf - b0, QS_LIST_CHUNK);
            e = cudaMemcpyAsync(d_lo, leaf_lo.data() + b0, 8 * cnt, cudaMemcpyHostToDevice, st);
            if (e == cudaSuccess) e = cudaMemcpyAsync(d_len, leaf_len.data() + b0, 4 * cnt, cudaMemcpyHostToDevice, st);
            if (e != cudaSuccess) return cuda_fail(e, "quicksort leaves H2D");
            if (P.leaf_algo == 1) {
                const size_t smem = sizeof(K) * LC::LEAF;
                cudaFuncSetAttribute(qs_leaf_kernel<K, LC::LEAF, LC::NT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem);
                qs_leaf_kernel<K, LC::LEAF, LC::NT><<<(unsigned)cnt, LC::NT, smem, st>>>(keys, d_lo, d_len);
            } else if (LEAF <= (uint64_t)LC::LEAF / 2) {  // small leaves: half-size CTAs, more per SM
                constexpr int HL = LC::LEAF / 2, HN = HL / LEAF_E;
                const size_t smem = 2 * sizeof(K) * (HL + HL / 8);
                cudaFuncSetAttribute(qs_leaf_merge_kernel<K, HL, HN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem);
                qs_leaf_merge_kernel<K, HL, HN><<<(unsigned)cnt, HN, smem, st>>>(keys, d_lo, d_len);
            } else {
                const size_t smem = 2 * sizeof(K) * (LC::LEAF + LC::LEAF / 8);
                cudaFuncSetAttribute(qs_leaf_merge_kernel<K, LC::LEAF, LC::NT>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                qs_leaf_merge_kernel<K, LC::LEAF, LC::NT><<<(unsigned)cnt, LC::NT, smem, st>>>(keys, d_lo, d_len);
            }
            note_launches(1);
            e = cudaGetLastError();
            if (e != cudaSuccess) return cuda_fail(e, "quicksort leaf launch");
        }
    }
    // the host vectors must outlive the async copies
    e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return cuda_fail(e, "quicksort leaves");
    {
        void* uw = nullptr;
        size_t ub = 0;
        last_stats().aux_bytes = user_workspace(&uw, &ub) ? g_qs_user_base + g_qs_peak : g_qws_bytes;
    }
    return PP_OK;
}

template pp_status quicksort_device<uint64_t>(uint64_t*, uint64_t, cudaStream_t);
template pp_status quicksort_device<uint32_t>(uint32_t*, uint64_t, cudaStream_t);

}  // namespace pp
