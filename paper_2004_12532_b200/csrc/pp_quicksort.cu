// pp_quicksort.cu -- in-place quicksort layered on the partition
// (§5 "Example Application: A Full Quicksort").
//
// The paper runs the parallel partition at the top levels of the recursion
// and a serial partition once subproblems are small.
// The GPU analogue is a breadth-first level loop:
//   - big segments (>= 2^27 keys): the full multi-CTA partition pipeline of
//     pp_partition.cu, one segment at a time;
//   - mid segments: ONE launch for all of them: the Smoothed Striding group
//     kernel with (segment, group) tasks, then the batched multi-CTA cleanup
//     (heavy segments) or one CTA per segment reducing its groups and
//     cleaning its (small) window by the rank-matched walk;
//   - small segments (<= 2^16 keys): one CTA each runs the rest of the
//     recursion (qs_small_kernel) and packs the leaves (<= 16384 keys) into
//     bins; every bin is sorted by a counting sort in shared memory
//     (qs_leaf_bidx_kernel; crowded bins by the merge sort of
//     qs_leaf_handoff_kernel).
// Pivot: median of A[lo], A[lo+(len-1)/2], A[hi-1]; split by x < p; when that
// split is empty (p is the segment minimum) the next level splits by x <= p
// and the left part (all == p) is final (reading R14).  Every
// segment carries the bounds [kmin, kmax] its ancestors' pivots imply; when
// they collapse to one value the segment is all equal keys and final.
#include <algorithm>
#include <chrono>
#include <functional>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "pp_engine.cuh"

namespace pp {

void note_launches(uint64_t k);

struct QSeg {
    uint64_t lo, hi;   // [lo, hi)
    uint64_t pivot;    // effective strict pivot (key < pivot goes left)
    uint64_t gbase;    // first task (CTA) of this segment in the group launch
    uint64_t g;        // groups of this segment
    uint32_t mode;     // 0: pivot = median-of-3 (computed on device); 1: pivot given (x <= p step);
                       // 2: pivot = ninther; 3: median of 31 samples (computed on device; param
                       // qs_pivot, and segments deeper than QS_DEEP take at least the ninther)
    uint32_t pad;      // device-built levels (qs_dev): the segment's depth
    uint64_t kmin;     // every key of the segment is >= kmin (the pivots above it)
};

// Counts of a device-built level list (qs_dev): the kernels of the level read
// them instead of launch arguments, so the host can enqueue the level before
// the list exists (grids are host-side upper bounds; surplus CTAs exit).
struct QDevCtl {
    uint64_t nmid, gtot, err, pad;
};

template <typename K>
__device__ __forceinline__ K median3(K a, K b, K c) {
    if (a > b) { K t = a; a = b; b = t; }
    if (b > c) b = c;
    return a > b ? a : b;
}

// Tukey's ninther: the median of the medians of three triples at the nine
// positions lo + j (len - 1) / 8, j = 0..8 (deep segments, see QS_DEEP)
template <typename K>
__host__ __device__ __forceinline__ uint64_t ninther_pos(uint64_t lo, uint64_t len, int j) {
    return lo + (len - 1) / 8 * (uint64_t)j + ((len - 1) % 8) * (uint64_t)j / 8;
}

// One warp per segment: mode 0 median of 3, 2 ninther, 3 the median of 31
// evenly spaced samples (warp bitonic sort of 31 samples + one +inf pad).
// the median of 31 evenly spaced keys (sample j at lo + j (len - 1) / 30)
template <typename K>
__device__ __forceinline__ K warp_median31(const K* keys, uint64_t lo, uint64_t len, int lane) {
    const K KMAX = (K)~(K)0;
    K v = lane < 31 ? keys[lo + (len - 1) / 30 * (uint64_t)lane + ((len - 1) % 30) * (uint64_t)lane / 30] : KMAX;
#pragma unroll
    for (int k = 2; k <= 32; k <<= 1)
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
            const K o = __shfl_xor_sync(0xffffffffu, v, j);
            const bool up = ((lane & k) == 0), lower = ((lane & j) == 0);
            v = (lower == up) ? (v < o ? v : o) : (v < o ? o : v);
        }
    return __shfl_sync(0xffffffffu, v, 15);  // the 16th smallest of the 31 samples
}

// A sampled pivot equal to the segment's lower bound kmin (every key >= kmin)
// would make the x < p split empty and cost a pass before the x <= p step
// (reading R14); splitting by x < kmin + 1 instead is that x <= p step at
// once: the left part (all == kmin, non-empty since p is a key) is final, the
// right part strictly smaller.  kmin < KMAX here (a segment whose bounds are
// one value is dropped as all equal).
template <typename K>
__host__ __device__ __forceinline__ uint64_t pivot_above_bound(K p, uint64_t kmin) {
    return (uint64_t)p == kmin ? (uint64_t)(K)(p + 1) : (uint64_t)p;
}

// Sample keys of a big segment (host-computed pivot): one launch writing into
// pinned host memory (mapped, UVA) instead of one pageable 8-byte copy each.
struct QsSamplePos {
    uint64_t p[31];
};
template <typename K>
__global__ void qs_sample_kernel(const K* __restrict__ keys, QsSamplePos pos, int ns, uint64_t* out) {
    if ((int)threadIdx.x < ns) out[threadIdx.x] = (uint64_t)keys[pos.p[threadIdx.x]];
}

template <typename K>
__global__ void __launch_bounds__(256) qs_pivot_kernel(const K* __restrict__ keys, QSeg* __restrict__ segs,
                                                       uint64_t nseg, const QDevCtl* __restrict__ dc = nullptr) {
    const int lane = threadIdx.x & 31;
    if (dc) nseg = dc->nmid;
    for (uint64_t s = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; s < nseg;
         s += ((uint64_t)gridDim.x * blockDim.x) >> 5) {
        const QSeg q = segs[s];  // uniform over the warp
        const uint64_t len = q.hi - q.lo;
        if (q.mode == 3) {
            const K p = warp_median31<K>(keys, q.lo, len, lane);
            if (lane == 0) segs[s].pivot = pivot_above_bound<K>(p, q.kmin);
        } else if (lane == 0 && q.mode == 0) {
            segs[s].pivot = pivot_above_bound<K>(
                median3<K>(keys[q.lo], keys[q.lo + (len - 1) / 2], keys[q.hi - 1]), q.kmin);
        } else if (lane == 0 && q.mode == 2) {
            K m[3];
#pragma unroll
            for (int t = 0; t < 3; ++t)
                m[t] = median3<K>(keys[ninther_pos<K>(q.lo, len, 3 * t)], keys[ninther_pos<K>(q.lo, len, 3 * t + 1)],
                                  keys[ninther_pos<K>(q.lo, len, 3 * t + 2)]);
            segs[s].pivot = pivot_above_bound<K>(median3<K>(m[0], m[1], m[2]), q.kmin);
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
                                                                   uint64_t seed, GroupOut* __restrict__ gout,
                                                                   const QDevCtl* __restrict__ dc = nullptr) {
    extern __shared__ __align__(128) unsigned char smem[];
    using C = GroupCfg<K>;
    griddep_wait();  // PDL launch: the pivots come from qs_pivot_kernel
    const uint64_t task = blockIdx.x;
    if (dc) {  // device-built level: the grid is an upper bound
        if (task >= dc->gtot) return;
        nseg = dc->nmid;
    }
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
template <typename K, int NT, int EPT>
__global__ void __launch_bounds__(NT) qs_cleanup_kernel(K* __restrict__ keys, const QSeg* __restrict__ segs,
                                                         const GroupOut* __restrict__ gout,
                                                         uint64_t* __restrict__ splits, uint64_t heavy,
                                                         const QDevCtl* __restrict__ dc = nullptr) {
    using C = GroupCfg<K>;
    extern __shared__ __align__(16) unsigned char csm[];
    griddep_wait();  // PDL launch: gout comes from qs_group_kernel
    if (dc && blockIdx.x >= dc->nmid) return;  // device-built level: the grid is an upper bound
    if (heavy && segs[blockIdx.x].hi - segs[blockIdx.x].lo >= heavy) return;  // batched multi-CTA cleanup
    StreamBuf<NT, EPT>& sb = *reinterpret_cast<StreamBuf<NT, EPT>*>(csm);
    __shared__ uint64_t red[4][NT / 32];
    const QSeg q = segs[blockIdx.x];
    K* seg = keys + q.lo;
    const uint64_t len = q.hi - q.lo;
    const K pivot = (K)q.pivot;
    const uint64_t h = seg_head<K>(keys, q.lo, len);
    const uint64_t n_lines = (len - h) / C::LK;
    const uint64_t region_end = n_lines * C::LK;
    uint64_t T = 0, vmin = region_end, vmax = 0, ht = 0;
    for (uint64_t i = threadIdx.x; i < q.g; i += NT) {
        const GroupOut o = gout[q.gbase + i];
        T += o.T;
        vmin = o.vlo < vmin ? o.vlo : vmin;
        vmax = o.vhi > vmax ? o.vhi : vmax;
    }
    for (uint64_t x = threadIdx.x; x < h; x += NT) ht += is_pred(seg[x], pivot) ? 1 : 0;
    for (uint64_t x = h + region_end + threadIdx.x; x < len; x += NT) ht += is_pred(seg[x], pivot) ? 1 : 0;
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
    for (int w = 0; w < NT / 32; ++w) {
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
    walk_swap_stream<K, NT, EPT>(seg, d, pivot, 0, c.Kv, c.Kv, c.W, sb);
    if (threadIdx.x == 0) splits[blockIdx.x] = Ks;
}

// ---------------------------------------------------------------------------
// Heavy mid segments (>= qs_heavy keys): their dirty windows are long (the
// window grows with the segment's chunk of g_s lines), so one CTA walking it
// is latency bound.  They get the multi-CTA cleanup pipeline of the
// partition (reduce+count, tile scan, locate, rank-matched swap; the device
// bodies of pp_engine.cuh), batched: blockIdx.y = heavy segment, each with
// its own control block and tile arrays (QS_HEAVY_TILES tiles per side, the
// tile size grows with the window).
// ---------------------------------------------------------------------------
constexpr uint64_t QS_HEAVY_TILES = 512;
struct HvLayout {
    size_t ctl, cntL, cntR, PL, PR, posL, posR, rk, ttl, ttr, stride;
};
static HvLayout hv_layout() {
    const uint64_t tiles = QS_HEAVY_TILES + 1, tasks = 2 * QS_HEAVY_TILES + 2;
    HvLayout L;
    size_t o = 0;
    auto take = [&](size_t b) {
        const size_t at = o;
        o += (b + 255) & ~size_t(255);
        return at;
    };
    L.ctl = take(sizeof(Ctl));
    L.cntL = take(4 * tiles);
    L.cntR = take(4 * tiles);
    L.PL = take(8 * tiles);
    L.PR = take(8 * tiles);
    L.posL = take(8 * tasks);
    L.posR = take(8 * tasks);
    L.rk = take(8 * tasks);
    L.ttl = take(4 * tasks);
    L.ttr = take(4 * tasks);
    L.stride = o;
    return L;
}
#define HV_PTR(T, f) reinterpret_cast<T*>(w + L.f)

template <typename K>
__global__ void __launch_bounds__(256) qs_hv_reduce_kernel(K* __restrict__ keys, const QSeg* __restrict__ segs,
                                                           const uint32_t* __restrict__ hidx,
                                                           const GroupOut* __restrict__ gout,
                                                           uint64_t* __restrict__ splits, unsigned char* ws,
                                                           HvLayout L) {
    using C = GroupCfg<K>;
    const uint32_t si = hidx[blockIdx.y];
    const QSeg q = segs[si];
    unsigned char* w = ws + (size_t)blockIdx.y * L.stride;
    const uint64_t len = q.hi - q.lo;
    const uint64_t h = seg_head<K>(keys, q.lo, len);
    reduce_count_body<K, true>(keys + q.lo, len, h, (len - h) / C::LK, (uint32_t)C::LK, gout + q.gbase,
                               (uint32_t)q.g, nullptr, 0, (K)q.pivot, HV_PTR(Ctl, ctl), splits + si,
                               HV_PTR(uint32_t, cntL), HV_PTR(uint32_t, cntR), QS_HEAVY_TILES, blockIdx.x, gridDim.x);
}

__global__ void __launch_bounds__(1024) qs_hv_scan_kernel(unsigned char* ws, HvLayout L) {
    extern __shared__ uint64_t hsp[];
    unsigned char* w = ws + (size_t)blockIdx.x * L.stride;
    tile_scan_body(HV_PTR(Ctl, ctl), HV_PTR(uint32_t, cntL), HV_PTR(uint32_t, cntR), HV_PTR(uint64_t, PL),
                   HV_PTR(uint64_t, PR), HV_PTR(uint64_t, rk), HV_PTR(uint32_t, ttl), HV_PTR(uint32_t, ttr), hsp);
}

template <typename K>
__global__ void __launch_bounds__(SW_NT, 3) qs_hv_locate_kernel(K* __restrict__ keys, const QSeg* __restrict__ segs,
                                                                const uint32_t* __restrict__ hidx,
                                                                unsigned char* ws, HvLayout L) {
    const QSeg q = segs[hidx[blockIdx.y]];
    unsigned char* w = ws + (size_t)blockIdx.y * L.stride;
    locate_body<K>(keys + q.lo, HV_PTR(Ctl, ctl), (K)q.pivot, HV_PTR(uint64_t, PL), HV_PTR(uint64_t, PR),
                   HV_PTR(uint64_t, posL), HV_PTR(uint64_t, posR), HV_PTR(uint64_t, rk), HV_PTR(uint32_t, ttl),
                   HV_PTR(uint32_t, ttr), blockIdx.x, gridDim.x);
}

template <typename K>
__global__ void __launch_bounds__(SW_NT, 3) qs_hv_swap_kernel(K* __restrict__ keys, const QSeg* __restrict__ segs,
                                                              const uint32_t* __restrict__ hidx, unsigned char* ws,
                                                              HvLayout L) {
    const QSeg q = segs[hidx[blockIdx.y]];
    unsigned char* w = ws + (size_t)blockIdx.y * L.stride;
    swap_body<K>(keys + q.lo, HV_PTR(Ctl, ctl), (K)q.pivot, HV_PTR(uint64_t, posL), HV_PTR(uint64_t, posR),
                 HV_PTR(uint64_t, rk), blockIdx.x, gridDim.x);
}
#undef HV_PTR

// ---------------------------------------------------------------------------
// Device-built levels (param qs_dev; SURVEY §8(a) a9 "next-level segment list
// compacted by scan"): one CTA turns a level's list, its pivots and its splits
// into the next level's list of mid segments -- the same children (P:1701-1732
// with reading R14's x <= p step), group counts, straggler take-back and
// longest-first order as the host loop (launch_level / finish_level) -- so the
// host can enqueue the next level before this one has run.  Small and leaf
// children stay with the host, which reads every level back one level behind
// (their per-CTA recursion and bin sorts run on other streams anyway).
// Deterministic: block scans and a stable per-warp counting sort, no atomics.
// ---------------------------------------------------------------------------
struct QBuildArgs {
    uint64_t small;     // mid children are longer than this (SMALL)
    uint64_t g_target;  // G_TARGET
    uint64_t minl;      // MINL: at least this many lines per group
    uint64_t slots;     // G_TARGET / qs_waves: CTA slots of one wave
    uint64_t nmax;      // capacity of the next list (<= QB_NMAX)
    uint32_t rule;      // level pivot rule (QSeg.mode of new segments) ...
    uint32_t deep;      // ... and the depth past which median of 3 becomes the ninther
    uint32_t pivots;    // 1: compute the next level's pivots here (rules 0 and 2; no pivot kernel then)
};
constexpr int QB_NT = 1024, QB_NW = QB_NT / 32, QB_NBK = 512;
constexpr uint64_t QB_NMAX = (uint64_t)QB_NBK * QB_NW;  // histogram entries; lists of <= QB_NMAX / 2 (shared memory)

// exclusive scan of one value per thread over the CTA; *tot = the sum
__device__ __forceinline__ uint64_t qb_scan(uint64_t v, uint64_t* wsum, uint64_t* tot) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint64_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint64_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) wsum[w] = x;
    __syncthreads();
    if (w == 0) {
        uint64_t z = wsum[lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint64_t y = __shfl_up_sync(0xffffffffu, z, o);
            if (lane >= o) z += y;
        }
        wsum[lane] = z;
    }
    __syncthreads();
    const uint64_t r = x - v + (w ? wsum[w - 1] : 0);
    *tot = wsum[QB_NW - 1];
    __syncthreads();
    return r;
}

// maximum over the CTA
__device__ __forceinline__ uint64_t qb_max(uint64_t v, uint64_t* wsum) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = max(v, (uint64_t)__shfl_xor_sync(0xffffffffu, v, o));
    if (lane == 0) wsum[w] = v;
    __syncthreads();
    uint64_t r = 0;
#pragma unroll 8
    for (int i = 0; i < QB_NW; ++i) r = max(r, wsum[i]);
    __syncthreads();
    return r;
}

struct QChild {
    uint64_t lo, hi, pivot, kmin, kmax;
    uint32_t mode;
};
// the mid children of one segment (host: finish_level's visit + add_child)
template <typename K>
__device__ __forceinline__ int qb_children(const QSeg& q, uint64_t k, uint64_t kmin, uint64_t kmax,
                                           const QBuildArgs& a, QChild (&c)[2]) {
    const K KMAX = (K)~(K)0;
    const uint32_t d = q.pad + 1;
    const uint32_t mrule = (d > a.deep && a.rule == 0) ? 2u : a.rule;
    int n = 0;
    auto add = [&](uint64_t lo, uint64_t hi, uint64_t kmn, uint64_t kmx) {
        if (hi - lo > a.small && kmn != kmx) c[n++] = QChild{lo, hi, 0, kmn, kmx, mrule};  // kmn == kmx: all equal
    };
    const uint64_t p = q.pivot;
    if (q.mode != 1) {
        if (k == 0) {
            // p is the segment minimum: split by x <= p next (unless p is the bound: all equal)
            if (p != kmax) c[n++] = QChild{q.lo, q.hi, (uint64_t)(K)(p + 1), p, kmax, 1u};
        } else {
            add(q.lo, q.lo + k, kmin, p - 1);  // keys < p
            add(q.lo + k, q.hi, p, kmax);      // keys >= p
        }
    } else {
        add(q.lo + k, q.hi, q.pivot, kmax);  // [lo, lo+k) is all equal: final
    }
    return n;
}

__device__ __forceinline__ uint32_t qb_bucket(uint64_t nl, uint64_t g) {  // host: launch_level's LPT buckets
    const uint64_t lpg = max((uint64_t)1, (nl << 10) / g);
    const int oct = 63 - __clzll((long long)lpg);
    const int sub = oct >= 3 ? (int)((lpg >> (oct - 3)) & 7) : (int)((lpg << (3 - oct)) & 7);
    return (uint32_t)(QB_NBK - 1 - (oct * 8 + sub));
}

template <typename K>
__global__ void __launch_bounds__(QB_NT) qs_build_kernel(const K* __restrict__ keys, const QSeg* __restrict__ cur,
                                                         const uint64_t* __restrict__ ckb,
                                                         const QDevCtl* __restrict__ cc,
                                                         const uint64_t* __restrict__ splits, QSeg* tmp,
                                                         uint64_t* tkb, QSeg* __restrict__ nxt,
                                                         uint64_t* __restrict__ nkb, QDevCtl* __restrict__ nc,
                                                         QBuildArgs a) {
    using C = GroupCfg<K>;
    extern __shared__ __align__(16) uint32_t qbs[];
    uint32_t* hist = qbs;                 // [QB_NBK][QB_NW] counts, then offsets; later g by list position
    uint32_t* pos = qbs + QB_NMAX;        // per child: rank in its warp's bucket, then its list position
    uint32_t* gs = pos + a.nmax;          // per child: groups
    uint32_t* nls = gs + a.nmax;          // per child: lines of its aligned region
    __shared__ uint64_t wsum[QB_NW];
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    const uint64_t N = cc->nmid;
    // 1. mid children of this thread's segments (contiguous runs: list order), compacted by a scan
    const uint64_t ipt = (N + QB_NT - 1) / QB_NT;
    const uint64_t s0 = min(N, (uint64_t)t * ipt), s1 = min(N, s0 + ipt);
    uint64_t cnt = 0;
    for (uint64_t i = s0; i < s1; ++i) {
        QChild c[2];
        cnt += qb_children<K>(cur[i], splits[i], ckb[2 * i], ckb[2 * i + 1], a, c);
    }
    uint64_t M = 0;
    uint64_t off = qb_scan(cnt, wsum, &M);
    if (M > a.nmax) {  // impossible: mid children are disjoint and longer than SMALL
        if (t == 0) *nc = QDevCtl{0, 0, 1, 0};
        return;
    }
    uint64_t lines = 0;
    for (uint64_t i = s0; i < s1; ++i) {
        QChild c[2];
        const QSeg q = cur[i];
        const int m = qb_children<K>(q, splits[i], ckb[2 * i], ckb[2 * i + 1], a, c);
        for (int j = 0; j < m; ++j, ++off) {
            const uint64_t len = c[j].hi - c[j].lo;
            const uint64_t nl = (len - seg_head<K>(keys, c[j].lo, len)) / C::LK;  // lines of the aligned region
            QSeg x;
            x.lo = c[j].lo;
            x.hi = c[j].hi;
            x.pivot = c[j].pivot;
            if (a.pivots && c[j].mode != 1u) {
                // the next level's pivot (its keys are final now): median of 3,
                // or the ninther past the depth guard; at the lower bound, kmin + 1
                K pk;
                if (c[j].mode == 2u) {
                    K m[3];
#pragma unroll
                    for (int t3 = 0; t3 < 3; ++t3)
                        m[t3] = median3<K>(keys[ninther_pos<K>(x.lo, len, 3 * t3)],
                                           keys[ninther_pos<K>(x.lo, len, 3 * t3 + 1)],
                                           keys[ninther_pos<K>(x.lo, len, 3 * t3 + 2)]);
                    pk = median3<K>(m[0], m[1], m[2]);
                } else {
                    pk = median3<K>(keys[x.lo], keys[x.lo + (len - 1) / 2], keys[x.hi - 1]);
                }
                x.pivot = pivot_above_bound<K>(pk, c[j].kmin);
            }
            x.gbase = nl;  // (lines until the list is ordered)
            x.g = 0;
            x.mode = c[j].mode;
            x.pad = q.pad + 1;
            x.kmin = c[j].kmin;
            tmp[off] = x;
            tkb[2 * off] = c[j].kmin;
            tkb[2 * off + 1] = c[j].kmax;
            nls[off] = (uint32_t)nl;
            lines += nl;
        }
    }
    uint64_t mid_lines = 0;
    qb_scan(lines, wsum, &mid_lines);  // (its barriers publish tmp to the CTA)
    // 2. groups per child: round(lines / L*) within [1, lines / MINL], L* = lines of the level / G_TARGET
    const double Lstar = fmax(1.0, (double)mid_lines / (double)a.g_target);
    uint64_t gsum = 0;
    for (uint64_t j = t; j < M; j += QB_NT) {
        const uint64_t nl = nls[j];
        const uint64_t cap = max((uint64_t)1, nl / a.minl);
        const uint64_t want = (uint64_t)((double)nl / Lstar + 0.5);
        const uint64_t g = max((uint64_t)1, min(cap, want));
        gs[j] = (uint32_t)g;
        gsum += g;
    }
    uint64_t gtot = 0;
    qb_scan(gsum, wsum, &gtot);
    // 3. a few CTAs past a whole number of waves: take them back round robin over
    //    the children by groups, descending (ties: list order), as the host does.
    //    Pass r takes one from every child with g >= r + 2, so R full passes and
    //    then the first m children of that order (all have g >= R + 2).
    const uint64_t excess = gtot > a.slots ? gtot % a.slots : 0;
    if (excess > 0 && excess <= a.slots / 16) {
        uint64_t left = excess, R = 0, m = 0;
        for (;;) {
            uint64_t c = 0, cr = 0;
            for (uint64_t j = t; j < M; j += QB_NT) c += gs[j] >= R + 2 ? 1 : 0;
            qb_scan(c, wsum, &cr);
            if (cr == 0) break;         // nothing left to take (the host's loop ends there too)
            if (cr >= left) { m = left; break; }
            left -= cr;
            ++R;
        }
        // the m-th largest g (Gs) and the children above it (above < m)
        uint64_t Gs = 0, above = 0;
        if (m > 0) {
            uint64_t lo = R + 2, hi = 1;  // count(g >= lo) >= m holds; find the largest such lo
            uint64_t gm = 0;
            for (uint64_t j = t; j < M; j += QB_NT) gm = max(gm, (uint64_t)gs[j]);
            hi = qb_max(gm, wsum) + 1;  // count(g >= hi) = 0 < m
            while (hi - lo > 1) {
                const uint64_t mid = (lo + hi) >> 1;
                uint64_t c = 0, cm = 0;
                for (uint64_t j = t; j < M; j += QB_NT) c += gs[j] >= mid ? 1 : 0;
                qb_scan(c, wsum, &cm);
                if (cm >= m) lo = mid; else hi = mid;
            }
            Gs = lo;
            uint64_t c = 0;
            for (uint64_t j = t; j < M; j += QB_NT) c += gs[j] > Gs ? 1 : 0;
            qb_scan(c, wsum, &above);
        }
        // ties at Gs in list order: contiguous runs per thread for the scan
        const uint64_t ipm = (M + QB_NT - 1) / QB_NT;
        const uint64_t j0 = min(M, (uint64_t)t * ipm), j1 = min(M, j0 + ipm);
        uint64_t ties = 0, tot = 0;
        for (uint64_t j = j0; j < j1; ++j) ties += (m > 0 && gs[j] == Gs) ? 1 : 0;
        uint64_t trank = qb_scan(ties, wsum, &tot);
        uint64_t dsum = 0;
        for (uint64_t j = j0; j < j1; ++j) {
            const uint64_t g = gs[j];
            uint64_t dec = min(R, g - 1);
            if (m > 0 && (g > Gs || (g == Gs && trank++ < m - above))) dec += 1;
            gs[j] = (uint32_t)(g - dec);
            dsum += dec;
        }
        uint64_t dtot = 0;
        qb_scan(dsum, wsum, &dtot);
        gtot -= dtot;
    }
    // 4. longest-first order: stable counting sort by bucket of lines per group
    //    (each warp owns a contiguous run of children and its own histogram row)
    for (uint64_t e = t; e < QB_NMAX; e += QB_NT) hist[e] = 0;
    __syncthreads();
    const uint64_t ipw = (M + QB_NW - 1) / QB_NW;
    const uint64_t w0 = min(M, (uint64_t)w * ipw), w1 = min(M, w0 + ipw);
    for (uint64_t b = w0; b < w1; b += 32) {
        const uint64_t j = b + lane;
        const bool act = j < w1;
        const uint32_t bk = act ? qb_bucket(nls[j], gs[j]) : 0xffffffffu;
        const uint32_t peers = __match_any_sync(0xffffffffu, bk);
        uint32_t base = 0;
        if (act) base = hist[bk * QB_NW + w];
        __syncwarp();
        const uint32_t rank = __popc(peers & ((1u << lane) - 1));
        if (act && rank == 0) hist[bk * QB_NW + w] = base + __popc(peers);
        __syncwarp();
        if (act) pos[j] = base + rank;
    }
    __syncthreads();
    {   // bucket-major, warp-minor offsets
        constexpr int EPT = (int)(QB_NMAX / QB_NT);
        uint32_t loc[EPT];
        uint64_t sum = 0;
#pragma unroll
        for (int i = 0; i < EPT; ++i) {
            loc[i] = hist[t * EPT + i];
            sum += loc[i];
        }
        uint64_t tot = 0;
        uint64_t ex = qb_scan(sum, wsum, &tot);
#pragma unroll
        for (int i = 0; i < EPT; ++i) {
            hist[t * EPT + i] = (uint32_t)ex;
            ex += loc[i];
        }
    }
    __syncthreads();
    for (uint64_t b = w0; b < w1; b += 32) {
        const uint64_t j = b + lane;
        if (j < w1) pos[j] += hist[qb_bucket(nls[j], gs[j]) * QB_NW + w];
    }
    __syncthreads();
    // 5. first task of each child: exclusive scan of g in list order (hist now holds g by position)
    for (uint64_t j = t; j < M; j += QB_NT) hist[pos[j]] = gs[j];
    __syncthreads();
    {
        const uint64_t ipm = (M + QB_NT - 1) / QB_NT;
        const uint64_t j0 = min(M, (uint64_t)t * ipm), j1 = min(M, j0 + ipm);
        uint64_t sum = 0, tot = 0;
        for (uint64_t j = j0; j < j1; ++j) sum += hist[j];
        uint64_t ex = qb_scan(sum, wsum, &tot);
        for (uint64_t j = j0; j < j1; ++j) {
            const uint32_t g = hist[j];
            hist[j] = (uint32_t)ex;
            ex += g;
        }
    }
    __syncthreads();
    for (uint64_t j = t; j < M; j += QB_NT) {
        const uint32_t d = pos[j];
        QSeg x = tmp[j];
        x.g = gs[j];
        x.gbase = hist[d];
        nxt[d] = x;
        nkb[2 * (uint64_t)d] = tkb[2 * j];
        nkb[2 * (uint64_t)d + 1] = tkb[2 * j + 1];
    }
    if (t == 0) *nc = QDevCtl{M, gtot, 0, 0};
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
static inline uint32_t lpad_host(uint32_t i) { return i + (i >> 3); }

template <typename K>
__device__ __forceinline__ void sort8(K (&v)[8]) {  // Batcher's 19-comparator network
    cmpx(v[0], v[1]); cmpx(v[2], v[3]); cmpx(v[4], v[5]); cmpx(v[6], v[7]);
    cmpx(v[0], v[2]); cmpx(v[1], v[3]); cmpx(v[4], v[6]); cmpx(v[5], v[7]);
    cmpx(v[1], v[2]); cmpx(v[5], v[6]);
    cmpx(v[0], v[4]); cmpx(v[1], v[5]); cmpx(v[2], v[6]); cmpx(v[3], v[7]);
    cmpx(v[2], v[4]); cmpx(v[3], v[5]);
    cmpx(v[1], v[2]); cmpx(v[3], v[4]); cmpx(v[5], v[6]);
}

// The 8 outputs starting at `base` of one merge step: runs of length L in
// src (padded layout) -> c[0..8).  Runs A = [blk, blk+La), B = [blk+La, +Lb)
// (the last pair may be short); the start is found on the merge path by
// binary search (ties: A first).
template <typename K>
__device__ __forceinline__ void merge_chunk_regs(const K* __restrict__ src, uint32_t base, uint32_t L, uint32_t P,
                                                 K (&c)[8]) {
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
}

template <typename K>
__device__ __forceinline__ void merge_chunk(const K* __restrict__ src, K* __restrict__ dst, uint32_t base,
                                            uint32_t L, uint32_t P) {
    K c[8];
    merge_chunk_regs<K>(src, base, L, P, c);
#pragma unroll
    for (int i = 0; i < 8; ++i) dst[lpad(base + i)] = c[i];
}

// Sorts the 256 keys of a warp held as 8 consecutive keys per lane (lane l
// holds positions 8l..8l+7, each lane's 8 already ascending) in registers:
// bitonic merges of ascending runs 8 -> 16 -> ... -> 256.  Each merge of two
// ascending runs of k/2 is a "flip" stage (position i against i ^ (k-1), the
// reversed partner, so no descending runs are needed) then half-cleaners
// i ^ j for j = k/4 .. 1; partners in other lanes come by __shfl_xor_sync,
// j < 8 stays inside the lane.
template <typename K>
__device__ __forceinline__ void warp_sort256(K (&v)[8]) {
    const uint32_t lane = threadIdx.x & 31;
#pragma unroll
    for (uint32_t k = 16; k <= 256; k <<= 1) {
        {  // flip: element (lane, r) vs (lane ^ (k/8 - 1), 7 - r)
            const uint32_t m = k / 8 - 1;
            const bool lower = (lane & (k / 16)) == 0;
            K y[8];
#pragma unroll
            for (int r = 0; r < 8; ++r) y[r] = __shfl_xor_sync(0xffffffffu, v[7 - r], m);
#pragma unroll
            for (int r = 0; r < 8; ++r) v[r] = lower ? (v[r] < y[r] ? v[r] : y[r]) : (v[r] < y[r] ? y[r] : v[r]);
        }
#pragma unroll
        for (uint32_t j = k / 4; j >= 8; j >>= 1) {  // half-cleaners across lanes
            const uint32_t m = j / 8;
            const bool lower = (lane & m) == 0;
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                const K y = __shfl_xor_sync(0xffffffffu, v[r], m);
                v[r] = lower ? (v[r] < y ? v[r] : y) : (v[r] < y ? y : v[r]);
            }
        }
        // half-cleaners j = 4, 2, 1 inside the lane
#pragma unroll
        for (int r = 0; r < 4; ++r) cmpx(v[r], v[r + 4]);
#pragma unroll
        for (int r = 0; r < 8; r += 4) {
            cmpx(v[r], v[r + 2]);
            cmpx(v[r + 1], v[r + 3]);
        }
#pragma unroll
        for (int r = 0; r < 8; r += 2) cmpx(v[r], v[r + 1]);
    }
}

// Sorts the P (a multiple of 256) keys of a padded shared-memory buffer
// (index lpad(i)) with nthr = P/8 threads: 8 consecutive keys per thread
// sorted in registers, runs of 256 per warp by the shuffle bitonic merge,
// then merge rounds in place (outputs staged in registers across a barrier).
// Ends with a barrier: buf holds the sorted keys.
template <typename K>
__device__ __forceinline__ void smem_merge_sort(K* buf, uint32_t P, uint32_t nthr) {
    const uint32_t base = threadIdx.x * LEAF_E;
    K v[LEAF_E];
#pragma unroll
    for (int r = 0; r < LEAF_E; ++r) v[r] = buf[lpad(base + r)];
    sort8(v);
    warp_sort256(v);  // runs of 256 (one warp) sorted in registers
    leaf_bar(nthr);
#pragma unroll
    for (int r = 0; r < LEAF_E; ++r) buf[lpad(base + r)] = v[r];
    leaf_bar(nthr);
    for (uint32_t L = 32 * LEAF_E; L < P; L <<= 1) {
        merge_chunk_regs<K>(buf, base, L, P, v);
        leaf_bar(nthr);
#pragma unroll
        for (int r = 0; r < LEAF_E; ++r) buf[lpad(base + r)] = v[r];
        leaf_bar(nthr);
    }
}


// The bins another bin sort handed over (length word tagged BIN_HANDOFF):
// a persistent grid walks all slots (one per thread) and merge-sorts the
// tagged ones (rare: keys clustered inside a wide range), so the untagged
// majority costs one load each instead of one CTA launch each.  Bins of up
// to 2 LEAF keys: each half is merge-sorted in its part of one padded buffer
// (the second half right after the first, so the pair is laid out as two
// adjacent runs) and one merge-path round writes the result to global memory.
constexpr uint32_t BIN_HANDOFF = 0x80000000u;
template <typename K, int LEAF, int NT>
__global__ void __launch_bounds__(NT) qs_leaf_handoff_kernel(K* __restrict__ keys,
                                                             const uint64_t* __restrict__ leaf_lo,
                                                             const uint32_t* __restrict__ leaf_len, uint64_t cnt) {
    static_assert(LEAF == NT * LEAF_E, "one block holds LEAF keys per half");
    extern __shared__ __align__(16) unsigned char lsm[];
    K* buf = reinterpret_cast<K*>(lsm);  // [lpad(2 LEAF)]
    const K KMAX = (K)~(K)0;
    __shared__ uint32_t tags[NT];
    const uint32_t tid = threadIdx.x;
    for (uint64_t base = (uint64_t)blockIdx.x * NT; base < cnt; base += (uint64_t)gridDim.x * NT) {
        const uint32_t t = base + tid < cnt ? leaf_len[base + tid] : 0u;  // one slot per thread
        tags[tid] = t;
        if (!__syncthreads_or((t & BIN_HANDOFF) != 0u)) continue;
        for (uint32_t k = 0; k < (uint32_t)NT; ++k) {
            const uint32_t tagged = tags[k];
            if (!(tagged & BIN_HANDOFF)) continue;  // uniform over the CTA
            const uint32_t len = tagged & ~BIN_HANDOFF;
            const uint64_t lo = leaf_lo[base + k];
            const uint32_t h1 = len < (uint32_t)LEAF ? len : (uint32_t)LEAF, h2 = len - h1;
            const uint32_t P1 = (h1 + 32 * LEAF_E - 1) / (32 * LEAF_E) * (32 * LEAF_E);
            const uint32_t P2 = (h2 + 32 * LEAF_E - 1) / (32 * LEAF_E) * (32 * LEAF_E);
            K* buf2 = buf + lpad(LEAF);
#pragma unroll
            for (int r = 0; r < LEAF_E; ++r) {
                const uint32_t i = (uint32_t)r * NT + tid;
                if (i < P1) buf[lpad(i)] = i < h1 ? __ldcs(keys + lo + i) : KMAX;
                if (i < P2) buf2[lpad(i)] = i < h2 ? __ldcs(keys + lo + LEAF + i) : KMAX;
            }
            __syncthreads();
            if (tid < P1 / LEAF_E) smem_merge_sort<K>(buf, P1, P1 / LEAF_E);
            __syncthreads();
            if (h2 == 0) {
#pragma unroll
                for (int r = 0; r < LEAF_E; ++r) {
                    const uint32_t i = (uint32_t)r * NT + tid;
                    if (i < len) __stcs(keys + lo + i, buf[lpad(i)]);
                }
            } else {
                if (tid < P2 / LEAF_E) smem_merge_sort<K>(buf2, P2, P2 / LEAF_E);
                __syncthreads();
                // runs [0, LEAF) and [LEAF, LEAF + P2): 8 outputs per chunk, two chunks per thread
                for (uint32_t c = tid; c < (LEAF + P2) / LEAF_E; c += NT) {
                    K v[LEAF_E];
                    merge_chunk_regs<K>(buf, c * LEAF_E, LEAF, LEAF + P2, v);
#pragma unroll
                    for (int r = 0; r < LEAF_E; ++r)
                        if (c * LEAF_E + r < len) __stcs(keys + lo + c * LEAF_E + r, v[r]);
                }
            }
            __syncthreads();  // buf is reused by the next tagged bin
        }
        __syncthreads();  // tags[] is rewritten by the next chunk
    }
}


constexpr uint32_t BK_MAX_RUN = 48;
// buckets per key slot of a bin (1 -- 176 KiB, room for a co-resident per-CTA
// recursion CTA -- measured +0.3%; 2 also leaves the run list its space)
#define PP_BIN_BX 2
template <typename K>
__device__ __forceinline__ int key_bits(K v) {
    return sizeof(K) == 8 ? 64 - __clzll((long long)v) : 32 - __clz((int)v);
}

// Bin sort: a counting sort of one bin (<= PLEAF keys) in shared memory.  The
// keys are staged in input order; bucket d = (key - min) >> sh over 2 PLEAF
// buckets (16-bit counts packed two per word, one shared-memory atomic per
// key returns its slot in the bucket); one block scan gives the bucket starts;
// every key keeps (position, slot, bucket size) packed in one register, so the
// 16-bit INDEX array scattered next reuses the counters' memory.  The key in
// slot 0 of a bucket of c > 1 keys marks the run [start, start + c) in a
// byte array; the thread owning the run's first position (16 positions per
// thread) insertion-sorts that run of indices by key (runs are disjoint; c <=
// BK_MAX_RUN).  The keys are then gathered through the indices into
// coalesced stores.  16384-key bins: 1024 threads, 208 KiB, one CTA per SM;
// 8192-key bins: 512 threads, two CTAs per SM.  A bin with a crowded bucket
// (> BK_MAX_RUN keys while sh > 0) is left untouched and tagged (BIN_HANDOFF
// in its length word) for qs_leaf_handoff_kernel, launched right after.
// (Round 2: the per-run insertion sort replaced a per-key rank loop -- each
// key of a multi-key bucket counted the bucket's smaller keys, divergent
// across the warp -- 37% of the kernel's instructions; the kernel time barely
// moved, 3.69 -> 3.66 ms per 2^28-key sort: it is bound by its HBM load
// latency at one CTA per SM, not by issue.)
template <typename K, int PLEAF, int NT>
__global__ void __launch_bounds__(NT, PLEAF >= 16384 ? 1 : 2) qs_leaf_bidx_kernel(K* __restrict__ keys,
                                                            const uint64_t* __restrict__ leaf_lo,
                                                            uint32_t* __restrict__ leaf_len,
                                                            const uint64_t* __restrict__ leaf_kb) {
    constexpr int E = PLEAF / NT, NW = NT / 32, NB = PP_BIN_BX * PLEAF, NWD = NB / 2, WPT = NWD / NT;
    constexpr int NBITS = (PLEAF == 16384 ? 14 : PLEAF == 8192 ? 13 : PLEAF == 4096 ? 12 : PLEAF == 2048 ? 11 : 10) +
                          (PP_BIN_BX == 2 ? 1 : 0);
    static_assert((1 << NBITS) == NB && WPT >= 1 && PLEAF <= (1 << 14), "bin geometry");
    static_assert(BK_MAX_RUN < 64, "bucket size fits the 6-bit field");
    extern __shared__ __align__(16) unsigned char lsm[];
    __shared__ K rmn[NW], rmx[NW];
    __shared__ uint64_t sw[32];
    __shared__ int handoff;
    __shared__ uint32_t nruns;  // runs of >= 3 keys listed for pass B of the run sort
    __shared__ __align__(8) uint64_t lbar;
    const K KMAX = (K)~(K)0;
    const uint64_t lo = leaf_lo[blockIdx.x];
    const uint32_t len = leaf_len[blockIdx.x];
    if (len < 2) return;
    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    // the 32-B aligned body of the bin arrives by ONE bulk copy (TMA) and
    // leaves by 32-B stores; the < 32 / sizeof(K) keys before it and after it
    // by plain loads / stores.  The keys are staged at lsm + 32 - head *
    // sizeof(K) so that the body lands aligned in shared memory too.
    constexpr uint32_t VK = 32 / sizeof(K);
    uint32_t head = (uint32_t)(((32u - ((uint32_t)reinterpret_cast<uintptr_t>(keys + lo) & 31u)) & 31u) / sizeof(K));
    head = head < len ? head : len;
    const uint32_t nbody = (len - head) / VK * VK, tail0 = head + nbody;
    K* ks = reinterpret_cast<K*>(lsm + 32) - head;               // [PLEAF] keys, input order
    uint32_t* cw = reinterpret_cast<uint32_t*>(lsm + 32 + sizeof(K) * PLEAF);  // [NWD + 1] packed counts, then starts
    uint16_t* ix = reinterpret_cast<uint16_t*>(cw);             // [PLEAF] key indices (after the starts are read)
    uint8_t* rs = reinterpret_cast<uint8_t*>(cw + NWD + 4);     // [PLEAF] size of the bucket starting here (> 1 only)
    constexpr int RW = PLEAF / NT / 16;  // 16-byte run-start words per thread
    static_assert(RW >= 1 && RW * 16 * NT == PLEAF, "16-byte run-start words per thread");
    if (tid == 0) {
        mbar_init(&lbar, 1);
        fence_mbar_init();
        if (nbody > 0) {
            mbar_expect_tx(&lbar, nbody * (uint32_t)sizeof(K));
            bulk_g2s(ks + head, keys + lo + head, nbody * (uint32_t)sizeof(K), &lbar);
        }
    }
    if (tid < head) ks[tid] = __ldcs(keys + lo + tid);
    if (tid < len - tail0) ks[tail0 + tid] = __ldcs(keys + lo + tail0 + tid);
#pragma unroll
    for (int j = 0; j < WPT; ++j) cw[j * NT + tid] = 0u;
#pragma unroll
    for (int j = 0; j < RW; ++j) reinterpret_cast<uint4*>(rs)[tid * RW + j] = make_uint4(0u, 0u, 0u, 0u);
    if (tid == 0) {
        handoff = 0;
        nruns = 0u;
        cw[NWD] = len;  // the end of the last bucket
    }
    __syncthreads();  // the barrier is initialised (and the head / tail keys are staged)
    if (nbody > 0) mbar_wait(&lbar, 0);
    K mn = KMAX, mx = 0;
    if (leaf_kb) {
        // key bounds of the bin from the quicksort's pivots (every key in
        // [kmin, kmax]): no min / max pass over the keys
        mn = (K)leaf_kb[2 * (uint64_t)blockIdx.x];
        mx = (K)leaf_kb[2 * (uint64_t)blockIdx.x + 1];
    } else {
#pragma unroll
    for (int r = 0; r < E; ++r) {
        const uint32_t i = (uint32_t)r * NT + tid;
        if (i < len) {
            const K v = ks[i];
            mn = v < mn ? v : mn;
            mx = v > mx ? v : mx;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const K a = __shfl_xor_sync(0xffffffffu, mn, o), b = __shfl_xor_sync(0xffffffffu, mx, o);
        mn = a < mn ? a : mn;
        mx = b > mx ? b : mx;
    }
    if (lane == 0) {
        rmn[warp] = mn;
        rmx[warp] = mx;
    }
    __syncthreads();
    if (warp == 0) {
        mn = lane < NW ? rmn[lane] : KMAX;
        mx = lane < NW ? rmx[lane] : (K)0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const K a = __shfl_xor_sync(0xffffffffu, mn, o), b = __shfl_xor_sync(0xffffffffu, mx, o);
            mn = a < mn ? a : mn;
            mx = b > mx ? b : mx;
        }
        if (lane == 0) {
            rmn[0] = mn;
            rmx[0] = mx;
        }
    }
    __syncthreads();
    mn = rmn[0];
    mx = rmx[0];
    }
    if (mn == mx) return;
    const int bits = key_bits<K>(mx - mn);
    const int sh = bits > NBITS ? bits - NBITS : 0;
    // per key: pos (14 bits) | slot in its bucket (6 bits) << 14 | min(bucket size, 63) << 20
    uint32_t meta[E];
#pragma unroll
    for (int r = 0; r < E; ++r) {
        const uint32_t i = (uint32_t)r * NT + tid;
        meta[r] = 0u;
        if (i < len) {
            const uint32_t d = (uint32_t)((ks[i] - mn) >> sh), hs = (d & 1u) * 16u;
            // the slot (14 bits) and the bucket (15 bits), kept for the next phase
            meta[r] = ((atomicAdd(&cw[d >> 1], 1u << hs) >> hs) & 0xFFFFu) | (d << 16);
        }
    }
    __syncthreads();
    {  // bucket starts: thread t owns words [WPT t, WPT t + WPT)
        uint32_t c[WPT], s = 0;
#pragma unroll
        for (int j = 0; j < WPT; ++j) {
            c[j] = cw[tid * WPT + j];
            s += (c[j] & 0xFFFFu) + (c[j] >> 16);
        }
        uint64_t tot;
        uint32_t e = (uint32_t)block_exscan<NT>(s, sw, tot);
        if (sh > 0) {
#pragma unroll
            for (int j = 0; j < WPT; ++j)
                if ((c[j] & 0xFFFFu) > BK_MAX_RUN || (c[j] >> 16) > BK_MAX_RUN) handoff = 1;
        }
#pragma unroll
        for (int j = 0; j < WPT; ++j) {
            const uint32_t e1 = e + (c[j] & 0xFFFFu);
            cw[tid * WPT + j] = e | (e1 << 16);
            e = e1 + (c[j] >> 16);
        }
    }
    __syncthreads();
    if (handoff) {  // crowded buckets: the handoff merge sort takes this bin (keys untouched)
        if (tid == 0) leaf_len[blockIdx.x] = len | BIN_HANDOFF;
        return;
    }
#pragma unroll
    for (int r = 0; r < E; ++r) {
        const uint32_t i = (uint32_t)r * NT + tid;
        if (i < len) {
            const uint32_t d = meta[r] >> 16;
            const uint32_t w = cw[d >> 1];
            const uint32_t b0 = (d & 1u) ? w >> 16 : w & 0xFFFFu;
            const uint32_t b1 = (d & 1u) ? cw[(d >> 1) + 1] & 0xFFFFu : w >> 16;
            const uint32_t slot = meta[r] & 0xFFFFu;
            meta[r] = (b0 + slot) | ((slot & 63u) << 14) | (min(b1 - b0, 63u) << 20);
        }
    }
    __syncthreads();  // the counters are dead: ix takes their memory
#pragma unroll
    for (int r = 0; r < E; ++r) {
        const uint32_t i = (uint32_t)r * NT + tid;
        if (i < len) {
            const uint32_t p = meta[r] & 0x3FFFu, c = meta[r] >> 20;
            ix[p] = (uint16_t)i;
            if (sh > 0 && ((meta[r] >> 14) & 63u) == 0u && c > 1u) rs[p] = (uint8_t)c;  // slot 0 marks the run
        }
    }
    __syncthreads();
    if (sh > 0) {
        // keys of one bucket sit in scatter order at [b0, b0 + c): sort each
        // such run of indices by key (runs are disjoint; equal keys are equal
        // bytes, their order never shows).  Pass A: the thread owning position
        // b0 (16 consecutive positions per thread) orders every run of TWO
        // with one predicated compare-exchange; runs of >= 3 (c <= BK_MAX_RUN:
        // a crowded bin was handed off) are appended to a list in the
        // counters' free second half.  Pass B: the list, one run per thread,
        // insertion sort -- so a warp's lanes never idle behind one lane's
        // long run.
        static_assert(PP_BIN_BX == 2, "the run list lives in the counters' second half");
        uint32_t* runs = cw + NWD / 2;  // ix takes the first half; room for PLEAF runs
#pragma unroll 1
        for (int rw = 0; rw < RW; ++rw) {
            const uint4 w4 = reinterpret_cast<const uint4*>(rs)[tid * RW + rw];
            if ((w4.x | w4.y | w4.z | w4.w) != 0u) {
                const uint32_t wv[4] = {w4.x, w4.y, w4.z, w4.w};
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    // visit only the run starts (nonzero bytes) of this word
                    for (uint32_t w = wv[q]; w != 0u;) {
                        const uint32_t bb = (uint32_t)(__ffs(w) - 1) >> 3;
                        const uint32_t c = (w >> (8 * bb)) & 0xFFu;
                        w &= ~(0xFFu << (8 * bb));
                        const uint32_t b0 = (tid * RW + rw) * 16u + (uint32_t)q * 4u + bb;
                        if (c == 2u) {
                            const uint16_t a = ix[b0], b = ix[b0 + 1];
                            if (ks[b] < ks[a]) {
                                ix[b0] = b;
                                ix[b0 + 1] = a;
                            }
                        } else {
                            runs[atomicAdd(&nruns, 1u)] = b0 | (c << 16);
                        }
                    }
                }
            }
        }
        __syncthreads();
        const uint32_t nr = nruns;
        for (uint32_t r = tid; r < nr; r += NT) {
            const uint32_t b0 = runs[r] & 0xFFFFu, c = runs[r] >> 16;
#pragma unroll 1
            for (uint32_t m = 1; m < c; ++m) {
                const uint16_t x = ix[b0 + m];
                const K kx = ks[x];
                uint32_t j = m;
                while (j > 0) {
                    const uint16_t y = ix[b0 + j - 1];
                    if (!(ks[y] > kx)) break;
                    ix[b0 + j] = y;
                    --j;
                }
                ix[b0 + j] = x;
            }
        }
        __syncthreads();
    }
    // gather through the indices; 32-B stores (STG.256) for the aligned body
    for (uint32_t q = tid; q < nbody / VK; q += NT) {
        const uint32_t j = head + q * VK;
        union {
            K k[VK];
            unsigned long long w[4];
        } v;
#pragma unroll
        for (int e = 0; e < (int)VK; ++e) v.k[e] = ks[ix[j + e]];
        asm volatile("st.global.cs.v4.u64 [%0], {%1, %2, %3, %4};" ::"l"(keys + lo + j), "l"(v.w[0]), "l"(v.w[1]),
                     "l"(v.w[2]), "l"(v.w[3])
                     : "memory");
    }
    if (tid < head) __stcs(keys + lo + tid, ks[ix[tid]]);
    if (tid < len - tail0) __stcs(keys + lo + tail0 + tid, ks[ix[tail0 + tid]]);
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
// 128 threads, 4 KiB lines with 4 in flight per end (refills issued by one
// lane per line), 32 KiB sort buffers: 4 CTAs per SM (independent recursions
// hide each other's latency).  (256-thread / 8 KiB-line and 2-in-flight
// configurations measured slower in round 1 and were removed.)
#ifndef PP_SMALL_PF  // A/B builds only (tools/ab_build.py; 3 and 2 measured slower)
#define PP_SMALL_PF 4
#endif
#ifndef PP_SMALL_MINB
#define PP_SMALL_MINB 4
#endif
#ifndef PP_SMALL_LINE  // A/B builds only (8 KiB / 2 in flight: -0.7%, not adopted)
#define PP_SMALL_LINE 4096
#endif
template <typename K>
struct SmallCfg {
    static constexpr int NT = 128, MINB = PP_SMALL_MINB;
    using GC = GroupCfgT<K, PP_SMALL_LINE, 128, PP_SMALL_PF, false, false, true>;
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
template <typename K>
__device__ uint64_t cta_partition(K* __restrict__ seg, uint64_t len, K pivot, uint64_t seed, unsigned char* smem,
                                  GroupOut* scratch, Ctl* sc, uint64_t* red, uint64_t* pr = nullptr) {
    using S = SmallCfg<K>;
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
    uint64_t tw = pr ? clock64() : 0;
    walk_swap_stream<K, NT, SW_EPT2>(seg, d, pivot, 0, Kv, Kv, W,
                                     *reinterpret_cast<StreamBuf<NT, SW_EPT2>*>(smem));
    __syncthreads();
    if (pr) pr[3] += clock64() - tw;
    return Ks;
}

// Bin slots a small segment of len keys may fill: greedy packing of its
// leaves (in array order) into bins of <= leaf keys leaves consecutive bins
// summing to > leaf, so <= 2*ceil(len/leaf) + 1 bins, plus one per range that
// is skipped (all keys equal) -- the rest of the slack; a CTA that runs out
// sorts the overflowing bin itself (qs_small_kernel).
__host__ __device__ __forceinline__ uint64_t qs_bin_cap(uint64_t len, uint64_t leaf) {
    return 2 * ((len + leaf - 1) / leaf) + 4;
}

// Stack entry modes of qs_small_kernel.
constexpr int QM_PIVOT = 0;   // pivot = median-of-3, split by x < p
constexpr int QM_LE = 1;      // split by x < p with p = (segment minimum) + 1, i.e. x <= min
constexpr int QM_INCTA = 2;   // flag: this range is sorted inside the CTA (bin slots exhausted)

// One CTA per small segment (leaf < len <= qs_small): the rest of its
// recursion, depth first with an explicit stack, left part first so that the
// leaves (pieces <= leaf keys) appear in array order.  Leaves are not sorted
// here: adjacent leaves are packed greedily into bins of <= leaf keys, and
// each bin (a contiguous range that is a union of whole leaves, so sorting it
// whole sorts each leaf) is written to this segment's slots [slot_base[i],
// +qs_bin_cap); unused slots get length 0.  One wide shared-memory sort
// launch then sorts every bin (qs_leaf_bidx_kernel).  Ranges whose keys are
// all equal (the x <= min split, reading R14) are final and skipped.  If the
// slots run out, the overflowing bin is pushed back with QM_INCTA and sorted
// by this CTA itself (partition down to LEAFC, merge sort in shared memory).
template <typename K>
__global__ void __launch_bounds__(SmallCfg<K>::NT, SmallCfg<K>::MINB)
    qs_small_kernel(K* __restrict__ keys, const uint64_t* __restrict__ seg_lo, const uint32_t* __restrict__ seg_len,
                    const uint64_t* __restrict__ slot_base, uint64_t* __restrict__ bin_lo,
                    uint32_t* __restrict__ bin_len, uint32_t leaf, uint64_t seed, GroupOut* __restrict__ scratch,
                    uint64_t* __restrict__ prof, int ninther, const uint64_t* __restrict__ seg_kb,
                    uint64_t* __restrict__ bin_kb) {
    using S = SmallCfg<K>;
    constexpr int DEPTH = 64, LEFT_FIRST_MAX = 40;
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ Ctl sc;
    __shared__ uint64_t red[S::NT / 32];
    __shared__ uint64_t st_lo[DEPTH], st_hi[DEPTH], st_p[DEPTH];
    __shared__ uint64_t st_kmin[DEPTH], st_kmax[DEPTH];  // key bounds of the range (from the pivots above it)
    __shared__ int st_mode[DEPTH];
    __shared__ int sp;
    const K KMAX = (K)~(K)0;
    K* A = reinterpret_cast<K*>(smem);
    K* B = A + lpad(S::LEAFC);
    // bin state (thread 0 only): open bin [blo, bhi) with key bounds [bkmin, bkmax], slots used
    uint64_t blo = 0, bhi = 0, bkmin = 0, bkmax = 0;
    uint32_t used = 0;
    const uint64_t base = slot_base[blockIdx.x];
    const uint32_t cap = (uint32_t)qs_bin_cap(seg_len[blockIdx.x], leaf);
    auto push = [&](uint64_t lo, uint64_t hi, int mode, uint64_t p, uint64_t kmn, uint64_t kmx) {  // thread 0
        const int s = sp;
        st_lo[s] = lo; st_hi[s] = hi; st_mode[s] = mode; st_p[s] = p;
        st_kmin[s] = kmn; st_kmax[s] = kmx;
        sp = s + 1;
    };
    auto emit = [&]() {  // thread 0: close the open bin
        if (bhi > blo) {
            if (used < cap) {
                bin_lo[base + used] = blo;
                bin_len[base + used] = (uint32_t)(bhi - blo);
                if (bin_kb) {
                    bin_kb[2 * (base + used)] = bkmin;
                    bin_kb[2 * (base + used) + 1] = bkmax;
                }
                ++used;
            } else {
                push(blo, bhi, QM_PIVOT | QM_INCTA, 0, bkmin, bkmax);
            }
        }
        blo = bhi = 0;
    };
    if (threadIdx.x == 0) {
        sp = 0;
        push(seg_lo[blockIdx.x], seg_lo[blockIdx.x] + seg_len[blockIdx.x], QM_PIVOT, 0,
             seg_kb ? seg_kb[2 * (uint64_t)blockIdx.x] : 0, seg_kb ? seg_kb[2 * (uint64_t)blockIdx.x + 1] : (uint64_t)KMAX);
    }
    __syncthreads();
    // optional phase profile (debug, PP_QS_PROF): cycles in pivot / partition / merge sort, counts
    uint64_t pr[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    uint64_t t0 = prof ? clock64() : 0;
    for (;;) {
        if (sp == 0) {  // uniform: sp is only written by thread 0 before a barrier
            __syncthreads();
            if (threadIdx.x == 0) emit();
            __syncthreads();
            if (sp == 0) break;
        }
        const int top = sp - 1;
        const uint64_t lo = st_lo[top], hi = st_hi[top], pm = st_p[top];
        const uint64_t kmn = st_kmin[top], kmx = st_kmax[top];
        const int mode = st_mode[top];
        __syncthreads();
        if (threadIdx.x == 0) sp = top;
        const uint64_t len = hi - lo;
        const int incta = mode & QM_INCTA;
        if (!incta && len <= leaf) {  // a leaf: into the open bin (thread 0), or a new bin
            if (threadIdx.x == 0 && len > 0) {
                if (bhi == lo && hi - blo <= leaf) {
                    bhi = hi;
                    bkmax = kmx > bkmax ? kmx : bkmax;
                } else if (blo == hi && bhi - lo <= leaf) {
                    blo = lo;
                    bkmin = kmn < bkmin ? kmn : bkmin;
                } else {
                    emit();
                    blo = lo; bhi = hi; bkmin = kmn; bkmax = kmx;
                }
            }
            __syncthreads();
            continue;
        }
        if (len <= 1 || (kmn == kmx && !incta)) {
            // (kmn == kmx: the pivots above it pin every key to one value --
            // all equal and final, like the x <= p step's left part)
            __syncthreads();
            continue;
        }
        if (incta && len <= S::LEAFC) {
            cta_merge_sort<K, S::NT>(keys + lo, (uint32_t)len, A, B);
            if (prof) { const uint64_t t1 = clock64(); pr[2] += t1 - t0; pr[5] += 1; pr[7] += len; t0 = t1; }
            continue;
        }
        K p;
        if ((mode & QM_LE) == 0 && ninther == 2) {  // median of 31 samples (param qs_pivot = 2): warp 0
            __shared__ K p31;
            if (threadIdx.x < 32) {
                const K v = warp_median31<K>(keys, lo, len, (int)threadIdx.x);
                if (threadIdx.x == 0) p31 = v;
            }
            __syncthreads();
            p = p31;
            __syncthreads();  // p31 is rewritten by the next partition
        } else if ((mode & QM_LE) == 0) {
            if (ninther) {  // Tukey's ninther (param qs_deep = 0, qs_pivot = 1)
                const K m0 = median3<K>(keys[ninther_pos<K>(lo, len, 0)], keys[ninther_pos<K>(lo, len, 1)],
                                        keys[ninther_pos<K>(lo, len, 2)]);
                const K m1 = median3<K>(keys[ninther_pos<K>(lo, len, 3)], keys[ninther_pos<K>(lo, len, 4)],
                                        keys[ninther_pos<K>(lo, len, 5)]);
                const K m2 = median3<K>(keys[ninther_pos<K>(lo, len, 6)], keys[ninther_pos<K>(lo, len, 7)],
                                        keys[ninther_pos<K>(lo, len, 8)]);
                p = median3<K>(m0, m1, m2);
            } else {
                p = median3<K>(keys[lo], keys[lo + (len - 1) / 2], keys[hi - 1]);
            }
        }
        else p = (K)pm;
        if ((mode & QM_LE) == 0 && kmn < kmx) p = (K)pivot_above_bound<K>(p, kmn);  // (p == kmn: the x <= p step now)
        if (prof) { const uint64_t t1 = clock64(); pr[0] += t1 - t0; t0 = t1; }
        const uint64_t k = cta_partition<K>(keys + lo, len, p, seed, smem, scratch + blockIdx.x, &sc, red,
                                               prof ? pr : nullptr);
        if (prof) { const uint64_t t1 = clock64(); pr[1] += t1 - t0; pr[4] += 1; pr[6] += len; t0 = t1; }
        if (threadIdx.x == 0) {
            // key bounds of the parts: left keys < p, right keys >= p
            const uint64_t pu = (uint64_t)p;
            if ((mode & QM_LE) == 0 && k == 0) {
                // p is the minimum: split by x <= p next (reading R14); p == kmx (e.g. all == MAX): final
                if (pu != kmx) push(lo, hi, QM_LE | incta, (uint64_t)(K)(p + 1), pu, kmx);  // (== kmx: all equal)
            } else if (mode & QM_LE) {
                push(lo + k, hi, QM_PIVOT | incta, 0, pu, kmx);  // [lo, lo+k) is all == p - 1: final, skipped
            } else if (incta || sp >= LEFT_FIRST_MAX) {
                // smaller part first (stack depth <= log2 len from here)
                const bool left_small = k < len - k;
                if (left_small) {
                    push(lo + k, hi, QM_PIVOT | incta, 0, pu, kmx);
                    push(lo, lo + k, QM_PIVOT | incta, 0, kmn, pu - 1);
                } else {
                    push(lo, lo + k, QM_PIVOT | incta, 0, kmn, pu - 1);
                    push(lo + k, hi, QM_PIVOT | incta, 0, pu, kmx);
                }
            } else {
                // left part first: leaves come out in array order
                push(lo + k, hi, QM_PIVOT, 0, pu, kmx);
                push(lo, lo + k, QM_PIVOT, 0, kmn, pu - 1);
            }
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        for (uint32_t u = used; u < cap; ++u) bin_len[base + u] = 0;
    }
    if (prof && threadIdx.x == 0) {
#pragma unroll
        for (int i = 0; i < 8; ++i) prof[8 * (uint64_t)blockIdx.x + i] = pr[i];
    }
}



template <typename K>
struct LeafCfg {
    static constexpr int LEAF = 8192;
    static constexpr int NT = LEAF / LEAF_E;
};

// Launch with programmatic stream serialization: the launch overlaps the
// previous kernel's tail; the kernel calls griddep_wait() before reading
// what its predecessor wrote (the shared cleanup bodies do so themselves).
template <typename... KArgs, typename... Args>
static cudaError_t qs_launch_pdl(void (*kern)(KArgs...), dim3 grid, unsigned block, size_t smem, cudaStream_t st,
                                 Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

// quicksort workspace (separate from the partition workspace)
static void* g_qws = nullptr;
static size_t g_qws_bytes = 0;
// With a caller workspace (pp_set_workspace) the quicksort's region starts
// after the partition region of the top-level call: [partition | quicksort].
static size_t g_qs_user_base = 0;
static size_t g_qs_peak = 0;
// work statistics of the last quicksort (pp_quicksort_last_stats)
struct QsStats {
    uint64_t n = 0, levels = 0, level_keys = 0, small_keys = 0, leaf_keys = 0, nsmall = 0;
};
static QsStats g_qs_stats;
pp_status quicksort_last_stats(uint64_t* out6) {
    if (!out6) return PP_E_INVAL;
    const QsStats& q = g_qs_stats;
    const uint64_t v[6] = {q.n, q.levels, q.level_keys, q.small_keys, q.leaf_keys, q.nsmall};
    for (int i = 0; i < 6; ++i) out6[i] = v[i];
    return PP_OK;
}
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

// Pinned host staging for the level loop's small transfers (segment list
// up, splits and device-computed pivots down): pageable copies are staged
// synchronously by the driver and lengthen every level's host round trip.
static unsigned char* g_qs_pin = nullptr;
static size_t g_qs_pin_bytes = 0;
static unsigned char* qs_pinned(size_t bytes) {
    if (bytes <= g_qs_pin_bytes) return g_qs_pin;
    if (g_qs_pin) cudaFreeHost(g_qs_pin);
    g_qs_pin = nullptr;
    g_qs_pin_bytes = 0;
    const size_t want = std::max<size_t>(bytes + (bytes >> 1), 1 << 16);
    if (cudaMallocHost(&g_qs_pin, want) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    g_qs_pin_bytes = want;
    return g_qs_pin;
}

// Size thresholds of the quicksort driver (current params).
struct QsGeom {
    uint64_t LEAF;      // segments <= LEAF: one smem sort
    uint64_t SMALL;     // segments in (LEAF, SMALL]: per-CTA recursion
    uint64_t BIG;       // segments >= BIG: full multi-CTA partition
    uint64_t G_TARGET;  // CTAs of one batched mid-level group launch
    uint64_t HEAVY;     // mid segments >= HEAVY: batched multi-CTA cleanup (0 = off)
};
template <typename K>
static QsGeom qs_geom() {
    using C = GroupCfg<K>;
    using LC = LeafCfg<K>;
    const Params& P = params();
    QsGeom q;
    // leaf capacity: LC::LEAF (8192 keys) for the bin sorts 1-5; the default
    // bin sort (6) takes bins of up to 2 LC::LEAF and defaults to that;
    // "leaf" may lower it
    const uint64_t lmax = 2 * (uint64_t)LC::LEAF;
    q.LEAF = (P.leaf > 0 && (uint64_t)P.leaf <= lmax) ? (uint64_t)P.leaf : lmax;
    q.BIG = P.qs_cta_max > 0 ? (uint64_t)P.qs_cta_max : (uint64_t)1 << 27;
    q.SMALL = P.qs_small > 0 ? std::max<uint64_t>((uint64_t)P.qs_small, q.LEAF) : q.LEAF;
    q.HEAVY = P.qs_heavy > 0 ? std::max<uint64_t>((uint64_t)P.qs_heavy, q.SMALL + 1) : 0;
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
static size_t qs_level_bound(uint64_t n) {  // one level's region (any level, any lane)
    const QsGeom q = qs_geom<K>();
    const uint64_t nmid = n / (q.SMALL + 1) + 1, nbig = n / q.BIG + 1;
    const uint64_t gtot = q.G_TARGET + 2 * nmid + 1;
    const uint64_t nh = q.HEAVY ? n / q.HEAVY + 1 : 0;
    return al256(al256(sizeof(QSeg) * nmid) + al256(sizeof(GroupOut) * gtot) + al256(8 * (nmid + nbig + 1)) +
                 al256(4 * (nh + 1)) + hv_layout().stride * nh);
}
// Device-built levels (qs_dev): per lane, two level lists and their key
// bounds (ping-pong), the builder's scratch list, two count blocks, the group
// outputs and the splits; pinned: one readback per list parity.
struct QDevLayout {
    size_t listB, kbB, goutB, splB, laneB, pinParB, pinB;
};
template <typename K>
static QDevLayout qdev_layout(uint64_t nm, uint64_t g_target) {
    QDevLayout D;
    D.listB = al256(sizeof(QSeg) * nm);
    D.kbB = al256(16 * nm);
    D.goutB = al256(sizeof(GroupOut) * (g_target + nm + 2));
    D.splB = al256(8 * nm);
    D.laneB = 3 * D.listB + 3 * D.kbB + 256 + D.goutB + D.splB;
    D.pinParB = D.listB + D.kbB + D.splB + 256;
    D.pinB = 2 * D.pinParB + 256;
    return D;
}
template <typename K>
static bool qdev_on(uint64_t n) {  // param qs_dev (default off) and a list that fits the builder
    const QsGeom q = qs_geom<K>();
    return params().qs_dev != 0 && n / (q.SMALL + 1) + 1 <= QB_NMAX / 2 && q.SMALL >= q.LEAF;
}
template <typename K>
uint64_t quicksort_workspace_bound(uint64_t n) {
    const QsGeom q = qs_geom<K>();
    const size_t level = qs_level_bound<K>(n);
    const uint64_t cl = std::min<uint64_t>(n / 2 + 1, QS_LIST_CHUNK);
    const uint64_t cs = std::min<uint64_t>(n / (q.LEAF + 1) + 1, QS_LIST_CHUNK);
    // bin slots of one chunk of small segments: sum of qs_bin_cap <= 2 n / LEAF + 6 per segment
    // bin slots of all small segments: sum of qs_bin_cap <= 2 n / LEAF + 6 per segment
    const uint64_t nslot = 2 * (n / q.LEAF) + 6 * (n / (q.LEAF + 1) + 1) + 6;
    const size_t lists = al256(8 * cl) + al256(4 * cl) + al256(8 * cs) + al256(4 * cs) + al256(8 * cs) +
                         al256(sizeof(GroupOut) * cs) + al256(8 * nslot) + al256(4 * nslot) + 256;
    // early per-CTA recursion lists (every small segment, all bin slots), beside the lanes
    const uint64_t s_max = n / (q.LEAF + 1) + 1, slot_max = 2 * (n / q.LEAF) + 6 * s_max + 6;
    const size_t early = al256(8 * s_max) + al256(4 * s_max) + al256(8 * s_max) + al256(sizeof(GroupOut) * s_max) +
                         al256(8 * slot_max) + al256(4 * slot_max) + al256(16 * s_max) + al256(16 * slot_max);
    const size_t dev = qdev_on<K>(n) ? 2 * qdev_layout<K>(n / (q.SMALL + 1) + 1, q.G_TARGET).laneB : 0;
    // two level lanes + early lists + device-built lanes (quicksort_device), or the final lists
    return std::max(2 * level + early + dev, lists);
}
template uint64_t quicksort_workspace_bound<uint64_t>(uint64_t);
template uint64_t quicksort_workspace_bound<uint32_t>(uint64_t);

template <typename K>
static pp_status quicksort_device_impl(K* keys, uint64_t n, cudaStream_t st) {
    using C = GroupCfg<K>;
    using LC = LeafCfg<K>;
    const Params& P = params();
    const QsGeom geom = qs_geom<K>();
    const uint64_t LEAF = geom.LEAF, BIG = geom.BIG, G_TARGET = geom.G_TARGET, HEAVY = geom.HEAVY;
    const HvLayout HVL = hv_layout();
    // at least this many lines per group (mid segments); auto: 64 lines (512 KiB
    // of keys per group u64, 256 KiB u32 -- re-swept at the end of round 2: fewer,
    // longer groups for the small late segments; was 128 KiB)
    const uint64_t MINL = P.qs_minl > 0 ? (uint64_t)P.qs_minl : 64;
    const K KMAX = (K)~(K)0;
    g_qs_user_base = al256(partition_workspace_bound(n));
    g_qs_peak = 0;
    g_qs_stats = QsStats();
    g_qs_stats.n = n;

    struct HSeg {
        uint64_t lo, hi, pivot;
        uint32_t mode, depth;
        uint64_t kmin, kmax;  // every key of the segment is in [kmin, kmax] (the pivots above it)
    };
    // Deep segments (an adversarial order can make median-of-3 peel off a few
    // keys per level) take the ninther instead (R14 fixes only the default
    // rule; the sorted output is unique, so parity is unaffected).  Uniform
    // and structured inputs never get this deep.
    uint32_t lg = 0;
    while ((1ull << lg) < n) ++lg;
    const uint32_t QS_DEEP = P.qs_deep >= 0 ? (uint32_t)P.qs_deep : 2 * lg + 16;
    // pivot rule of the level loop: param qs_pivot 0 median of 3 (BJ config 5), 1 ninther, 2 median of 31
    const uint32_t RULE = P.qs_pivot == 2 ? 3u : P.qs_pivot == 1 ? 2u : 0u;
    auto rule_at = [&](uint32_t depth) -> uint32_t { return depth > QS_DEEP && RULE == 0 ? 2u : RULE; };
    std::vector<uint64_t> leaf_lo, small_lo;
    std::vector<uint32_t> leaf_len, small_len;
    std::vector<uint64_t> small_base_v{0};  // bin-slot offset of each small segment (prefix of qs_bin_cap)
    std::vector<uint64_t> small_kb;         // key bounds (kmin, kmax) of each small segment
    // segments in (LEAF, SMALL] finish in one CTA each (qs_small_kernel)
    const uint64_t SMALL = geom.SMALL;
    auto add_child = [&](std::vector<HSeg>& next, uint64_t lo, uint64_t hi, uint32_t depth, uint64_t kmin,
                         uint64_t kmax) {
        const uint64_t len = hi - lo;
        if (len <= 1) return;
        // the pivots above it pin every key to [kmin, kmax]: a single value
        // means the segment is all equal keys -- final, no pass
        if (kmin == kmax) return;
        if (len <= LEAF) {
            leaf_lo.push_back(lo);
            leaf_len.push_back((uint32_t)len);
            g_qs_stats.leaf_keys += len;
        } else if (len <= SMALL) {
            g_qs_stats.small_keys += len;
            ++g_qs_stats.nsmall;
            small_lo.push_back(lo);
            small_len.push_back((uint32_t)len);
            small_base_v.push_back(small_base_v.back() + qs_bin_cap(len, LEAF));
            small_kb.push_back(kmin);
            small_kb.push_back(kmax);
        } else {
            next.push_back({lo, hi, 0, rule_at(depth), depth, kmin, kmax});
        }
    };
    // The level loop runs in up to two LANES: while some segment takes the
    // big-segment path (or fewer than two segments exist) one lane runs on
    // the caller's stream; then the segment list is split in two array-disjoint
    // halves, each recursing independently on its own stream with its own
    // workspace and pinned regions.  While the host waits on one lane's
    // level and builds its next list, the other lane's kernels keep the GPU
    // busy, and each lane's kernel tails overlap the other's work.
    struct Lane {
        std::vector<HSeg> cur, next;
        std::vector<QSeg> mids, m2;
        std::vector<uint64_t> splits_h, pivots_h, seg_nl;
        std::vector<size_t> big_idx, mid_idx, ordi, i2;
        std::vector<uint32_t> bk, cnt, hidx;
        cudaStream_t st = nullptr;
        cudaEvent_t done = nullptr;
        cudaEvent_t lev[3] = {nullptr, nullptr, nullptr};
        unsigned char* pin = nullptr;
        uint64_t nmid = 0, nbig = 0, gtot = 0, depth = 0;
        bool inflight = false;
        int id = 0;
        // device-built levels (qs_dev): up to two levels in flight, oldest first
        bool dev = false;
        int dq = 0;
        int qpar[2] = {0, 1};           // list parity of each level in flight
        uint64_t qexact = 0;            // segments of the oldest level in flight (the host knows it exactly)
        unsigned char* dreg = nullptr;  // device region (QDevLayout)
        unsigned char* dpin = nullptr;  // pinned readbacks
        std::vector<QSeg> dev_expect;   // qs_dev_check: the host's plan of the next device-built list
        std::vector<uint64_t> dev_expect_kb;
        bool dev_expect_valid = false;
    };
    static cudaStream_t lane_st1 = nullptr, lane_hi1 = nullptr;
    static cudaEvent_t lane_ev[3] = {nullptr, nullptr, nullptr};
    if (!lane_st1) {
        int least = 0, greatest = 0;
        cudaDeviceGetStreamPriorityRange(&least, &greatest);
        cudaStreamCreateWithFlags(&lane_st1, cudaStreamNonBlocking);
        cudaStreamCreateWithPriority(&lane_hi1, cudaStreamNonBlocking, greatest);
        for (auto& x : lane_ev) cudaEventCreateWithFlags(&x, cudaEventDisableTiming);
    }
    Lane lanes[2];
    lanes[0].st = st;
    lanes[0].done = lane_ev[0];
    lanes[1].st = P.qs_prio != 0 ? lane_hi1 : lane_st1;
    cudaStream_t lane_st1_used = lanes[1].st;
    lanes[1].done = lane_ev[1];
    lanes[1].id = 1;
    lanes[0].cur.push_back({0, n, 0, rule_at(0), 0, 0, (uint64_t)KMAX});
    if (n <= SMALL) {
        lanes[0].cur.clear();
        add_child(lanes[0].cur, 0, n, 0, 0, (uint64_t)KMAX);
    }
    cudaError_t e;
    cudaFuncSetAttribute(qs_group_kernel<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
    static const bool lvl_prof = getenv("PP_QS_PROF") != nullptr;
    if (lvl_prof)
        for (Lane& L : lanes)
            for (auto& x : L.lev) cudaEventCreate(&x);
    // sorts `cnt` bins (lo, len) of <= LEAF keys each, len 0 = empty slot:
    // the index-staged counting sort, then the merge sort of the bins it handed
    // off (crowded buckets)
    // PP_QS_SKIP (measurement only, the output is then NOT sorted): bit 0
    // skips the bin sorts, bit 1 the per-CTA recursion and the bin sorts -- the
    // time the rest takes
    static const int qs_skip = getenv("PP_QS_SKIP") ? atoi(getenv("PP_QS_SKIP")) : 0;
    // d_kb (optional): key bounds (kmin, kmax) per slot -- the bin sort skips its min / max pass
    auto sort_bins = [&](const uint64_t* d_lo, const uint32_t* d_len, uint64_t cnt, cudaStream_t bst,
                         const uint64_t* d_kb = nullptr) -> cudaError_t {
        if (cnt == 0 || (qs_skip & 3)) return cudaSuccess;
        static const bool bin_stats = getenv("PP_QS_BINSTATS") != nullptr;  // measurement only: bin sizes
        if (bin_stats) {
            std::vector<uint32_t> h(cnt);
            cudaStreamSynchronize(bst);
            cudaMemcpy(h.data(), d_len, 4 * cnt, cudaMemcpyDeviceToHost);
            uint64_t hist[6] = {0, 0, 0, 0, 0, 0}, keys_in = 0, nonempty = 0;
            for (uint32_t x : h) {
                const uint32_t l = x & ~0x80000000u;
                if (l >= 2) ++nonempty;
                keys_in += l;
                hist[l < 2 ? 0 : l <= 2048 ? 1 : l <= 4096 ? 2 : l <= 8192 ? 3 : l <= 12288 ? 4 : 5]++;
            }
            fprintf(stderr, "qs bins: slots=%llu nonempty=%llu keys=%llu  <2:%llu <=2K:%llu <=4K:%llu <=8K:%llu <=12K:%llu >12K:%llu\n",
                    (unsigned long long)cnt, (unsigned long long)nonempty, (unsigned long long)keys_in,
                    (unsigned long long)hist[0], (unsigned long long)hist[1], (unsigned long long)hist[2],
                    (unsigned long long)hist[3], (unsigned long long)hist[4], (unsigned long long)hist[5]);
        }
        constexpr int HL = LC::LEAF, HN = HL / LEAF_E;
        if (LEAF > (uint64_t)HL) {  // bins of <= 2 LC::LEAF keys: 1024 threads, one CTA per SM
#ifndef PP_BIN16_NT  // A/B builds only (512 threads x 32 keys measured 6% slower: the bin sort needs the warps)
#define PP_BIN16_NT 1024
#endif
            constexpr int PL = 2 * HL, BNT = PP_BIN16_NT;
            const size_t smem = 32 + sizeof(K) * PL + 2 * PP_BIN_BX * PL + 16 + PL;
            cudaFuncSetAttribute(qs_leaf_bidx_kernel<K, PL, BNT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem);
            qs_leaf_bidx_kernel<K, PL, BNT><<<(unsigned)cnt, BNT, smem, bst>>>(keys, d_lo, const_cast<uint32_t*>(d_len),
                                                                               d_kb);
        } else {  // bins of <= LC::LEAF keys: 512 threads, two CTAs per SM
            constexpr int PL = HL, BNT = 512;
            const size_t smem = 32 + sizeof(K) * PL + 2 * PP_BIN_BX * PL + 16 + PL;
            cudaFuncSetAttribute(qs_leaf_bidx_kernel<K, PL, BNT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem);
            qs_leaf_bidx_kernel<K, PL, BNT><<<(unsigned)cnt, BNT, smem, bst>>>(keys, d_lo, const_cast<uint32_t*>(d_len),
                                                                               d_kb);
        }
        const size_t msmem = sizeof(K) * lpad_host(2 * HL);
        cudaFuncSetAttribute(qs_leaf_handoff_kernel<K, HL, HN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)msmem);
        const unsigned hg = (unsigned)std::min<uint64_t>((cnt + HN - 1) / HN, 2 * (uint64_t)sm_count());
        qs_leaf_handoff_kernel<K, HL, HN><<<hg, HN, msmem, bst>>>(keys, d_lo, d_len, cnt);
        note_launches(2);
        return cudaGetLastError();
    };
    // the per-CTA recursion over `cnt` small segments (lists on the device)
    auto launch_small = [&](uint64_t cnt, const uint64_t* slo, const uint32_t* sln, const uint64_t* sbase,
                            uint64_t* blo, uint32_t* bln, GroupOut* scr, uint64_t* prof, cudaStream_t s3,
                            const uint64_t* skb = nullptr, uint64_t* bkb = nullptr) {
        using S = SmallCfg<K>;
        if (qs_skip & 2) return cudaSuccess;  // (measurement only; the bin sorts are skipped too)
        cudaFuncSetAttribute(qs_small_kernel<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S::SMEM);
        qs_small_kernel<K><<<(unsigned)cnt, S::NT, S::SMEM, s3>>>(keys, slo, sln, sbase, blo, bln, (uint32_t)LEAF,
                                                                  P.seed, scr, prof,
                                                                  P.qs_pivot == 2 ? 2 : (P.qs_deep == 0 || P.qs_pivot == 1) ? 1 : 0,
                                                                  skb, bkb);
        note_launches(1);
        return cudaGetLastError();
    };
    // pinned staging per lane, sized once from the level bound (a lane's
    // readback may be in flight while the other lane builds its level)
    const uint64_t nmid_max = n / (SMALL + 1) + 1, nbig_max = n / BIG + 1;
    const uint64_t nh_max = HEAVY ? n / HEAVY + 1 : 1;
    const size_t pin_sB = al256(sizeof(QSeg) * nmid_max), pin_spB = al256(8 * (nmid_max + nbig_max + 1));
    const size_t pin_lane = pin_sB + pin_spB + al256(4 * nh_max);
    // device-built levels (param qs_dev): regions per lane
    const bool dev_on = qdev_on<K>(n);
    const uint64_t NM = nmid_max;
    const QDevLayout DL = qdev_layout<K>(NM, G_TARGET);
    unsigned char* pin_all = qs_pinned(2 * pin_lane + (dev_on ? 2 * DL.pinB : 0));
    if (!pin_all) return PP_E_NOMEM;
    lanes[0].pin = pin_all;
    lanes[1].pin = pin_all + pin_lane;
    if (dev_on)
        for (int i = 0; i < 2; ++i) lanes[i].dpin = pin_all + 2 * pin_lane + (size_t)i * DL.pinB;
    // bytes of each lane's device region: the level bound up front (a few MB
    // at 2^28 keys), so a growing level never has to drain the other lane
    const size_t lane_half = qs_level_bound<K>(n);
    // early per-CTA recursion (param qs_early): the lists of every small
    // segment and all bin slots, indexed globally, after the two lane regions;
    // a batch runs on a third stream as soon as its segments are final
    const bool early = P.qs_early != 0;  // -1 auto = on
    // batch size of the early recursion: x #SM segments (auto: 4 for u64, 2 for u32 -- measured)
    const uint64_t early_min =
        (uint64_t)(P.qs_early_min > 0 ? P.qs_early_min : (sizeof(K) == 8 ? 8 : 2)) * (uint64_t)sm_count();
    const uint64_t s_max = n / (LEAF + 1) + 1, slot_max = 2 * (n / LEAF) + 6 * s_max + 6;
    const size_t e_sloB = al256(8 * s_max), e_slnB = al256(4 * s_max), e_sbB = al256(8 * s_max);
    const size_t e_scrB = al256(sizeof(GroupOut) * s_max), e_bloB = al256(8 * slot_max), e_blnB = al256(4 * slot_max);
    const size_t e_skbB = al256(16 * s_max), e_bkbB = al256(16 * slot_max);  // key bounds: segments, bins
    const size_t earlyB = early ? e_sloB + e_slnB + e_sbB + e_scrB + e_bloB + e_blnB + e_skbB + e_bkbB : 0;
    const size_t devB = dev_on ? 2 * DL.laneB : 0;
    unsigned char* ws_all = static_cast<unsigned char*>(qs_workspace(2 * lane_half + earlyB + devB));
    if (!ws_all) return PP_E_NOMEM;
    unsigned char* ew = ws_all + 2 * lane_half;
    if (dev_on)
        for (int i = 0; i < 2; ++i) lanes[i].dreg = ws_all + 2 * lane_half + earlyB + (size_t)i * DL.laneB;
    uint64_t* d_eslo = reinterpret_cast<uint64_t*>(ew);
    uint32_t* d_esln = reinterpret_cast<uint32_t*>(ew + e_sloB);
    uint64_t* d_esbase = reinterpret_cast<uint64_t*>(ew + e_sloB + e_slnB);
    GroupOut* d_escr = reinterpret_cast<GroupOut*>(ew + e_sloB + e_slnB + e_sbB);
    uint64_t* d_eblo = reinterpret_cast<uint64_t*>(ew + e_sloB + e_slnB + e_sbB + e_scrB);
    uint32_t* d_ebln = reinterpret_cast<uint32_t*>(ew + e_sloB + e_slnB + e_sbB + e_scrB + e_bloB);
    uint64_t* d_eskb = reinterpret_cast<uint64_t*>(ew + e_sloB + e_slnB + e_sbB + e_scrB + e_bloB + e_blnB);
    uint64_t* d_ebkb = reinterpret_cast<uint64_t*>(ew + e_sloB + e_slnB + e_sbB + e_scrB + e_bloB + e_blnB + e_skbB);
    static cudaStream_t early_st = nullptr, early_bst = nullptr;  // recursion; bin sorts
    static cudaEvent_t early_ev[64];
    if (!early_st) {
        cudaStreamCreateWithFlags(&early_st, cudaStreamNonBlocking);
        cudaStreamCreateWithFlags(&early_bst, cudaStreamNonBlocking);
        for (auto& x : early_ev) cudaEventCreateWithFlags(&x, cudaEventDisableTiming);
    }
    uint64_t early_nb = 0;  // batches so far (events recycled: a batch's bins wait on its recursion)
    uint64_t small_done = 0;
    // small segments [b, en) (their levels have completed: the host synchronised on them)
    auto small_batch = [&](uint64_t b, uint64_t en) -> pp_status {
        if (en <= b) return PP_OK;
        const uint64_t cnt = en - b;
        e = cudaMemcpyAsync(d_eslo + b, small_lo.data() + b, 8 * cnt, cudaMemcpyHostToDevice, early_st);
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(d_esln + b, small_len.data() + b, 4 * cnt, cudaMemcpyHostToDevice, early_st);
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(d_esbase + b, small_base_v.data() + b, 8 * cnt, cudaMemcpyHostToDevice, early_st);
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(d_eskb + 2 * b, small_kb.data() + 2 * b, 16 * cnt, cudaMemcpyHostToDevice, early_st);
        if (e == cudaSuccess)
            e = launch_small(cnt, d_eslo + b, d_esln + b, d_esbase + b, d_eblo, d_ebln, d_escr + b, nullptr, early_st,
                             d_eskb + 2 * b, d_ebkb);
        cudaEvent_t ev = early_ev[early_nb++ % 64];
        if (e == cudaSuccess) e = cudaEventRecord(ev, early_st);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(early_bst, ev, 0);
        if (e == cudaSuccess)
            e = sort_bins(d_eblo + small_base_v[b], d_ebln + small_base_v[b], small_base_v[en] - small_base_v[b],
                          early_bst, d_ebkb + 2 * small_base_v[b]);
        return e == cudaSuccess ? PP_OK : cuda_fail(e, "quicksort early small batch");
    };

    // classify a lane's segments, upload its level, launch its kernels and
    // the readback; records L.done (L.inflight = false if nothing to do)
    // the level's mid segments with their group counts, in launch order (LPT);
    // big ones into L.big_idx; returns the level's total groups
    auto plan_mids = [&](Lane& L) -> uint64_t {
        L.mids.clear();
        L.big_idx.clear();
        L.mid_idx.clear();
        L.seg_nl.clear();
        uint64_t gtot = 0, mid_lines = 0;
        // mid segments share one launch.  Every CTA should carry about the
        // same number of lines: L* = (lines of all mid segments) / G_TARGET,
        // a segment gets round(lines / L*) groups (>= 1, <= lines / MINL);
        // the tasks are then ordered by lines per group, longest first, so the
        // in-order CTA dispatch approximates longest-processing-time-first
        // scheduling over the SMs' slots (balanced waves, no straggler wave).
        for (size_t i = 0; i < L.cur.size(); ++i) {
            const uint64_t len = L.cur[i].hi - L.cur[i].lo;
            if (len >= BIG) {
                L.big_idx.push_back(i);
                continue;
            }
            L.mid_idx.push_back(i);
            QSeg q;
            q.lo = L.cur[i].lo;
            q.hi = L.cur[i].hi;
            q.pivot = L.cur[i].pivot;
            q.mode = L.cur[i].mode;
            q.pad = 0;
            q.kmin = L.cur[i].kmin;
            // lines of the aligned region (host mirror of seg_head)
            const uint64_t addr = (uint64_t)(uintptr_t)(keys + q.lo);
            uint64_t h = ((16 - (addr & 15)) & 15) / sizeof(K);
            if (h > len) h = len;
            const uint64_t nl = (len - h) / C::LK;
            L.seg_nl.push_back(nl);
            mid_lines += nl;
            L.mids.push_back(q);
        }
        std::vector<QSeg>& mids = L.mids;
        {
            const double Lstar = std::max(1.0, (double)mid_lines / (double)G_TARGET);
            for (size_t i = 0; i < mids.size(); ++i) {
                const uint64_t cap = std::max<uint64_t>(1, L.seg_nl[i] / MINL);
                const uint64_t want = (uint64_t)((double)L.seg_nl[i] / Lstar + 0.5);
                mids[i].g = std::max<uint64_t>(1, std::min<uint64_t>(cap, want));
                gtot += mids[i].g;
            }
            // a few CTAs past a whole number of waves would run as a straggler
            // wave: take them back from the segments with the most groups
            const uint64_t slots = G_TARGET / (uint64_t)std::max<int64_t>(P.qs_waves, 1);
            uint64_t excess = gtot > slots ? gtot % slots : 0;
            if (excess > 0 && excess <= slots / 16) {
                // segments by group count, descending (ties: segment order): counting sort
                uint64_t gmax = 0;
                for (const QSeg& q : mids) gmax = std::max<uint64_t>(gmax, q.g);
                std::vector<uint32_t> gc(gmax + 2, 0);
                for (const QSeg& q : mids) ++gc[gmax - q.g + 1];
                for (uint64_t b = 0; b <= gmax; ++b) gc[b + 1] += gc[b];
                std::vector<size_t> byg(mids.size());
                for (size_t i = 0; i < mids.size(); ++i) byg[gc[gmax - mids[i].g]++] = i;
                for (bool any = true; excess > 0 && any;) {  // round robin, most groups first
                    any = false;
                    for (size_t k : byg) {
                        if (excess == 0) break;
                        if (mids[k].g > 1) {
                            --mids[k].g;
                            --excess;
                            any = true;
                        }
                    }
                }
            }
            gtot = 0;
            // lines per group, descending, to 1/8 of an octave (ties: segment
            // order) -- the order only steers the LPT dispatch, so a counting
            // sort over 8 x 64 log-scale buckets replaces a comparison sort
            // (O(segments); the host sits on the critical path between levels)
            constexpr int NBK = 8 * 64;
            L.bk.resize(mids.size());
            L.cnt.assign(NBK + 1, 0);
            for (size_t i = 0; i < mids.size(); ++i) {
                const uint64_t lpg = std::max<uint64_t>(1, (L.seg_nl[i] << 10) / mids[i].g);
                const int oct = 63 - __builtin_clzll(lpg);
                const int sub = oct >= 3 ? (int)((lpg >> (oct - 3)) & 7) : (int)((lpg << (3 - oct)) & 7);
                L.bk[i] = (uint32_t)(NBK - 1 - (oct * 8 + sub));  // descending
                ++L.cnt[L.bk[i] + 1];
            }
            for (int b = 0; b < NBK; ++b) L.cnt[b + 1] += L.cnt[b];
            L.ordi.resize(mids.size());
            for (size_t i = 0; i < mids.size(); ++i) L.ordi[L.cnt[L.bk[i]]++] = i;
            L.m2.clear();
            L.i2.clear();
            for (size_t k : L.ordi) {
                L.m2.push_back(mids[k]);
                L.i2.push_back(L.mid_idx[k]);
            }
            mids.swap(L.m2);
            L.mid_idx.swap(L.i2);
            for (QSeg& q : mids) {
                q.gbase = gtot;
                gtot += q.g;
            }
        }
        return gtot;
    };
    auto launch_level = [&](Lane& L) -> pp_status {
        L.inflight = false;
        if (L.cur.empty()) return PP_OK;
        g_qs_stats.levels = std::max<uint64_t>(g_qs_stats.levels, ++L.depth);
        const uint64_t gtot = plan_mids(L);
        std::vector<QSeg>& mids = L.mids;
        const uint64_t nmid = mids.size(), nbig = L.big_idx.size();
        L.nmid = nmid;
        for (const HSeg& sg : L.cur) g_qs_stats.level_keys += sg.hi - sg.lo;  // every key of the level is partitioned
        L.nbig = nbig;
        L.gtot = gtot;
        // heavy mid segments: batched multi-CTA cleanup
        L.hidx.clear();
        for (size_t mi = 0; mi < mids.size(); ++mi)
            if (HEAVY && mids[mi].hi - mids[mi].lo >= HEAVY) L.hidx.push_back((uint32_t)mi);
        const uint64_t nh = L.hidx.size();
        // ---- workspace: this lane's region [segs][gout][splits][heavy index][heavy blocks] ----
        const size_t segB = al256(sizeof(QSeg) * std::max<uint64_t>(nmid, 1));
        const size_t goB = al256(sizeof(GroupOut) * std::max<uint64_t>(gtot, 1));
        const size_t spB = al256(8 * (nmid + nbig + 1));
        const size_t hiB = al256(4 * std::max<uint64_t>(nh, 1));
        const size_t hvB = HVL.stride * nh;
        const size_t need = al256(segB + goB + spB + hiB + hvB);
        if (need > lane_half) {
            // impossible by construction (lane_half is the level bound: gtot <=
            // G_TARGET + nmid, nmid <= n / (SMALL + 1) + 1, nh <= n / HEAVY + 1);
            // growing the lanes would overlap the early-recursion lists in flight
            set_error("quicksort: a level exceeds its workspace bound");
            return PP_E_INVAL;
        }
        unsigned char* wsb = static_cast<unsigned char*>(qs_workspace(2 * lane_half));
        if (!wsb) return PP_E_NOMEM;
        unsigned char* ws = wsb + (size_t)L.id * lane_half;
        QSeg* d_segs = reinterpret_cast<QSeg*>(ws);
        GroupOut* d_gout = reinterpret_cast<GroupOut*>(ws + segB);
        uint64_t* d_splits = reinterpret_cast<uint64_t*>(ws + segB + goB);
        uint32_t* d_hidx = reinterpret_cast<uint32_t*>(ws + segB + goB + spB);
        unsigned char* d_hv = ws + segB + goB + spB + hiB;
        // pinned staging: [segs][splits][heavy index]
        QSeg* pin_segs = reinterpret_cast<QSeg*>(L.pin);
        uint64_t* pin_splits = reinterpret_cast<uint64_t*>(L.pin + pin_sB);
        uint32_t* pin_hidx = reinterpret_cast<uint32_t*>(L.pin + pin_sB + pin_spB);
        if (nmid > 0) memcpy(pin_segs, mids.data(), sizeof(QSeg) * nmid);
        if (nh > 0) memcpy(pin_hidx, L.hidx.data(), 4 * nh);
        cudaStream_t lst = L.st;
        // ---- big segments: full multi-CTA partition, one at a time (lane 0 only) ----
        L.pivots_h.assign(L.cur.size(), 0);
        for (size_t bi = 0; bi < nbig; ++bi) {
            HSeg& sg = L.cur[L.big_idx[bi]];
            uint64_t p = sg.pivot;
            if (sg.mode != 1) {  // median of 3 (mode 0), ninther (2) or median of 31 (3) of host-read samples
                const uint64_t len = sg.hi - sg.lo;
                const int ns = sg.mode == 3 ? 31 : sg.mode == 2 ? 9 : 3;
                QsSamplePos sp;
                uint64_t* pos = sp.p;
                if (ns == 3) {
                    pos[0] = sg.lo;
                    pos[1] = sg.lo + (len - 1) / 2;
                    pos[2] = sg.hi - 1;
                } else if (ns == 9) {
                    for (int j = 0; j < 9; ++j) pos[j] = ninther_pos<K>(sg.lo, len, j);
                } else {
                    for (int j = 0; j < 31; ++j)
                        pos[j] = sg.lo + (len - 1) / 30 * (uint64_t)j + ((len - 1) % 30) * (uint64_t)j / 30;
                }
                // the lane's pinned split area is idle until this level's splits come down
                volatile uint64_t* hs = reinterpret_cast<uint64_t*>(L.pin + pin_sB);
                qs_sample_kernel<K><<<1, 32, 0, lst>>>(keys, sp, ns, const_cast<uint64_t*>(hs));
                note_launches(1);
                e = cudaGetLastError();
                if (e == cudaSuccess) e = cudaStreamSynchronize(lst);
                if (e != cudaSuccess) return cuda_fail(e, "quicksort pivot");
                K v[31];
                for (int j = 0; j < ns; ++j) v[j] = (K)hs[j];
                auto med3 = [](K a, K b, K c) {
                    if (a > b) std::swap(a, b);
                    if (b > c) b = c;
                    return a > b ? a : b;
                };
                if (ns == 3) {
                    p = (uint64_t)med3(v[0], v[1], v[2]);
                } else if (ns == 9) {
                    p = (uint64_t)med3(med3(v[0], v[1], v[2]), med3(v[3], v[4], v[5]), med3(v[6], v[7], v[8]));
                } else {
                    std::sort(v, v + 31);
                    p = (uint64_t)v[15];
                }
                p = pivot_above_bound<K>((K)p, sg.kmin);
            }
            L.pivots_h[L.big_idx[bi]] = p;
            pp_status ps = partition_device<K>(keys + sg.lo, sg.hi - sg.lo, (K)p, lst, d_splits + nmid + bi, nullptr);
            if (ps != PP_OK) return ps;
        }
        // ---- mid segments: one batched pass ----
        if (nmid > 0) {
            // host lists up first, then the level's kernels back to back (PDL-chained;
            // with the profiling events in between they run plainly serialized)
            e = cudaMemcpyAsync(d_segs, pin_segs, sizeof(QSeg) * nmid, cudaMemcpyHostToDevice, lst);
            if (e == cudaSuccess && nh > 0) e = cudaMemcpyAsync(d_hidx, pin_hidx, 4 * nh, cudaMemcpyHostToDevice, lst);
            if (e != cudaSuccess) return cuda_fail(e, "quicksort H2D");
            qs_pivot_kernel<K><<<(unsigned)((nmid + 7) / 8), 256, 0, lst>>>(keys, d_segs, nmid);
            if (lvl_prof) cudaEventRecord(L.lev[0], lst);
            e = qs_launch_pdl(qs_group_kernel<K>, dim3((unsigned)gtot), C::NT, C::SMEM, lst, keys, d_segs, nmid,
                              P.seed, d_gout, (const QDevCtl*)nullptr);
            if (e != cudaSuccess) return cuda_fail(e, "quicksort group launch");
            if (lvl_prof) cudaEventRecord(L.lev[1], lst);
            if (nh > 0) {
                const unsigned X = (unsigned)std::min<uint64_t>(
                    2 * QS_HEAVY_TILES, std::max<uint64_t>(2, ((uint64_t)sm_count() * 4 + nh - 1) / nh));
                const dim3 grid(X, (unsigned)nh);
                e = qs_launch_pdl(qs_hv_reduce_kernel<K>, grid, 256, 0, lst, keys, (const QSeg*)d_segs,
                                  (const uint32_t*)d_hidx, (const GroupOut*)d_gout, d_splits, d_hv, HVL);
                if (e == cudaSuccess)
                    e = qs_launch_pdl(qs_hv_scan_kernel, dim3((unsigned)nh), 1024, 2 * 8 * (QS_HEAVY_TILES + 1), lst,
                                      d_hv, HVL);
                if (e == cudaSuccess)
                    e = qs_launch_pdl(qs_hv_locate_kernel<K>, grid, SW_NT, 0, lst, keys, (const QSeg*)d_segs,
                                      (const uint32_t*)d_hidx, d_hv, HVL);
                if (e == cudaSuccess)
                    e = qs_launch_pdl(qs_hv_swap_kernel<K>, grid, SW_NT, 0, lst, keys, (const QSeg*)d_segs,
                                      (const uint32_t*)d_hidx, d_hv, HVL);
                if (e != cudaSuccess) return cuda_fail(e, "quicksort heavy cleanup launch");
                note_launches(4);
            }
            if (nh == nmid) {
                // every mid segment was heavy
            } else if (nmid <= (uint64_t)sm_count()) {
                // few (large) segments, long walks: 512-thread CTAs, 4096 keys per side per round trip
                constexpr int NT = 512, EPT = 8;
                const size_t sm = sizeof(StreamBuf<NT, EPT>);
                cudaFuncSetAttribute(qs_cleanup_kernel<K, NT, EPT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)sm);
                e = qs_launch_pdl(qs_cleanup_kernel<K, NT, EPT>, dim3((unsigned)nmid), NT, sm, lst, keys,
                                  (const QSeg*)d_segs, (const GroupOut*)d_gout, d_splits, HEAVY,
                                  (const QDevCtl*)nullptr);
            } else {
                const size_t sm = sizeof(StreamBuf<SW_NT, SW_EPT2>);
                e = qs_launch_pdl(qs_cleanup_kernel<K, SW_NT, SW_EPT2>, dim3((unsigned)nmid), SW_NT, sm, lst, keys,
                                  (const QSeg*)d_segs, (const GroupOut*)d_gout, d_splits, HEAVY,
                                  (const QDevCtl*)nullptr);
            }
            if (e != cudaSuccess) return cuda_fail(e, "quicksort cleanup launch");
            if (lvl_prof) cudaEventRecord(L.lev[2], lst);
            note_launches(3);
            e = cudaGetLastError();
            if (e != cudaSuccess) return cuda_fail(e, "quicksort mid launch");
        }
        // ---- read back splits (and mid pivots) ----
        if (nmid + nbig > 0) {
            e = cudaMemcpyAsync(pin_splits, d_splits, 8 * (nmid + nbig), cudaMemcpyDeviceToHost, lst);
            if (e != cudaSuccess) return cuda_fail(e, "quicksort D2H");
        }
        if (nmid > 0) {
            e = cudaMemcpyAsync(pin_segs, d_segs, sizeof(QSeg) * nmid, cudaMemcpyDeviceToHost, lst);
            if (e != cudaSuccess) return cuda_fail(e, "quicksort D2H");
        }
        e = cudaEventRecord(L.done, lst);
        if (e != cudaSuccess) return cuda_fail(e, "quicksort level event");
        L.inflight = true;
        return PP_OK;
    };

    // the children of a partitioned segment (pivot p, split k): mid ones into
    // `next`, small and leaf ones into the lists of the per-CTA recursion
    // (qs_build_kernel computes the same mid children on the device)
    auto visit = [&](std::vector<HSeg>& next, const HSeg& sg, uint64_t p, uint64_t k) {
        const uint32_t d = sg.depth + 1;
        // key bounds of the parts: left keys < p, right keys >= p
        if (sg.mode != 1) {
            if (k == 0) {
                // p is the segment minimum; split by x <= p next (p == kmax, e.g.
                // all == MAX: every key equals p -- final)
                if (p != sg.kmax) next.push_back({sg.lo, sg.hi, (uint64_t)(K)(p + 1), 1, d, p, sg.kmax});
            } else {
                add_child(next, sg.lo, sg.lo + k, d, sg.kmin, p - 1);
                add_child(next, sg.lo + k, sg.hi, d, p, sg.kmax);
            }
        } else {
            // split by x < sg.pivot (= min + 1): [lo, lo+k) is all equal: final
            add_child(next, sg.lo + k, sg.hi, d, sg.pivot, sg.kmax);
        }
    };
    // wait for a lane's level, read its splits and build its next segment list
    auto finish_level = [&](Lane& L) -> pp_status {
        e = cudaEventSynchronize(L.done);
        if (e != cudaSuccess) return cuda_fail(e, "quicksort level");
        L.inflight = false;
        const uint64_t nmid = L.nmid, nbig = L.nbig;
        const QSeg* pin_segs = reinterpret_cast<const QSeg*>(L.pin);
        const uint64_t* pin_splits = reinterpret_cast<const uint64_t*>(L.pin + pin_sB);
        L.splits_h.assign(pin_splits, pin_splits + nmid + nbig);
        for (size_t mi = 0; mi < nmid; ++mi) L.pivots_h[L.mid_idx[mi]] = pin_segs[mi].pivot;
        if (lvl_prof && nmid > 0) {  // debug: per-level times of the batched mid pass
            float tg = 0, tc = 0;
            cudaEventElapsedTime(&tg, L.lev[0], L.lev[1]);
            cudaEventElapsedTime(&tc, L.lev[1], L.lev[2]);
            uint64_t mk = 0, mx = 0;
            for (const QSeg& q : L.mids) { mk += q.hi - q.lo; mx = std::max<uint64_t>(mx, q.hi - q.lo); }
            fprintf(stderr, "qs level: lane=%d nmid=%llu nbig=%llu gtot=%llu keys=%llu maxseg=%llu group=%.3f ms "
                    "(%.2f TB/s) cleanup=%.3f ms\n", L.id, (unsigned long long)nmid, (unsigned long long)nbig,
                    (unsigned long long)L.gtot, (unsigned long long)mk, (unsigned long long)mx, tg,
                    16.0 * mk / (tg * 1e9), tc);
        }
        // ---- next level ----
        L.next.clear();
        for (size_t mi = 0; mi < nmid; ++mi)
            visit(L.next, L.cur[L.mid_idx[mi]], L.pivots_h[L.mid_idx[mi]], L.splits_h[mi]);
        for (size_t bi = 0; bi < nbig; ++bi)
            visit(L.next, L.cur[L.big_idx[bi]], L.pivots_h[L.big_idx[bi]], L.splits_h[nmid + bi]);
        L.cur.swap(L.next);
        return PP_OK;
    };

    // ---- device-built levels (param qs_dev) ----
    // Once a lane's segments are all below HEAVY (one CTA cleans each), every
    // next level is built on the device by qs_build_kernel, and the host keeps
    // two levels in flight per lane: it enqueues level l+2 (grids sized by the
    // bound 2 x its parent level's count, surplus CTAs exit) as soon as it has
    // read level l back, and takes the small and leaf children from that
    // readback (same visit as the host loop; the device's count of mid
    // children is checked against the host's).  No host round trip sits
    // between two levels of a lane.
    static cudaEvent_t dev_ev[2][2];
    static bool dev_ev_made = false;
    if (dev_on && !dev_ev_made) {
        for (auto& a : dev_ev)
            for (auto& x : a) cudaEventCreateWithFlags(&x, cudaEventDisableTiming);
        dev_ev_made = true;
    }
    struct DevPtr {
        QSeg* list[2];
        QSeg* tmp;
        uint64_t* kb[2];
        uint64_t* tkb;
        QDevCtl* ctl;  // [2]: the count block of list 0 and list 1
        GroupOut* gout;
        uint64_t* splits;
    };
    auto dev_ptr = [&](const Lane& L) {
        DevPtr D;
        unsigned char* b = L.dreg;
        D.list[0] = reinterpret_cast<QSeg*>(b);
        D.list[1] = reinterpret_cast<QSeg*>(b + DL.listB);
        D.tmp = reinterpret_cast<QSeg*>(b + 2 * DL.listB);
        b += 3 * DL.listB;
        D.kb[0] = reinterpret_cast<uint64_t*>(b);
        D.kb[1] = reinterpret_cast<uint64_t*>(b + DL.kbB);
        D.tkb = reinterpret_cast<uint64_t*>(b + 2 * DL.kbB);
        b += 3 * DL.kbB;
        D.ctl = reinterpret_cast<QDevCtl*>(b);
        b += 256;
        D.gout = reinterpret_cast<GroupOut*>(b);
        D.splits = reinterpret_cast<uint64_t*>(b + DL.goutB);
        return D;
    };
    // pinned readback of parity par: [segs][kb][splits][next count block]
    auto pin_segs = [&](const Lane& L, int par) { return reinterpret_cast<QSeg*>(L.dpin + (size_t)par * DL.pinParB); };
    auto pin_kb = [&](const Lane& L, int par) {
        return reinterpret_cast<uint64_t*>(L.dpin + (size_t)par * DL.pinParB + DL.listB);
    };
    auto pin_spl = [&](const Lane& L, int par) {
        return reinterpret_cast<uint64_t*>(L.dpin + (size_t)par * DL.pinParB + DL.listB + DL.kbB);
    };
    auto pin_ctl = [&](const Lane& L, int par) {
        return reinterpret_cast<QDevCtl*>(L.dpin + (size_t)par * DL.pinParB + DL.listB + DL.kbB + DL.splB);
    };
    QBuildArgs QA;
    QA.small = SMALL;
    QA.g_target = G_TARGET;
    QA.minl = MINL;
    QA.slots = G_TARGET / (uint64_t)std::max<int64_t>(P.qs_waves, 1);
    QA.nmax = NM;
    QA.rule = RULE;
    QA.deep = QS_DEEP;
    QA.pivots = RULE != 3 ? 1u : 0u;  // the median of 31 needs a warp per segment: the pivot kernel keeps it
    const bool dev_pivot_kernel = QA.pivots == 0;
    const size_t qb_smem = 4 * (QB_NMAX + 3 * NM);
    if (dev_on) cudaFuncSetAttribute(qs_build_kernel<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)qb_smem);
    // enqueue the level whose list has parity par (at most `bound` segments)
    auto dev_enqueue = [&](Lane& L, int par, uint64_t bound, bool need_pivots) -> pp_status {
        const DevPtr D = dev_ptr(L);
        const cudaStream_t lst = L.st;
        QSeg* segs = D.list[par];
        const QDevCtl* cc = D.ctl + par;
        bound = std::max<uint64_t>(bound, 1);
        if (need_pivots) qs_pivot_kernel<K><<<(unsigned)((bound + 7) / 8), 256, 0, lst>>>(keys, segs, 0, cc);
        e = qs_launch_pdl(qs_group_kernel<K>, dim3((unsigned)(G_TARGET + bound + 1)), C::NT, C::SMEM, lst, keys,
                          (const QSeg*)segs, (uint64_t)0, P.seed, D.gout, cc);
        if (e == cudaSuccess) {
            if (bound <= (uint64_t)sm_count()) {
                constexpr int NT = 512, EPT = 8;
                const size_t sm = sizeof(StreamBuf<NT, EPT>);
                cudaFuncSetAttribute(qs_cleanup_kernel<K, NT, EPT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)sm);
                e = qs_launch_pdl(qs_cleanup_kernel<K, NT, EPT>, dim3((unsigned)bound), NT, sm, lst, keys,
                                  (const QSeg*)segs, (const GroupOut*)D.gout, D.splits, HEAVY, cc);
            } else {
                const size_t sm = sizeof(StreamBuf<SW_NT, SW_EPT2>);
                e = qs_launch_pdl(qs_cleanup_kernel<K, SW_NT, SW_EPT2>, dim3((unsigned)bound), SW_NT, sm, lst, keys,
                                  (const QSeg*)segs, (const GroupOut*)D.gout, D.splits, HEAVY, cc);
            }
        }
        if (e == cudaSuccess) {
            qs_build_kernel<K><<<1, QB_NT, qb_smem, lst>>>(keys, segs, D.kb[par], cc, D.splits, D.tmp, D.tkb,
                                                           D.list[par ^ 1], D.kb[par ^ 1], D.ctl + (par ^ 1), QA);
            e = cudaGetLastError();
        }
        note_launches(need_pivots ? 4 : 3);
        if (e == cudaSuccess) e = cudaMemcpyAsync(pin_segs(L, par), segs, sizeof(QSeg) * bound, cudaMemcpyDeviceToHost, lst);
        if (e == cudaSuccess) e = cudaMemcpyAsync(pin_kb(L, par), D.kb[par], 16 * bound, cudaMemcpyDeviceToHost, lst);
        if (e == cudaSuccess) e = cudaMemcpyAsync(pin_spl(L, par), D.splits, 8 * bound, cudaMemcpyDeviceToHost, lst);
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(pin_ctl(L, par), D.ctl + (par ^ 1), sizeof(QDevCtl), cudaMemcpyDeviceToHost, lst);
        if (e == cudaSuccess) e = cudaEventRecord(dev_ev[L.id][par], lst);
        return e == cudaSuccess ? PP_OK : cuda_fail(e, "quicksort device-built level");
    };
    // switch a lane to device-built levels: its current list goes up once
    auto dev_start = [&](Lane& L) -> pp_status {
        const uint64_t gtot = plan_mids(L);
        const uint64_t nm = L.mids.size();
        const DevPtr D = dev_ptr(L);
        QSeg* ps = pin_segs(L, 0);
        uint64_t* pk = pin_kb(L, 0);
        for (uint64_t i = 0; i < nm; ++i) {
            const HSeg& sg = L.cur[L.mid_idx[i]];
            ps[i] = L.mids[i];
            ps[i].pad = sg.depth;
            pk[2 * i] = sg.kmin;
            pk[2 * i + 1] = sg.kmax;
        }
        QDevCtl* pc = reinterpret_cast<QDevCtl*>(L.dpin + 2 * DL.pinParB);
        *pc = QDevCtl{nm, gtot, 0, 0};
        const cudaStream_t lst = L.st;
        e = cudaMemcpyAsync(D.list[0], ps, sizeof(QSeg) * nm, cudaMemcpyHostToDevice, lst);
        if (e == cudaSuccess) e = cudaMemcpyAsync(D.kb[0], pk, 16 * nm, cudaMemcpyHostToDevice, lst);
        if (e == cudaSuccess) e = cudaMemcpyAsync(D.ctl, pc, sizeof(QDevCtl), cudaMemcpyHostToDevice, lst);
        if (e != cudaSuccess) return cuda_fail(e, "quicksort device-built level H2D");
        L.dev = true;
        L.cur.clear();
        pp_status ps0 = dev_enqueue(L, 0, nm, true);  // (the host's list: pivots on the device)
        if (ps0 != PP_OK) return ps0;
        if ((ps0 = dev_enqueue(L, 1, std::min<uint64_t>(NM, 2 * nm), dev_pivot_kernel)) != PP_OK) return ps0;
        L.qpar[0] = 0;
        L.qpar[1] = 1;
        L.dq = 2;
        L.qexact = nm;
        L.inflight = true;
        return PP_OK;
    };
    // read the oldest level of a device-built lane back, take its small and
    // leaf children, enqueue the level after the next one
    auto dev_step = [&](Lane& L) -> pp_status {
        const int par = L.qpar[0];
        e = cudaEventSynchronize(dev_ev[L.id][par]);
        if (e != cudaSuccess) return cuda_fail(e, "quicksort device-built level");
        const uint64_t nm = L.qexact;
        const QSeg* ps = pin_segs(L, par);
        const uint64_t* pk = pin_kb(L, par);
        const uint64_t* pspl = pin_spl(L, par);
        const QDevCtl pc = *pin_ctl(L, par);
        if (nm > 0) g_qs_stats.levels = std::max<uint64_t>(g_qs_stats.levels, ++L.depth);
        if (P.qs_dev_check && L.dev_expect_valid) {
            // test hook (param qs_dev_check): this device-built list must be the
            // host's plan of the same children -- order, groups, first tasks,
            // depth, mode, bounds (pivots of modes 0 / 2 / 3 are device data)
            bool same = L.dev_expect.size() == nm;
            for (uint64_t i = 0; same && i < nm; ++i) {
                const QSeg& a = ps[i];
                const QSeg& b = L.dev_expect[i];
                same = a.lo == b.lo && a.hi == b.hi && a.g == b.g && a.gbase == b.gbase && a.mode == b.mode &&
                       a.pad == b.pad && a.kmin == b.kmin && (a.mode != 1 || a.pivot == b.pivot) &&
                       pk[2 * i] == L.dev_expect_kb[2 * i] && pk[2 * i + 1] == L.dev_expect_kb[2 * i + 1];
            }
            if (!same) {
                set_error("quicksort: the device-built level list differs from the host's plan (qs_dev_check)");
                return PP_E_INTERNAL;
            }
        }
        L.next.clear();
        for (uint64_t i = 0; i < nm; ++i) {
            const QSeg& q = ps[i];
            const HSeg sg{q.lo, q.hi, q.pivot, q.mode, q.pad, pk[2 * i], pk[2 * i + 1]};
            g_qs_stats.level_keys += q.hi - q.lo;
            visit(L.next, sg, q.pivot, pspl[i]);
        }
        const uint64_t nnext = L.next.size();
        L.dev_expect_valid = false;
        if (P.qs_dev_check && nnext > 0) {
            // the host's plan of these children, checked against the list the
            // device builds from them when that level is read back (the next
            // step of this lane)
            std::swap(L.cur, L.next);
            plan_mids(L);
            L.dev_expect = L.mids;
            L.dev_expect_kb.clear();
            for (size_t i = 0; i < L.mids.size(); ++i) {
                const HSeg& sg = L.cur[L.mid_idx[i]];
                L.dev_expect[i].pad = sg.depth;
                L.dev_expect_kb.push_back(sg.kmin);
                L.dev_expect_kb.push_back(sg.kmax);
            }
            std::swap(L.cur, L.next);
            L.dev_expect_valid = true;
        }
        L.next.clear();
        if (pc.err != 0 || pc.nmid != nnext) {
            set_error("quicksort: the device-built level list disagrees with the host's children");
            return PP_E_INTERNAL;
        }
        L.qpar[0] = L.qpar[1];
        L.dq = 1;
        L.qexact = nnext;
        if (nnext == 0) {  // the level in flight has no segments: the lane is done
            L.dq = 0;
            L.inflight = false;
            return PP_OK;
        }
        const int np = L.qpar[0] ^ 1;
        pp_status s2 = dev_enqueue(L, np, std::min<uint64_t>(NM, 2 * nnext), dev_pivot_kernel);
        if (s2 != PP_OK) return s2;
        L.qpar[1] = np;
        L.dq = 2;
        return PP_OK;
    };
    auto dev_ready = [&](const Lane& L) {
        if (!dev_on || L.cur.empty()) return false;
        for (const HSeg& sg : L.cur)
            if (sg.hi - sg.lo >= BIG || (HEAVY && sg.hi - sg.lo >= HEAVY)) return false;
        return true;
    };

    // phase 1: one lane while big segments exist (or fewer than two segments)
    auto needs_one_lane = [&](const Lane& L) {
        const int64_t nl = P.qs_lanes > 0 ? P.qs_lanes : 2;
        if (nl < 2 || L.cur.size() < 2) return true;
        for (const HSeg& sg : L.cur)
            if (sg.hi - sg.lo >= BIG) return true;
        return false;
    };
    pp_status ps = PP_OK;
    while (!lanes[0].cur.empty() && needs_one_lane(lanes[0])) {
        if ((ps = launch_level(lanes[0])) != PP_OK) return ps;
        if ((ps = finish_level(lanes[0])) != PP_OK) return ps;
    }
    if (!lanes[0].cur.empty()) {
        // phase 2: split by keys (array order), lane 1 starts after the work so far on `st`
        std::vector<HSeg>& c0 = lanes[0].cur;
        uint64_t total = 0, acc = 0;
        for (const HSeg& sg : c0) total += sg.hi - sg.lo;
        size_t cut = 0;
        while (cut + 1 < c0.size() && acc + (c0[cut].hi - c0[cut].lo) <= total / 2) {
            acc += c0[cut].hi - c0[cut].lo;
            ++cut;
        }
        if (cut == 0) cut = 1;
        lanes[1].cur.assign(c0.begin() + cut, c0.end());
        lanes[1].depth = lanes[0].depth;
        c0.resize(cut);
        e = cudaEventRecord(lane_ev[2], st);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(lane_st1_used, lane_ev[2], 0);
        if (e != cudaSuccess) return cuda_fail(e, "quicksort lanes");
        for (Lane& L : lanes)
            if ((ps = dev_ready(L) ? dev_start(L) : launch_level(L)) != PP_OK) return ps;
        while (lanes[0].inflight || lanes[1].inflight) {
            for (Lane& L : lanes) {
                if (!L.inflight) continue;
                if (L.dev) {
                    if ((ps = dev_step(L)) != PP_OK) return ps;
                } else {
                    if ((ps = finish_level(L)) != PP_OK) return ps;
                    if ((ps = dev_ready(L) ? dev_start(L) : launch_level(L)) != PP_OK) return ps;
                }
                if (early && small_lo.size() - small_done >= early_min) {
                    if ((ps = small_batch(small_done, small_lo.size())) != PP_OK) return ps;
                    small_done = small_lo.size();
                }
            }
        }
        // lane 1's last work precedes whatever follows on `st`
        e = cudaEventRecord(lane_ev[2], lane_st1_used);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(st, lane_ev[2], 0);
        if (e != cudaSuccess) return cuda_fail(e, "quicksort lanes");
    }
    if (early) {  // the rest of the small segments, then `st` waits for the early stream
        if ((ps = small_batch(small_done, small_lo.size())) != PP_OK) return ps;
        small_done = small_lo.size();
        e = cudaEventRecord(lane_ev[2], early_bst);  // the bin sorts follow their recursions
        if (e == cudaSuccess) e = cudaStreamWaitEvent(st, lane_ev[2], 0);
        if (e != cudaSuccess) return cuda_fail(e, "quicksort early join");
    }
    // ---- small segments (one CTA each: recursion down to leaves, packed into
    //      bins) and leaves (sorted in shared memory, one CTA per bin); lists
    //      uploaded in chunks of QS_LIST_CHUNK (stream order makes reuse safe) ----
    const uint64_t nleaf = leaf_lo.size(), nsmall = early ? 0 : small_lo.size();
    const uint64_t cl = std::min<uint64_t>(nleaf, QS_LIST_CHUNK), cs = std::min<uint64_t>(nsmall, QS_LIST_CHUNK);
    // bin slots of every small segment (global offsets: chunks of the
    // per-CTA recursion and their bin sorts are pipelined on two streams, so
    // no chunk reuses another's slots)
    std::vector<uint64_t> small_base(nsmall + 1, 0);
    for (uint64_t i = 0; i < nsmall; ++i) small_base[i + 1] = small_base[i] + qs_bin_cap(small_len[i], LEAF);
    const uint64_t max_slots = small_base[nsmall];
    const size_t loB = al256(8 * cl), lnB = al256(4 * cl), sloB = al256(8 * cs), slnB = al256(4 * cs);
    const size_t sbB = al256(8 * cs), scrB = al256(sizeof(GroupOut) * cs);
    const size_t bloB = al256(8 * max_slots), blnB = al256(4 * max_slots);
    unsigned char* qws =
        static_cast<unsigned char*>(qs_workspace(loB + lnB + sloB + slnB + sbB + scrB + bloB + blnB + 256));
    if (!qws) return PP_E_NOMEM;
    if (nsmall > 0) {
        unsigned char* w = qws + loB + lnB;
        uint64_t* d_slo = reinterpret_cast<uint64_t*>(w);
        uint32_t* d_sln = reinterpret_cast<uint32_t*>(w + sloB);
        uint64_t* d_sbase = reinterpret_cast<uint64_t*>(w + sloB + slnB);
        GroupOut* d_scr = reinterpret_cast<GroupOut*>(w + sloB + slnB + sbB);
        uint64_t* d_blo = reinterpret_cast<uint64_t*>(w + sloB + slnB + sbB + scrB);
        uint32_t* d_bln = reinterpret_cast<uint32_t*>(w + sloB + slnB + sbB + scrB + bloB);
        uint64_t* d_prof = nullptr;  // debug phase profile (env PP_QS_PROF)
        static const bool qs_prof = getenv("PP_QS_PROF") != nullptr;
        if (qs_prof) cudaMalloc(&d_prof, 64 * cs);
        // pipeline: chunk c's bins are sorted on a second stream while the
        // per-CTA recursion of chunk c+1 runs (disjoint segments)
        static cudaStream_t st2 = nullptr;
        static std::vector<cudaEvent_t> evs;
        if (!st2) cudaStreamCreateWithFlags(&st2, cudaStreamNonBlocking);
        const uint64_t chunk = QS_LIST_CHUNK;
        const uint64_t nchunks = (nsmall + chunk - 1) / chunk;
        while (evs.size() < nchunks + 1) {
            cudaEvent_t ev;
            cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
            evs.push_back(ev);
        }
        for (uint64_t c = 0, b0 = 0; b0 < nsmall; ++c, b0 += chunk) {
            const uint64_t cnt = std::min<uint64_t>(nsmall - b0, chunk);
            const uint64_t slot0 = small_base[b0], nslots = small_base[b0 + cnt] - slot0;
            e = cudaMemcpyAsync(d_slo, small_lo.data() + b0, 8 * cnt, cudaMemcpyHostToDevice, st);
            if (e == cudaSuccess)
                e = cudaMemcpyAsync(d_sln, small_len.data() + b0, 4 * cnt, cudaMemcpyHostToDevice, st);
            if (e == cudaSuccess)
                e = cudaMemcpyAsync(d_sbase, small_base.data() + b0, 8 * cnt, cudaMemcpyHostToDevice, st);
            if (e != cudaSuccess) return cuda_fail(e, "quicksort small H2D");
            e = launch_small(cnt, d_slo, d_sln, d_sbase, d_blo, d_bln, d_scr, d_prof, st);
            if (e != cudaSuccess) return cuda_fail(e, "quicksort small launch");
            if (d_prof) {
                std::vector<uint64_t> h(8 * cnt);
                cudaMemcpy(h.data(), d_prof, 64 * cnt, cudaMemcpyDeviceToHost);
                uint64_t tot[8] = {0, 0, 0, 0, 0, 0, 0, 0};
                for (uint64_t i = 0; i < cnt; ++i)
                    for (int j = 0; j < 8; ++j) tot[j] += h[8 * i + j];
                fprintf(stderr,
                        "qs_small prof: ctas=%llu slots=%llu cycles pivot=%.3g part=%.3g (walk=%.3g) merge=%.3g; "
                        "partitions=%llu merges=%llu part_keys=%llu merge_keys=%llu\n",
                        (unsigned long long)cnt, (unsigned long long)nslots, (double)tot[0], (double)tot[1],
                        (double)tot[3], (double)tot[2], (unsigned long long)tot[4], (unsigned long long)tot[5],
                        (unsigned long long)tot[6], (unsigned long long)tot[7]);
            }
            e = cudaEventRecord(evs[c], st);
            if (e == cudaSuccess) e = cudaStreamWaitEvent(st2, evs[c], 0);
            if (e == cudaSuccess) e = sort_bins(d_blo + slot0, d_bln + slot0, nslots, st2);
            if (e != cudaSuccess) return cuda_fail(e, "quicksort bin sort launch");
        }
        e = cudaEventRecord(evs[nchunks], st2);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(st, evs[nchunks], 0);
        if (e != cudaSuccess) return cuda_fail(e, "quicksort pipeline join");
        if (d_prof) cudaFree(d_prof);
    }
    if (nleaf > 0) {
        uint64_t* d_lo = reinterpret_cast<uint64_t*>(qws);
        uint32_t* d_len = reinterpret_cast<uint32_t*>(qws + loB);
        for (uint64_t b0 = 0; b0 < nleaf; b0 += QS_LIST_CHUNK) {
            const uint64_t cnt = std::min<uint64_t>(nleaf - b0, QS_LIST_CHUNK);
            e = cudaMemcpyAsync(d_lo, leaf_lo.data() + b0, 8 * cnt, cudaMemcpyHostToDevice, st);
            if (e == cudaSuccess) e = cudaMemcpyAsync(d_len, leaf_len.data() + b0, 4 * cnt, cudaMemcpyHostToDevice, st);
            if (e != cudaSuccess) return cuda_fail(e, "quicksort leaves H2D");
            e = sort_bins(d_lo, d_len, cnt, st);
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

// Stream priorities (param qs_prio, default on): the level loop -- the
// critical path -- runs on high-priority streams (lane 0 on an internal one
// ordered after the caller's stream by events, lane 1 on its own), the early
// per-CTA recursion and bin sorts stay at the lowest priority, so whenever
// CTAs of both are pending the SMs that free up go to the level kernels (a
// 16384-key bin sort holds a whole SM: 208 KiB of shared memory).
template <typename K>
pp_status quicksort_device(K* keys, uint64_t n, cudaStream_t st) {
    if (params().qs_prio == 0) return quicksort_device_impl<K>(keys, n, st);
    static cudaStream_t hi0 = nullptr;
    static cudaEvent_t ev_in = nullptr, ev_out = nullptr;
    if (!hi0) {
        int least = 0, greatest = 0;
        cudaDeviceGetStreamPriorityRange(&least, &greatest);
        if (cudaStreamCreateWithPriority(&hi0, cudaStreamNonBlocking, greatest) != cudaSuccess ||
            cudaEventCreateWithFlags(&ev_in, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&ev_out, cudaEventDisableTiming) != cudaSuccess)
            return cuda_fail(cudaGetLastError(), "quicksort priority stream");
    }
    cudaError_t e = cudaEventRecord(ev_in, st);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(hi0, ev_in, 0);
    if (e != cudaSuccess) return cuda_fail(e, "quicksort priority stream order");
    const pp_status s = quicksort_device_impl<K>(keys, n, hi0);
    e = cudaEventRecord(ev_out, hi0);  // whatever the caller enqueues next sees the sorted keys
    if (e == cudaSuccess) e = cudaStreamWaitEvent(st, ev_out, 0);
    if (e != cudaSuccess && s == PP_OK) return cuda_fail(e, "quicksort priority stream join");
    return s;
}

template pp_status quicksort_device<uint64_t>(uint64_t*, uint64_t, cudaStream_t);
template pp_status quicksort_device<uint32_t>(uint32_t*, uint64_t, cudaStream_t);

}  // namespace pp
