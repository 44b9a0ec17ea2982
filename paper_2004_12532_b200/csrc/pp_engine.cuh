// pp_engine.cuh -- device building blocks shared by the partition and the
// quicksort translation units:
//   * ss_group_engine (pp_group.cuh): one CTA's Smoothed Striding group
//     partition (Fig. 3);
//   * the dirty-set helpers and finish_ctl (window bookkeeping,
//     PAPER.md:979-1001);
//   * the cleanup building blocks, generic over the CTA size NT and the keys
//     per thread EPT: one-round-trip two-sided range scans, select, the
//     rank-matched tile-pair swap and the streaming walk (the r-th misplaced
//     successor left of K <-> the r-th misplaced predecessor right of K).
#pragma once
#include "pp_device.cuh"
#include "pp_group.cuh"
#include "pp_internal.h"

namespace pp {

// ===========================================================================
// Dirty set helpers.
// ===========================================================================
struct Dirty {
    uint64_t s[3], l[3];
};
__device__ __forceinline__ Dirty load_dirty(const Ctl* c) {
    Dirty d;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        d.s[k] = c->ds[k];
        d.l[k] = c->dl[k];
    }
    return d;
}
__device__ __forceinline__ uint64_t vreal(const Dirty& d, uint64_t u) {
    if (u < d.l[0]) return d.s[0] + u;
    u -= d.l[0];
    if (u < d.l[1]) return d.s[1] + u;
    u -= d.l[1];
    return d.s[2] + u;
}

constexpr uint64_t CLEANUP_MIN_TILE = 2048;  // keys per cleanup tile (multi-kernel path)
constexpr uint64_t CLEANUP_MAX_TILES = 8192; // tiles per side, at most (=> O(1) aux)
// tiles per side for an n-key segment: n/2^14 clamped to [64, 8192]
__host__ __device__ __forceinline__ uint64_t cleanup_max_tiles(uint64_t n) {
    uint64_t c = n >> 14;
    return c < 64 ? 64 : (c > CLEANUP_MAX_TILES ? CLEANUP_MAX_TILES : c);
}

// Build the sorted, merged dirty set from up to 3 intervals [a,b) and fill
// K, W, Kv and the cleanup geometry of the control block.  The tile size
// (>= min_tile) grows with the dirty-set size so that each side has
// <= cleanup_max_tiles(n) tiles (aux memory independent of n).
static __device__ void finish_ctl(Ctl* c, uint64_t n, uint64_t K, uint64_t a[3], uint64_t b[3],
                                  uint64_t min_tile = CLEANUP_MIN_TILE, uint64_t max_tiles = 0) {
    // sort by start (3 elements), drop empties, merge overlaps / adjacency
    for (int i = 0; i < 3; ++i)
        for (int j = i + 1; j < 3; ++j)
            if (a[j] < a[i]) {
                uint64_t t = a[i]; a[i] = a[j]; a[j] = t;
                t = b[i]; b[i] = b[j]; b[j] = t;
            }
    uint64_t ms[3], me[3];
    int m = 0;
    for (int i = 0; i < 3; ++i) {
        if (b[i] <= a[i]) continue;
        if (m > 0 && a[i] <= me[m - 1]) {
            if (b[i] > me[m - 1]) me[m - 1] = b[i];
        } else {
            ms[m] = a[i];
            me[m] = b[i];
            ++m;
        }
    }
    uint64_t W = 0, Kv = 0;
    for (int i = 0; i < 3; ++i) {
        if (i < m) {
            c->ds[i] = ms[i];
            c->dl[i] = me[i] - ms[i];
            W += me[i] - ms[i];
            if (K > ms[i]) Kv += (K < me[i] ? K : me[i]) - ms[i];
        } else {
            c->ds[i] = n;
            c->dl[i] = 0;
        }
    }
    uint64_t side = Kv > W - Kv ? Kv : W - Kv;
    const uint64_t cap = max_tiles ? max_tiles : cleanup_max_tiles(n);
    uint64_t tile = (side + cap - 1) / cap;
    if (tile < min_tile) tile = min_tile;
    c->n = n;
    c->K = K;
    c->W = W;
    c->Kv = Kv;
    c->tile = tile;
    c->R = 0;
    c->nL = (Kv + tile - 1) / tile;
    c->nR = (W - Kv + tile - 1) / tile;
    c->ML = c->MR = 0;
    c->nTasks = 0;
    c->err = 0;
}

// ===========================================================================
// Two-sided range scan: the next <= NT*EPT keys of a left range and of a
// right range, all loads of both sides in flight together (one memory round
// trip).  Left items = successors (misplaced left of K), right items =
// predecessors; ranks in ascending position order per side.  Element k of a
// thread is at offset k*NT + tid (coalesced per k).
// ===========================================================================
template <typename K, int EPT>
struct PairScan {
    K xl[EPT], xr[EPT];
    uint32_t rl[EPT], rr[EPT];
    uint32_t fl, fr;  // item flags per element slot
    uint32_t tl, tr;  // item totals
};

template <int NT, int EPT>
struct ScanCnt {
    uint32_t cnt[2][EPT][NT / 32];
};

template <typename K, int NT, int EPT>
__device__ __forceinline__ void scan_pair(const K* __restrict__ keys, const Dirty& d, K pivot, uint64_t uL,
                                          uint64_t uLend, uint64_t uR, uint64_t uRend, ScanCnt<NT, EPT>& sc,
                                          PairScan<K, EPT>& ps) {
    constexpr int NW = NT / 32;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
#pragma unroll
    for (int k = 0; k < EPT; ++k) {
        const uint64_t a = uL + (uint64_t)k * NT + tid, b = uR + (uint64_t)k * NT + tid;
        ps.xl[k] = a < uLend ? __ldcg(keys + vreal(d, a)) : (K)0;
        ps.xr[k] = b < uRend ? __ldcg(keys + vreal(d, b)) : (K)0;
    }
    uint32_t bl[EPT], br[EPT];
    ps.fl = ps.fr = 0;
#pragma unroll
    for (int k = 0; k < EPT; ++k) {
        const uint64_t a = uL + (uint64_t)k * NT + tid, b = uR + (uint64_t)k * NT + tid;
        const bool fl = a < uLend && !is_pred(ps.xl[k], pivot);
        const bool fr = b < uRend && is_pred(ps.xr[k], pivot);
        bl[k] = __ballot_sync(0xffffffffu, fl);
        br[k] = __ballot_sync(0xffffffffu, fr);
        ps.fl |= (fl ? 1u : 0u) << k;
        ps.fr |= (fr ? 1u : 0u) << k;
    }
    if (lane == 0) {
#pragma unroll
        for (int k = 0; k < EPT; ++k) {
            sc.cnt[0][k][warp] = __popc(bl[k]);
            sc.cnt[1][k][warp] = __popc(br[k]);
        }
    }
    __syncthreads();
    const uint32_t lt = lanemask_lt();
    uint32_t beforeL = 0, beforeR = 0;
#pragma unroll
    for (int k = 0; k < EPT; ++k) {
        uint32_t wl = 0, wr = 0, kl = 0, kr = 0;
#pragma unroll
        for (int w = 0; w < NW; ++w) {
            const uint32_t cl = sc.cnt[0][k][w], cr = sc.cnt[1][k][w];
            wl += (w < warp) ? cl : 0u;
            wr += (w < warp) ? cr : 0u;
            kl += cl;
            kr += cr;
        }
        ps.rl[k] = beforeL + wl + __popc(bl[k] & lt);
        ps.rr[k] = beforeR + wr + __popc(br[k] & lt);
        beforeL += kl;
        beforeR += kr;
    }
    ps.tl = beforeL;
    ps.tr = beforeR;
    __syncthreads();  // cnt reusable
}

template <typename K, int NT, int EPT>
struct PairBuf {
    static constexpr int RNG = NT * EPT;
    K lval[RNG], rval[RNG];
    ScanCnt<NT, EPT> sc;
    uint64_t sel[2];
};

// Positions of the left item of rank rl in [uL, uLend) and the right item of
// rank rr in [uR, uRend), scanning NT*EPT keys per side per round trip;
// returns uLend / uRend for a side whose item is absent.
template <typename K, int NT, int EPT>
__device__ void select_pair(const K* __restrict__ keys, const Dirty& d, K pivot, uint64_t uL, uint64_t uLend,
                            uint64_t rl, uint64_t uR, uint64_t uRend, uint64_t rr, PairBuf<K, NT, EPT>& pb,
                            uint64_t& pl, uint64_t& pr) {
    constexpr int RNG = NT * EPT;
    if (threadIdx.x == 0) {
        pb.sel[0] = uLend;
        pb.sel[1] = uRend;
    }
    bool doneL = uL >= uLend, doneR = uR >= uRend;
    while (!(doneL && doneR)) {
        PairScan<K, EPT> ps;
        const uint64_t eL = doneL ? uL : min(uL + RNG, uLend), eR = doneR ? uR : min(uR + RNG, uRend);
        scan_pair<K, NT, EPT>(keys, d, pivot, uL, eL, uR, eR, pb.sc, ps);
#pragma unroll
        for (int k = 0; k < EPT; ++k) {
            const uint64_t off = (uint64_t)k * NT + threadIdx.x;
            if (!doneL && ((ps.fl >> k) & 1u) && ps.rl[k] == rl) pb.sel[0] = uL + off;
            if (!doneR && ((ps.fr >> k) & 1u) && ps.rr[k] == rr) pb.sel[1] = uR + off;
        }
        if (!doneL) {
            if (rl < ps.tl) doneL = true; else { rl -= ps.tl; uL = eL; doneL = uL >= uLend; }
        }
        if (!doneR) {
            if (rr < ps.tr) doneR = true; else { rr -= ps.tr; uR = eR; doneR = uR >= uRend; }
        }
    }
    __syncthreads();
    pl = pb.sel[0];
    pr = pb.sel[1];
    __syncthreads();
}

// Swap the i-th misplaced successor of [uL, uLend) with the i-th misplaced
// predecessor of [uR, uRend), for i < npairs (ranges <= NT*EPT; all items
// of both ranges belong to this CTA).  Values cross through shared memory
// by rank; each thread writes back its own items' positions.
template <typename K, int NT, int EPT>
__device__ __forceinline__ void swap_pair(K* __restrict__ keys, const Dirty& d, K pivot, uint64_t uL,
                                          uint64_t uLend, uint64_t uR, uint64_t uRend, uint64_t npairs,
                                          PairBuf<K, NT, EPT>& pb) {
    PairScan<K, EPT> ps;
    scan_pair<K, NT, EPT>(keys, d, pivot, uL, uLend, uR, uRend, pb.sc, ps);
#pragma unroll
    for (int k = 0; k < EPT; ++k) {
        if (((ps.fl >> k) & 1u) && ps.rl[k] < npairs) pb.lval[ps.rl[k]] = ps.xl[k];
        if (((ps.fr >> k) & 1u) && ps.rr[k] < npairs) pb.rval[ps.rr[k]] = ps.xr[k];
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < EPT; ++k) {
        const uint64_t off = (uint64_t)k * NT + threadIdx.x;
        if (((ps.fl >> k) & 1u) && ps.rl[k] < npairs) keys[vreal(d, uL + off)] = pb.rval[ps.rl[k]];
        if (((ps.fr >> k) & 1u) && ps.rr[k] < npairs) keys[vreal(d, uR + off)] = pb.lval[ps.rr[k]];
    }
    __syncthreads();
}

// ===========================================================================
// Streaming rank-matched walk for one CTA over a whole (possibly long) left
// range and right range: every round scans the next NT*EPT keys of BOTH
// sides at once (one memory round trip), appends the misplaced keys'
// offsets to two rings, and swaps min(#left, #right) pairs.  Offsets are
// 32-bit relative to the range starts (ranges < 2^32 keys); values are
// re-read at swap time.  Pairs the i-th item of each side.
// ===========================================================================
template <int NT, int EPT>
struct StreamBuf {
    static constexpr uint32_t Q = 2 * NT * EPT;  // ring capacity per side
    uint32_t ql[Q], qr[Q];
    ScanCnt<NT, EPT> sc;
};

template <typename K, int NT, int EPT>
__device__ void walk_swap_stream(K* __restrict__ keys, const Dirty& d, K pivot, uint64_t uL0, uint64_t uLend,
                                 uint64_t uR0, uint64_t uRend, StreamBuf<NT, EPT>& sb) {
    constexpr uint32_t RNG = NT * EPT, Q = StreamBuf<NT, EPT>::Q;
    uint64_t uL = uL0, uR = uR0;
    uint32_t hl = 0, tl = 0, hr = 0, tr = 0;  // ring head / tail counters
    for (;;) {
        const bool scanL = (tl - hl) < RNG && uL < uLend;
        const bool scanR = (tr - hr) < RNG && uR < uRend;
        if (scanL || scanR) {
            PairScan<K, EPT> ps;
            scan_pair<K, NT, EPT>(keys, d, pivot, uL, scanL ? min(uL + RNG, uLend) : uL, uR,
                                  scanR ? min(uR + RNG, uRend) : uR, sb.sc, ps);
#pragma unroll
            for (int k = 0; k < EPT; ++k) {
                const uint32_t off = (uint32_t)k * NT + threadIdx.x;
                if ((ps.fl >> k) & 1u) sb.ql[(tl + ps.rl[k]) % Q] = (uint32_t)(uL - uL0) + off;
                if ((ps.fr >> k) & 1u) sb.qr[(tr + ps.rr[k]) % Q] = (uint32_t)(uR - uR0) + off;
            }
            tl += ps.tl;
            tr += ps.tr;
            if (scanL) uL = min(uL + RNG, uLend);
            if (scanR) uR = min(uR + RNG, uRend);
            __syncthreads();
        }
        const uint32_t m = min(tl - hl, tr - hr);
        if (m == 0) {
            if (!(uL < uLend && (tl - hl) < RNG) && !(uR < uRend && (tr - hr) < RNG)) break;
            continue;
        }
        for (uint32_t t = threadIdx.x; t < m; t += NT) {
            const uint64_t pl = vreal(d, uL0 + sb.ql[(hl + t) % Q]);
            const uint64_t pr = vreal(d, uR0 + sb.qr[(hr + t) % Q]);
            const K a = keys[pl], b = keys[pr];
            keys[pl] = b;
            keys[pr] = a;
        }
        hl += m;
        hr += m;
        __syncthreads();
    }
}

template <typename K, int NT, int EPT>
union CleanupSmem {
    PairBuf<K, NT, EPT> pb;
    StreamBuf<NT, EPT> sb;
};

// The 256-thread cleanup CTAs of the multi-kernel path: 2048 keys per side
// per round trip (= CLEANUP_MIN_TILE, the one-round-trip tile).
constexpr int SW_NT = 256;
constexpr int SW_EPT2 = 8;
constexpr int SW_RNG = SW_NT * SW_EPT2;
static_assert(SW_RNG == (int)CLEANUP_MIN_TILE, "tile = one round trip");

}  // namespace pp
