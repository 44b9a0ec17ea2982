// pp_engine.cuh -- device building blocks shared by the partition and the
// quicksort translation units:
//   * ss_group_engine (pp_group.cuh): one CTA's Smoothed Striding group
//     partition (Fig. 3);
//   * the dirty-set helpers and finish_ctl (window bookkeeping,
//     PAPER.md:979-1001);
//   * the CTA chunk scanner, select and the rank-matched walk used by the
//     cleanup (the r-th misplaced successor left of K <-> the r-th misplaced
//     predecessor right of K).
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

constexpr uint64_t CLEANUP_MIN_TILE = 2048;  // keys per cleanup tile (at least)
constexpr uint64_t CLEANUP_MAX_TILES = 8192; // tiles per side, at most (=> O(1) aux)
// tiles per side for an n-key segment: n/2^14 clamped to [64, 8192]
__host__ __device__ __forceinline__ uint64_t cleanup_max_tiles(uint64_t n) {
    uint64_t c = n >> 14;
    return c < 64 ? 64 : (c > CLEANUP_MAX_TILES ? CLEANUP_MAX_TILES : c);
}

// Build the sorted, merged dirty set from up to 3 intervals [a,b) and fill
// K, W, Kv and the cleanup geometry of the control block.  The tile size
// grows with the dirty-set size so that each side has <= CLEANUP_MAX_TILES
// tiles (aux memory independent of n).
static __device__ void finish_ctl(Ctl* c, uint64_t n, uint64_t K, uint64_t a[3], uint64_t b[3]) {
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
    const uint64_t cap = cleanup_max_tiles(n);
    uint64_t tile = (side + cap - 1) / cap;
    if (tile < CLEANUP_MIN_TILE) tile = CLEANUP_MIN_TILE;
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
// CTA chunk scanner for the cleanup (SW_NT threads, SW_EPT elements each).
// Element e of the chunk starting at virtual index u is u + k*SW_NT + tid
// (k = 0..SW_EPT-1): coalesced per k.  Items (elements whose predicate equals
// want_pred) are ranked in ascending position order.
// ===========================================================================
constexpr int SW_NT = 256;   // threads of the walk / cleanup CTAs
constexpr int SW_EPT = 4;    // elements per thread per chunk
constexpr int SW_CH = SW_NT * SW_EPT;

template <typename K>
struct WalkBuf {
    uint64_t lpos[SW_CH], rpos[SW_CH];
    K lval[SW_CH], rval[SW_CH];
    uint32_t cnt[SW_EPT][SW_NT / 32];
    uint64_t sel;
};

template <typename K>
struct ChunkItems {
    K x[SW_EPT];
    uint32_t rank[SW_EPT];  // rank within the chunk (valid where the item flag is set)
    uint32_t flags;         // bit k: element k is an item
    uint32_t total;         // items in the chunk
};

template <typename K>
__device__ __forceinline__ void scan_chunk(const K* __restrict__ keys, const Dirty& d, K pivot, bool want_pred,
                                           uint64_t u, uint64_t uend, uint32_t (*cnt)[SW_NT / 32],
                                           ChunkItems<K>& it) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    uint32_t ball[SW_EPT];
    it.flags = 0;
#pragma unroll
    for (int k = 0; k < SW_EPT; ++k) {
        const uint64_t uu = u + (uint64_t)k * SW_NT + tid;
        it.x[k] = 0;
        if (uu < uend) it.x[k] = keys[vreal(d, uu)];
    }
#pragma unroll
    for (int k = 0; k < SW_EPT; ++k) {
        const uint64_t uu = u + (uint64_t)k * SW_NT + tid;
        const bool f = uu < uend && (is_pred(it.x[k], pivot) == want_pred);
        ball[k] = __ballot_sync(0xffffffffu, f);
        it.flags |= (f ? 1u : 0u) << k;
    }
    if (lane == 0) {
#pragma unroll
        for (int k = 0; k < SW_EPT; ++k) cnt[k][warp] = __popc(ball[k]);
    }
    __syncthreads();
    uint32_t before = 0;
    const uint32_t lt = lanemask_lt();
#pragma unroll
    for (int k = 0; k < SW_EPT; ++k) {
        uint32_t wbefore = 0, ktot = 0;
#pragma unroll
        for (int w = 0; w < SW_NT / 32; ++w) {
            const uint32_t c = cnt[k][w];
            wbefore += (w < warp) ? c : 0u;
            ktot += c;
        }
        it.rank[k] = before + wbefore + __popc(ball[k] & lt);
        before += ktot;
    }
    it.total = before;
    __syncthreads();  // cnt may be rewritten by the next chunk
}

// Collect up to `need` items from [u, uend) in order into pos/val; advances u
// to just past the last collected item (or to the end of the scanned range).
// Only elements at positions before the last collected item influence the
// result, so elements past it may be concurrently rewritten by another CTA.
template <typename K>
__device__ uint32_t collect_items(const K* __restrict__ keys, const Dirty& d, K pivot, bool want_pred, uint64_t& u,
                                  uint64_t uend, uint32_t need, uint64_t* pos, K* val, WalkBuf<K>& wb) {
    uint32_t got = 0;
    while (got < need && u < uend) {
        ChunkItems<K> it;
        scan_chunk<K>(keys, d, pivot, want_pred, u, uend, wb.cnt, it);
        const uint32_t want = need - got;
#pragma unroll
        for (int k = 0; k < SW_EPT; ++k) {
            if ((it.flags >> k) & 1u) {
                const uint32_t r = it.rank[k];
                const uint64_t uu = u + (uint64_t)k * SW_NT + threadIdx.x;
                if (r < want) {
                    pos[got + r] = uu;
                    val[got + r] = it.x[k];
                }
                if (r == want - 1) wb.sel = uu;
            }
        }
        if (it.total >= want) {
            __syncthreads();
            u = wb.sel + 1;
            got = need;
        } else {
            got += it.total;
            const uint64_t nu = u + SW_CH;
            u = nu < uend ? nu : uend;
        }
        __syncthreads();
    }
    return got;
}

// Position (virtual) of the item of the given rank in [u0, u1), or u1.
template <typename K>
__device__ uint64_t select_item(const K* __restrict__ keys, const Dirty& d, K pivot, bool want_pred, uint64_t u0,
                                uint64_t u1, uint64_t rank, WalkBuf<K>& wb) {
    uint64_t u = u0;
    while (u < u1) {
        ChunkItems<K> it;
        scan_chunk<K>(keys, d, pivot, want_pred, u, u1, wb.cnt, it);
        if (rank < it.total) {
#pragma unroll
            for (int k = 0; k < SW_EPT; ++k)
                if (((it.flags >> k) & 1u) && it.rank[k] == rank) wb.sel = u + (uint64_t)k * SW_NT + threadIdx.x;
            __syncthreads();
            const uint64_t r = wb.sel;
            __syncthreads();
            return r;
        }
        rank -= it.total;
        u += SW_CH;
    }
    return u1;
}

// ===========================================================================
// One-round-trip scan of a left range and a right range of <= SW_RNG
// elements each (both sides' loads in flight together): the cleanup's fast
// path when the tile size is CLEANUP_MIN_TILE.  Left items are successors,
// right items predecessors; ranks in ascending position order per side.
// ===========================================================================
constexpr int SW_EPT2 = 8;
constexpr int SW_RNG = SW_NT * SW_EPT2;  // == CLEANUP_MIN_TILE

template <typename K>
struct PairScan {
    K xl[SW_EPT2], xr[SW_EPT2];
    uint32_t rl[SW_EPT2], rr[SW_EPT2];
    uint32_t fl, fr;     // item flags per element slot
    uint32_t tl, tr;     // item totals
};

template <typename K>
__device__ __forceinline__ void scan_pair(const K* __restrict__ keys, const Dirty& d, K pivot, uint64_t uL,
                                          uint64_t uLend, uint64_t uR, uint64_t uRend,
                                          uint32_t (*cnt)[SW_EPT2][SW_NT / 32], PairScan<K>& ps) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
#pragma unroll
    for (int k = 0; k < SW_EPT2; ++k) {
        const uint64_t a = uL + (uint64_t)k * SW_NT + tid, b = uR + (uint64_t)k * SW_NT + tid;
        ps.xl[k] = a < uLend ? keys[vreal(d, a)] : (K)0;
        ps.xr[k] = b < uRend ? keys[vreal(d, b)] : (K)0;
    }
    uint32_t bl[SW_EPT2], br[SW_EPT2];
    ps.fl = ps.fr = 0;
#pragma unroll
    for (int k = 0; k < SW_EPT2; ++k) {
        const uint64_t a = uL + (uint64_t)k * SW_NT + tid, b = uR + (uint64_t)k * SW_NT + tid;
        const bool fl = a < uLend && !is_pred(ps.xl[k], pivot);
        const bool fr = b < uRend && is_pred(ps.xr[k], pivot);
        bl[k] = __ballot_sync(0xffffffffu, fl);
        br[k] = __ballot_sync(0xffffffffu, fr);
        ps.fl |= (fl ? 1u : 0u) << k;
        ps.fr |= (fr ? 1u : 0u) << k;
    }
    if (lane == 0) {
#pragma unroll
        for (int k = 0; k < SW_EPT2; ++k) {
            cnt[0][k][warp] = __popc(bl[k]);
            cnt[1][k][warp] = __popc(br[k]);
        }
    }
    __syncthreads();
    const uint32_t lt = lanemask_lt();
    uint32_t beforeL = 0, beforeR = 0;
#pragma unroll
    for (int k = 0; k < SW_EPT2; ++k) {
        uint32_t wl = 0, wr = 0, kl = 0, kr = 0;
#pragma unroll
        for (int w = 0; w < SW_NT / 32; ++w) {
            const uint32_t cl = cnt[0][k][w], cr = cnt[1][k][w];
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

template <typename K>
struct PairBuf {
    K lval[SW_RNG], rval[SW_RNG];
    uint32_t cnt[2][SW_EPT2][SW_NT / 32];
    uint64_t sel[2];
};

// Positions of the left item of rank rl in [uL, uLend) and the right item of
// rank rr in [uR, uRend) (ranges <= SW_RNG); returns uLend / uRend if absent.
template <typename K>
__device__ __forceinline__ void select_pair(const K* __restrict__ keys, const Dirty& d, K pivot, uint64_t uL,
                                            uint64_t uLend, uint64_t rl, uint64_t uR, uint64_t uRend, uint64_t rr,
                                            PairBuf<K>& pb, uint64_t& pl, uint64_t& pr) {
    PairScan<K> ps;
    if (threadIdx.x == 0) {
        pb.sel[0] = uLend;
        pb.sel[1] = uRend;
    }
    scan_pair<K>(keys, d, pivot, uL, uLend, uR, uRend, pb.cnt, ps);
#pragma unroll
    for (int k = 0; k < SW_EPT2; ++k) {
        const uint64_t off = (uint64_t)k * SW_NT + threadIdx.x;
        if (((ps.fl >> k) & 1u) && ps.rl[k] == rl) pb.sel[0] = uL + off;
        if (((ps.fr >> k) & 1u) && ps.rr[k] == rr) pb.sel[1] = uR + off;
    }
    __syncthreads();
    pl = pb.sel[0];
    pr = pb.sel[1];
    __syncthreads();
}

// ===========================================================================
// Streaming rank-matched walk for one CTA over a whole (possibly long) left
// range and right range: every round scans the next SW_RNG keys of BOTH
// sides at once (one memory round trip), appends the misplaced keys'
// offsets to two rings, and swaps min(#left, #right) pairs.  Offsets are
// 32-bit relative to the range starts (ranges < 2^32 keys); values are
// re-read at swap time.  Pairs the i-th item of each side, like walk_swap.
// ===========================================================================
constexpr uint32_t SWQ = 2 * SW_RNG;  // ring capacity per side

struct StreamBuf {
    uint32_t ql[SWQ], qr[SWQ];
    uint32_t cnt[2][SW_EPT2][SW_NT / 32];
};

template <typename K>
__device__ void walk_swap_stream(K* __restrict__ keys, const Dirty& d, K pivot, uint64_t uL0, uint64_t uLend,
                                 uint64_t uR0, uint64_t uRend, StreamBuf& sb) {
    uint64_t uL = uL0, uR = uR0;
    uint32_t hl = 0, tl = 0, hr = 0, tr = 0;  // ring head / tail counters
    for (;;) {
        const bool scanL = (tl - hl) < SW_RNG && uL < uLend;
        const bool scanR = (tr - hr) < SW_RNG && uR < uRend;
        if (scanL || scanR) {
            PairScan<K> ps;
            scan_pair<K>(keys, d, pivot, uL, scanL ? min(uL + SW_RNG, uLend) : uL, uR,
                         scanR ? min(uR + SW_RNG, uRend) : uR, sb.cnt, ps);
#pragma unroll
            for (int k = 0; k < SW_EPT2; ++k) {
                const uint32_t off = (uint32_t)k * SW_NT + threadIdx.x;
                if ((ps.fl >> k) & 1u) sb.ql[(tl + ps.rl[k]) % SWQ] = (uint32_t)(uL - uL0) + off;
                if ((ps.fr >> k) & 1u) sb.qr[(tr + ps.rr[k]) % SWQ] = (uint32_t)(uR - uR0) + off;
            }
            tl += ps.tl;
            tr += ps.tr;
            if (scanL) uL = min(uL + SW_RNG, uLend);
            if (scanR) uR = min(uR + SW_RNG, uRend);
            __syncthreads();
        }
        const uint32_t m = min(tl - hl, tr - hr);
        if (m == 0) {
            if (!(uL < uLend && (tl - hl) < SW_RNG) && !(uR < uRend && (tr - hr) < SW_RNG)) break;
            continue;
        }
        for (uint32_t t = threadIdx.x; t < m; t += SW_NT) {
            const uint64_t pl = vreal(d, uL0 + sb.ql[(hl + t) % SWQ]);
            const uint64_t pr = vreal(d, uR0 + sb.qr[(hr + t) % SWQ]);
            const K a = keys[pl], b = keys[pr];
            keys[pl] = b;
            keys[pr] = a;
        }
        hl += m;
        hr += m;
        __syncthreads();
    }
}

template <typename K>
union CleanupSmem {
    WalkBuf<K> wb;
    PairBuf<K> pb;
    StreamBuf sb;
};

// Swap the i-th misplaced successor of [uL, uLend) with the i-th misplaced
// predecessor of [uR, uRend), for i < npairs (ranges <= SW_RNG; all items of
// both ranges belong to this CTA).  Values cross through shared memory by
// rank; each thread writes back its own items' positions.
template <typename K>
__device__ __forceinline__ void swap_pair(K* __restrict__ keys, const Dirty& d, K pivot, uint64_t uL,
                                          uint64_t uLend, uint64_t uR, uint64_t uRend, uint64_t npairs,
                                          PairBuf<K>& pb) {
    PairScan<K> ps;
    scan_pair<K>(keys, d, pivot, uL, uLend, uR, uRend, pb.cnt, ps);
#pragma unroll
    for (int k = 0; k < SW_EPT2; ++k) {
        if (((ps.fl >> k) & 1u) && ps.rl[k] < npairs) pb.lval[ps.rl[k]] = ps.xl[k];
        if (((ps.fr >> k) & 1u) && ps.rr[k] < npairs) pb.rval[ps.rr[k]] = ps.xr[k];
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < SW_EPT2; ++k) {
        const uint64_t off = (uint64_t)k * SW_NT + threadIdx.x;
        if (((ps.fl >> k) & 1u) && ps.rl[k] < npairs) keys[vreal(d, uL + off)] = pb.rval[ps.rl[k]];
        if (((ps.fr >> k) & 1u) && ps.rr[k] < npairs) keys[vreal(d, uR + off)] = pb.lval[ps.rr[k]];
    }
    __syncthreads();
}

// Rank-matched walk: pairs the i-th misplaced successor of [uL, uLend) with
// the i-th misplaced predecessor of [uR, uRend), for up to max_pairs pairs,
// and swaps each pair (one thread per pair).  Only this CTA writes inside
// the two ranges, so the swaps are exclusive (EREW).
template <typename K>
__device__ void walk_swap(K* __restrict__ keys, const Dirty& d, K pivot, uint64_t uL, uint64_t uLend, uint64_t uR,
                          uint64_t uRend, uint64_t max_pairs, WalkBuf<K>& wb) {
    uint64_t remaining = max_pairs;
    while (remaining > 0) {
        const uint32_t need = (uint32_t)(remaining < (uint64_t)SW_CH ? remaining : (uint64_t)SW_CH);
        const uint32_t cl = collect_items<K>(keys, d, pivot, false, uL, uLend, need, wb.lpos, wb.lval, wb);
        const uint32_t cr = collect_items<K>(keys, d, pivot, true, uR, uRend, need, wb.rpos, wb.rval, wb);
        const uint32_t c = cl < cr ? cl : cr;
        for (uint32_t t = threadIdx.x; t < c; t += SW_NT) {
            keys[vreal(d, wb.lpos[t])] = wb.rval[t];
            keys[vreal(d, wb.rpos[t])] = wb.lval[t];
        }
        __syncthreads();
        remaining -= c;
        if (c < need) break;
    }
}

}  // namespace pp
