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
    tile = (tile + min_tile - 1) / min_tile * min_tile;  // a multiple of the one-round-trip tile
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
// (ra, rb: the pairs are the items of ranks [ra, ra+npairs) on the left and
// [rb, rb+npairs) on the right -- a task that starts inside its tiles.)
template <typename K, int NT, int EPT>
__device__ __forceinline__ void swap_pair(K* __restrict__ keys, const Dirty& d, K pivot, uint64_t uL,
                                          uint64_t uLend, uint64_t uR, uint64_t uRend, uint64_t npairs,
                                          PairBuf<K, NT, EPT>& pb, uint32_t ra = 0, uint32_t rb = 0) {
    PairScan<K, EPT> ps;
    scan_pair<K, NT, EPT>(keys, d, pivot, uL, uLend, uR, uRend, pb.sc, ps);
#pragma unroll
    for (int k = 0; k < EPT; ++k) {
        const uint32_t il = ps.rl[k] - ra, ir = ps.rr[k] - rb;  // wraps (large) below the window
        if (((ps.fl >> k) & 1u) && il < npairs) pb.lval[il] = ps.xl[k];
        if (((ps.fr >> k) & 1u) && ir < npairs) pb.rval[ir] = ps.xr[k];
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < EPT; ++k) {
        const uint64_t off = (uint64_t)k * NT + threadIdx.x;
        const uint32_t il = ps.rl[k] - ra, ir = ps.rr[k] - rb;
        if (((ps.fl >> k) & 1u) && il < npairs) {
            keys[vreal(d, uL + off)] = pb.rval[il];
            PP_AUDIT_W(keys + vreal(d, uL + off), AUDIT_CLEANUP);
        }
        if (((ps.fr >> k) & 1u) && ir < npairs) {
            keys[vreal(d, uR + off)] = pb.lval[ir];
            PP_AUDIT_W(keys + vreal(d, uR + off), AUDIT_CLEANUP);
        }
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
                                 uint64_t uR0, uint64_t uRend, StreamBuf<NT, EPT>& sb,
                                 uint64_t max_pairs = ~0ull) {
    constexpr uint32_t RNG = NT * EPT, Q = StreamBuf<NT, EPT>::Q;
    uint64_t uL = uL0, uR = uR0;
    uint32_t hl = 0, tl = 0, hr = 0, tr = 0;  // ring head / tail counters
    uint64_t done = 0;
    for (;;) {
        if (done >= max_pairs) break;
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
        uint32_t m = min(tl - hl, tr - hr);
        if ((uint64_t)m > max_pairs - done) m = (uint32_t)(max_pairs - done);
        if (m == 0) {
            if (done >= max_pairs) break;
            if (!(uL < uLend && (tl - hl) < RNG) && !(uR < uRend && (tr - hr) < RNG)) break;
            continue;
        }
        for (uint32_t t = threadIdx.x; t < m; t += NT) {
            const uint64_t pl = vreal(d, uL0 + sb.ql[(hl + t) % Q]);
            const uint64_t pr = vreal(d, uR0 + sb.qr[(hr + t) % Q]);
            const K a = keys[pl], b = keys[pr];
            keys[pl] = b;
            keys[pr] = a;
            PP_AUDIT_W(keys + pl, AUDIT_CLEANUP);
            PP_AUDIT_W(keys + pr, AUDIT_CLEANUP);
        }
        hl += m;
        hr += m;
        done += m;
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

// ===========================================================================
// The multi-CTA cleanup pipeline, as device functions
// over (block index bx, block count gx) so that both the single-array kernels
// of pp_partition.cu and the per-segment batched kernels of the quicksort
// (blockIdx.y = segment) run the same code.
// ===========================================================================
// K4 + K1: window reduction (redundantly in every CTA; CTA bx == 0 publishes
// the control block) fused with the tile counts over the dirty set:
//   left tiles  [t*T, min((t+1)T, Kv))      count successors (misplaced)
//   right tiles [Kv + t*T, min(.., W))       count predecessors (misplaced)
// FROM_GROUPS: K = head_T + sum T_i + tail_T from the group outputs;
// otherwise (cleanup-only path) K = sum of the count_kernel partials and
// D = [0, n).  max_tiles: tiles per side (0 = cleanup_max_tiles(n)).
// Misplaced-flag bitmap of the dirty set (fused cleanup tail): one bit per
// dirty position, left side [0, Kv) then right side [Kv, W), each side
// bm_side_words(cap) words; written only when W <= cap.
__host__ __device__ __forceinline__ uint64_t bm_side_words(uint64_t cap) { return cap / 32 + 64; }

template <typename K, bool FROM_GROUPS>
__device__ void reduce_count_body(const K* __restrict__ keys, uint64_t n, uint64_t h, uint64_t n_lines, uint32_t LK,
                                  const GroupOut* __restrict__ go, uint32_t g, const uint64_t* __restrict__ partial,
                                  int np, K pivot, Ctl* __restrict__ ctl, uint64_t* __restrict__ d_split,
                                  uint32_t* __restrict__ cntL, uint32_t* __restrict__ cntR, uint64_t max_tiles,
                                  uint32_t bx, uint32_t gx, uint32_t* __restrict__ flags = nullptr,
                                  uint32_t nflags = 0, uint32_t* __restrict__ bm = nullptr, uint64_t bm_cap = 0) {
    __shared__ uint64_t sT[8], sMin[8], sMax[8], sHT[8];
    __shared__ Ctl sc;
    __shared__ uint32_t s[8];
    griddep_wait();
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint64_t region_end = n_lines * LK;
    uint64_t T = 0, vmin = region_end, vmax = 0, ht = 0;
    if (FROM_GROUPS) {
        for (uint32_t i = tid; i < g; i += 256) {
            const GroupOut o = go[i];
            T += o.T;
            vmin = o.vlo < vmin ? o.vlo : vmin;
            vmax = o.vhi > vmax ? o.vhi : vmax;
        }
        // head [0,h) and tail [h + region_end, n) predecessors
        for (uint64_t x = tid; x < h; x += 256) ht += is_pred(keys[x], pivot) ? 1 : 0;
        for (uint64_t x = h + region_end + tid; x < n; x += 256) ht += is_pred(keys[x], pivot) ? 1 : 0;
    } else {
        for (int i = tid; i < np; i += 256) T += partial[i];
    }
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
        sT[warp] = T;
        sMin[warp] = vmin;
        sMax[warp] = vmax;
        sHT[warp] = ht;
    }
    __syncthreads();
    if (tid == 0) {
        for (int w = 1; w < 8; ++w) {
            T += sT[w];
            ht += sHT[w];
            vmin = sMin[w] < vmin ? sMin[w] : vmin;
            vmax = sMax[w] > vmax ? sMax[w] : vmax;
        }
        const uint64_t Ksplit = T + ht;
        uint64_t a[3], b[3];
        if (FROM_GROUPS) {
            a[0] = 0; b[0] = h;                                // head
            const uint64_t lo = h + vmin, hi = h + vmax;       // partial-partition window
            a[1] = lo < Ksplit ? lo : Ksplit;
            b[1] = hi > Ksplit ? hi : Ksplit;
            if (vmin > vmax) { a[1] = b[1] = 0; }             // no non-empty group: no window
            a[2] = h + region_end; b[2] = n;                   // tail
            finish_ctl(&sc, n, Ksplit, a, b, CLEANUP_MIN_TILE, max_tiles);
            sc.vmin = lo;
            sc.vmax = hi;
        } else {
            a[0] = 0; b[0] = n;
            a[1] = a[2] = b[1] = b[2] = n;
            finish_ctl(&sc, n, Ksplit, a, b, CLEANUP_MIN_TILE, max_tiles);
            sc.vmin = 0;
            sc.vmax = n;
        }
        if (bx == 0) {
            *ctl = sc;
            if (d_split) *d_split = Ksplit;
        }
    }
    // the next kernel's grid barrier starts from zeroed flags
    if (bx == 0)
        for (uint32_t i = tid; i < nflags; i += 256) flags[i] = 0;
    __syncthreads();
    griddep_launch();
    Dirty d;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        d.s[k] = sc.ds[k];
        d.l[k] = sc.dl[k];
    }
    const uint64_t Kv = sc.Kv, W = sc.W, TT = sc.tile, nL = sc.nL, nR = sc.nR;
    const bool use_bm = bm != nullptr && W <= bm_cap;
    for (uint64_t t = bx; t < nL + nR; t += gx) {
        const bool left = t < nL;
        const uint64_t u0 = left ? t * TT : Kv + (t - nL) * TT;
        const uint64_t u1 = left ? min(u0 + TT, Kv) : min(u0 + TT, W);
        uint32_t c = 0;
        for (uint64_t ub = u0; ub < u1; ub += 8 * 256) {
            K x[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const uint64_t u = ub + (uint64_t)k * 256 + tid;
                x[k] = u < u1 ? keys[vreal(d, u)] : (K)0;
            }
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const uint64_t u = ub + (uint64_t)k * 256 + tid;
                const bool p = is_pred(x[k], pivot);
                const bool f = u < u1 && (left ? !p : p);
                c += f ? 1u : 0u;
                if (use_bm) {  // misplaced-flag bitmap of the dirty set (tiles start at multiples of 32)
                    const uint32_t b = __ballot_sync(0xffffffffu, f);
                    const uint64_t w = (u - lane - (left ? 0 : Kv)) >> 5;
                    if (lane == 0 && u - lane < u1) (left ? bm : bm + bm_side_words(bm_cap))[w] = b;
                }
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
        if (lane == 0) s[warp] = c;
        __syncthreads();
        if (tid == 0) {
            uint32_t tot = 0;
            for (int w = 0; w < 8; ++w) tot += s[w];
            if (left) cntL[t] = tot; else cntR[t - nL] = tot;
        }
        __syncthreads();
    }
}


// K2: exclusive scan of the tile counts (1 CTA, 1024 threads, fixed order).
static __device__ __forceinline__ uint64_t block_exclusive_scan_1024(uint64_t v, uint64_t* sw, uint64_t& total) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    uint64_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint64_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) sw[warp] = x;
    __syncthreads();
    if (warp == 0) {
        uint64_t w = sw[lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint64_t y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += y;
        }
        sw[lane] = w;  // inclusive over warps
    }
    __syncthreads();
    total = sw[31];
    const uint64_t wpre = warp > 0 ? sw[warp - 1] : 0;
    __syncthreads();
    return wpre + x - v;
}

static __device__ __forceinline__ uint64_t lower_bound_u64(const uint64_t* a, uint64_t n, uint64_t x) {
    uint64_t lo = 0, hi = n;
    while (lo < hi) {
        const uint64_t mid = (lo + hi) >> 1;
        if (a[mid] < x) lo = mid + 1; else hi = mid;
    }
    return lo;
}
static __device__ __forceinline__ uint64_t upper_bound_u64(const uint64_t* a, uint64_t n, uint64_t x) {
    uint64_t lo = 0, hi = n;
    while (lo < hi) {
        const uint64_t mid = (lo + hi) >> 1;
        if (a[mid] <= x) lo = mid + 1; else hi = mid;
    }
    return lo;
}

// Scans the tile counts into PL / PR (exclusive rank starts of each tile)
// and builds the swap task list: the stable merge of PL and PR (left entries
// first on ties).  Left tile t lands at t + #{PR < PL[t]}, right tile t' at
// t' + #{PL <= PR[t']} (binary searches in shared memory); each task stores
// its start rank and the left / right tile holding that rank.
// Dynamic shared memory: 2 * (cap + 1) u64.
static __device__ void tile_scan_body(Ctl* __restrict__ ctl, const uint32_t* __restrict__ cntL,
                                      const uint32_t* __restrict__ cntR, uint64_t* __restrict__ PL,
                                      uint64_t* __restrict__ PR, uint64_t* __restrict__ rk,
                                      uint32_t* __restrict__ ttl, uint32_t* __restrict__ ttr,
                                      uint64_t* sp /* smem [nL] PL, then [nR] PR */) {
    __shared__ uint64_t sw[32];
    griddep_wait();
    griddep_launch();
    const uint64_t nL = ctl->nL, nR = ctl->nR;
    uint64_t* sPL = sp;
    uint64_t* sPR = sp + nL;
    uint64_t carry = 0;
    for (uint64_t b = 0; b < nL; b += 1024) {
        const uint64_t i = b + threadIdx.x;
        uint64_t tot;
        const uint64_t ex = block_exclusive_scan_1024(i < nL ? cntL[i] : 0, sw, tot);
        if (i < nL) PL[i] = sPL[i] = carry + ex;
        carry += tot;
    }
    const uint64_t ML = carry;
    carry = 0;
    for (uint64_t b = 0; b < nR; b += 1024) {
        const uint64_t i = b + threadIdx.x;
        uint64_t tot;
        const uint64_t ex = block_exclusive_scan_1024(i < nR ? cntR[i] : 0, sw, tot);
        if (i < nR) PR[i] = sPR[i] = carry + ex;
        carry += tot;
    }
    __syncthreads();
    const bool ok = (ML == carry && ML > 0);
    if (ok) {
        for (uint64_t t = threadIdx.x; t < nL; t += 1024) {
            const uint64_t r = sPL[t];
            const uint64_t m = t + lower_bound_u64(sPR, nR, r);
            rk[m] = r;
            ttl[m] = (uint32_t)t;
            ttr[m] = (uint32_t)(upper_bound_u64(sPR, nR, r) - 1);
        }
        for (uint64_t t = threadIdx.x; t < nR; t += 1024) {
            const uint64_t r = sPR[t];
            const uint64_t ub = upper_bound_u64(sPL, nL, r);
            const uint64_t m = t + ub;
            rk[m] = r;
            ttl[m] = (uint32_t)(ub - 1);
            ttr[m] = (uint32_t)t;
        }
    }
    if (threadIdx.x == 0) {
        ctl->ML = ML;
        ctl->MR = carry;
        if (ML != carry) ctl->err = 1;  // #misplaced successors must equal #misplaced predecessors
        // one swap task per breakpoint of the merged tile rank boundaries
        ctl->nTasks = ok ? nL + nR : 0;
        rk[ok ? nL + nR : 0] = ML;  // sentinel
    }
}

template <typename K>
__device__ void locate_body(const K* __restrict__ keys, Ctl* __restrict__ ctl, K pivot,
                            const uint64_t* __restrict__ PL, const uint64_t* __restrict__ PR,
                            uint64_t* __restrict__ posL, uint64_t* __restrict__ posR, const uint64_t* __restrict__ rk,
                            const uint32_t* __restrict__ ttl, const uint32_t* __restrict__ ttr, uint32_t bx,
                            uint32_t gx) {
    __shared__ CleanupSmem<K, SW_NT, SW_EPT2> sm;
    griddep_wait();
    griddep_launch();
    const Dirty d = load_dirty(ctl);
    const uint64_t Kv = ctl->Kv, W = ctl->W, T = ctl->tile, M = ctl->ML;
    const uint64_t nTasks = ctl->nTasks;
    for (uint64_t j = bx; j <= nTasks; j += gx) {
        const uint64_t r = rk[j];
        uint64_t pl = Kv, pr = W;
        if (j < nTasks && r < M) {
            const uint64_t tl = ttl[j], tr = ttr[j];
            // one round trip per side when the tile is SW_RNG keys
            select_pair<K, SW_NT, SW_EPT2>(keys, d, pivot, tl * T, min(tl * T + T, Kv), r - PL[tl], Kv + tr * T,
                                           min(Kv + tr * T + T, W), r - PR[tr], sm.pb, pl, pr);
        }
        if (threadIdx.x == 0) {
            posL[j] = pl;
            posR[j] = pr;
        }
    }
}

// K5b: rank-matched swap, one CTA per task (grid-stride over bx, gx).
template <typename K>
__device__ void swap_body(K* __restrict__ keys, const Ctl* __restrict__ ctl, K pivot, const uint64_t* __restrict__ posL,
                          const uint64_t* __restrict__ posR, const uint64_t* __restrict__ rk, uint32_t bx,
                          uint32_t gx) {
    __shared__ CleanupSmem<K, SW_NT, SW_EPT2> sm;
    griddep_wait();
    const Dirty d = load_dirty(ctl);
    const uint64_t nTasks = ctl->nTasks, T = ctl->tile, Kv = ctl->Kv, W = ctl->W;
    for (uint64_t j = bx; j < nTasks; j += gx) {
        const uint64_t pairs = rk[j + 1] - rk[j];
        if (pairs == 0) continue;
        const uint64_t uL = posL[j], uR = posR[j];
        // the task's items lie in the tiles of its first items: clamp to them
        const uint64_t tle = min((uL / T + 1) * T, Kv), tre = min(Kv + ((uR - Kv) / T + 1) * T, W);
        const uint64_t eL = min(posL[j + 1], tle), eR = min(posR[j + 1], tre);
        if (T == (uint64_t)SW_RNG) {
            swap_pair<K, SW_NT, SW_EPT2>(keys, d, pivot, uL, eL, uR, eR, pairs, sm.pb);
        } else {
            walk_swap_stream<K, SW_NT, SW_EPT2>(keys, d, pivot, uL, eL, uR, eR, sm.sb);
        }
    }
}


// ===========================================================================
// K2+K5 fused (the default cleanup tail): every CTA redundantly scans the
// tile counts (<= FUSED_MAX_TILES per side) into shared memory, finds its
// tasks -- the breakpoints U_j of the stable merge of the left and right tile
// rank boundaries -- by a merge-path co-rank search, and swaps task j's pairs
// (ranks [U_j, U_j+1)), which lie in ONE left and ONE right tile, in one
// round trip over the two tiles (rank offsets instead of a separate locate
// pass).  Tiles larger than one round trip (huge dirty sets) locate the
// task's first items, then walk with a pair limit.  CTA bx == 0 publishes the
// totals.  Dynamic shared memory: 2 * (FUSED_MAX_TILES + 1) u64.
// ===========================================================================
constexpr uint64_t FUSED_MAX_TILES = 2048;

template <int NT>
__device__ __forceinline__ uint64_t block_exscan(uint64_t v, uint64_t* sw, uint64_t& total) {
    constexpr int NW = NT / 32;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint64_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint64_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) sw[warp] = x;
    __syncthreads();
    if (warp == 0) {
        uint64_t w = lane < NW ? sw[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint64_t y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += y;
        }
        if (lane < NW) sw[lane] = w;
    }
    __syncthreads();
    total = sw[NW - 1];
    const uint64_t wpre = warp > 0 ? sw[warp - 1] : 0;
    __syncthreads();
    return wpre + x - v;
}

// Two independent exclusive scans in one pass (the same barriers): the
// left and right tile counts, or the left and right bitmap words.
template <int NT>
__device__ __forceinline__ void block_exscan2(uint64_t va, uint64_t vb, uint64_t* sw /* [64] */, uint64_t& exa,
                                              uint64_t& exb, uint64_t& tota, uint64_t& totb) {
    constexpr int NW = NT / 32;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint64_t xa = va, xb = vb;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint64_t ya = __shfl_up_sync(0xffffffffu, xa, o), yb = __shfl_up_sync(0xffffffffu, xb, o);
        if (lane >= o) {
            xa += ya;
            xb += yb;
        }
    }
    if (lane == 31) {
        sw[warp] = xa;
        sw[32 + warp] = xb;
    }
    __syncthreads();
    uint64_t pa = 0, pb = 0;
    tota = 0;
    totb = 0;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
        const uint64_t ca = sw[w], cb = sw[32 + w];
        pa += w < warp ? ca : 0;
        pb += w < warp ? cb : 0;
        tota += ca;
        totb += cb;
    }
    __syncthreads();
    exa = pa + xa - va;
    exb = pb + xb - vb;
}

// the j-th value of the sorted merge of a[0..na) and b[0..nb)
__device__ __forceinline__ uint64_t merged_at(const uint64_t* a, uint64_t na, const uint64_t* b, uint64_t nb,
                                             uint64_t j) {
    uint64_t lo = j > nb ? j - nb : 0, hi = j < na ? j : na;
    while (lo < hi) {
        const uint64_t mid = (lo + hi) >> 1;
        if (a[mid] <= b[j - 1 - mid]) lo = mid + 1; else hi = mid;
    }
    return (lo < na && (j - lo >= nb || a[lo] <= b[j - lo])) ? a[lo] : b[j - lo];
}

// Grid barrier over nb co-resident CTAs (cooperative launch): every CTA
// release-stores 1 into its own flag (the flags were zeroed by the previous
// kernel of the stream), then acquire-polls all flags.  No atomics.
__device__ __forceinline__ void grid_barrier_flags(uint32_t* flags, uint32_t bx, uint32_t nb) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        st_release_gpu(flags + bx, 1u);
    }
    for (uint32_t i = threadIdx.x; i < nb; i += blockDim.x)
        while (ld_acquire_gpu(flags + i) == 0u) __nanosleep(32);
    __threadfence();
    __syncthreads();
}

constexpr int FUSED_TASKS_PER_CTA = 32;  // task slots per CTA (grid >= 2*FUSED_MAX_TILES / 32)

// position (0..31) of the k-th set bit of w (k < popc(w))
__device__ __forceinline__ uint32_t select_bit(uint32_t w, uint32_t k) {
    uint32_t pos = 0;
#pragma unroll
    for (int sh = 16; sh > 0; sh >>= 1) {
        const uint32_t lo = w & ((1u << sh) - 1u);
        const uint32_t c = __popc(lo);
        if (k >= c) {
            k -= c;
            w >>= sh;
            pos += sh;
        } else {
            w = lo;
        }
    }
    return pos;
}

// bitmap path: tiles of <= FUSED_BM_TILE_WORDS * 32 keys (W <= the bitmap cap
// <= FUSED_MAX_TILES * that, so the tile size stays within it)
constexpr int FUSED_BM_TILE_WORDS = 512;
__host__ __device__ __forceinline__ uint64_t fused_bm_cap(uint64_t n) {
    const uint64_t c = n / 128, mx = FUSED_MAX_TILES * (uint64_t)FUSED_BM_TILE_WORDS * 32;
    return c < mx ? c : mx;
}

template <typename K>
__device__ void scan_swap_body(K* __restrict__ keys, Ctl* __restrict__ ctl, K pivot,
                               const uint32_t* __restrict__ cntL, const uint32_t* __restrict__ cntR,
                               uint32_t* __restrict__ flags, const uint32_t* __restrict__ bm, uint64_t bm_cap,
                               uint64_t* sp, uint32_t bx, uint32_t gx) {
    __shared__ uint64_t sw[64];
    __shared__ uint64_t posLs[FUSED_TASKS_PER_CTA], posRs[FUSED_TASKS_PER_CTA];
    __shared__ CleanupSmem<K, SW_NT, SW_EPT2> sm;
    griddep_wait();
    griddep_launch();
    const int tid = threadIdx.x;
    const Dirty d = load_dirty(ctl);
    const uint64_t Kv = ctl->Kv, W = ctl->W, T = ctl->tile, nL = ctl->nL, nR = ctl->nR;
    uint64_t* sPL = sp;
    uint64_t* sPR = sp + nL + 1;
    uint64_t ML = 0, MR = 0;  // both sides' counts scanned in one pass per chunk
    for (uint64_t b = 0; b < nL || b < nR; b += SW_NT) {
        const uint64_t i = b + tid;
        uint64_t exl, exr, tl, tr;
        block_exscan2<SW_NT>(i < nL ? cntL[i] : 0, i < nR ? cntR[i] : 0, sw, exl, exr, tl, tr);
        if (i < nL) sPL[i] = ML + exl;
        if (i < nR) sPR[i] = MR + exr;
        ML += tl;
        MR += tr;
    }
    __syncthreads();
    const bool ok = ML == MR && ML > 0;  // identical in every CTA: all return or none
    if (bx == 0 && tid == 0) {
        ctl->ML = ML;
        ctl->MR = MR;
        if (ML != MR) ctl->err = 1;  // #misplaced successors must equal #misplaced predecessors
        ctl->nTasks = ok ? nL + nR : 0;
    }
    if (!ok) return;
    const uint64_t nT = nL + nR;
    // task j covers ranks [U_j, U_j+1) of the stable merge of the tile rank
    // boundaries; its items lie in left tile tl and right tile tr
    struct Task {
        uint64_t np, ra, rb, uL, uLe, uR, uRe;
    };
    auto task = [&](uint64_t j) {
        Task t;
        const uint64_t U = merged_at(sPL, nL, sPR, nR, j);
        const uint64_t U1 = j + 1 < nT ? merged_at(sPL, nL, sPR, nR, j + 1) : ML;
        t.np = U1 - U;
        const uint64_t tl = upper_bound_u64(sPL, nL, U) - 1, tr = upper_bound_u64(sPR, nR, U) - 1;
        t.ra = U - sPL[tl];
        t.rb = U - sPR[tr];
        t.uL = tl * T;
        t.uLe = min(t.uL + T, Kv);
        t.uR = Kv + tr * T;
        t.uRe = min(t.uR + T, W);
        return t;
    };
    if (bm != nullptr && W <= bm_cap) {
        // bitmap path: the misplaced flags of the dirty set were recorded by
        // the count kernel and are never changed by a swap, so every task
        // locates its pairs from its two tiles' bitmap words (popcount
        // prefix + bit select) and swaps them -- no key scan, no barrier
        __shared__ uint32_t bwL[FUSED_BM_TILE_WORDS], bwR[FUSED_BM_TILE_WORDS];
        __shared__ uint32_t bpL[FUSED_BM_TILE_WORDS], bpR[FUSED_BM_TILE_WORDS];
        const uint32_t* bmL = bm;
        const uint32_t* bmR = bm + bm_side_words(bm_cap);
        for (uint64_t j = bx; j < nT; j += gx) {
            const Task t = task(j);
            if (t.np == 0) continue;  // uniform
            const uint32_t nwL = (uint32_t)((t.uLe - t.uL + 31) / 32), nwR = (uint32_t)((t.uRe - t.uR + 31) / 32);
            const uint64_t wL0 = t.uL / 32, wR0 = (t.uR - Kv) / 32;
            const uint32_t nw = nwL > nwR ? nwL : nwR;
            uint64_t cL = 0, cR = 0;
            for (uint32_t b = 0; b < nw; b += SW_NT) {
                const uint32_t i = b + tid;
                const uint32_t wl = i < nwL ? bmL[wL0 + i] : 0u, wr = i < nwR ? bmR[wR0 + i] : 0u;
                uint64_t tl, tr, el, er;
                block_exscan2<SW_NT>(__popc(wl), __popc(wr), sw, el, er, tl, tr);
                if (i < nwL) { bwL[i] = wl; bpL[i] = (uint32_t)(cL + el); }
                if (i < nwR) { bwR[i] = wr; bpR[i] = (uint32_t)(cR + er); }
                cL += tl;
                cR += tr;
            }
            __syncthreads();
            for (uint64_t i = tid; i < t.np; i += SW_NT) {
                const uint32_t rl = (uint32_t)(t.ra + i), rr = (uint32_t)(t.rb + i);
                uint32_t lo = 0, hi = nwL;  // last word with prefix <= rl
                while (hi - lo > 1) {
                    const uint32_t mid = (lo + hi) >> 1;
                    if (bpL[mid] <= rl) lo = mid; else hi = mid;
                }
                const uint64_t uL = t.uL + 32ull * lo + select_bit(bwL[lo], rl - bpL[lo]);
                lo = 0;
                hi = nwR;
                while (hi - lo > 1) {
                    const uint32_t mid = (lo + hi) >> 1;
                    if (bpR[mid] <= rr) lo = mid; else hi = mid;
                }
                const uint64_t uR = t.uR + 32ull * lo + select_bit(bwR[lo], rr - bpR[lo]);
                const uint64_t pl = vreal(d, uL), pr = vreal(d, uR);
                const K a = keys[pl], b = keys[pr];
                keys[pl] = b;
                keys[pr] = a;
                PP_AUDIT_W(keys + pl, AUDIT_CLEANUP);
                PP_AUDIT_W(keys + pr, AUDIT_CLEANUP);
            }
            __syncthreads();
        }
        return;
    }
    // barrier path (dirty set beyond the bitmap cap)
    // phase 1 (read only): the positions of every task's first items
    int k = 0;
    for (uint64_t j = bx; j < nT; j += gx, ++k) {
        const Task t = task(j);
        if (t.np == 0) continue;  // uniform
        uint64_t pl, pr;
        select_pair<K, SW_NT, SW_EPT2>(keys, d, pivot, t.uL, t.uLe, t.ra, t.uR, t.uRe, t.rb, sm.pb, pl, pr);
        if (tid == 0) {
            posLs[k] = pl;
            posRs[k] = pr;
        }
    }
    // no swap may change a key another CTA is still classifying
    grid_barrier_flags(flags, bx, gx);
    // phase 2: swap each task's pairs, scanning from its first items
    k = 0;
    for (uint64_t j = bx; j < nT; j += gx, ++k) {
        const Task t = task(j);
        if (t.np == 0) continue;
        const uint64_t pl = posLs[k], pr = posRs[k];
        if (T == (uint64_t)SW_RNG) {
            swap_pair<K, SW_NT, SW_EPT2>(keys, d, pivot, pl, t.uLe, pr, t.uRe, t.np, sm.pb);
        } else {
            walk_swap_stream<K, SW_NT, SW_EPT2>(keys, d, pivot, pl, t.uLe, pr, t.uRe, sm.sb, t.np);
        }
    }
}

}  // namespace pp
