// pp_engine.cuh -- device building blocks shared by the partition and the
// quicksort translation units:
//   * ss_group_engine: one CTA's Smoothed Striding group partition
//     (Fig. 3);
//   * the dirty-set helpers and finish_ctl (window bookkeeping,
//     PAPER.md:979-1001);
//   * the CTA chunk scanner, select and the rank-matched walk used by the
//     cleanup (the r-th misplaced successor left of K <-> the r-th misplaced
//     predecessor right of K).
#pragma once
#include "pp_device.cuh"
#include "pp_internal.h"

namespace pp {

// ===========================================================================
// K3: Smoothed Striding group partition.
// ===========================================================================
// LINE_BYTES = b * sizeof(K) (the paper's cache line of b elements,
// PAPER.md:747, 814-816; b = 512 elements there).
// NT threads; PF lines in flight per end; TMA_STORE: resolved lines leave
// shared memory through the bulk-copy engine instead of thread stores.
template <typename K, int LINE_BYTES, int NT_, int PF_, bool TMA_STORE_>
struct GroupCfgT {
    using Key = K;
    static constexpr int LK = LINE_BYTES / (int)sizeof(K);
    static constexpr int NT = NT_;
    static constexpr int PF = PF_;
    static constexpr bool TMA_STORE = TMA_STORE_;
    static constexpr int VEC = 16 / (int)sizeof(K);
    static constexpr int VPT = LK / (NT * VEC);  // 16-B vectors per thread per line
    static constexpr int KPT = VPT * VEC;
    static constexpr int NW = NT / 32;
    static constexpr int POOL = 2 * LK;          // pool ring capacity (occupancy <= 2b)
    static constexpr int LTAB = 16;              // line-index table entries per end
    static constexpr size_t SMEM =
        (size_t)(2 * PF * LK + 2 * POOL) * sizeof(K) + 2 * PF * 8 + 4 * ((NW + 7) / 8 * 8) + 4 * 2 * LTAB + 16;
    static_assert(VPT >= 1 && VPT * NT * VEC == LK, "line must be a multiple of NT 16-B vectors");
    static_assert((POOL & (POOL - 1)) == 0, "pool ring must be a power of two");
    static_assert(PF + 3 < LTAB, "line table too small for the prefetch depth");
};

// the default configuration (used by quicksort and by variant 0)
template <typename K>
using GroupCfg = GroupCfgT<K, 8192, 256, 4, false>;

// Line index of the j-th line (group order) of group gi: G_i(j) of
// PAPER.md:963-969 in 0-based form, j*g + ((X[j] + i) mod g).
__device__ __forceinline__ uint64_t group_line(uint64_t seed, uint32_t g, uint32_t gi, uint32_t j) {
    uint32_t x = ss_offset(seed, (uint64_t)j, g) + gi;
    if (x >= g) x -= g;
    return (uint64_t)j * g + x;
}

// One CTA partitions group gi of the region (n_lines full lines of LK keys).
// The group's lines in group order are consumed from both ends; predecessors
// and successors are appended to two shared-memory pools; a front line is
// written back (all predecessors) when the predecessor pool holds a line's
// worth and a consumed-but-unwritten front slot exists, a back line likewise
// with successors.  At the end the <= 2 open lines get the remaining
// predecessors then successors.  => the group's first T_i elements (group
// order) are predecessors: exactly the Partial Partition Step's postcondition
// (PAPER.md:979-1001), with every line read once and written once.
//
// Control state is uniform (every thread tracks it); only thread 0 issues the
// bulk copies.  Line indices are hashed once, at claim time, into a small
// shared table (ltab) that the write phase reads back.
template <typename C>
__device__ void ss_group_engine(typename C::Key* __restrict__ region, uint64_t n_lines, uint32_t g, uint32_t gi,
                                uint64_t seed, typename C::Key pivot, GroupOut* __restrict__ out,
                                unsigned char* smem) {
    using K = typename C::Key;
    constexpr int LK = C::LK, NT = C::NT, PF = C::PF, VEC = C::VEC, VPT = C::VPT, KPT = C::KPT, NW = C::NW;
    constexpr uint32_t PMASK = C::POOL - 1;
    constexpr uint32_t LBYTES = LK * sizeof(K);
    constexpr int LT = C::LTAB;

    K* ring = reinterpret_cast<K*>(smem);         // [2][PF][LK]: front ring, back ring
    K* tpool = ring + 2 * PF * LK;                // predecessor pool (ring of 2 lines)
    K* fpool = tpool + C::POOL;                   // successor pool
    uint64_t* bars = reinterpret_cast<uint64_t*>(fpool + C::POOL);
    uint32_t* wtrue = reinterpret_cast<uint32_t*>(bars + 2 * PF);
    uint32_t* ltab = wtrue + (NW + 7) / 8 * 8;    // [2][LT] line indices (front, back)

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t lt = lanemask_lt();

    // number of lines of this group: s-1 full chunks + the last chunk's line if it exists
    const uint32_t s = (uint32_t)((n_lines + g - 1) / g);
    int S = 0;
    if (s > 0) S = (int)s - 1 + (group_line(seed, g, gi, s - 1) < n_lines ? 1 : 0);

    if (tid == 0) {
        for (int k = 0; k < 2 * PF; ++k) mbar_init(&bars[k], 1);
        fence_mbar_init();
    }
    __syncthreads();

    int fpf = 0, bpf = S - 1;  // next line to claim for the front / back ring
    int fc = 0, bc = S - 1;    // next line to consume from the front / back
    int fw = 0, bw = S - 1;    // front lines [0,fw) and back lines (bw,S-1] are written
    uint32_t th = 0, tt = 0, fh = 0, ft = 0;  // pool head/tail counters (mod 2^32)

    auto claim_front = [&]() {
        if (tid == 0) {
            const uint32_t slot = (uint32_t)fpf % PF;
            const uint32_t line = (uint32_t)group_line(seed, g, gi, (uint32_t)fpf);
            ltab[fpf & (LT - 1)] = line;
            mbar_expect_tx(&bars[slot], LBYTES);
            bulk_g2s(ring + slot * LK, region + (uint64_t)line * LK, LBYTES, &bars[slot]);
        }
        ++fpf;
    };
    auto claim_back = [&]() {
        if (tid == 0) {
            const uint32_t kk = (uint32_t)(S - 1 - bpf);
            const uint32_t slot = kk % PF;
            const uint32_t line = (uint32_t)group_line(seed, g, gi, (uint32_t)bpf);
            ltab[LT + (kk & (LT - 1))] = line;
            mbar_expect_tx(&bars[PF + slot], LBYTES);
            bulk_g2s(ring + (PF + slot) * LK, region + (uint64_t)line * LK, LBYTES, &bars[PF + slot]);
        }
        --bpf;
    };
    // array line index of group line j (claimed by the front ring iff j < fpf)
    auto line_index = [&](int j) -> uint32_t {
        return j < fpf ? ltab[j & (LT - 1)] : ltab[LT + ((S - 1 - j) & (LT - 1))];
    };
    auto store_line = [&](const K* pool, uint32_t head, int j) {
        K* dst = region + (uint64_t)line_index(j) * LK;
        const K* src = pool + (head & PMASK);
        if constexpr (C::TMA_STORE) {
            if (tid == 0) {
                bulk_s2g(dst, src, LBYTES);
                bulk_commit();
            }
        } else {
#pragma unroll
            for (int q = 0; q < VPT; ++q) {
                const int off = (q * NT + tid) * VEC;
                *reinterpret_cast<uint4*>(dst + off) = *reinterpret_cast<const uint4*>(src + off);
            }
        }
    };
    for (int k = 0; k < PF; ++k) {
        if (fpf <= bpf) claim_front();
        if (fpf <= bpf) claim_back();
    }

    while (fc <= bc) {
        // ---- choose the end to consume (uniform across the CTA) ----
        const uint32_t tocc = tt - th, focc = ft - fh;
        const int nF = fc - fw, nB = bw - bc;  // consumed-but-unwritten slots
        bool front;
        if (tocc >= (uint32_t)LK && nF == 0) front = true;
        else if (focc >= (uint32_t)LK && nB == 0) front = false;
        else front = (nF <= nB);
        const int l = front ? fc : bc;
        uint32_t bi, par;
        if (l < fpf) {
            bi = (uint32_t)l % PF;
            par = ((uint32_t)l / PF) & 1u;
        } else {
            const uint32_t kk = (uint32_t)(S - 1 - l);
            bi = PF + kk % PF;
            par = (kk / PF) & 1u;
        }
        const K* src = ring + bi * LK;
        mbar_wait(&bars[bi], par);

        // ---- classify: warp ballots, slot-major order within the warp ----
        K x[KPT];
#pragma unroll
        for (int q = 0; q < VPT; ++q) {
            Vec16<K> v = *reinterpret_cast<const Vec16<K>*>(src + (q * NT + tid) * VEC);
#pragma unroll
            for (int e = 0; e < VEC; ++e) x[q * VEC + e] = v.v[e];
        }
        uint32_t ball[KPT];
        uint32_t wt = 0;
#pragma unroll
        for (int k = 0; k < KPT; ++k) {
            ball[k] = __ballot_sync(0xffffffffu, is_pred(x[k], pivot));
            wt += __popc(ball[k]);
        }
        if (lane == 0) wtrue[warp] = wt;
        if constexpr (C::TMA_STORE) {
            // pool slots written out by the bulk engine must be read before reuse
            if (tid == 0) bulk_wait_read<0>();
        }
        __syncthreads();  // (A) warp totals visible; previous write phase finished
        uint32_t woff = 0, tot = 0;
#pragma unroll
        for (int w = 0; w < NW; ++w) {
            const uint32_t c = wtrue[w];
            woff += (w < warp) ? c : 0u;
            tot += c;
        }
        const uint32_t toff = tt + woff;
        const uint32_t foff = ft + (uint32_t)(warp * 32 * KPT) - woff;
        uint32_t acc = 0;
#pragma unroll
        for (int k = 0; k < KPT; ++k) {
            const uint32_t b = ball[k];
            const uint32_t rt = acc + __popc(b & lt);
            const uint32_t before = (uint32_t)(k * 32 + lane);
            if ((b >> lane) & 1u) tpool[(toff + rt) & PMASK] = x[k];
            else fpool[(foff + before - rt) & PMASK] = x[k];
            acc += __popc(b);
        }
        __syncthreads();  // (B) pools complete; ring slot free for reuse
        tt += tot;
        ft += (uint32_t)LK - tot;
        if (front) ++fc; else --bc;

        // ---- refill the rings (thread 0 issues, everyone tracks) ----
        while (fpf <= bpf && fpf - fc < PF) claim_front();
        while (bpf >= fpf && bc - bpf < PF) claim_back();

        // ---- write resolved lines ----
        if constexpr (C::TMA_STORE) {
            if (tid == 0) fence_proxy_async();  // generic smem writes -> async-proxy reads
        }
        for (;;) {
            if (tt - th >= (uint32_t)LK && fw < fc) {
                store_line(tpool, th, fw);
                th += LK;
                ++fw;
            } else if (ft - fh >= (uint32_t)LK && bw > bc) {
                store_line(fpool, fh, bw);
                fh += LK;
                --bw;
            } else {
                break;
            }
        }
    }

    // ---- final flush: open lines [fw, bw] get predecessors then successors ----
    const uint32_t tp = tt - th;
    for (int jl = fw; jl <= bw; ++jl) {
        K* dst = region + (uint64_t)line_index(jl) * LK;
        const uint32_t base = (uint32_t)(jl - fw) * LK;
        for (int e = tid; e < LK; e += NT) {
            const uint32_t q = base + e;
            dst[e] = (q < tp) ? tpool[(th + q) & PMASK] : fpool[(fh + (q - tp)) & PMASK];
        }
    }
    if constexpr (C::TMA_STORE) {
        if (tid == 0) bulk_wait<0>();
    }
    if (tid == 0) {
        const uint64_t T = (uint64_t)fw * LK + tp;
        GroupOut o;
        o.T = T;
        if (S == 0) {
            o.vlo = n_lines * LK;
            o.vhi = 0;
        } else if (T == (uint64_t)S * LK) {
            o.vlo = o.vhi = group_line(seed, g, gi, (uint32_t)(S - 1)) * LK + LK;
        } else {
            o.vlo = o.vhi = group_line(seed, g, gi, (uint32_t)(T / LK)) * LK + T % LK;
        }
        *out = o;
    }
}

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
