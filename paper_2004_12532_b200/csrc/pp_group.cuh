// pp_group.cuh -- K3, the Smoothed Striding group partition engine: one CTA
// partitions one group U_i (Fig. 3).
#pragma once
#include "pp_device.cuh"
#include "pp_internal.h"

namespace pp {

// LINE_BYTES = b * sizeof(K) (the paper's cache line of b elements,
// PAPER.md:747, 814-816; b = 512 elements there).
// NT threads; PF lines in flight per end; TMA_STORE: resolved lines leave
// shared memory through the bulk-copy engine instead of thread stores;
// STRIDED: X[j] = 0 for every chunk, the Strided Algorithm (PAPER.md:796-825,
// the SURVEY §8(f) ablation) -- a separate instantiation, so the default
// engine carries no branch for it.
// PAR_ISSUE: the refill bulk copies are issued by one lane of warp 0 per new
// line instead of serially by thread 0 (measured: +3% for u32 4 KiB lines,
// -7% for u64 8 KiB lines).
template <typename K, int LINE_BYTES, int NT_, int PF_, bool TMA_STORE_, bool STRIDED_ = false,
          bool PAR_ISSUE_ = false>
struct GroupCfgT {
    using Key = K;
    static constexpr bool STRIDED = STRIDED_;
    static constexpr bool PAR_ISSUE = PAR_ISSUE_;
    static constexpr int LK = LINE_BYTES / (int)sizeof(K);
    static constexpr int NT = NT_;
    static constexpr int PF = PF_;
    static constexpr bool TMA_STORE = TMA_STORE_;
    static constexpr int VEC = 16 / (int)sizeof(K);
    static constexpr int VPT = LK / (NT * VEC);  // 16-B vectors per thread per line
    static constexpr int KPT = VPT * VEC;
    static constexpr int NW = NT / 32;
    static constexpr int NW8 = (NW + 7) / 8 * 8;  // warp-total slots (u16), padded to 16 B
    static constexpr int POOL = 2 * LK;          // pool ring capacity (occupancy <= 2b)
    static constexpr size_t SMEM =
        (size_t)(2 * PF * LK + 2 * POOL) * sizeof(K) + 2 * PF * 8 + 2 * NW8 + 4 * 2 * PF + 16;
    static_assert(VPT >= 1 && VPT * NT * VEC == LK, "line must be a multiple of NT 16-B vectors");
    static_assert((POOL & (POOL - 1)) == 0, "pool ring must be a power of two");
    static_assert(NW <= 16, "warp totals are packed into at most two 16-byte words");
    static_assert(PF <= 16, "refills: one lane of warp 0 per new line, <= 16 per end");
};

// the default configuration (used by quicksort and by variant 0), measured
// fastest on B200 (tools/tune.py): 8 KiB lines for u64 (b = 1024 keys),
// 4 KiB lines for u32 (b = 1024 keys, 4 CTAs per SM); 128 threads.
#ifndef PP_U32_LINE  // A/B builds only (tools/)
#define PP_U32_LINE 4096
#endif
#ifndef PP_U32_NT
#define PP_U32_NT 128
#endif
#ifndef PP_U32_PF
#define PP_U32_PF 4
#endif
#ifndef PP_U64_LINE
#define PP_U64_LINE 8192
#endif
#ifndef PP_U64_NT
#define PP_U64_NT 128
#endif
#ifndef PP_U64_PF
#define PP_U64_PF 4
#endif
template <typename K>
using GroupCfg = GroupCfgT<K, sizeof(K) == 8 ? PP_U64_LINE : PP_U32_LINE, sizeof(K) == 8 ? PP_U64_NT : PP_U32_NT,
                           sizeof(K) == 8 ? PP_U64_PF : PP_U32_PF, false, false, sizeof(K) == 4>;
// The partition's own group kernel for u32: 8 KiB lines (b = 2048 keys), 256
// threads, 2 lines in flight per end (64 KiB of shared memory, 3 CTAs per
// SM).  The u32 engine is issue-bound (per-line control and barriers over
// 1024 keys with 4 KiB lines); twice the keys per line halve that overhead.
// Config 4 (round 2, profiles/r06_u32_part_configs.txt): 1.37-1.40 ms with
// 4 KiB / 128 threads / 3 in flight (itself -2-3% from 4 in flight) ->
// 1.32-1.37 ms.  The quicksort's level kernel keeps GroupCfg.
#ifndef PP_U32_PART_PF
#define PP_U32_PART_PF 2
#endif
#ifndef PP_U32_PART_LINE
#define PP_U32_PART_LINE 8192
#endif
#ifndef PP_U32_PART_NT
#define PP_U32_PART_NT 256
#endif
#ifndef PP_U64_PART_TMA_STORE  // A/B builds only (TMA bulk stores measured 7% slower, profiles/r06_u64_tma_store_ab.txt)
#define PP_U64_PART_TMA_STORE 0
#endif
template <typename K>
using PartGroupCfg = GroupCfgT<K, sizeof(K) == 8 ? PP_U64_LINE : PP_U32_PART_LINE, sizeof(K) == 8 ? PP_U64_NT : PP_U32_PART_NT,
                               sizeof(K) == 8 ? PP_U64_PF : PP_U32_PART_PF,
                               sizeof(K) == 8 ? (PP_U64_PART_TMA_STORE != 0) : false, false, sizeof(K) == 4>;

// Line index of the j-th line (group order) of group gi: G_i(j) of
// PAPER.md:963-969 in 0-based form, j*g + ((X[j] + i) mod g).
template <bool STRIDED = false>
__device__ __forceinline__ uint64_t group_line(uint64_t seed, uint32_t g, uint32_t gi, uint32_t j) {
    if (STRIDED) return (uint64_t)j * g + gi;
    uint32_t x = ss_offset(seed, (uint64_t)j, g) + gi;
    if (x >= g) x -= g;
    return (uint64_t)j * g + x;
}

// Exclusive prefix (for warp w) and total of up to 16 u16 warp counts held in
// two 16-byte words (lanes of 16 bits; x * 0x0001000100010001 forms the
// inclusive prefix of the four lanes of a 64-bit word).
__device__ __forceinline__ void warp_prefix16(const uint16_t* cnt16, int nw, int warp, uint32_t& woff,
                                              uint32_t& tot) {
    constexpr uint64_t M = 0x0001000100010001ULL;
    uint32_t carry = 0;
    woff = 0;
    for (int q = 0; q < (nw + 7) / 8; ++q) {
        const uint4 v = reinterpret_cast<const uint4*>(cnt16)[q];
        const uint64_t lo = ((uint64_t)v.y << 32) | v.x, hi = ((uint64_t)v.w << 32) | v.z;
        const uint64_t plo = lo * M, phi = hi * M;
        const uint32_t slo = (uint32_t)(plo >> 48), shi = (uint32_t)(phi >> 48);
        const int w = warp - 8 * q;  // position of this warp inside the word pair
        if (w >= 0 && w < 8) {
            uint32_t ex;
            if (w == 0) ex = 0;
            else if (w < 4) ex = (uint32_t)(plo >> (16 * (w - 1))) & 0xFFFFu;
            else if (w == 4) ex = slo;
            else ex = slo + ((uint32_t)(phi >> (16 * (w - 5))) & 0xFFFFu);
            woff = carry + ex;
        }
        carry += slo + shi;
    }
    tot = carry;
}

// The same by warp shuffles: lane i < NW holds warp i's count, an inclusive
// shuffle scan over the NW lanes, two broadcasts -- ~12 instructions per warp
// and line instead of the packed-word arithmetic's ~45, but a longer chain of
// dependent shuffles (used where the engine is issue-bound: 8+ warps).
template <int NW>
__device__ __forceinline__ void warp_prefix_shfl(const uint16_t* cnt16, int warp, int lane, uint32_t& woff,
                                                 uint32_t& tot) {
    uint32_t c = lane < NW ? (uint32_t)cnt16[lane] : 0u;
#pragma unroll
    for (int o = 1; o < NW; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, c, o);
        if (lane >= o) c += y;
    }
    tot = __shfl_sync(0xffffffffu, c, NW - 1);
    const uint32_t before = __shfl_sync(0xffffffffu, c, warp > 0 ? warp - 1 : 0);
    woff = warp > 0 ? before : 0u;
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
// Invariant (checked by simulation and by the parity tests): after
// each consumption at most ONE front and ONE back line are consumed but not
// yet written, and the pools hold <= 2b keys.  Control state is uniform
// (every thread tracks it); only thread 0 issues the bulk copies.  Line
// indices are hashed once, at claim time, into a per-ring-slot table.
template <typename C>
__device__ void ss_group_engine(typename C::Key* __restrict__ region, uint64_t n_lines, uint32_t g, uint32_t gi,
                                uint64_t seed, typename C::Key pivot, GroupOut* __restrict__ out,
                                unsigned char* smem) {
    using K = typename C::Key;
    constexpr int LK = C::LK, NT = C::NT, PF = C::PF, VEC = C::VEC, VPT = C::VPT, KPT = C::KPT, NW = C::NW;
    constexpr uint32_t PMASK = C::POOL - 1;
    constexpr uint32_t LBYTES = LK * sizeof(K);

    K* ring = reinterpret_cast<K*>(smem);         // [2][PF][LK]: front ring, back ring
    K* tpool = ring + 2 * PF * LK;                // predecessor pool (ring of 2 lines)
    K* fpool = tpool + C::POOL;                   // successor pool
    uint64_t* bars = reinterpret_cast<uint64_t*>(fpool + C::POOL);
    uint16_t* wcnt = reinterpret_cast<uint16_t*>(bars + 2 * PF);  // 16-B aligned
    uint32_t* slot_line = reinterpret_cast<uint32_t*>(wcnt + C::NW8);  // [2*PF] line of each ring slot
    const uint32_t bars_s = smem_u32(bars);

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t lt = lanemask_lt();

    // number of lines of this group: s-1 full chunks + the last chunk's line if it exists
    const uint32_t s = (uint32_t)((n_lines + g - 1) / g);
    int S = 0;
    if (s > 0) S = (int)s - 1 + (group_line<C::STRIDED>(seed, g, gi, s - 1) < n_lines ? 1 : 0);

    if (tid == 0) {
        for (int k = 0; k < 2 * PF; ++k) mbar_init(&bars[k], 1);
        fence_mbar_init();
    }
    if (tid < C::NW8) wcnt[tid] = 0;  // padding slots beyond NW are read by warp_prefix16
    __syncthreads();

    int fpf = 0, bpf = S - 1;  // next line to claim for the front / back ring
    int fc = 0, bc = S - 1;    // next line to consume from the front / back
    int fw = 0, bw = S - 1;    // front lines [0,fw) and back lines (bw,S-1] are written
    uint32_t fopen = 0, bopen = 0;            // array line of the open front / back slot
    uint32_t th = 0, tt = 0, fh = 0, ft = 0;  // pool head/tail counters (mod 2^32)

    // issue the load of group line j into ring slot bi (one thread per line)
    auto issue = [&](uint32_t bi, int j) {
        const uint32_t line = (uint32_t)group_line<C::STRIDED>(seed, g, gi, (uint32_t)j);
        slot_line[bi] = line;
        mbar_expect_tx(&bars[bi], LBYTES);
        bulk_g2s(ring + bi * LK, region + (uint64_t)line * LK, LBYTES, &bars[bi]);
    };
    auto store_line = [&](const K* pool, uint32_t head, uint32_t line) {
        K* dst = region + (uint64_t)line * LK;
        const K* src = pool + (head & PMASK);
        if constexpr (C::TMA_STORE) {
            if (tid == 0) {
                bulk_s2g(dst, src, LBYTES);
                bulk_commit();
            }
#if PP_AUDIT
            for (int e = tid; e < LK; e += NT) PP_AUDIT_W(dst + e, AUDIT_GROUP);
#endif
        } else {
#pragma unroll
            for (int q = 0; q < VPT; ++q) {
                const int off = (q * NT + tid) * VEC;
                *reinterpret_cast<uint4*>(dst + off) = *reinterpret_cast<const uint4*>(src + off);
#if PP_AUDIT
                for (int e = 0; e < VEC; ++e) PP_AUDIT_W(dst + off + e, AUDIT_GROUP);
#endif
            }
        }
    };
    for (int k = 0; k < PF; ++k) {
        if (fpf <= bpf) {
            if (tid == 0) issue((uint32_t)fpf % PF, fpf);
            ++fpf;
        }
        if (fpf <= bpf) {
            if (tid == 0) issue(PF + (uint32_t)(S - 1 - bpf) % PF, bpf);
            --bpf;
        }
    }
    __syncthreads();  // slot_line entries of the initial claims visible

    while (fc <= bc) {
        // ---- choose the end to consume (uniform across the CTA) ----
        const uint32_t tocc = tt - th, focc = ft - fh;
        const int nF = fc - fw, nB = bw - bc;  // consumed-but-unwritten slots (0 or 1 each)
        bool front;
        if (tocc >= (uint32_t)LK && nF == 0) front = true;
        else if (focc >= (uint32_t)LK && nB == 0) front = false;
        else front = (nF <= nB);
        const int l = front ? fc : bc;
        uint32_t bi, par;
        if (l < fpf) {  // claimed by the front ring
            bi = (uint32_t)l % PF;
            par = ((uint32_t)l / PF) & 1u;
        } else {        // claimed by the back ring
            const uint32_t kk = (uint32_t)(S - 1 - l);
            bi = PF + kk % PF;
            par = (kk / PF) & 1u;
        }
        const K* src = ring + bi * LK;
        mbar_wait_s(bars_s + bi * 8, par);

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
        if (lane == 0) wcnt[warp] = (uint16_t)wt;
        if constexpr (C::TMA_STORE) {
            // pool slots written out by the bulk engine must be read before reuse
            if (tid == 0) bulk_wait_read<0>();
        }
        __syncthreads();  // (A) warp totals visible; previous write phase finished
        const uint32_t cur_line = slot_line[bi];  // written by thread 0 before an earlier barrier
        uint32_t woff, tot;
        // 8+ warps (the u32 partition engine, issue-bound): shuffles, -0.5-1% on
        // config 4; 4 warps (u64, the quicksort levels): the packed words, whose
        // shorter dependency chain measured 7% faster at config 2
        if constexpr (NW >= 8) warp_prefix_shfl<NW>(wcnt, warp, lane, woff, tot);
        else warp_prefix16(wcnt, NW, warp, woff, tot);
        const uint32_t toff = tt + woff;
        const uint32_t foff = ft + (uint32_t)(warp * 32 * KPT) - woff;
        uint32_t acc = 0;
#pragma unroll
        for (int k = 0; k < KPT; ++k) {
            const uint32_t b = ball[k];
            const uint32_t rt = acc + __popc(b & lt);
            const bool p = (b >> lane) & 1u;
            const uint32_t idx = p ? (toff + rt) : (foff + (uint32_t)(k * 32 + lane) - rt);
            (p ? tpool : fpool)[idx & PMASK] = x[k];
            acc += __popc(b);
        }
        __syncthreads();  // (B) pools complete; ring slot free for reuse
        tt += tot;
        ft += (uint32_t)LK - tot;
        if (front) {
            fopen = cur_line;
            ++fc;
        } else {
            bopen = cur_line;
            --bc;
        }

        // ---- refill the rings: front up to fc+PF, back down to bc-PF ----
        {
            int fnew = min(fc + PF, bpf + 1);
            if (fnew < fpf) fnew = fpf;
            int bnew = max(bc - PF, fnew - 1);
            if (bnew > bpf) bnew = bpf;
            if constexpr (C::PAR_ISSUE) {
                // one lane of warp 0 per new line (front: lanes 0..15, back:
                // 16..31): the hashes and bulk-copy issues run in parallel
                // instead of serially in thread 0, which the other warps wait for
                if (warp == 0) {
                    if (lane < 16) {
                        const int j = fpf + lane;
                        if (j < fnew) issue((uint32_t)j % PF, j);
                    } else {
                        const int j = bpf - (lane - 16);
                        if (j > bnew) issue(PF + (uint32_t)(S - 1 - j) % PF, j);
                    }
                }
            } else if (tid == 0) {
                for (int j = fpf; j < fnew; ++j) issue((uint32_t)j % PF, j);
                for (int j = bpf; j > bnew; --j) issue(PF + (uint32_t)(S - 1 - j) % PF, j);
            }
            fpf = fnew;
            bpf = bnew;
        }

        // ---- write resolved lines (at most one per end) ----
        if constexpr (C::TMA_STORE) {
            if (tid == 0) fence_proxy_async();  // generic smem writes -> async-proxy reads
        }
        if (tt - th >= (uint32_t)LK && fw < fc) {
            store_line(tpool, th, fopen);
            th += LK;
            ++fw;
        }
        if (ft - fh >= (uint32_t)LK && bw > bc) {
            store_line(fpool, fh, bopen);
            fh += LK;
            --bw;
        }
    }

    // ---- final flush: open lines (front's, then back's) get predecessors
    //      then successors ----
    const uint32_t tp = tt - th;
    const bool has_f = fw < fc, has_b = bw > bc;
    const int nopen = (has_f ? 1 : 0) + (has_b ? 1 : 0);
    for (int o = 0; o < nopen; ++o) {
        const uint32_t line = (o == 0 && has_f) ? fopen : bopen;
        K* dst = region + (uint64_t)line * LK;
        const uint32_t base = (uint32_t)o * LK;
        for (int e = tid; e < LK; e += NT) {
            const uint32_t q = base + e;
            dst[e] = (q < tp) ? tpool[(th + q) & PMASK] : fpool[(fh + (q - tp)) & PMASK];
            PP_AUDIT_W(dst + e, AUDIT_GROUP);
        }
    }
    if constexpr (C::TMA_STORE) {
        if (tid == 0) bulk_wait<0>();
    }
    // all loads were waited for: retire the barriers so the shared memory
    // may be reused by a caller (the fused kernel's later phases)
    __syncthreads();
    if (tid == 0) {
        for (int k = 0; k < 2 * PF; ++k) mbar_inval(&bars[k]);
    }
    if (tid == 0) {
        const uint64_t T = (uint64_t)fw * LK + tp;
        GroupOut o;
        o.T = T;
        if (S == 0) {
            o.vlo = n_lines * LK;
            o.vhi = 0;
        } else if (T == (uint64_t)S * LK) {
            o.vlo = o.vhi = group_line<C::STRIDED>(seed, g, gi, (uint32_t)(S - 1)) * LK + LK;
        } else {
            o.vlo = o.vhi = group_line<C::STRIDED>(seed, g, gi, (uint32_t)(T / LK)) * LK + T % LK;
        }
        *out = o;
    }
}

}  // namespace pp
