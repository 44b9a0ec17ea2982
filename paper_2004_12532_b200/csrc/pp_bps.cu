// pp_bps.cu -- the paper's Blocked-Prefix-Sum partition (PAPER.md:319-478,
// §3, Figs. 1-2) in the form of its "low-space implementation"
// (§5): the prefix sums of blocks of B = 4096 keys are
// kept in an explicit array (n/4096 + 1 words: the implicit bit-pair codec of
// Lemma 3.2 is not used), the Preprocessing and Reordering
// phases run in place.  SURVEY §8(f) #3: the paper's own low-aux algorithm as
// a comparison row to the Smoothed Striding path (it needs several passes:
// count, MakeSuccessorHeavy (~2n reads), block counts, reorder).
//
//   bps_count_kernel   predecessors per block (physical ranges)
//   bps_scan_kernel    exclusive block prefix S[0..nb] (one CTA, fixed order)
//   bps_msh_kernel     one level of MakeSuccessorHeavy: for
//                      i < m/2, V[i] pred and V[m-1-i] succ -> swap; the last
//                      levels (m <= BPS_MSH_CTA) run in one CTA
//   bps_base_kernel    Reorder's serial base case (one CTA): the r-th
//                      successor of V[0,K') <-> the r-th predecessor of
//                      V[K',m) (reading R22)
//   bps_tail_kernel    one Reorder level: CTA per block i
//                      of the tail, its j-th predecessor <-> V[S[i] + j]
//
// V is the view: V(i) = A[i], or A[n-1-i] with the roles of predecessors and
// successors swapped when fewer than half of the keys are successors (the
// role swap); every kernel derives it from the device-side
// count, so the whole sequence runs without a host round trip.  Each step
// follows the paper's definition with the DESIGN.md readings (R21-R23),
// which the CPU oracle implements independently, so the output is compared
// with it byte for byte.  No atomics.
#include <vector>

#include "pp_engine.cuh"

namespace pp {

void note_launches(uint64_t k);

constexpr uint64_t BPS_B = 4096;        // block size (the paper's 4096)
constexpr uint64_t BPS_MSH_CTA = 1 << 14;  // MakeSuccessorHeavy levels with m <= this: one CTA

struct BpsView {
    uint64_t n;
    bool rev;
    __device__ __forceinline__ uint64_t at(uint64_t i) const { return rev ? n - 1 - i : i; }
};
template <typename K>
__device__ __forceinline__ bool bps_pred(K x, K pivot, bool rev) {
    return rev ? !(x < pivot) : (x < pivot);
}
// role swap: fewer than half of the keys are successors
__device__ __forceinline__ BpsView bps_view(uint64_t n, const uint64_t* K) {
    BpsView v;
    v.n = n;
    v.rev = 2 * (n - *K) < n;
    return v;
}

// predecessors (by the original predicate) per block of BPS_B physical keys:
// their total K decides the role swap
template <typename K>
__global__ void __launch_bounds__(256) bps_count_kernel(const K* __restrict__ keys, uint64_t n, K pivot,
                                                        uint32_t* __restrict__ cnt) {
    __shared__ uint32_t s[8];
    const uint64_t lo = (uint64_t)blockIdx.x * BPS_B;
    const uint64_t hi = lo + BPS_B < n ? lo + BPS_B : n;
    uint32_t c = 0;
    for (uint64_t q = lo + threadIdx.x; q < hi; q += 256) c += is_pred(keys[q], pivot) ? 1u : 0u;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t t = 0;
        for (int w = 0; w < 8; ++w) t += s[w];
        cnt[blockIdx.x] = t;
    }
}

// total K of the original predicate (for the role swap)
__global__ void __launch_bounds__(1024) bps_total_kernel(const uint32_t* __restrict__ cnt, uint64_t nblk,
                                                         uint64_t* __restrict__ K) {
    __shared__ uint64_t sw[32];
    uint64_t acc = 0;
    for (uint64_t b = 0; b < nblk; b += 1024) {
        const uint64_t i = b + threadIdx.x;
        uint64_t tot;
        block_exclusive_scan_1024(i < nblk ? cnt[i] : 0, sw, tot);
        acc += tot;
    }
    if (threadIdx.x == 0) *K = acc;
}

// One MakeSuccessorHeavy level on V[0, m) (grid-stride over i < m/2).
template <typename K>
__global__ void __launch_bounds__(256) bps_msh_kernel(K* __restrict__ keys, uint64_t n, K pivot, uint64_t m,
                                                      const uint64_t* __restrict__ dK) {
    const BpsView v = bps_view(n, dK);
    for (uint64_t i = (uint64_t)blockIdx.x * 256 + threadIdx.x; i < m / 2; i += (uint64_t)gridDim.x * 256) {
        const uint64_t a = v.at(i), b = v.at(m - 1 - i);
        const K x = keys[a], y = keys[b];
        if (bps_pred(x, pivot, v.rev) && !bps_pred(y, pivot, v.rev)) {
            keys[a] = y;
            keys[b] = x;
        }
    }
}

// The remaining MakeSuccessorHeavy levels (m <= BPS_MSH_CTA) in one CTA.
template <typename K>
__global__ void __launch_bounds__(1024) bps_msh_tail_kernel(K* __restrict__ keys, uint64_t n, K pivot, uint64_t m,
                                                            const uint64_t* __restrict__ dK) {
    const BpsView v = bps_view(n, dK);
    while (m > 1) {
        for (uint64_t i = threadIdx.x; i < m / 2; i += 1024) {
            const uint64_t a = v.at(i), b = v.at(m - 1 - i);
            const K x = keys[a], y = keys[b];
            if (bps_pred(x, pivot, v.rev) && !bps_pred(y, pivot, v.rev)) {
                keys[a] = y;
                keys[b] = x;
            }
        }
        __syncthreads();  // the next level reads what this one wrote (same CTA, global memory)
        m = (m + 1) / 2;
    }
}

// Explicit block prefix: S[0] = 0, S[i+1] = view
// predecessors in view blocks 0..i (inclusive scan of the counts, one CTA,
// fixed order).
__global__ void __launch_bounds__(1024) bps_scan_kernel(const uint32_t* __restrict__ cnt, uint64_t nb,
                                                        uint64_t* __restrict__ S) {
    __shared__ uint64_t sw[32];
    uint64_t carry = 0;
    if (threadIdx.x == 0) S[0] = 0;
    for (uint64_t b = 0; b < nb; b += 1024) {
        const uint64_t i = b + threadIdx.x;
        const uint64_t c = i < nb ? cnt[i] : 0;
        uint64_t tot;
        const uint64_t ex = block_exclusive_scan_1024(c, sw, tot);
        if (i < nb) S[i + 1] = carry + ex + c;
        carry += tot;
    }
}

// View-block predecessor counts (view predicate): CTA per view block.
template <typename K>
__global__ void __launch_bounds__(256) bps_vcount_kernel(const K* __restrict__ keys, uint64_t n, K pivot, uint64_t nb,
                                                         const uint64_t* __restrict__ dK, uint32_t* __restrict__ cnt) {
    __shared__ uint32_t s[8];
    const BpsView v = bps_view(n, dK);
    const uint64_t i = blockIdx.x;
    const uint64_t lo = i * BPS_B, hi = (i == nb - 1) ? n : lo + BPS_B;
    uint32_t c = 0;
    for (uint64_t q = lo + threadIdx.x; q < hi; q += 256) c += bps_pred(keys[v.at(q)], pivot, v.rev) ? 1u : 0u;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t t = 0;
        for (int w = 0; w < 8; ++w) t += s[w];
        cnt[i] = t;
    }
}

// Reorder's base case on V[0, m), K' = S[tb] view predecessors: the r-th
// successor of V[0,K') <-> the r-th predecessor of V[K',m), streamed in
// rounds of 1024 positions per side (ranks by ballots + warp totals).
template <typename K>
__global__ void __launch_bounds__(1024) bps_base_kernel(K* __restrict__ keys, uint64_t n, K pivot, uint64_t m,
                                                        const uint64_t* __restrict__ S, uint64_t tb,
                                                        const uint64_t* __restrict__ dK) {
    constexpr uint32_t NT = 1024, Q = 2 * NT;
    __shared__ uint32_t ql[Q], qr[Q];
    __shared__ uint32_t wl[32], wr[32];
    const BpsView v = bps_view(n, dK);
    const uint64_t Kp = S[tb];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t lt = lanemask_lt();
    uint64_t uL = 0, uR = Kp;
    uint32_t hl = 0, tl = 0, hr = 0, tr = 0;
    for (;;) {
        const bool sL = (tl - hl) < NT && uL < Kp, sR = (tr - hr) < NT && uR < m;
        if (sL || sR) {
            const uint64_t a = uL + tid, b = uR + tid;
            const bool fl = sL && a < Kp && !bps_pred(keys[v.at(a)], pivot, v.rev);
            const bool fr = sR && b < m && bps_pred(keys[v.at(b)], pivot, v.rev);
            const uint32_t bl = __ballot_sync(0xffffffffu, fl), br = __ballot_sync(0xffffffffu, fr);
            if (lane == 0) {
                wl[warp] = __popc(bl);
                wr[warp] = __popc(br);
            }
            __syncthreads();
            uint32_t pl = 0, pr = 0, totl = 0, totr = 0;
            for (int w = 0; w < 32; ++w) {
                pl += w < warp ? wl[w] : 0u;
                pr += w < warp ? wr[w] : 0u;
                totl += wl[w];
                totr += wr[w];
            }
            if (fl) ql[(tl + pl + __popc(bl & lt)) % Q] = (uint32_t)(a);
            if (fr) qr[(tr + pr + __popc(br & lt)) % Q] = (uint32_t)(b);
            tl += totl;
            tr += totr;
            if (sL) uL = uL + NT < Kp ? uL + NT : Kp;
            if (sR) uR = uR + NT < m ? uR + NT : m;
            __syncthreads();
        }
        const uint32_t cnt = min(tl - hl, tr - hr);
        if (cnt == 0) {
            if (!(uL < Kp && (tl - hl) < NT) && !(uR < m && (tr - hr) < NT)) break;
            continue;
        }
        for (uint32_t t = tid; t < cnt; t += NT) {
            const uint64_t x = v.at(ql[(hl + t) % Q]), y = v.at(qr[(hr + t) % Q]);
            const K kx = keys[x], ky = keys[y];
            keys[x] = ky;
            keys[y] = kx;
        }
        hl += cnt;
        hr += cnt;
        __syncthreads();
    }
}

// One Reorder level: CTA per tail block i in [t, tb): its j-th view
// predecessor (position order) is swapped with V[S[i] + j] (Lemma 3.4: a
// successor of the already reordered prefix).  Blocks hold < 2B keys.
template <typename K, int NT>
__global__ void __launch_bounds__(NT) bps_tail_kernel(K* __restrict__ keys, uint64_t n, K pivot, uint64_t nb,
                                                      uint64_t t0, const uint64_t* __restrict__ S,
                                                      const uint64_t* __restrict__ dK) {
    constexpr int NW = NT / 32, EPT = 8, CH = NT * EPT;  // positions per pass; blocks hold < 2B
    __shared__ uint32_t wc[EPT][NW];
    const BpsView v = bps_view(n, dK);
    const uint64_t i = t0 + blockIdx.x;
    const uint64_t lo = i * BPS_B, hi = (i == nb - 1) ? n : lo + BPS_B;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t lt = lanemask_lt();
    const uint64_t base = S[i];
    uint32_t before = 0;  // the block's predecessors at earlier positions (earlier passes)
    for (uint64_t c0 = lo; c0 < hi; c0 += CH) {
        K x[EPT];
        uint32_t ball[EPT];
#pragma unroll
        for (int k = 0; k < EPT; ++k) {
            const uint64_t q = c0 + (uint64_t)k * NT + tid;
            x[k] = q < hi ? keys[v.at(q)] : (K)0;
            ball[k] = __ballot_sync(0xffffffffu, q < hi && bps_pred(x[k], pivot, v.rev));
            if (lane == 0) wc[k][warp] = __popc(ball[k]);
        }
        __syncthreads();
        // all targets first, then all target loads (independent, in flight
        // together), then the stores: no load waits behind another pair's store
        uint64_t tgt[EPT];
#pragma unroll
        for (int k = 0; k < EPT; ++k) {
            uint32_t wpre = 0, row = 0;
            for (int w = 0; w < NW; ++w) {
                const uint32_t cc = wc[k][w];
                wpre += w < warp ? cc : 0u;
                row += cc;
            }
            tgt[k] = v.at(base + before + wpre + __popc(ball[k] & lt));
            before += row;
        }
        __syncthreads();  // wc reusable by the next pass
        K y[EPT];
#pragma unroll
        for (int k = 0; k < EPT; ++k)
            if ((ball[k] >> lane) & 1u) y[k] = keys[tgt[k]];
#pragma unroll
        for (int k = 0; k < EPT; ++k) {
            if ((ball[k] >> lane) & 1u) {
                keys[tgt[k]] = x[k];
                keys[v.at(c0 + (uint64_t)k * NT + tid)] = y[k];
            }
        }
    }
}

template <typename K>
pp_status partition_bps_device(K* keys, uint64_t n, K pivot, cudaStream_t st, uint64_t* d_split) {
    const uint64_t nblk = (n + BPS_B - 1) / BPS_B;  // physical count blocks
    const uint64_t nb = n / BPS_B;                   // view blocks (last takes the remainder)
    const size_t cntB = (4 * std::max<uint64_t>(nblk, 1) + 255) & ~size_t(255);
    const size_t SB = (8 * (nb + 2) + 255) & ~size_t(255);
    unsigned char* ws = static_cast<unsigned char*>(workspace(cntB + SB + 256, st));
    if (!ws) return PP_E_NOMEM;
    uint32_t* cnt = reinterpret_cast<uint32_t*>(ws);
    uint64_t* S = reinterpret_cast<uint64_t*>(ws + cntB);
    uint64_t* dK = d_split ? d_split : reinterpret_cast<uint64_t*>(ws + cntB + SB);
    LastStats& LS = last_stats();
    LS = LastStats();
    LS.n = n;
    LS.aux_bytes = cntB + SB + 256;
    LS.path = 6;
    uint64_t launches = 0;
    // 1. count (original predicate) -> K, the role swap
    bps_count_kernel<K><<<(unsigned)nblk, 256, 0, st>>>(keys, n, pivot, cnt);
    bps_total_kernel<<<1, 1024, 0, st>>>(cnt, nblk, dK);
    launches += 2;
    // 2. MakeSuccessorHeavy
    uint64_t m = n;
    const int grid = sm_count() * 8;
    while (m > BPS_MSH_CTA) {
        const uint64_t pairs = m / 2;
        const unsigned g = (unsigned)std::min<uint64_t>((pairs + 255) / 256, (uint64_t)grid);
        bps_msh_kernel<K><<<g, 256, 0, st>>>(keys, n, pivot, m, dK);
        ++launches;
        m = (m + 1) / 2;
    }
    bps_msh_tail_kernel<K><<<1, 1024, 0, st>>>(keys, n, pivot, m, dK);
    ++launches;
    if (nb == 0) {  // one short block: the base case on the whole view
        // S = {0, view predecessors}: count them with one view block
        bps_vcount_kernel<K><<<1, 256, 0, st>>>(keys, n, pivot, 1, dK, cnt);
        bps_scan_kernel<<<1, 1024, 0, st>>>(cnt, 1, S);
        bps_base_kernel<K><<<1, 1024, 0, st>>>(keys, n, pivot, n, S, 1, dK);
        launches += 3;
    } else {
        // 3. explicit block prefix over the view blocks
        bps_vcount_kernel<K><<<(unsigned)nb, 256, 0, st>>>(keys, n, pivot, nb, dK, cnt);
        bps_scan_kernel<<<1, 1024, 0, st>>>(cnt, nb, S);
        launches += 2;
        // 4. Reorder: prefix sizes top down, then bottom up
        std::vector<uint64_t> tbs{nb};
        for (;;) {
            const uint64_t tb = tbs.back();
            const uint64_t mm = (tb == nb) ? n : tb * BPS_B;
            const uint64_t t = (4 * mm) / (5 * BPS_B) + 1;
            if (mm <= 5 * BPS_B || t >= tb) break;
            tbs.push_back(t);
        }
        const uint64_t tbL = tbs.back();
        bps_base_kernel<K><<<1, 1024, 0, st>>>(keys, n, pivot, (tbL == nb) ? n : tbL * BPS_B, S, tbL, dK);
        ++launches;
        for (size_t k = tbs.size() - 1; k-- > 0;) {
            const uint64_t t = tbs[k + 1], tb = tbs[k];
            if (params().bps_nt == 1024)
                bps_tail_kernel<K, 1024><<<(unsigned)(tb - t), 1024, 0, st>>>(keys, n, pivot, nb, t, S, dK);
            else if (params().bps_nt == 512)
                bps_tail_kernel<K, 512><<<(unsigned)(tb - t), 512, 0, st>>>(keys, n, pivot, nb, t, S, dK);
            else if (params().bps_nt == 128)
                bps_tail_kernel<K, 128><<<(unsigned)(tb - t), 128, 0, st>>>(keys, n, pivot, nb, t, S, dK);
            else
                bps_tail_kernel<K, 256><<<(unsigned)(tb - t), 256, 0, st>>>(keys, n, pivot, nb, t, S, dK);
            ++launches;
        }
    }
    note_launches(launches);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "bps partition launch");
    return PP_OK;
}

template pp_status partition_bps_device<uint64_t>(uint64_t*, uint64_t, uint64_t, cudaStream_t, uint64_t*);
template pp_status partition_bps_device<uint32_t>(uint32_t*, uint64_t, uint32_t, cudaStream_t, uint64_t*);

}  // namespace pp
