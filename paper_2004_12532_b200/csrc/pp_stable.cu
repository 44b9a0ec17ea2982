// pp_stable.cu -- the paper's Standard Algorithm (§2 "The
// Parallel Partition Problem"): a STABLE, out-of-place partition by prefix
// sums.  D[i] = [A[i] < p]; S = prefix sums of D; predecessor i goes to
// C[S[i] - 1], successor i to C[t + i - S[i]] with t = S[n-1] (0-based form
// of PAPER.md:301-305, reading R9).  The SURVEY §8(f) #4 comparison row: it
// needs Theta(n) extra memory (the output array) and reads the input twice
// (count, then scatter): 3*n*w bytes of traffic against the in-place
// partition's 2*n*w.
//
// On the GPU the prefix sum is blocked: tiles of ST_TILE keys,
//   st_count_kernel   D summed per tile (warp ballots),
//   st_scan_kernel    exclusive scan of the tile sums (one CTA, fixed order),
//   st_scatter_kernel per tile: ranks inside the tile in position order
//                     (ballot prefix per warp + warp totals), then the
//                     destinations above -- every output written once.
// No atomics; the output is unique (stability), so it is compared byte for
// byte with the oracle's Standard Algorithm.
//
// The in-place STABLE variant (SURVEY §8(f) #4 "stable in-place variants";
// of the algorithms there only the out-of-place Standard
// Algorithm is stable): O(n log n) work, O(n / 4096) aux words.
//   sti_leaf_kernel      every tile of ST_TILE keys stable-partitioned in
//                        place (the tile is held in registers, then the
//                        Standard Algorithm's placement inside the tile);
//   merge levels         adjacent stable-partitioned segments [P1 S1][P2 S2]
//                        become [P1 P2 S1 S2] by rotating the middle
//                        [S1 P2] with three in-place reversals (reverse S1
//                        and P2: sti_reverse2_kernel; reverse the whole
//                        middle: sti_reverse_mid_kernel), one swap per
//                        thread; segment sizes double each level.
// Relative order is kept by every step, so the result is the Standard
// Algorithm's output, byte for byte.  The price of stability in place: about
// 2 passes over the array per level, log2(n / 4096) levels.
#include <algorithm>

#include "pp_engine.cuh"

namespace pp {

void note_launches(uint64_t k);

constexpr int ST_NT = 256;
constexpr int ST_EPT = 16;
constexpr uint64_t ST_TILE = (uint64_t)ST_NT * ST_EPT;  // 4096 keys

// position of element k of thread tid inside a tile: k-major, then thread
__device__ __forceinline__ uint64_t st_pos(uint64_t tile, int k, int tid) {
    return tile * ST_TILE + (uint64_t)k * ST_NT + tid;
}

template <typename K>
__global__ void __launch_bounds__(ST_NT) st_count_kernel(const K* __restrict__ in, uint64_t n, K pivot,
                                                         uint32_t* __restrict__ cnt) {
    __shared__ uint32_t s[ST_NT / 32];
    const uint64_t t = blockIdx.x;
    const int tid = threadIdx.x;
    K x[ST_EPT];
#pragma unroll
    for (int k = 0; k < ST_EPT; ++k) {
        const uint64_t p = st_pos(t, k, tid);
        x[k] = p < n ? __ldcs(in + p) : (K)0;
    }
    uint32_t c = 0;
#pragma unroll
    for (int k = 0; k < ST_EPT; ++k) c += (st_pos(t, k, tid) < n && is_pred(x[k], pivot)) ? 1u : 0u;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if ((tid & 31) == 0) s[tid >> 5] = c;
    __syncthreads();
    if (tid == 0) {
        uint32_t tot = 0;
        for (int w = 0; w < ST_NT / 32; ++w) tot += s[w];
        cnt[t] = tot;
    }
}

// Exclusive prefix of the tile sums (S at tile granularity) and t = S[n-1].
__global__ void __launch_bounds__(1024) st_scan_kernel(const uint32_t* __restrict__ cnt, uint64_t ntiles,
                                                       uint64_t* __restrict__ pre, uint64_t* __restrict__ total) {
    __shared__ uint64_t sw[32];
    uint64_t carry = 0;
    for (uint64_t b = 0; b < ntiles; b += 1024) {
        const uint64_t i = b + threadIdx.x;
        uint64_t tot;
        const uint64_t ex = block_exclusive_scan_1024(i < ntiles ? cnt[i] : 0, sw, tot);
        if (i < ntiles) pre[i] = carry + ex;
        carry += tot;
    }
    if (threadIdx.x == 0) *total = carry;
}

template <typename K>
__global__ void __launch_bounds__(ST_NT) st_scatter_kernel(const K* __restrict__ in, K* __restrict__ out, uint64_t n,
                                                           K pivot, const uint64_t* __restrict__ pre,
                                                           const uint64_t* __restrict__ total) {
    constexpr int NW = ST_NT / 32;
    __shared__ uint32_t wc[ST_EPT][NW];
    const uint64_t t = blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t lt = lanemask_lt();
    K x[ST_EPT];
    uint32_t ball[ST_EPT];
#pragma unroll
    for (int k = 0; k < ST_EPT; ++k) {
        const uint64_t p = st_pos(t, k, tid);
        x[k] = p < n ? __ldcs(in + p) : (K)0;
    }
#pragma unroll
    for (int k = 0; k < ST_EPT; ++k) {
        ball[k] = __ballot_sync(0xffffffffu, st_pos(t, k, tid) < n && is_pred(x[k], pivot));
        if (lane == 0) wc[k][warp] = __popc(ball[k]);
    }
    __syncthreads();
    const uint64_t Tt = pre[t], Kt = *total;
    const uint64_t false_base = Kt + (t * ST_TILE - Tt);  // successors before this tile: t*TILE - Tt
    uint32_t before = 0;  // predecessors of this tile at positions before element k's row
#pragma unroll
    for (int k = 0; k < ST_EPT; ++k) {
        uint32_t wpre = 0, rowtot = 0;
#pragma unroll
        for (int w = 0; w < NW; ++w) {
            const uint32_t c = wc[k][w];
            wpre += (w < warp) ? c : 0u;
            rowtot += c;
        }
        const uint64_t p = st_pos(t, k, tid);
        if (p < n) {
            const uint32_t rt = before + wpre + __popc(ball[k] & lt);  // predecessors before p in the tile
            const uint32_t off = (uint32_t)k * ST_NT + tid;             // p - tile start
            if ((ball[k] >> lane) & 1u) __stcs(out + Tt + rt, x[k]);
            else __stcs(out + false_base + (off - rt), x[k]);
        }
        before += rowtot;
    }
}

// ---- in-place stable variant ----
template <typename K>
__global__ void __launch_bounds__(ST_NT) sti_leaf_kernel(K* __restrict__ keys, uint64_t n, K pivot,
                                                         uint64_t* __restrict__ cnt) {
    constexpr int NW = ST_NT / 32;
    __shared__ uint32_t wc[ST_EPT][NW];
    const uint64_t t = blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t lt = lanemask_lt();
    K x[ST_EPT];
    uint32_t ball[ST_EPT];
#pragma unroll
    for (int k = 0; k < ST_EPT; ++k) {
        const uint64_t p = st_pos(t, k, tid);
        x[k] = p < n ? keys[p] : (K)0;
    }
#pragma unroll
    for (int k = 0; k < ST_EPT; ++k) {
        ball[k] = __ballot_sync(0xffffffffu, st_pos(t, k, tid) < n && is_pred(x[k], pivot));
        if (lane == 0) wc[k][warp] = __popc(ball[k]);
    }
    __syncthreads();  // every key of the tile is in registers: the tile may be overwritten
    uint32_t tt = 0;  // predecessors in the tile
#pragma unroll
    for (int k = 0; k < ST_EPT; ++k)
#pragma unroll
        for (int w = 0; w < NW; ++w) tt += wc[k][w];
    const uint64_t base = t * ST_TILE;
    uint32_t before = 0;
#pragma unroll
    for (int k = 0; k < ST_EPT; ++k) {
        uint32_t wpre = 0, rowtot = 0;
#pragma unroll
        for (int w = 0; w < NW; ++w) {
            const uint32_t c = wc[k][w];
            wpre += (w < warp) ? c : 0u;
            rowtot += c;
        }
        const uint64_t p = st_pos(t, k, tid);
        if (p < n) {
            const uint32_t rt = before + wpre + __popc(ball[k] & lt);
            const uint32_t off = (uint32_t)k * ST_NT + tid;
            keys[base + (((ball[k] >> lane) & 1u) ? rt : tt + (off - rt))] = x[k];
        }
        before += rowtot;
    }
    if (tid == 0) cnt[t] = tt;
}

// Pair i of level with segment size seg: left [2i seg, +len1), right after it
// (+len2); t1, t2 their predecessor counts.  x = pair-local thread index.
template <typename K>
__global__ void __launch_bounds__(256) sti_reverse2_kernel(K* __restrict__ keys, uint64_t n, uint64_t seg,
                                                           uint64_t npairs, const uint64_t* __restrict__ cnt) {
    const uint64_t total = npairs * seg;
    for (uint64_t g = (uint64_t)blockIdx.x * 256 + threadIdx.x; g < total; g += (uint64_t)gridDim.x * 256) {
        const uint64_t i = g / seg, x = g - i * seg;
        const uint64_t s0 = 2 * i * seg, len1 = seg, len2 = min(seg, n - s0 - len1);
        const uint64_t t1 = cnt[2 * i], t2 = cnt[2 * i + 1];
        const uint64_t a = len1 - t1;  // |S1|
        if (x < a / 2) {               // reverse S1 = [s0 + t1, s0 + len1)
            K* p = keys + s0 + t1 + x;
            K* q = keys + s0 + len1 - 1 - x;
            const K u = *p, v = *q;
            *p = v;
            *q = u;
        }
        if (x < t2 / 2) {  // reverse P2 = [s0 + len1, s0 + len1 + t2)
            K* p = keys + s0 + len1 + x;
            K* q = keys + s0 + len1 + t2 - 1 - x;
            const K u = *p, v = *q;
            *p = v;
            *q = u;
        }
        (void)len2;
    }
}

template <typename K>
__global__ void __launch_bounds__(256) sti_reverse_mid_kernel(K* __restrict__ keys, uint64_t seg, uint64_t npairs,
                                                              const uint64_t* __restrict__ cnt,
                                                              uint64_t* __restrict__ cnt_next) {
    const uint64_t total = npairs * seg;
    for (uint64_t g = (uint64_t)blockIdx.x * 256 + threadIdx.x; g < total; g += (uint64_t)gridDim.x * 256) {
        const uint64_t i = g / seg, x = g - i * seg;
        const uint64_t s0 = 2 * i * seg, len1 = seg;
        const uint64_t t1 = cnt[2 * i], t2 = cnt[2 * i + 1];
        const uint64_t m = len1 - t1 + t2;  // the middle [S1 P2] (both reversed): reverse it whole
        if (x < m / 2) {
            K* p = keys + s0 + t1 + x;
            K* q = keys + s0 + t1 + m - 1 - x;
            const K u = *p, v = *q;
            *p = v;
            *q = u;
        }
        if (x == 0) cnt_next[i] = t1 + t2;
    }
}

// the unpaired last segment of a level keeps its count
__global__ void sti_carry_kernel(const uint64_t* __restrict__ cnt, uint64_t* __restrict__ cnt_next, uint64_t nseg) {
    if (threadIdx.x == 0 && (nseg & 1)) cnt_next[nseg / 2] = cnt[nseg - 1];
}

template <typename K>
pp_status partition_stable_inplace_device(K* keys, uint64_t n, K pivot, cudaStream_t st, uint64_t* d_split) {
    const uint64_t ntiles = (n + ST_TILE - 1) / ST_TILE;
    const size_t cB = (8 * (ntiles + 1) + 255) & ~size_t(255);
    unsigned char* ws = static_cast<unsigned char*>(workspace(2 * cB, st));
    if (!ws) return PP_E_NOMEM;
    uint64_t* ca = reinterpret_cast<uint64_t*>(ws);
    uint64_t* cb = reinterpret_cast<uint64_t*>(ws + cB);
    LastStats& S = last_stats();
    S = LastStats();
    S.n = n;
    S.aux_bytes = 2 * cB;
    S.path = 6;
    sti_leaf_kernel<K><<<(unsigned)ntiles, ST_NT, 0, st>>>(keys, n, pivot, ca);
    uint64_t launches = 1;
    uint64_t nseg = ntiles, seg = ST_TILE;
    const unsigned grid_cap = (unsigned)sm_count() * 16;
    while (nseg > 1) {
        const uint64_t npairs = nseg / 2;
        const unsigned grid = (unsigned)std::min<uint64_t>((npairs * seg + 255) / 256, grid_cap);
        sti_reverse2_kernel<K><<<grid, 256, 0, st>>>(keys, n, seg, npairs, ca);
        sti_reverse_mid_kernel<K><<<grid, 256, 0, st>>>(keys, seg, npairs, ca, cb);
        sti_carry_kernel<<<1, 32, 0, st>>>(ca, cb, nseg);
        launches += 3;
        std::swap(ca, cb);
        nseg = (nseg + 1) / 2;
        seg *= 2;
    }
    note_launches(launches + 1);
    cudaError_t e = cudaMemcpyAsync(d_split, ca, 8, cudaMemcpyDeviceToDevice, st);
    if (e == cudaSuccess) e = cudaGetLastError();
    return e == cudaSuccess ? PP_OK : cuda_fail(e, "stable in-place partition launch");
}
template pp_status partition_stable_inplace_device<uint64_t>(uint64_t*, uint64_t, uint64_t, cudaStream_t, uint64_t*);
template pp_status partition_stable_inplace_device<uint32_t>(uint32_t*, uint64_t, uint32_t, cudaStream_t, uint64_t*);

template <typename K>
pp_status partition_stable_device(const K* in, K* out, uint64_t n, K pivot, cudaStream_t st, uint64_t* d_split,
                                  uint64_t** total_out) {
    const uint64_t ntiles = (n + ST_TILE - 1) / ST_TILE;
    const size_t cntB = (4 * ntiles + 255) & ~size_t(255), preB = (8 * ntiles + 255) & ~size_t(255);
    unsigned char* ws = static_cast<unsigned char*>(workspace(cntB + preB + 256, st));
    if (!ws) return PP_E_NOMEM;
    uint32_t* cnt = reinterpret_cast<uint32_t*>(ws);
    uint64_t* pre = reinterpret_cast<uint64_t*>(ws + cntB);
    uint64_t* total = d_split ? d_split : reinterpret_cast<uint64_t*>(ws + cntB + preB);
    if (total_out) *total_out = total;
    LastStats& S = last_stats();
    S = LastStats();
    S.n = n;
    S.aux_bytes = cntB + preB + 256;
    S.path = 5;
    st_count_kernel<K><<<(unsigned)ntiles, ST_NT, 0, st>>>(in, n, pivot, cnt);
    st_scan_kernel<<<1, 1024, 0, st>>>(cnt, ntiles, pre, total);
    st_scatter_kernel<K><<<(unsigned)ntiles, ST_NT, 0, st>>>(in, out, n, pivot, pre, total);
    note_launches(3);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "stable partition launch");
    return PP_OK;
}

template pp_status partition_stable_device<uint64_t>(const uint64_t*, uint64_t*, uint64_t, uint64_t, cudaStream_t,
                                                     uint64_t*, uint64_t**);
template pp_status partition_stable_device<uint32_t>(const uint32_t*, uint32_t*, uint64_t, uint32_t, cudaStream_t,
                                                     uint64_t*, uint64_t**);

}  // namespace pp
