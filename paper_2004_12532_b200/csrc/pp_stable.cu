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
