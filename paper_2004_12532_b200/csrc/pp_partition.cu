// pp_partition.cu -- B200 (sm_100a) in-place parallel partition.
//
// Pipeline for one array:
//   K3 ss_group_kernel   Smoothed Striding Partial Partition Step
//                        (Fig. 3): one CTA
//                        per group U_i, a two-ended in-place partition of the
//                        group's lines staged through shared memory by the TMA
//                        bulk-copy engine; every line read once, written once.
//   K4+K1 reduce_count   every CTA reduces the group outputs: K = sum T_i,
//                        v_min, v_max and the dirty set
//                        D = head U [v_min,v_max) U tail; then per-tile
//                        misplaced counts over D (PAPER.md:288-291 D array,
//                        counted per tile like the paper's per-64/4096 chunk
//                        counts).
//   K2 tile_scan         deterministic exclusive scan of the tile counts
//                        (PAPER.md:288-297, 1488-1496).
//   K5a locate / K5b swap  rank-matched cleanup: the r-th misplaced
//                        successor left of K is swapped with the r-th
//                        misplaced predecessor right of K; each pair owned by
//                        exactly one CTA (EREW).
// No atomics anywhere; all reductions are fixed-order.  The cleanup kernels
// are chained with programmatic dependent launch (griddepcontrol).
#include <atomic>
#include <algorithm>
#include <cstdio>
#include <vector>

#include "pp_engine.cuh"

namespace pp {

template <typename C>
__global__ void __launch_bounds__(C::NT) ss_group_kernel(typename C::Key* __restrict__ region, uint64_t n_lines,
                                                         uint32_t g, uint64_t seed, typename C::Key pivot,
                                                         GroupOut* __restrict__ out) {
    extern __shared__ __align__(128) unsigned char smem[];
    griddep_wait();  // PDL launch: the previous kernel on the stream may still be finishing
    ss_group_engine<C>(region, n_lines, g, blockIdx.x, seed, pivot, out + blockIdx.x, smem);
}

// Cleanup-only path (SURVEY §7 minimum slice / ablation): K by a count pass.
template <typename K>
__global__ void __launch_bounds__(256) count_kernel(const K* __restrict__ keys, uint64_t n, K pivot,
                                                    uint64_t* __restrict__ partial) {
    __shared__ uint64_t s[8];
    uint64_t c = 0;
    for (uint64_t x = (uint64_t)blockIdx.x * 256 + threadIdx.x; x < n; x += (uint64_t)gridDim.x * 256)
        c += is_pred(keys[x], pivot) ? 1 : 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < 8; ++w) c += s[w];
        partial[blockIdx.x] = c;
    }
}

// ===========================================================================
// K4 + K1: window reduction (redundantly in every CTA; CTA 0 publishes the
// control block) fused with the tile counts over the dirty set:
//   left tiles  [t*T, min((t+1)T, Kv))      count successors (misplaced)
//   right tiles [Kv + t*T, min(.., W))       count predecessors (misplaced)
// FROM_GROUPS: K = head_T + sum T_i + tail_T from the group outputs;
// otherwise (cleanup-only path) K = sum of the count_kernel partials and
// D = [0, n).
// ===========================================================================
template <typename K, bool FROM_GROUPS>
__global__ void __launch_bounds__(256) reduce_count_kernel(const K* __restrict__ keys, uint64_t n, uint64_t h,
                                                           uint64_t n_lines, uint32_t LK,
                                                           const GroupOut* __restrict__ go, uint32_t g,
                                                           const uint64_t* __restrict__ partial, int np, K pivot,
                                                           Ctl* __restrict__ ctl, uint64_t* __restrict__ d_split,
                                                           uint32_t* __restrict__ cntL, uint32_t* __restrict__ cntR,
                                                           uint64_t max_tiles, uint32_t* __restrict__ flags,
                                                           uint32_t nflags, uint32_t* __restrict__ bm,
                                                           uint64_t bm_cap) {
    reduce_count_body<K, FROM_GROUPS>(keys, n, h, n_lines, LK, go, g, partial, np, pivot, ctl, d_split, cntL, cntR,
                                      max_tiles, blockIdx.x, gridDim.x, flags, nflags, bm, bm_cap);
}

// K2+K5 fused cleanup tail (pp_engine.cuh scan_swap_body).
// Launched cooperatively (all CTAs co-resident: the grid barrier between
// its locate and swap phases needs it).
template <typename K>
__global__ void __launch_bounds__(SW_NT, 2) scan_swap_kernel(K* __restrict__ keys, Ctl* __restrict__ ctl, K pivot,
                                                          const uint32_t* __restrict__ cntL,
                                                          const uint32_t* __restrict__ cntR,
                                                          uint32_t* __restrict__ flags,
                                                          const uint32_t* __restrict__ bm, uint64_t bm_cap) {
    extern __shared__ uint64_t ssp[];
    scan_swap_body<K>(keys, ctl, pivot, cntL, cntR, flags, bm, bm_cap, ssp, blockIdx.x, gridDim.x);
}

// ===========================================================================
// K2: exclusive scan of the tile counts (1 CTA, 1024 threads, fixed order).
// ===========================================================================
// Dynamic shared memory: 2 * (cap + 1) u64.
__global__ void __launch_bounds__(1024) tile_scan_kernel(Ctl* __restrict__ ctl, const uint32_t* __restrict__ cntL,
                                                         const uint32_t* __restrict__ cntR,
                                                         uint64_t* __restrict__ PL, uint64_t* __restrict__ PR,
                                                         uint64_t* __restrict__ rk, uint32_t* __restrict__ ttl,
                                                         uint32_t* __restrict__ ttr) {
    extern __shared__ uint64_t sp[];
    tile_scan_body(ctl, cntL, cntR, PL, PR, rk, ttl, ttr, sp);
}

// ===========================================================================
// K5a: locate the start of every swap task (one CTA per task, grid-stride).
// Tasks are the breakpoints of the merged rank boundaries of the left tiles
// (PL) and the right tiles (PR): task k covers ranks [U_k, U_{k+1}) where U
// is the sorted merge of PL[0..nL) and PR[0..nR) (duplicates kept: empty
// tasks), so each task's items lie inside ONE left tile and ONE right tile
// -- every walk is bounded by the tile size, whatever the item density.
// rk[k] = U_k (written by tile_scan with the tiles ttl[k] / ttr[k] holding
// rank U_k); posL[k] / posR[k] = virtual index of the misplaced successor /
// predecessor of rank U_k (Kv / W if U_k = M): sentinels at k = nTasks.
// ===========================================================================
template <typename K>
__global__ void __launch_bounds__(SW_NT, 3) locate_kernel(const K* __restrict__ keys, Ctl* __restrict__ ctl,
                                                          K pivot, const uint64_t* __restrict__ PL,
                                                          const uint64_t* __restrict__ PR,
                                                          uint64_t* __restrict__ posL, uint64_t* __restrict__ posR,
                                                          const uint64_t* __restrict__ rk,
                                                          const uint32_t* __restrict__ ttl,
                                                          const uint32_t* __restrict__ ttr) {
    locate_body<K>(keys, ctl, pivot, PL, PR, posL, posR, rk, ttl, ttr, blockIdx.x, gridDim.x);
}

// ===========================================================================
// K5b: rank-matched swap, one CTA per task (grid-stride).
// ===========================================================================
template <typename K>
__global__ void __launch_bounds__(SW_NT, 3) swap_kernel(K* __restrict__ keys, const Ctl* __restrict__ ctl, K pivot,
                                                     const uint64_t* __restrict__ posL,
                                                     const uint64_t* __restrict__ posR,
                                                     const uint64_t* __restrict__ rk) {
    swap_body<K>(keys, ctl, pivot, posL, posR, rk, blockIdx.x, gridDim.x);
}

// ===========================================================================
// Single-CTA path for small n: count, then one walk over [0,K) x [K,n).
// ===========================================================================
template <typename K>
__global__ void __launch_bounds__(SW_NT) small_partition_kernel(K* __restrict__ keys, uint64_t n, K pivot,
                                                                Ctl* __restrict__ ctl,
                                                                uint64_t* __restrict__ d_split) {
    __shared__ StreamBuf<SW_NT, SW_EPT2> sb;
    __shared__ uint64_t sK[SW_NT / 32];
    uint64_t c = 0;
    for (uint64_t x = threadIdx.x; x < n; x += SW_NT) c += is_pred(keys[x], pivot) ? 1 : 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0) sK[threadIdx.x >> 5] = c;
    __syncthreads();
    uint64_t Ksplit = 0;
    for (int w = 0; w < SW_NT / 32; ++w) Ksplit += sK[w];
    Dirty d;
    d.s[0] = 0; d.l[0] = n;
    d.s[1] = d.s[2] = n; d.l[1] = d.l[2] = 0;
    walk_swap_stream<K, SW_NT, SW_EPT2>(keys, d, pivot, 0, Ksplit, Ksplit, n, sb);
    if (threadIdx.x == 0) {
        if (ctl) {
            uint64_t a[3] = {0, n, n}, b[3] = {n, n, n};
            finish_ctl(ctl, n, Ksplit, a, b);
            ctl->vmin = 0;
            ctl->vmax = n;
        }
        if (d_split) *d_split = Ksplit;
    }
}

// ===========================================================================
// Host driver.
// ===========================================================================
static std::atomic<uint64_t> g_launches{0};
uint64_t launch_count(int reset) {
    return reset ? g_launches.exchange(0) : g_launches.load();
}
void note_launches(uint64_t k) { g_launches += k; }

// launch with programmatic stream serialization (the kernel calls
// griddep_wait() before touching its predecessor's results)
template <typename... KArgs, typename... Args>
static cudaError_t launch_pdl_smem(void (*kern)(KArgs...), unsigned grid, unsigned block, size_t smem,
                                   cudaStream_t st, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    note_launches(1);
    return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}
template <typename... KArgs, typename... Args>
static cudaError_t launch_pdl(void (*kern)(KArgs...), unsigned grid, unsigned block, cudaStream_t st,
                              Args... args) {
    return launch_pdl_smem(kern, grid, block, 0, st, args...);
}

// Optional per-call phase timing with CUDA events recorded on the launch
// stream (bench.py's roofline: the group kernel's live duration).
static bool g_timing = false;
static std::vector<cudaEvent_t> g_ev_pool;
static size_t g_ev_used = 0;
static cudaEvent_t timing_event() {
    if (g_ev_used == g_ev_pool.size()) {
        cudaEvent_t e;
        cudaEventCreate(&e);
        g_ev_pool.push_back(e);
    }
    return g_ev_pool[g_ev_used++];
}
static void timing_mark(cudaStream_t st) {
    if (g_timing) cudaEventRecord(timing_event(), st);
}
void timing_enable(int on) {
    g_timing = on != 0;
    g_ev_used = 0;
}
// out = {calls, group_ms, rest_ms, total_ms}; events come in triples per call
int timing_read(double* out) {
    out[0] = out[1] = out[2] = out[3] = 0;
    if (g_ev_used % 3) return 1;
    for (size_t i = 0; i + 2 < g_ev_used; i += 3) {
        float a = 0, b = 0;
        if (cudaEventSynchronize(g_ev_pool[i + 2]) != cudaSuccess) return 2;
        cudaEventElapsedTime(&a, g_ev_pool[i], g_ev_pool[i + 1]);
        cudaEventElapsedTime(&b, g_ev_pool[i + 1], g_ev_pool[i + 2]);
        out[0] += 1;
        out[1] += a;
        out[2] += b;
        out[3] += a + b;
    }
    g_ev_used = 0;
    return 0;
}

// ---------------------------------------------------------------------------
// Group-kernel instantiations: the default and the Strided Algorithm (X = 0).
// (Line sizes 4-8 KiB, 64-256 threads, 3-6 lines in flight, TMA stores and
// parallel refill issue were measured in round 1 -- tools/tune.py -- and the
// default is the fastest; the alternatives were removed.)
// ---------------------------------------------------------------------------
template <typename C>
static int occupancy_of() {
    static int occ = -1;
    if (occ < 0) {
        cudaFuncSetAttribute(ss_group_kernel<C>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
        int o = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, ss_group_kernel<C>, C::NT, C::SMEM);
        occ = o > 0 ? o : 1;
    }
    return occ;
}

struct VariantInfo {
    uint64_t LK;
    int occ;
};

template <typename K, int V>
struct VariantCfg;
// 0: the default configuration (pp_group.cuh PartGroupCfg)
template <typename K> struct VariantCfg<K, 0> { using type = PartGroupCfg<K>; };
// 1: the same with X = 0 (the Strided Algorithm), selected by
// the "strided" param (seed 0): a separate instantiation, since a runtime
// branch on the seed made the compiler unswitch the whole engine (-7%)
template <typename K> struct VariantCfg<K, 1> {
    using D = PartGroupCfg<K>;
    using type = GroupCfgT<K, D::LK * (int)sizeof(K), D::NT, D::PF, D::TMA_STORE, true, D::PAR_ISSUE>;
};
constexpr int STRIDED_VARIANT = 1;

template <typename K, int V>
static VariantInfo variant_info_t() {
    using C = typename VariantCfg<K, V>::type;
    return {(uint64_t)C::LK, occupancy_of<C>()};
}
template <typename K>
static VariantInfo variant_info(int v) {
    return v == STRIDED_VARIANT ? variant_info_t<K, STRIDED_VARIANT>() : variant_info_t<K, 0>();
}
template <typename K, int V>
static void launch_group_t(K* region, uint64_t n_lines, uint32_t g, uint64_t seed, K pivot, GroupOut* out,
                           cudaStream_t st) {
    using C = typename VariantCfg<K, V>::type;
    occupancy_of<C>();
    // plain launch: with programmatic dependent launch the group CTAs became
    // resident while the previous call's cooperative cleanup still held SMs,
    // placing them unevenly -- the group kernel ran ~4% slower at 2^27 keys
    // (measured; its griddep_wait() is then a no-op)
    ss_group_kernel<C><<<g, C::NT, C::SMEM, st>>>(region, n_lines, g, seed, pivot, out);
    note_launches(1);
}
template <typename K>
static void launch_group(int v, K* region, uint64_t n_lines, uint32_t g, uint64_t seed, K pivot, GroupOut* out,
                         cudaStream_t st) {
    if (v == STRIDED_VARIANT)
        launch_group_t<K, STRIDED_VARIANT>(region, n_lines, g, seed, pivot, out, st);
    else
        launch_group_t<K, 0>(region, n_lines, g, seed, pivot, out, st);
}

static int cur_variant() { return params().seed == 0 ? STRIDED_VARIANT : 0; }  // "strided" param: X = 0

struct Layout {
    size_t ctl, gout, cntL, cntR, PL, PR, posL, posR, rk, ttl, ttr, partial, flags, bm, total;
};
constexpr uint64_t MAX_BARRIER_CTAS = 4096;  // grid-barrier flags of the fused cleanup tail

// Workspace: fixed-size cleanup arrays (cleanup_max_tiles(n) per side, the
// tile size adapts to the dirty set on the device) + one GroupOut per group:
// the auxiliary memory does not grow with n beyond the g <= #SM x occupancy
// groups and the <= 8192 tiles per side.
static Layout make_layout(uint64_t n, uint64_t g, bool cleanup, uint64_t nPartial) {
    const uint64_t maxTiles = cleanup ? cleanup_max_tiles(n) + 1 : 1;
    const uint64_t maxTasks = cleanup ? 2 * cleanup_max_tiles(n) + 1 : 1;
    Layout L;
    size_t o = 0;
    auto take = [&](size_t bytes) {
        size_t at = o;
        o += (bytes + 255) & ~size_t(255);
        return at;
    };
    L.ctl = take(sizeof(Ctl));
    L.gout = take(sizeof(GroupOut) * std::max<uint64_t>(g, 1));
    L.cntL = take(4 * maxTiles);
    L.cntR = take(4 * maxTiles);
    L.PL = take(8 * maxTiles);
    L.PR = take(8 * maxTiles);
    L.posL = take(8 * (maxTasks + 1));
    L.posR = take(8 * (maxTasks + 1));
    L.rk = take(8 * (maxTasks + 1));
    L.ttl = take(4 * (maxTasks + 1));
    L.ttr = take(4 * (maxTasks + 1));
    L.partial = take(8 * nPartial);
    L.flags = take(4 * MAX_BARRIER_CTAS);
    L.bm = take(cleanup ? 4 * 2 * bm_side_words(fused_bm_cap(n)) : 4);
    L.total = o;
    return L;
}

template <typename K>
static uint64_t choose_groups(uint64_t n_lines, int occ) {
    const Params& P = params();
    if (P.g > 0) return std::min<uint64_t>((uint64_t)P.g, std::max<uint64_t>(n_lines, 1));
    const uint64_t cap = (uint64_t)sm_count() * occ;
    uint64_t g = n_lines / (uint64_t)std::max<int64_t>(P.min_lines_per_group, 1);
    // small arrays are latency-bound: at least one group per SM while every
    // group keeps >= 2 lines (measured at 2^18-2^20 keys: 10-15% faster)
    g = std::max<uint64_t>(g, std::min<uint64_t>((uint64_t)sm_count(), n_lines / 2));
    return std::max<uint64_t>(1, std::min(g, cap));
}

// The fused cleanup tail runs on a co-resident grid (cooperative launch):
// #SM x its occupancy, capped so every CTA has <= FUSED_TASKS_PER_CTA tasks.
static constexpr size_t SCAN_SWAP_SMEM = 2 * 8 * (FUSED_MAX_TILES + 1);
static uint32_t fused_tail_grid() {
    static uint32_t G = 0;
    if (!G) {
        int occ = 0;
        cudaFuncSetAttribute(scan_swap_kernel<uint64_t>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)SCAN_SWAP_SMEM);
        cudaFuncSetAttribute(scan_swap_kernel<uint32_t>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)SCAN_SWAP_SMEM);
        int o64 = 0, o32 = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o64, scan_swap_kernel<uint64_t>, SW_NT, SCAN_SWAP_SMEM);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o32, scan_swap_kernel<uint32_t>, SW_NT, SCAN_SWAP_SMEM);
        occ = std::max(1, std::min(o64, o32));
        G = (uint32_t)std::min<uint64_t>((uint64_t)sm_count() * (uint64_t)occ, MAX_BARRIER_CTAS);
        static_assert(2 * FUSED_MAX_TILES <= 148 * (uint64_t)FUSED_TASKS_PER_CTA, "task slots per CTA");
    }
    return G;
}

template <typename K>
static cudaError_t launch_scan_swap(uint32_t G, cudaStream_t st, K* keys, Ctl* ctl, K pivot, const uint32_t* cntL,
                                    const uint32_t* cntR, uint32_t* flags, const uint32_t* bm, uint64_t bm_cap) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(G);
    cfg.blockDim = dim3(SW_NT);
    cfg.dynamicSmemBytes = SCAN_SWAP_SMEM;
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    note_launches(1);
    cudaError_t e = cudaLaunchKernelEx(&cfg, scan_swap_kernel<K>, keys, ctl, pivot, cntL, cntR, flags, bm, bm_cap);
    if (e != cudaSuccess) {  // cooperative + programmatic serialization refused: plain cooperative
        cudaGetLastError();
        cfg.numAttrs = 1;
        e = cudaLaunchKernelEx(&cfg, scan_swap_kernel<K>, keys, ctl, pivot, cntL, cntR, flags, bm, bm_cap);
    }
    return e;
}

template <typename K>
pp_status partition_device(K* keys, uint64_t n, K pivot, cudaStream_t st, uint64_t* d_split, Ctl** ctl_out) {
    const Params& P = params();
    const int variant = cur_variant();
    const VariantInfo vi = variant_info<K>(variant);
    const uint64_t LK = vi.LK;
    LastStats& S = last_stats();
    S = LastStats();
    S.n = n;
    S.line_keys = LK;
    const uint64_t addr = (uint64_t)(uintptr_t)keys;
    uint64_t h = ((16 - (addr & 15)) & 15) / sizeof(K);
    if (h > n) h = n;
    const uint64_t n_lines = (n - h) / LK;

    int path = (int)P.path;
    if (path == 0) path = (n < (uint64_t)P.small_n || n_lines < 2) ? 1 : 2;
    if (path == 2 && n_lines == 0) path = 1;
    S.path = path;

    const unsigned grid_cleanup = (unsigned)sm_count() * 4;
    const uint64_t g = path == 2 ? choose_groups<K>(n_lines, vi.occ) : 0;
    const int nPartial = sm_count() * 2;
    Layout L = make_layout(n, g, path != 1, nPartial);
    unsigned char* ws = static_cast<unsigned char*>(workspace(L.total, st));
    if (!ws) return PP_E_NOMEM;
    Ctl* ctl = reinterpret_cast<Ctl*>(ws + L.ctl);
    if (ctl_out) *ctl_out = ctl;
    S.g = g;
    S.head = h;
    S.n_lines = n_lines;
    S.aux_bytes = L.total;

    cudaError_t e = cudaSuccess;
    timing_mark(st);
    if (path == 1) {
        small_partition_kernel<K><<<1, SW_NT, 0, st>>>(keys, n, pivot, ctl, d_split);
        note_launches(1);
        timing_mark(st);
    } else {
        GroupOut* gout = reinterpret_cast<GroupOut*>(ws + L.gout);
        uint64_t* partial = reinterpret_cast<uint64_t*>(ws + L.partial);
        uint32_t* cntL = reinterpret_cast<uint32_t*>(ws + L.cntL);
        uint32_t* cntR = reinterpret_cast<uint32_t*>(ws + L.cntR);
        uint64_t* PL = reinterpret_cast<uint64_t*>(ws + L.PL);
        uint64_t* PR = reinterpret_cast<uint64_t*>(ws + L.PR);
        uint64_t* posL = reinterpret_cast<uint64_t*>(ws + L.posL);
        uint64_t* posR = reinterpret_cast<uint64_t*>(ws + L.posR);
        uint64_t* rk = reinterpret_cast<uint64_t*>(ws + L.rk);
        uint32_t* ttl = reinterpret_cast<uint32_t*>(ws + L.ttl);
        uint32_t* ttr = reinterpret_cast<uint32_t*>(ws + L.ttr);
        // cleanup tail: fused scan+locate+barrier+swap (default) or the 3-kernel chain
        // (the fused tail needs a grid with <= FUSED_TASKS_PER_CTA tasks per CTA)
        // auto: the 3-kernel chain below 1 GiB of keys, the fused tail from
        // 1 GiB (measured crossover between 2^26 and 2^27 u64 keys)
        const bool want_fused =
            P.cleanup_chain == 0 || (P.cleanup_chain < 0 && n * sizeof(K) >= (uint64_t(1) << 30));
        const bool fused_tail =
            want_fused && (uint64_t)fused_tail_grid() * FUSED_TASKS_PER_CTA >= 2 * FUSED_MAX_TILES;
        const uint64_t max_tiles = fused_tail ? std::min<uint64_t>(cleanup_max_tiles(n), FUSED_MAX_TILES) : 0;
        const uint32_t nflags = fused_tail ? fused_tail_grid() : 0;
        uint32_t* flags = reinterpret_cast<uint32_t*>(ws + L.flags);
        uint32_t* bm = fused_tail && P.cleanup_bitmap ? reinterpret_cast<uint32_t*>(ws + L.bm) : nullptr;
        const uint64_t bm_cap = fused_bm_cap(n);
        if (path == 2) {
            launch_group<K>(variant, keys + h, n_lines, (uint32_t)g, P.seed, pivot, gout, st);
            timing_mark(st);
            e = launch_pdl(reduce_count_kernel<K, true>, grid_cleanup, 256, st, keys, n, h, n_lines, (uint32_t)LK,
                           gout, (uint32_t)g, partial, nPartial, pivot, ctl, d_split, cntL, cntR, max_tiles, flags,
                           nflags, bm, bm_cap);
        } else {
            count_kernel<K><<<nPartial, 256, 0, st>>>(keys, n, pivot, partial);
            note_launches(1);
            timing_mark(st);
            e = launch_pdl(reduce_count_kernel<K, false>, grid_cleanup, 256, st, keys, n, (uint64_t)0, (uint64_t)0,
                           (uint32_t)LK, gout, (uint32_t)0, partial, nPartial, pivot, ctl, d_split, cntL, cntR,
                           max_tiles, flags, nflags, bm, bm_cap);
        }
        if (fused_tail) {
            if (e == cudaSuccess) e = launch_scan_swap<K>(nflags, st, keys, ctl, pivot, cntL, cntR, flags, bm, bm_cap);
        } else {
            const size_t scan_smem = 2 * 8 * (cleanup_max_tiles(n) + 1);
            static size_t scan_smem_set = 0;
            if (scan_smem > 48 * 1024 && scan_smem > scan_smem_set) {
                cudaFuncSetAttribute(tile_scan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)scan_smem);
                scan_smem_set = scan_smem;
            }
            if (e == cudaSuccess)
                e = launch_pdl_smem(tile_scan_kernel, 1, 1024, scan_smem, st, ctl, cntL, cntR, PL, PR, rk, ttl, ttr);
            if (e == cudaSuccess)
                e = launch_pdl(locate_kernel<K>, grid_cleanup, SW_NT, st, keys, ctl, pivot, PL, PR, posL, posR, rk,
                               ttl, ttr);
            if (e == cudaSuccess)
                e = launch_pdl(swap_kernel<K>, grid_cleanup, SW_NT, st, keys, ctl, pivot, posL, posR, rk);
        }
    }
    timing_mark(st);
    if (e != cudaSuccess) return cuda_fail(e, "partition launch");
    e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "partition launch");
    return PP_OK;
}

template <typename K>
pp_status ss_groups_device(K* keys, uint64_t n, K pivot, uint64_t g_req, cudaStream_t st, uint64_t* T_host,
                           uint64_t* vlo_host, uint64_t* vhi_host, uint64_t* info) {
    const int variant = cur_variant();
    const VariantInfo vi = variant_info<K>(variant);
    const uint64_t addr = (uint64_t)(uintptr_t)keys;
    uint64_t h = ((16 - (addr & 15)) & 15) / sizeof(K);
    if (h > n) h = n;
    const uint64_t n_lines = (n - h) / vi.LK;
    const uint64_t g = g_req > 0 ? g_req : choose_groups<K>(n_lines, vi.occ);
    info[0] = g;
    info[1] = h;
    info[2] = n_lines;
    info[3] = vi.LK;
    info[4] = params().seed;
    info[5] = (uint64_t)variant;
    if (n_lines == 0) return PP_OK;
    GroupOut* gout = static_cast<GroupOut*>(workspace(sizeof(GroupOut) * g, st));
    if (!gout) return PP_E_NOMEM;
    launch_group<K>(variant, keys + h, n_lines, (uint32_t)g, params().seed, pivot, gout, st);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "ss_group launch");
    std::vector<GroupOut> host(g);
    e = cudaMemcpyAsync(host.data(), gout, sizeof(GroupOut) * g, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return cuda_fail(e, "ss_group readback");
    for (uint64_t i = 0; i < g; ++i) {
        T_host[i] = host[i].T;
        vlo_host[i] = host[i].vlo;
        vhi_host[i] = host[i].vhi;
    }
    return PP_OK;
}

uint64_t max_groups() {
    int occ = 1;
    for (int v : {0, STRIDED_VARIANT}) {
        occ = std::max(occ, variant_info<uint64_t>(v).occ);
        occ = std::max(occ, variant_info<uint32_t>(v).occ);
    }
    return (uint64_t)sm_count() * (uint64_t)occ;
}

// Largest make_layout any partition_device / ss_groups_device call on <= n
// keys requests: g <= max(max_groups(), min(param g, n)), the cleanup arrays
// grow monotonically with n (cleanup_max_tiles).
uint64_t partition_workspace_bound(uint64_t n) {
    const Params& P = params();
    uint64_t g = max_groups();
    if (P.g > 0) g = std::max<uint64_t>(g, std::min<uint64_t>((uint64_t)P.g, n));
    return make_layout(n, g, true, (uint64_t)sm_count() * 2).total;
}

template pp_status partition_device<uint64_t>(uint64_t*, uint64_t, uint64_t, cudaStream_t, uint64_t*, Ctl**);
template pp_status partition_device<uint32_t>(uint32_t*, uint64_t, uint32_t, cudaStream_t, uint64_t*, Ctl**);
template pp_status ss_groups_device<uint64_t>(uint64_t*, uint64_t, uint64_t, uint64_t, cudaStream_t, uint64_t*,
                                              uint64_t*, uint64_t*, uint64_t*);
template pp_status ss_groups_device<uint32_t>(uint32_t*, uint64_t, uint32_t, uint64_t, cudaStream_t, uint64_t*,
                                              uint64_t*, uint64_t*, uint64_t*);

// EREW shadow-writer audit (libpp_audit.so only): point this translation
// unit's kernels (the partition pipeline) at a counter array; nullptr stops it.
pp_status audit_set_partition(uint32_t* shadow, const void* base, uint64_t n, uint32_t key_bytes) {
#if PP_AUDIT
    AuditState a{shadow, (uint64_t)(uintptr_t)base, n, key_bytes};
    const cudaError_t e = cudaMemcpyToSymbol(g_audit, &a, sizeof(a));
    return e == cudaSuccess ? PP_OK : cuda_fail(e, "audit state");
#else
    (void)shadow; (void)base; (void)n; (void)key_bytes;
    set_error("pp_audit_set: this is the product library; the EREW audit lives in libpp_audit.so");
    return PP_E_INVAL;
#endif
}

}  // namespace pp
