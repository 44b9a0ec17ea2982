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
// Fused single-kernel partition (default path): ONE cooperative launch runs
// the group partition and the whole cleanup; the phases are separated by a
// flag-array grid barrier (each CTA release-stores its own flag, then
// acquire-polls all flags: no atomics).  Phases after the group step reuse
// the group engine's shared memory.  Cleanup tiles are NT*EPT = 1024 keys
// (one round trip per side), <= FU_MAX_TILES per side.
// ===========================================================================
constexpr int FU_EPT = 8;
constexpr uint64_t FU_MAX_TILES = 4096;

template <typename K>
struct FusedArgs {
    K* keys;
    uint64_t n, h, n_lines, seed;
    uint32_t g, epoch, stop;  // stop: debug, return after phase `stop` (0 = run all)
    K pivot;
    GroupOut* gout;
    Ctl* ctl;
    uint64_t* d_split;
    uint32_t *cntL, *cntR, *ttl, *ttr, *flags;
    uint64_t *PL, *PR, *rk, *posL, *posR;
};

__device__ __forceinline__ void grid_sync(uint32_t* flags, uint32_t nb, uint32_t epoch) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        st_release_gpu(flags + blockIdx.x, epoch);
    }
    for (uint32_t i = threadIdx.x; i < nb; i += blockDim.x)
        while ((int32_t)(ld_acquire_gpu(flags + i) - epoch) < 0) __nanosleep(64);
    __threadfence();
    __syncthreads();
}

template <typename C>
__global__ void __launch_bounds__(C::NT) fused_partition_kernel(const FusedArgs<typename C::Key> a) {
    using K = typename C::Key;
    constexpr int NT = C::NT, NW = NT / 32, EPT = FU_EPT, RNG = NT * EPT;
    extern __shared__ __align__(128) unsigned char smem[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint64_t LK = C::LK;

    // ---- phase 1: Smoothed Striding group partition ----
    ss_group_engine<C>(a.keys + a.h, a.n_lines, a.g, blockIdx.x, a.seed, a.pivot, a.gout + blockIdx.x, smem);
    if (a.stop == 1) return;
    grid_sync(a.flags, a.g, a.epoch + 1);

    // ---- phase 2: window reduction (every CTA) + tile counts ----
    Ctl* sc = reinterpret_cast<Ctl*>(smem);
    uint64_t* red = reinterpret_cast<uint64_t*>(smem + 512);    // [4][NW]
    uint32_t* s32 = reinterpret_cast<uint32_t*>(smem + 1536);   // [NW]
    unsigned char* work = smem + 2048;                          // phase buffers
    const uint64_t region_end = a.n_lines * LK;
    {
        uint64_t T = 0, vmin = region_end, vmax = 0, ht = 0;
        for (uint32_t i = tid; i < a.g; i += NT) {
            T += __ldcg(&a.gout[i].T);
            const uint64_t lo = __ldcg(&a.gout[i].vlo), hi = __ldcg(&a.gout[i].vhi);
            vmin = lo < vmin ? lo : vmin;
            vmax = hi > vmax ? hi : vmax;
        }
        for (uint64_t x = tid; x < a.h; x += NT) ht += is_pred(__ldcg(a.keys + x), a.pivot) ? 1 : 0;
        for (uint64_t x = a.h + region_end + tid; x < a.n; x += NT) ht += is_pred(__ldcg(a.keys + x), a.pivot) ? 1 : 0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            T += __shfl_xor_sync(0xffffffffu, T, o);
            ht += __shfl_xor_sync(0xffffffffu, ht, o);
            const uint64_t p = __shfl_xor_sync(0xffffffffu, vmin, o), q = __shfl_xor_sync(0xffffffffu, vmax, o);
            vmin = p < vmin ? p : vmin;
            vmax = q > vmax ? q : vmax;
        }
        if (lane == 0) {
            red[0 * NW + warp] = T;
            red[1 * NW + warp] = ht;
            red[2 * NW + warp] = vmin;
            red[3 * NW + warp] = vmax;
        }
        __syncthreads();
        if (tid == 0) {
            for (int w = 1; w < NW; ++w) {
                T += red[0 * NW + w];
                ht += red[1 * NW + w];
                vmin = red[2 * NW + w] < vmin ? red[2 * NW + w] : vmin;
                vmax = red[3 * NW + w] > vmax ? red[3 * NW + w] : vmax;
            }
            const uint64_t Ksplit = T + ht;
            uint64_t lo[3], hi[3];
            lo[0] = 0; hi[0] = a.h;
            const uint64_t wlo = a.h + vmin, whi = a.h + vmax;
            lo[1] = wlo < Ksplit ? wlo : Ksplit;
            hi[1] = whi > Ksplit ? whi : Ksplit;
            if (vmin > vmax) { lo[1] = hi[1] = 0; }
            lo[2] = a.h + region_end; hi[2] = a.n;
            const uint64_t cap = cleanup_max_tiles(a.n) < FU_MAX_TILES ? cleanup_max_tiles(a.n) : FU_MAX_TILES;
            finish_ctl(sc, a.n, Ksplit, lo, hi, (uint64_t)RNG, cap);
            sc->vmin = wlo;
            sc->vmax = whi;
            if (blockIdx.x == 0) {
                *a.ctl = *sc;
                if (a.d_split) *a.d_split = Ksplit;
            }
        }
        __syncthreads();
    }
    Dirty d;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        d.s[k] = sc->ds[k];
        d.l[k] = sc->dl[k];
    }
    const uint64_t Kv = sc->Kv, W = sc->W, TT = sc->tile, nL = sc->nL, nR = sc->nR;
    for (uint64_t t = blockIdx.x; t < nL + nR; t += gridDim.x) {
        const bool left = t < nL;
        const uint64_t u0 = left ? t * TT : Kv + (t - nL) * TT;
        const uint64_t u1 = left ? min(u0 + TT, Kv) : min(u0 + TT, W);
        uint32_t c = 0;
        for (uint64_t ub = u0; ub < u1; ub += (uint64_t)EPT * NT) {
            K x[EPT];
#pragma unroll
            for (int k = 0; k < EPT; ++k) {
                const uint64_t u = ub + (uint64_t)k * NT + tid;
                x[k] = u < u1 ? __ldcg(a.keys + vreal(d, u)) : (K)0;
            }
#pragma unroll
            for (int k = 0; k < EPT; ++k) {
                const uint64_t u = ub + (uint64_t)k * NT + tid;
                const bool p = is_pred(x[k], a.pivot);
                c += (u < u1 && (left ? !p : p)) ? 1u : 0u;
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
        if (lane == 0) s32[warp] = c;
        __syncthreads();
        if (tid == 0) {
            uint32_t tot = 0;
            for (int w = 0; w < NW; ++w) tot += s32[w];
            if (left) a.cntL[t] = tot; else a.cntR[t - nL] = tot;
        }
        __syncthreads();
    }
    if (a.stop == 2) return;
    grid_sync(a.flags, a.g, a.epoch + 2);

    // ---- phase 3 (CTA 0): scans + merged task list ----
    if (blockIdx.x == 0) {
        uint64_t* sw = reinterpret_cast<uint64_t*>(smem + 1024);  // [NW]
        uint64_t* sPL = reinterpret_cast<uint64_t*>(work);
        uint64_t* sPR = sPL + nL;
        uint64_t carry = 0;
        for (uint64_t b = 0; b < nL; b += NT) {
            const uint64_t i = b + tid;
            uint64_t tot;
            const uint64_t ex = block_exscan<NT>(i < nL ? __ldcg(a.cntL + i) : 0, sw, tot);
            if (i < nL) a.PL[i] = sPL[i] = carry + ex;
            carry += tot;
        }
        const uint64_t ML = carry;
        carry = 0;
        for (uint64_t b = 0; b < nR; b += NT) {
            const uint64_t i = b + tid;
            uint64_t tot;
            const uint64_t ex = block_exscan<NT>(i < nR ? __ldcg(a.cntR + i) : 0, sw, tot);
            if (i < nR) a.PR[i] = sPR[i] = carry + ex;
            carry += tot;
        }
        __syncthreads();
        const bool ok = (ML == carry && ML > 0);
        if (ok) {
            for (uint64_t t = tid; t < nL; t += NT) {
                const uint64_t r = sPL[t];
                const uint64_t m = t + lower_bound_u64(sPR, nR, r);
                a.rk[m] = r;
                a.ttl[m] = (uint32_t)t;
                a.ttr[m] = (uint32_t)(upper_bound_u64(sPR, nR, r) - 1);
            }
            for (uint64_t t = tid; t < nR; t += NT) {
                const uint64_t r = sPR[t];
                const uint64_t ub = upper_bound_u64(sPL, nL, r);
                const uint64_t m = t + ub;
                a.rk[m] = r;
                a.ttl[m] = (uint32_t)(ub - 1);
                a.ttr[m] = (uint32_t)t;
            }
        }
        if (tid == 0) {
            a.ctl->ML = ML;
            a.ctl->MR = carry;
            if (ML != carry) a.ctl->err = 1;
            a.ctl->nTasks = ok ? nL + nR : 0;
            a.rk[ok ? nL + nR : 0] = ML;
        }
    }
    if (a.stop == 3) return;
    grid_sync(a.flags, a.g, a.epoch + 3);

    // ---- phase 4: locate the first item of every task ----
    const uint64_t nTasks = __ldcg(&a.ctl->nTasks), M = __ldcg(&a.ctl->ML);
    {
        PairBuf<K, NT, EPT>& pb = *reinterpret_cast<PairBuf<K, NT, EPT>*>(work);
        for (uint64_t j = blockIdx.x; j <= nTasks; j += gridDim.x) {
            const uint64_t r = __ldcg(a.rk + j);
            uint64_t pl = Kv, pr = W;
            if (j < nTasks && r < M) {
                const uint64_t tl = __ldcg(a.ttl + j), tr = __ldcg(a.ttr + j);
                select_pair<K, NT, EPT>(a.keys, d, a.pivot, tl * TT, min(tl * TT + TT, Kv), r - __ldcg(a.PL + tl),
                                        Kv + tr * TT, min(Kv + tr * TT + TT, W), r - __ldcg(a.PR + tr), pb, pl,
                                        pr);
            }
            if (tid == 0) {
                a.posL[j] = pl;
                a.posR[j] = pr;
            }
        }
    }
    if (a.stop == 4) return;
    grid_sync(a.flags, a.g, a.epoch + 4);

    // ---- phase 5: rank-matched swaps ----
    for (uint64_t j = blockIdx.x; j < nTasks; j += gridDim.x) {
        const uint64_t pairs = __ldcg(a.rk + j + 1) - __ldcg(a.rk + j);
        if (pairs == 0) continue;
        const uint64_t uL = __ldcg(a.posL + j), uR = __ldcg(a.posR + j);
        const uint64_t tle = min((uL / TT + 1) * TT, Kv), tre = min(Kv + ((uR - Kv) / TT + 1) * TT, W);
        const uint64_t eL = min(__ldcg(a.posL + j + 1), tle), eR = min(__ldcg(a.posR + j + 1), tre);
        if (TT == (uint64_t)RNG) {
            swap_pair<K, NT, EPT>(a.keys, d, a.pivot, uL, eL, uR, eR, pairs,
                                  *reinterpret_cast<PairBuf<K, NT, EPT>*>(work));
        } else {
            walk_swap_stream<K, NT, EPT>(a.keys, d, a.pivot, uL, eL, uR, eR,
                                         *reinterpret_cast<StreamBuf<NT, EPT>*>(work));
        }
    }
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
// Group-kernel variants (line size, threads, prefetch depth, store path),
// selectable with pp_set_param("variant", v) for tuning; 0 is the default.
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
template <typename K> struct VariantCfg<K, 0> { using type = GroupCfg<K>; };
template <typename K> struct VariantCfg<K, 1> { using type = GroupCfgT<K, 8192, 256, 4, false>; };
template <typename K> struct VariantCfg<K, 2> { using type = GroupCfgT<K, 4096, 128, 4, false>; };
template <typename K> struct VariantCfg<K, 3> { using type = GroupCfgT<K, 8192, 64, 4, false>; };
template <typename K> struct VariantCfg<K, 4> { using type = GroupCfgT<K, 8192, 128, 3, false>; };
template <typename K> struct VariantCfg<K, 5> { using type = GroupCfgT<K, 4096, 64, 6, false>; };
template <typename K> struct VariantCfg<K, 6> { using type = GroupCfgT<K, 8192, 128, 4, true>; };
// 7: the default configuration with X = 0 (Strided Algorithm), selected by
// the "strided" param (seed 0), not by "variant"
template <typename K> struct VariantCfg<K, 7> {
    using D = GroupCfg<K>;
    using type = GroupCfgT<K, D::LK * (int)sizeof(K), D::NT, D::PF, D::TMA_STORE, true, D::PAR_ISSUE>;
};
// 8: 8 KiB lines, 128 threads, 4 in flight per end, parallel refill issue
template <typename K> struct VariantCfg<K, 8> { using type = GroupCfgT<K, 8192, 128, 4, false, false, true>; };
// 9: 4 KiB lines, 256 threads, parallel refill issue
template <typename K> struct VariantCfg<K, 9> { using type = GroupCfgT<K, 4096, 256, 4, false, false, true>; };
constexpr int N_VARIANTS = 10;
constexpr int STRIDED_VARIANT = 7;

template <typename K, int V>
static VariantInfo variant_info_t() {
    using C = typename VariantCfg<K, V>::type;
    return {(uint64_t)C::LK, occupancy_of<C>()};
}
template <typename K>
static VariantInfo variant_info(int v) {
    switch (v) {
        case 1: return variant_info_t<K, 1>();
        case 2: return variant_info_t<K, 2>();
        case 3: return variant_info_t<K, 3>();
        case 4: return variant_info_t<K, 4>();
        case 5: return variant_info_t<K, 5>();
        case 6: return variant_info_t<K, 6>();
        case 7: return variant_info_t<K, 7>();
        case 8: return variant_info_t<K, 8>();
        case 9: return variant_info_t<K, 9>();
        default: return variant_info_t<K, 0>();
    }
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
    switch (v) {
        case 1: launch_group_t<K, 1>(region, n_lines, g, seed, pivot, out, st); break;
        case 2: launch_group_t<K, 2>(region, n_lines, g, seed, pivot, out, st); break;
        case 3: launch_group_t<K, 3>(region, n_lines, g, seed, pivot, out, st); break;
        case 4: launch_group_t<K, 4>(region, n_lines, g, seed, pivot, out, st); break;
        case 5: launch_group_t<K, 5>(region, n_lines, g, seed, pivot, out, st); break;
        case 6: launch_group_t<K, 6>(region, n_lines, g, seed, pivot, out, st); break;
        case 7: launch_group_t<K, 7>(region, n_lines, g, seed, pivot, out, st); break;
        case 8: launch_group_t<K, 8>(region, n_lines, g, seed, pivot, out, st); break;
        case 9: launch_group_t<K, 9>(region, n_lines, g, seed, pivot, out, st); break;
        default: launch_group_t<K, 0>(region, n_lines, g, seed, pivot, out, st); break;
    }
}

// Grid-barrier flags of the fused kernel: one u32 per CTA, zeroed once;
// every launch uses 4 fresh epochs (monotone, compared wrap-safely).
static uint32_t* g_flags = nullptr;
static uint64_t g_flags_cap = 0;
static uint32_t g_epoch = 0;
static uint32_t* grid_flags(uint64_t g) {
    if (g > g_flags_cap) {
        if (g_flags) {
            cudaDeviceSynchronize();
            cudaFree(g_flags);
        }
        g_flags = nullptr;
        g_flags_cap = 0;
        const uint64_t cap = std::max<uint64_t>(g, 1024);
        if (cudaMalloc(&g_flags, cap * 4) != cudaSuccess) {
            cudaGetLastError();
            set_error("grid flag allocation failed");
            return nullptr;
        }
        cudaMemset(g_flags, 0, cap * 4);
        cudaDeviceSynchronize();
        g_flags_cap = cap;
        g_epoch = 0;
    }
    return g_flags;
}
static uint32_t next_epoch() {
    const uint32_t e = g_epoch;
    g_epoch += 4;
    return e;
}

static int cur_variant() {
    if (params().seed == 0) return STRIDED_VARIANT;  // "strided" param: X = 0
    const int v = (int)params().variant;
    return (v >= 0 && v < N_VARIANTS) ? v : 0;
}

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
        if (path == 2 && P.fused && variant == 0 && g <= (uint64_t)sm_count() * (uint64_t)vi.occ) {
            // one cooperative launch: group partition + cleanup
            using C = GroupCfg<K>;
            uint32_t* flags = grid_flags(g);
            if (!flags) return PP_E_NOMEM;
            FusedArgs<K> fa;
            fa.keys = keys;
            fa.n = n;
            fa.h = h;
            fa.n_lines = n_lines;
            fa.seed = P.seed;
            fa.g = (uint32_t)g;
            fa.epoch = next_epoch();
            fa.stop = (uint32_t)P.fused_stop;
            fa.pivot = pivot;
            fa.gout = gout;
            fa.ctl = ctl;
            fa.d_split = d_split;
            fa.cntL = cntL;
            fa.cntR = cntR;
            fa.ttl = ttl;
            fa.ttr = ttr;
            fa.flags = flags;
            fa.PL = PL;
            fa.PR = PR;
            fa.rk = rk;
            fa.posL = posL;
            fa.posR = posR;
            static bool attr = false;
            if (!attr) {
                cudaFuncSetAttribute(fused_partition_kernel<C>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)C::SMEM);
                attr = true;
            }
            void* args[] = {&fa};
            e = cudaLaunchCooperativeKernel((void*)fused_partition_kernel<C>, dim3((unsigned)g), dim3(C::NT), args,
                                            C::SMEM, st);
            note_launches(1);
            S.path = 4;
            timing_mark(st);  // whole partition counted as the "group" phase
            timing_mark(st);
            if (e != cudaSuccess) return cuda_fail(e, "fused partition launch");
            e = cudaGetLastError();
            if (e != cudaSuccess) return cuda_fail(e, "fused partition launch");
            return PP_OK;
        }
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
    for (int v = 0; v < N_VARIANTS; ++v) {
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

}  // namespace pp
