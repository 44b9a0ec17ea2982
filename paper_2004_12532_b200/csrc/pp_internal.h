// pp_internal.h -- host-side internals shared by the C-ABI (pp_api.cu), the
// partition driver (pp_partition.cu) and the quicksort driver (pp_quicksort.cu).
#pragma once
#include <cstdint>
#include <string>
#include <cuda_runtime.h>

#include "../../include/pp.h"

namespace pp {

// Per-segment control block, resident in device workspace.  Written by the
// window-reduce kernel, read by the cleanup kernels (no host round trip).
struct Ctl {
    uint64_t n;          // segment length
    uint64_t K;          // split = #keys < pivot in the segment
    uint64_t W;          // |D|, size of the dirty set
    uint64_t Kv;         // #dirty positions < K
    uint64_t ds[3];      // dirty intervals [ds, ds+dl), sorted, disjoint
    uint64_t dl[3];
    uint64_t vmin, vmax; // window of the partial partition step (absolute)
    uint64_t ML, MR;     // misplaced falses left of K / trues right of K (equal)
    uint64_t nL, nR;     // cleanup tiles on each side
    uint64_t nTasks;     // rank-matched swap tasks
    uint64_t tile;       // tile size (keys) of the cleanup count
    uint64_t R;          // ranks per swap task
    uint64_t err;        // nonzero = internal invariant violated
};

// Per-group output of the Smoothed Striding partial partition step.
struct GroupOut {
    uint64_t T;    // #predecessors in the group
    uint64_t vlo;  // first successor position (region-relative), or sentinel
    uint64_t vhi;
};

struct Params {
    int64_t g = 0;                 // 0 = auto
    int64_t min_lines_per_group = 16;
    int64_t small_n = 1 << 15;     // below: single-CTA path
    int64_t path = 0;              // 0 auto, 1 single-CTA, 2 smoothed-striding, 3 cleanup-only
    int64_t tile = 0;              // 0 = auto
    int64_t ranks = 0;             // 0 = auto (ranks per swap task)
    uint64_t seed = 0x5EEDC0DE2004ULL;  // Smoothed Striding offset seed (fixed => deterministic)
    int64_t leaf = 0;              // quicksort: 0 = auto smem leaf size
    int64_t qs_cta_max = 0;        // quicksort: 0 = auto segment size handled by one CTA
    int64_t qs_waves = 2;          // quicksort mid levels: target CTA waves of the group launch
    int64_t qs_small = 1 << 16;    // quicksort: segments <= this finish in one CTA (0 = off)
    int64_t cleanup_chain = -1;    // partition cleanup tail: 0 fused scan+swap, 1 scan / locate / swap kernels,
                                   // -1 auto (chain below 1 GiB of keys, fused from 1 GiB: measured crossover)
    int64_t cleanup_bitmap = 1;    // fused tail: locate pairs from the dirty-set bitmap (0: locate + grid barrier)
    int64_t bps_nt = 256;          // Blocked-Prefix-Sum Reorder level kernel: threads per CTA (256/512/1024)
    int64_t qs_lanes = 0;          // quicksort level loop: 1 = one stream, 2 = two array-disjoint lanes on two
                                   // streams, 0 = auto (= 2)
    int64_t qs_early = -1;         // quicksort: run the per-CTA recursion + bin sort of small segments on two more
                                   // streams as soon as their levels complete (overlapping the remaining levels);
                                   // -1 auto (= on), 0 off, 1 on
    int64_t qs_early_min = 0;      // quicksort early recursion: batch when >= this x #SM small segments are final
                                   // (0 auto: 8 for u64, 2 for u32 -- measured)
    int64_t qs_minl = 0;           // quicksort: at least this many lines per group for mid segments (0 auto: 64)
    int64_t dist_p2p = 0;          // pp_partition_dist: 1 = one-sided exchange over CUDA-IPC peer mappings (no staging)
    int64_t dist_timeout_ms = 600000;  // distributed calls: a wait longer than this aborts (PP_E_NCCL on every rank)
    int64_t dist_fault = 0;        // test hook (loopback): 1 = rank dist_fault_rank fails its local step, 2 = it never arrives
    int64_t dist_fault_rank = -1;
    int64_t dist_overlap = 0;      // pp_partition_dist: 1 = count first, then chunked local partitions whose exchange
                                   // pieces move while the next chunk is partitioned
    int64_t dist_chunks = 8;       // dist_overlap: chunks per shard (the same on every rank)
    int64_t dist_split = 0;        // distributed quicksort: 1 = pivots of spanning segments at the sample quantile
                                   // of their rank boundary (63 samples; fewer distributed rounds), 0 = R14's rule
    int64_t dist_small = 1 << 16;  // distributed quicksort: spanning segments <= this are gathered and sorted locally
    int64_t host_chunk = 1 << 23;  // host-buffer partition: keys per streamed chunk (measured best at 1-8 GiB)
    int64_t qs_pivot = 0;          // quicksort level-loop pivot: 0 median of 3 (BJ config 5), 1 Tukey's ninther,
                                   // 2 median of 31 samples (the per-CTA recursion takes the ninther for 1, 2)
    int64_t qs_deep = -1;          // quicksort levels: segments deeper than this use the ninther pivot (-1 auto:
                                   // 2 log2(n) + 16; 0: always)
    int64_t qs_prio = -1;          // quicksort: level loop on high-priority streams, early recursion / bins low
                                   // (-1 auto = on, 0 off, 1 on)
    int64_t qs_heavy = 1 << 21;    // quicksort: mid segments >= this get the batched multi-CTA cleanup (0 = off)
    int64_t qs_dev_check = 0;      // test hook: compare each device-built level list with the host's plan of it
    int64_t qs_dev = 0;            // quicksort: 1 = levels whose segments are all < qs_heavy are built on the
                                   // device (qs_build_kernel), two levels in flight per lane; 0 (default) = the
                                   // host builds every level (measured 0.2-2% faster: the two lanes already hide
                                   // the host's work, the builder's ~13 us sit on a lane's critical path)
};
Params& params();

struct LastStats {
    uint64_t n = 0, K = 0, W = 0, vmin = 0, vmax = 0, M = 0, g = 0, line_keys = 0;
    uint64_t n_lines = 0, head = 0, aux_bytes = 0, path = 0, nTasks = 0;
};
LastStats& last_stats();

void set_error(const std::string& msg);
pp_status cuda_fail(cudaError_t e, const char* what);

// device workspace (grows; one per process / device)
void* workspace(size_t bytes, cudaStream_t st);
// caller-owned workspace (pp_set_workspace), if one is set
bool user_workspace(void** p, size_t* bytes);
int sm_count();
// upper bounds of the device workspace (current params), pp_workspace_bytes
uint64_t partition_workspace_bound(uint64_t n);
template <typename K>
uint64_t quicksort_workspace_bound(uint64_t n);

template <typename K>
pp_status partition_device(K* keys, uint64_t n, K pivot, cudaStream_t st, uint64_t* d_split, Ctl** ctl_out);
// EREW shadow-writer audit (libpp_audit.so; PP_E_INVAL in the product library)
pp_status audit_set_partition(uint32_t* shadow, const void* base, uint64_t n, uint32_t key_bytes);

template <typename K>
pp_status ss_groups_device(K* keys, uint64_t n, K pivot, uint64_t g, cudaStream_t st, uint64_t* T_host,
                           uint64_t* vlo_host, uint64_t* vhi_host, uint64_t* info_host);

template <typename K>
pp_status quicksort_device(K* keys, uint64_t n, cudaStream_t st);
pp_status quicksort_last_stats(uint64_t* out6);

// the paper's Blocked-Prefix-Sum partition, low-space form (pp_bps.cu)
template <typename K>
pp_status partition_bps_device(K* keys, uint64_t n, K pivot, cudaStream_t st, uint64_t* d_split);

// the Standard Algorithm, stable and out of place (pp_stable.cu)
template <typename K>
pp_status partition_stable_device(const K* in, K* out, uint64_t n, K pivot, cudaStream_t st, uint64_t* d_split,
                                  uint64_t** total_out);

// the in-place stable variant (pp_stable.cu): O(n log n) work, split to a device word
template <typename K>
pp_status partition_stable_inplace_device(K* keys, uint64_t n, K pivot, cudaStream_t st, uint64_t* d_split);

// multi-GPU (pp_dist.cu)
pp_status dist_unique_id(void* out128);
pp_status dist_init(const void* id128, int nranks, int rank, int device);
pp_status dist_finalize();
void dist_set_staging(uint64_t bytes);
template <typename K>
pp_status partition_dist(K* shard, uint64_t n_local, K pivot, cudaStream_t st, uint64_t* global_split);
pp_status dist_plan(const uint64_t* ns, const uint64_t* ts, int P, uint64_t cap, uint64_t* out, uint64_t out_cap,
                    uint64_t* n_out, uint64_t* K_out);
template <typename K>
pp_status quicksort_dist(K* shard, uint64_t n_local, cudaStream_t st, uint64_t small);
template <typename K>
pp_status partition_dist_loopback(K* keys, const uint64_t* ns, int P, K pivot, uint64_t* split_out);
template <typename K>
pp_status quicksort_dist_loopback(K* keys, const uint64_t* ns, int P, uint64_t small);
template <typename K>
pp_status swap_ranges(const uint64_t* host_tri, uint64_t np, cudaStream_t st);
pp_status dist_p2p_pieces(const uint64_t* ns, const uint64_t* ts, int P, int rank, uint64_t* out, uint64_t out_cap,
                          uint64_t* n_out);
pp_status ipc_export(const void* d_ptr, void* handle_out, uint64_t* offset_out);
pp_status ipc_import(const void* handle, uint64_t offset, void** d_ptr_out);
pp_status ipc_close_all();
pp_status dist_last_timing(double* out4);

}  // namespace pp
