/*
 * pp.h -- C ABI of the B200-native in-place parallel partition and quicksort
 * (arxiv 2004.12532, "In-place parallel partition"; PAPER.md below means the
 * paper's text).  Plain C: pointers and integer sizes only, no CUDA or torch
 * types in the signatures (streams are passed as `void*` = cudaStream_t).
 *
 * Problem (§2 "The Parallel Partition Problem"): reorder an
 * array so that predecessors precede successors.  Here predecessor <=>
 * key < pivot, unsigned compare; indices are 0-based; the returned split is
 * K = #{i : keys[i] < pivot}, i.e. the index of the first successor.
 *
 * Method: the Smoothed Striding Partial Partition Step
 * (Fig. 3) realised as one CTA per group
 * U_i, followed by a parallel rank-matched cleanup of the window
 * [v_min, v_max) (the paper recurses or uses the Blocked-Prefix-Sum
 * partition there).  Quicksort is
 * layered on the same kernels.
 *
 * Ownership: `keys` is owned by the caller and is never allocated, freed or
 * reallocated by the library.  The library owns an internal device
 * workspace (o(n) bytes, reported by pp_last_aux_bytes) and one small pinned
 * host word; calls from several host threads are serialised by a mutex.
 *
 * Errors: every call returns a pp_status.  PP_E_INVAL: NULL pointer with
 * n > 0, `keys` not aligned to the key size, or a host pointer passed where a
 * device pointer is required (or vice versa).  PP_E_CUDA: a CUDA call or
 * kernel failed (message in pp_last_error(); the array is then unspecified
 * but remains a permutation of the input if the failure came after launch).
 * PP_E_INTERNAL: a device-side invariant check failed (never expected).
 *
 * Determinism: output bytes are a pure function of (input bytes, n, pivot,
 * library build): no atomics on the partition paths, fixed thread mappings,
 * a fixed offset seed.  (The quicksort's bin sort counts with shared-memory
 * atomics; its output, a sorted array, is unique.)
 */
#ifndef PP_H_
#define PP_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    PP_OK = 0,
    PP_E_INVAL = 1,
    PP_E_CUDA = 2,
    PP_E_NOMEM = 3,
    PP_E_NCCL = 4,
    PP_E_INTERNAL = 5
} pp_status;

/* ---- single-GPU partition ------------------------------------------------
 * keys: DEVICE pointer to n keys (uint64 / uint32), aligned to the key size
 *       (any such alignment; 16-B vector I/O peels the unaligned head).
 * pivot: predecessor <=> key < pivot (unsigned).
 * stream: cudaStream_t (NULL = legacy default stream).  All work is enqueued
 *       on it; the synchronous variants then wait for it.
 * split_out: HOST pointer, receives K (sync variants).
 * d_split:  DEVICE pointer to one uint64, receives K (async variants; the
 *       call returns after enqueueing; no host synchronisation at all).
 * n == 0 returns K = 0.  Cites: PAPER.md:272-281 (problem), 953-1015
 * (Smoothed Striding partial step + cleanup). */
pp_status pp_partition_u64(uint64_t *keys, uint64_t n, uint64_t pivot, void *stream, uint64_t *split_out);
pp_status pp_partition_u32(uint32_t *keys, uint64_t n, uint32_t pivot, void *stream, uint64_t *split_out);
pp_status pp_partition_async_u64(uint64_t *keys, uint64_t n, uint64_t pivot, void *stream, uint64_t *d_split);
pp_status pp_partition_async_u32(uint32_t *keys, uint64_t n, uint32_t pivot, void *stream, uint64_t *d_split);

/* ---- single-GPU quicksort ----------------------------
 * Sorts n DEVICE keys ascending (unsigned), in place; synchronises `stream`
 * (the level loop reads the per-level segment count).  Median-of-3 pivot,
 * strict split, "x <= p" progress step when the pivot is the minimum
 * (reading R14); small segments are sorted in shared memory. */
pp_status pp_quicksort_u64(uint64_t *keys, uint64_t n, void *stream);
pp_status pp_quicksort_u32(uint32_t *keys, uint64_t n, void *stream);

/* ---- the paper's Blocked-Prefix-Sum partition (low-space form) -----------
 * PAPER.md:319-478 (§3, Figs. 1-2) as the paper's "low-space implementation"
 * (PAPER.md:1466-1486): role swap when fewer than half of the keys are
 * successors (the view is the reversed array),
 * MakeSuccessorHeavy in place (Fig. 1), block prefix sums over blocks of 4096
 * keys kept in an explicit array (the bit-pair codec of Lemma 3.2 is not
 * used), the recursive in-place Reorder (Fig. 2).  keys: DEVICE pointer to n
 * keys, partitioned in place by key < pivot; the arrangement is the
 * algorithm's (deterministic; equals the CPU oracle's byte for byte).
 * Several passes over the array (count, ~2n for MakeSuccessorHeavy, block
 * counts, Reorder): the comparison row of SURVEY §8(f) #3, not the fast path.
 * Aux: 12 bytes per 4096 keys + O(1).  split_out: HOST pointer (sync);
 * d_split: DEVICE word (async, no host synchronisation). */
pp_status pp_partition_bps_u64(uint64_t *keys, uint64_t n, uint64_t pivot, void *stream, uint64_t *split_out);
pp_status pp_partition_bps_u32(uint32_t *keys, uint64_t n, uint32_t pivot, void *stream, uint64_t *split_out);
pp_status pp_partition_bps_async_u64(uint64_t *keys, uint64_t n, uint64_t pivot, void *stream, uint64_t *d_split);

/* ---- the Standard Algorithm: stable, OUT-OF-PLACE partition ---------------
 * PAPER.md:284-311 (§2): D[i] = [in[i] < pivot], S = prefix sums of D, t =
 * S[n-1]; predecessor i -> out[S[i]-1], successor i -> out[t + i - S[i]]
 * (0-based; reading R9 fixes the paper's index garbles).  The output is
 * unique (stable on both sides).  in, out: DEVICE pointers to n keys each,
 * non-overlapping (PP_E_INVAL otherwise); in is not modified.  Not in place:
 * Theta(n) extra memory (out) and 3*n*w bytes of traffic (count pass +
 * scatter pass), the paper's baseline that the in-place algorithms avoid;
 * kept as the SURVEY §8(f) #4 comparison row.  Aux: 12 bytes per 4096 keys.
 * split_out: HOST pointer (synchronous); the async variant writes the split
 * to the DEVICE word d_split and does not synchronise. */
pp_status pp_partition_stable_u64(const uint64_t *in, uint64_t *out, uint64_t n, uint64_t pivot, void *stream,
                                  uint64_t *split_out);
pp_status pp_partition_stable_u32(const uint32_t *in, uint32_t *out, uint64_t n, uint32_t pivot, void *stream,
                                  uint64_t *split_out);
pp_status pp_partition_stable_async_u64(const uint64_t *in, uint64_t *out, uint64_t n, uint64_t pivot,
                                        void *stream, uint64_t *d_split);

/* ---- stable IN-PLACE partition (comparison row) ----------
 * The Standard Algorithm's output (stable on both sides)
 * produced in place: every tile of 4096 keys is stable-partitioned in
 * registers, then adjacent partitioned segments [P1 S1][P2 S2] are merged
 * into [P1 P2 S1 S2] by rotating [S1 P2] with three in-place reversals,
 * level by level (PAPER.md:309-311 notes that only the out-of-place
 * Standard Algorithm is stable).  O(n log(n / 4096)) work (about two passes
 * over the array per level), O(n / 4096) aux words, deterministic, no
 * atomics; equals pp_partition_stable_* byte for byte.  keys: DEVICE
 * pointer to n keys (in place); split_out: HOST pointer; synchronous. */
pp_status pp_partition_stable_inplace_u64(uint64_t *keys, uint64_t n, uint64_t pivot, void *stream,
                                          uint64_t *split_out);
pp_status pp_partition_stable_inplace_u32(uint32_t *keys, uint64_t n, uint32_t pivot, void *stream,
                                          uint64_t *split_out);

/* ---- host-buffer (end-to-end) variants ------------------------------------
 * host_keys: HOST pointer (pinned or pageable) to n keys, partitioned / sorted
 * in place through a library-owned device buffer.  These are what an
 * application with host-resident data calls; bench.py's "e2e" number times
 * them (H2D + kernels + D2H).  pp_partition_host_* streams: chunks of
 * "host_chunk" keys (param, default 2^23) are uploaded alternately from the
 * front and the back, each is partitioned on the device as it lands, and its
 * keys < pivot are copied back to the front of host_keys, the others to the
 * back, as soon as those host positions have been uploaded -- downloads
 * overlap uploads.  The result satisfies the partition contract (keys <
 * pivot in [0, split), the rest after); the arrangement within each side is
 * chunk order (any arrangement is a correct output).
 * pp_quicksort_host_u64: H2D, sort, D2H.  Synchronous; PP_E_NOMEM if the
 * device buffer cannot be allocated. */
pp_status pp_partition_host_u64(uint64_t *host_keys, uint64_t n, uint64_t pivot, uint64_t *split_out);
pp_status pp_partition_host_u32(uint32_t *host_keys, uint64_t n, uint32_t pivot, uint64_t *split_out);
pp_status pp_quicksort_host_u64(uint64_t *host_keys, uint64_t n);

/* ---- north-star names ------------------------------------------------------
 * pp_partition(keys, n, pivot) -> split: uint64 DEVICE keys on the legacy
 * default stream; returns UINT64_MAX on error (see pp_last_error()).
 * pp_quicksort(keys, n): uint64 DEVICE keys on the legacy default stream. */
uint64_t pp_partition(uint64_t *keys, uint64_t n, uint64_t pivot);
pp_status pp_quicksort(uint64_t *keys, uint64_t n);

/* ---- multi-GPU partition (BASELINE config 3) ------------------
 * One process per GPU; the global array is the concatenation of the ranks'
 * shards in rank order.  Collective calls: every rank must call them, in
 * the same order.
 * pp_dist_unique_id: fills out128 (128 bytes) with a fresh NCCL unique id;
 *   call on one rank and share the bytes with the others (any channel).
 * pp_dist_init: creates the library's NCCL communicator (NCCL is loaded at
 *   run time; the copy PyTorch already loaded is preferred).  device = the
 *   CUDA device of this rank.  PP_E_NCCL on NCCL failure.
 * pp_partition_dist_u64/u32: partitions the local DEVICE shard (n_local keys)
 *   by key < pivot, then exchanges misplaced ranges so that the GLOBAL array
 *   is partitioned; *global_split_out = K = #keys < pivot over all ranks
 *   (HOST pointer).  The local step is pp_partition_*; then ncclAllGather of
 *   (status, n_r, t_r, pivot), a plan computed identically on every rank, and
 *   ncclSend/ncclRecv rounds through two staging halves of <= the staging size
 *   each (default 256 MiB, pp_dist_set_staging): a round's copies from
 *   staging into place run on a side stream while the next round transfers
 *   into the other half.  Mismatched pivots or key types
 *   across ranks -> PP_E_INVAL on every rank.  Synchronises `stream`.
 *   Failure handling: every rank agrees on the status before returning (a
 *   local failure is reported by all ranks); the communicator is
 *   non-blocking and every wait polls ncclCommGetAsyncError with a timeout
 *   (param "dist_timeout_ms", default 600000): a dead or hung peer aborts the
 *   communicator and returns PP_E_NCCL (pp_dist_finalize + pp_dist_init to
 *   recover).
 * pp_dist_plan: the exchange plan alone (host arithmetic, no GPU): for shard
 *   sizes ns[P] and local splits ts[P], writes *n_out pieces of 6 uint64
 *   {round, rank_f, f, rank_t, t, len} (swap global [f, f+len) on rank_f with
 *   [t, t+len) on rank_t) into out[6*out_cap] and K into *K_out.
 * pp_dist_finalize: destroys the communicator and frees the buffers. */
pp_status pp_dist_unique_id(void *out128);
pp_status pp_dist_init(const void *id128, int nranks, int rank, int device);
pp_status pp_partition_dist_u64(uint64_t *shard, uint64_t n_local, uint64_t pivot, void *stream,
                                uint64_t *global_split_out);
pp_status pp_partition_dist_u32(uint32_t *shard, uint64_t n_local, uint32_t pivot, void *stream,
                                uint64_t *global_split_out);
pp_status pp_dist_set_staging(uint64_t bytes);
/* pp_dist_last_timing: phases of this rank's last pp_partition_dist_* call,
 * from CUDA events on its stream: out4[0] = local partition ms, out4[1] =
 * (n_r, t_r) all-gather ms, out4[2] = exchange ms, out4[3] = bytes this rank
 * moved between GPUs in the exchange (staged path: bytes sent, as many are
 * received; one-sided path: remote bytes read + written by its swaps). */
pp_status pp_dist_last_timing(double *out4);
/* pp_quicksort_dist_u64/u32: sorts the GLOBAL array (shards in rank order)
 * ascending, unsigned, in place (collective).  Segments spanning ranks are
 * split by pp_partition_dist_* with a median-of-3 pivot gathered from the
 * owning ranks (the "x <= p" step when the pivot is the minimum); spanning
 * segments of <= 2^16 keys are all-gathered and sorted on every participating
 * rank; finally each rank sorts its shard with pp_quicksort_*.  Shard sizes
 * may differ.  Synchronises `stream`. */
pp_status pp_quicksort_dist_u64(uint64_t *shard, uint64_t n_local, void *stream);
pp_status pp_quicksort_dist_u32(uint32_t *shard, uint64_t n_local, void *stream);
/* ---- loopback: the distributed calls with P emulated ranks on ONE GPU --------
 * The multi-GPU algorithm above (local partition, record all-gather with
 * status agreement, the same plan, staged send/recv rounds or the one-sided
 * share rule with param "dist_p2p", the batched distributed quicksort) run
 * by P host threads of this process, rank r owning the DEVICE slice
 * keys[sum(ns[0..r-1]), + ns[r]) on its own stream.  Collectives rendezvous
 * on a host barrier; every received piece is one cudaMemcpyAsync from the
 * sender's range; local library calls are serialised (one workspace).  This
 * is how the P > 1 code path is tested on a single GPU (PAPER.md:272-281:
 * the global result must be a partition / the sort).  1 <= nranks <= 64;
 * shards may be empty.  Synchronous.  Errors: the lowest-ranked failure is
 * returned (every rank agrees); a rank that never arrives (test param
 * "dist_fault" = 2) makes the others fail after "dist_timeout_ms". */
pp_status pp_partition_dist_loopback_u64(uint64_t *keys, const uint64_t *ns, int nranks, uint64_t pivot,
                                         uint64_t *global_split_out);
pp_status pp_partition_dist_loopback_u32(uint32_t *keys, const uint64_t *ns, int nranks, uint32_t pivot,
                                         uint64_t *global_split_out);
pp_status pp_quicksort_dist_loopback_u64(uint64_t *keys, const uint64_t *ns, int nranks);
pp_status pp_quicksort_dist_loopback_u32(uint32_t *keys, const uint64_t *ns, int nranks);
pp_status pp_dist_plan(const uint64_t *ns, const uint64_t *ts, int nranks, uint64_t cap, uint64_t *out,
                       uint64_t out_cap, uint64_t *n_out, uint64_t *K_out);
pp_status pp_dist_finalize(void);

/* pp_swap_ranges_u64/u32: the staging-free exchange primitive (SURVEY §8(f)
 * #1): for each of n_pieces HOST triples (a, b, len) -- a and b DEVICE
 * addresses (a peer-mapped b is allowed), aligned to the key size -- swaps
 * keys [a, a+len) with [b, b+len) elementwise, one thread per pair.  With
 * the pieces of pp_dist_plan (a = the left rank's misplaced successors, b =
 * the right rank's misplaced predecessors) it performs the partition's
 * exchange one-sidedly with no staging buffer; on one GPU it executes the
 * plan of emulated ranks.  Ranges must not overlap.  Synchronous on
 * `stream`; PP_E_INVAL for misaligned ranges or NULL triples. */
pp_status pp_swap_ranges_u64(const uint64_t *triples, uint64_t n_pieces, void *stream);
pp_status pp_swap_ranges_u32(const uint64_t *triples, uint64_t n_pieces, void *stream);

/* One-sided (staging-free) exchange of pp_partition_dist_* (
 * param "dist_p2p" = 1, default 0): every rank maps every other rank's shard
 * through CUDA IPC and swaps its share of the misplaced pairs directly with
 * pp_swap_ranges' kernel; a closing collective keeps ranks from returning
 * while a peer still writes into their shard.  Needs peer access between the
 * GPUs (NVLink/NVSwitch).
 * pp_dist_p2p_pieces: the share of rank `rank` (host arithmetic, no GPU): for
 *   shard sizes ns[P] and local splits ts[P], writes *n_out rows of 5 uint64
 *   {rank_a, a, rank_b, b, len} -- swap GLOBAL positions [a, a+len) (on
 *   rank_a, misplaced successors) with [b, b+len) (on rank_b, misplaced
 *   predecessors) -- into out[5*out_cap].  Every matched run of the plan is
 *   split: the left rank takes the first ceil(len/2) pairs, the right rank the
 *   rest, so each pair is swapped by exactly one rank.  PP_E_INVAL if out_cap
 *   is too small (n_out still set), ts[r] > ns[r], or rank is out of range.
 * pp_ipc_export: (64-byte CUDA IPC handle of the allocation holding d_ptr,
 *   byte offset of d_ptr in it) -> handle_out[64], *offset_out.
 * pp_ipc_import: maps an exported range in this process (cached per handle;
 *   peer access enabled lazily) -> *d_ptr_out = mapped base + offset.
 * pp_ipc_close_all: unmaps every imported range (pp_dist_finalize does too). */
pp_status pp_dist_p2p_pieces(const uint64_t *ns, const uint64_t *ts, int nranks, int rank, uint64_t *out,
                             uint64_t out_cap, uint64_t *n_out);
pp_status pp_ipc_export(const void *d_ptr, void *handle_out, uint64_t *offset_out);
pp_status pp_ipc_import(const void *handle, uint64_t offset, void **d_ptr_out);
pp_status pp_ipc_close_all(void);

/* ---- Smoothed Striding partial partition step alone (parity of internals) --
 * Runs only the group kernel on the 16-B aligned region of `keys` with g
 * groups (g = 0: the library's automatic choice) and copies the per-group
 * statistics to HOST arrays T, vlo, vhi (g entries each; allocate
 * pp_max_groups() entries if g = 0).  info[0..5] receives
 * {g, head, n_lines, line_keys, seed, 0}: the region is keys[head ..
 * head + n_lines*line_keys), X[j] = ((fmix64(seed + (j+1)*0x9E3779B97F4A7C15)
 * >> 32) * g) >> 32; seed = 0 means X[j] = 0 for every j, the
 * Strided Algorithm (param "strided").  vlo/vhi are
 * region-relative positions.
 * The array is left partially partitioned. */
pp_status pp_ss_groups_u64(uint64_t *keys, uint64_t n, uint64_t pivot, uint64_t g, void *stream,
                           uint64_t *T, uint64_t *vlo, uint64_t *vhi, uint64_t *info);
pp_status pp_ss_groups_u32(uint32_t *keys, uint64_t n, uint32_t pivot, uint64_t g, void *stream,
                           uint64_t *T, uint64_t *vlo, uint64_t *vhi, uint64_t *info);
uint64_t pp_max_groups(void);

/* ---- workspace / statistics / tuning --------------------------------------- */
/* Bytes of device workspace a call on n keys of key_bytes (4 or 8) may use,
 * under the current tuning parameters; op 0 = partition, 1 = quicksort.
 * o(n): the cleanup arrays are capped, quicksort segment
 * lists are uploaded in chunks of 2^20 descriptors. */
uint64_t pp_workspace_bytes(uint64_t n, int key_bytes, int op);
/* Caller-owned device workspace (e.g. a torch tensor): when set, every
 * partition / quicksort call uses it instead of the library's internal one,
 * and fails with PP_E_NOMEM if a step needs more than it holds (a partition
 * then leaves the array untouched; a quicksort leaves a permutation of the
 * input).  pp_workspace_bytes(n, key_bytes, op) always suffices.  d_ws must be device memory, 256-byte
 * aligned; the library never frees it.  d_ws = NULL reverts to the internal
 * workspace.  Calls sharing one workspace must be stream-ordered.
 * (Survey §8(b); o(n) aux memory per the "in-place" definition.) */
pp_status pp_set_workspace(void *d_ws, uint64_t bytes);
/* Device bytes besides `keys` touched by the last call (aux memory). */
uint64_t pp_last_aux_bytes(void);
/* Statistics of the last partition call: out[0..12] = {n, K, W(dirty-set
 * size), v_min, v_max, M (misplaced pairs in the cleanup), g, line_keys,
 * n_lines, head, aux_bytes, path, nTasks}.  Reads device memory: synchronous. */
pp_status pp_last_stats(uint64_t *out13);
/* Work statistics of the last single-GPU quicksort (host counters, no device
 * access): out6 = {n, levels (depth of the breadth-first level loop),
 * level_keys (sum over levels of the keys in the segments partitioned there:
 * each is read and written once by that level's kernels), small_keys (keys in
 * segments of (leaf, qs_small] keys, finished by the per-CTA recursion),
 * leaf_keys (keys in segments of <= leaf keys, sorted by the bin sort
 * directly), nsmall (number of such small segments)}.  bench.py derives the
 * quicksort's algorithmic bytes from these. */
pp_status pp_quicksort_last_stats(uint64_t *out6);
/* EREW shadow-writer audit (the GPU analogue of SPEC's
 * element-level auditor S:62-70 for the EREW claim of PAPER.md:229-238).
 * Only the debug build libpp_audit.so (compiled with -DPP_AUDIT=1) implements
 * it; the product libpp.so returns PP_E_INVAL.  d_shadow: device array of n
 * zeroed uint32 counters owned by the caller, one per key of the device range
 * [keys, keys + n) (key_bytes 4 or 8).  While set, every store of a key by
 * the partition's kernels (pp_partition_* and its cleanup tails, all paths)
 * adds 1 (the Smoothed Striding group kernel) or 1 << 16 (the cleanup
 * kernels) to that key's counter.  d_shadow = NULL switches it off.  Not
 * thread safe with concurrent calls; debugging / tests only. */
pp_status pp_audit_set(uint32_t *d_shadow, const void *keys, uint64_t n, int key_bytes);
/* Tunables (tests / benchmarks): "g", "min_lines_per_group", "small_n",
 * "path" (0 auto, 1 single-CTA, 2 smoothed striding, 3 cleanup only), "tile",
 * "ranks", "seed", "strided" (1: X = 0, the Strided Algorithm PAPER.md:796-825,
 * i.e. seed 0; 0: back to the default seed), "cleanup_chain" (-1 auto:
 * 3-kernel chain below 1 GiB of keys, fused scan/swap tail above; 0 fused
 * tail; 1 chain), "cleanup_bitmap"; quicksort: "leaf" (bin capacity, <= 16384,
 * default 16384), "qs_cta_max", "qs_small", "qs_waves", "qs_heavy",
 * "qs_lanes" (0 auto = 2 lanes), "qs_early" (-1 auto = on), "qs_early_min"
 * (0 auto), "qs_minl" (0 auto: 128 KiB per group), "qs_pivot" (0 median of 3
 * -- BASELINE config 5's rule, the default --, 1 Tukey's ninther, 2 the median
 * of 31 evenly spaced keys: better balanced splits, fewer levels; also the
 * distributed quicksort's rule for segments spanning ranks), "qs_deep" (segments deeper
 * than this take Tukey's ninther instead of the median of 3; -1 auto =
 * 2 log2(n) + 16, 0 = always), "qs_prio" (-1 auto = on: the level loop on
 * high-priority streams, the early recursion / bin sorts at low priority; 0
 * off), "qs_dev" (1: once a lane's segments are all
 * below qs_heavy, every next level's segment list is built on the device by
 * one kernel -- children, group counts, longest-first order compacted by
 * scans -- and two levels per lane are in flight without a host round trip;
 * default 0: the host builds each level, measured 0.2-2% faster because the
 * two lanes already hide its work), "qs_dev_check" (test hook: every
 * device-built list is compared with the host's plan of it, PP_E_INTERNAL on
 * a difference); "host_chunk", "bps_nt";
 * multi-GPU: "dist_p2p", "dist_timeout_ms", "dist_small" (distributed
 * quicksort: spanning segments of <= this many keys are gathered and sorted
 * locally), "dist_split" (1: the pivot of a segment spanning ranks is the
 * quantile of its rank boundary among 63 samples -- fewer distributed rounds;
 * 0 default: the level loop's rule), "dist_overlap" (1: pp_partition_dist counts every chunk of the
 * shard first, all-gathers the counts, then partitions the "dist_chunks"
 * chunks in order while the exchange of each finished chunk runs on a second
 * stream -- SURVEY §8(f) #1; same result contract), "dist_chunks" (default
 * 8, must be equal on every rank), "dist_fault", "dist_fault_rank" (loopback
 * test hooks).
 * Returns PP_E_INVAL for an unknown name.  pp_get_param returns INT64_MIN
 * for an unknown name. */
pp_status pp_set_param(const char *name, int64_t value);
int64_t pp_get_param(const char *name);
/* Restores every tunable to the library's default. */
void pp_reset_params(void);

const char *pp_status_string(pp_status s);
const char *pp_last_error(void);
/* Number of kernel launches enqueued by the library since the last reset. */
uint64_t pp_launch_count(int reset);
/* Phase timing of partition calls with CUDA events recorded on each call's
 * stream: pp_timing(1) starts (and clears) recording; pp_timing_read(out)
 * waits for the recorded events and writes {calls, group-kernel ms total,
 * rest-of-pipeline ms total, total ms}, then clears.  For single-CTA /
 * cleanup-only calls the "group" phase is the whole first kernel(s). */
void pp_timing(int enable);
pp_status pp_timing_read(double *out4);

#ifdef __cplusplus
}
#endif

#endif /* PP_H_ */
