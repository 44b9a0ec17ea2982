// pp_device.cuh -- device-side helpers for the B200 (sm_100a) in-place partition.
//
// Shares nothing with oracle/ (task rule): the offset hash below is this
// side's own implementation of the counter-based generator that DESIGN.md
// ("Random offsets") defines for the Smoothed Striding X[j] draws
// (§4 Formal Algorithm Description).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace pp {

// ---------------------------------------------------------------------------
// Predicate ("decider"; reading R1: predecessor <=> key < p,
// unsigned compare).
// ---------------------------------------------------------------------------
template <typename K>
__device__ __forceinline__ bool is_pred(K x, K pivot) { return x < pivot; }

// ---------------------------------------------------------------------------
// EREW shadow-writer audit (the GPU analogue of SPEC's
// element-level auditor S:62-70).  Only in the separate
// debug library libpp_audit.so (-DPP_AUDIT=1): every store of a key by the
// partition's kernels adds `inc` to a per-key counter -- 1 for the group
// kernel (the partial step), 1 << 16 for the cleanup kernels -- so the test
// can assert that each key is written at most once per phase.  The product
// library compiles every PP_AUDIT_W to nothing (and has no atomics).
// ---------------------------------------------------------------------------
#if PP_AUDIT
struct AuditState {
    uint32_t* shadow;  // one counter per key of [base, base + n keys)
    uint64_t base, n, kb;
};
static __device__ AuditState g_audit;  // per translation unit (set for pp_partition.cu's kernels)
__device__ __forceinline__ void audit_w(const void* p, uint32_t inc) {
    const AuditState a = g_audit;
    if (a.shadow == nullptr) return;
    const uint64_t off = (uint64_t)(uintptr_t)p - a.base;
    if (off % a.kb == 0 && off / a.kb < a.n) atomicAdd(a.shadow + off / a.kb, inc);
}
#define PP_AUDIT_W(p, inc) ::pp::audit_w((const void*)(p), (inc))
#else
#define PP_AUDIT_W(p, inc) ((void)0)
#endif
constexpr uint32_t AUDIT_GROUP = 1u, AUDIT_CLEANUP = 1u << 16;

// ---------------------------------------------------------------------------
// Smoothed Striding chunk offsets X[j] in {0..g-1}, computed on the fly (the
// paper stores s words of X; recomputing costs ~10 integer
// ops per line and no memory).
// ---------------------------------------------------------------------------
__host__ __device__ __forceinline__ uint64_t ss_fmix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
__host__ __device__ __forceinline__ uint32_t ss_offset(uint64_t seed, uint64_t j, uint32_t g) {
    uint64_t h = ss_fmix(seed + (j + 1) * 0x9E3779B97F4A7C15ULL);
    return (uint32_t)(((h >> 32) * (uint64_t)g) >> 32);
}

// ---------------------------------------------------------------------------
// PTX wrappers: mbarrier + 1-D bulk async copy (TMA engine, SASS UBLKCP).
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_inval(uint64_t* bar) {
    asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// gpu-scope release store / acquire load (flag-array grid barrier, no atomics)
__device__ __forceinline__ void st_release_gpu(uint32_t* p, uint32_t v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_gpu(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// same with a precomputed shared-window address
__device__ __forceinline__ void mbar_wait_s(uint32_t bar_s, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(bar_s),
        "r"(parity)
        : "memory");
}
// global -> shared bulk copy; bytes % 16 == 0, both addresses 16-B aligned.
__device__ __forceinline__ void bulk_g2s(void* dst_smem, const void* src_gmem, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst_smem)),
        "l"(src_gmem), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
// shared -> global bulk copy (bulk-group completion).
__device__ __forceinline__ void bulk_s2g(void* dst_gmem, const void* src_smem, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst_gmem),
                 "r"(smem_u32(src_smem)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait() {
    asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}

// Programmatic dependent launch: wait for the preceding grid's results /
// allow the next grid to start launching (no-ops without the PDL attribute).
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void griddep_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// 16-byte vector of keys.
template <typename K>
struct __align__(16) Vec16 {
    static constexpr int N = 16 / sizeof(K);
    K v[N];
};

__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

}  // namespace pp
