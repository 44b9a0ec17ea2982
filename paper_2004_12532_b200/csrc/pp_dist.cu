// pp_dist.cu -- multi-GPU partition of one array sharded contiguously over
// ranks (BASELINE config 3): local partition on every
// rank, ncclAllGather of (n_r, t_r, pivot), identical exchange plan on every
// rank, and ncclSend/ncclRecv of matched misplaced ranges through a bounded
// staging buffer.  NCCL is loaded at run time (dlopen) -- preferably the copy
// already loaded by PyTorch in this process -- so libpp.so has no link-time
// NCCL dependency and two NCCLs never end up in one process.
#include <dlfcn.h>

#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include <cuda.h>  // driver types only (cuMemGetAddressRange is fetched through the runtime)
#include <nccl.h>

#include "pp_internal.h"

namespace pp {

void note_launches(uint64_t k);

// ---------------------------------------------------------------------------
// The exchange plan (host arithmetic; mirrored independently in Python by
// paper_2004_12532_b200/dist.py and cross-checked by tests/test_dist.py).
// ---------------------------------------------------------------------------
struct Piece {
    uint64_t round, rank_f, f, rank_t, t, len;
};

// Pairs the i-th misplaced successor (global order, left of K) with the i-th
// misplaced predecessor (right of K); splits transfers into pieces <= cap and
// groups them into rounds where no rank moves more than cap keys.
static uint64_t plan_pieces(const uint64_t* ns, const uint64_t* ts, int P, uint64_t cap,
                            std::vector<Piece>& out) {
    uint64_t K = 0;
    for (int r = 0; r < P; ++r) K += ts[r];
    struct Iv {
        uint64_t rank, s, e;
    };
    std::vector<Iv> F, T;
    uint64_t base = 0;
    for (int r = 0; r < P; ++r) {
        const uint64_t b = base, n = ns[r], t = ts[r];
        const uint64_t fs = b + t, fe = std::min(K, b + n);
        if (fs < fe) F.push_back({(uint64_t)r, fs, fe});
        const uint64_t s2 = std::max(K, b), e2 = b + t;
        if (s2 < e2) T.push_back({(uint64_t)r, s2, e2});
        base += n;
    }
    out.clear();
    std::vector<uint64_t> used(P, 0);
    uint64_t round = 0;
    size_t i = 0, j = 0;
    while (i < F.size() && j < T.size()) {
        const uint64_t m = std::min(F[i].e - F[i].s, T[j].e - T[j].s);
        // split into pieces of <= cap, each placed in the current or a new round
        uint64_t s = 0;
        while (s < m) {
            const uint64_t len = std::min(cap, m - s);
            if (used[F[i].rank] + len > cap || used[T[j].rank] + len > cap) {
                ++round;
                std::fill(used.begin(), used.end(), 0);
            }
            out.push_back({round, F[i].rank, F[i].s + s, T[j].rank, T[j].s + s, len});
            used[F[i].rank] += len;
            used[T[j].rank] += len;
            s += len;
        }
        F[i].s += m;
        T[j].s += m;
        if (F[i].s == F[i].e) ++i;
        if (T[j].s == T[j].e) ++j;
    }
    return K;
}

// One-sided (staging-free) exchange: who executes which pairs.  The plan
// with no staging cap has one piece per matched run (the left rank's
// misplaced successors [f, f+len) against the right rank's misplaced
// predecessors [t, t+len); the two ranks always differ, because a shard's
// misplaced keys are all successors (shard ends left of K) or all
// predecessors).  The left rank swaps the first ceil(len/2) pairs, the right
// rank the rest, each reading and writing its partner's keys through the
// peer mapping, so both directions of every NVLink pair carry traffic.
// Mirrored by paper_2004_12532_b200/dist.py p2p_pieces (tests/test_dist.py).
struct P2PPiece {
    uint64_t rank_a, a, rank_b, b, len;
};
static uint64_t p2p_pieces(const uint64_t* ns, const uint64_t* ts, int P, int me, std::vector<P2PPiece>& out) {
    std::vector<Piece> pcs;
    const uint64_t K = plan_pieces(ns, ts, P, ~0ull, pcs);
    out.clear();
    for (const Piece& p : pcs) {
        const uint64_t h = (p.len + 1) / 2;
        if ((int)p.rank_f == me) out.push_back({p.rank_f, p.f, p.rank_t, p.t, h});
        if ((int)p.rank_t == me && p.len > h) out.push_back({p.rank_f, p.f + h, p.rank_t, p.t + h, p.len - h});
    }
    return K;
}

// ---------------------------------------------------------------------------
// CUDA IPC: a device range exported as (allocation handle, offset) and
// mapped in another process (peer access enabled lazily).  Mappings are
// cached by handle and released by ipc_close_all / dist_finalize.
// ---------------------------------------------------------------------------
struct IpcMap {
    cudaIpcMemHandle_t h;
    void* base;
};
static std::vector<IpcMap> g_ipc;

static pp_status alloc_base(const void* p, void** base) {
    using Fn = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
    static Fn fn = nullptr;
    if (!fn) {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        cudaError_t e = cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q);
        if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !f) {
            set_error("cuMemGetAddressRange unavailable");
            return PP_E_CUDA;
        }
        fn = reinterpret_cast<Fn>(f);
    }
    CUdeviceptr b = 0;
    size_t sz = 0;
    if (fn(&b, &sz, (CUdeviceptr)p) != CUDA_SUCCESS) {
        set_error("cuMemGetAddressRange failed (not a device allocation?)");
        return PP_E_INVAL;
    }
    *base = reinterpret_cast<void*>(b);
    return PP_OK;
}

pp_status ipc_export(const void* d_ptr, void* handle_out, uint64_t* offset_out) {
    if (!d_ptr || !handle_out || !offset_out) return PP_E_INVAL;
    void* base = nullptr;
    pp_status s = alloc_base(d_ptr, &base);
    if (s != PP_OK) return s;
    cudaIpcMemHandle_t h;
    cudaError_t e = cudaIpcGetMemHandle(&h, base);
    if (e != cudaSuccess) return cuda_fail(e, "cudaIpcGetMemHandle");
    static_assert(sizeof(cudaIpcMemHandle_t) == 64, "64-byte IPC handle");
    memcpy(handle_out, &h, 64);
    *offset_out = (uint64_t)(static_cast<const char*>(d_ptr) - static_cast<const char*>(base));
    return PP_OK;
}

pp_status ipc_import(const void* handle, uint64_t offset, void** d_ptr_out) {
    if (!handle || !d_ptr_out) return PP_E_INVAL;
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, 64);
    for (const IpcMap& m : g_ipc)
        if (memcmp(&m.h, &h, 64) == 0) {
            *d_ptr_out = static_cast<char*>(m.base) + offset;
            return PP_OK;
        }
    void* base = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return cuda_fail(e, "cudaIpcOpenMemHandle");
    g_ipc.push_back({h, base});
    *d_ptr_out = static_cast<char*>(base) + offset;
    return PP_OK;
}

pp_status ipc_close_all() {
    cudaError_t first = cudaSuccess;
    for (const IpcMap& m : g_ipc) {
        cudaError_t e = cudaIpcCloseMemHandle(m.base);
        if (first == cudaSuccess) first = e;
    }
    g_ipc.clear();
    return first == cudaSuccess ? PP_OK : cuda_fail(first, "cudaIpcCloseMemHandle");
}

// ---------------------------------------------------------------------------
// NCCL, loaded at run time.
// ---------------------------------------------------------------------------
struct NcclApi {
    void* lib = nullptr;
    decltype(&ncclGetUniqueId) GetUniqueId = nullptr;
    decltype(&ncclCommInitRank) CommInitRank = nullptr;
    decltype(&ncclCommDestroy) CommDestroy = nullptr;
    decltype(&ncclAllGather) AllGather = nullptr;
    decltype(&ncclSend) Send = nullptr;
    decltype(&ncclRecv) Recv = nullptr;
    decltype(&ncclGroupStart) GroupStart = nullptr;
    decltype(&ncclGroupEnd) GroupEnd = nullptr;
    decltype(&ncclGetErrorString) GetErrorString = nullptr;
};
static NcclApi g_nccl;

#ifndef PP_NCCL_LIB
#define PP_NCCL_LIB "libnccl.so.2"
#endif

static bool nccl_load() {
    if (g_nccl.lib) return true;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // torch's copy, if loaded
    if (!h) h = dlopen(PP_NCCL_LIB, RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
        set_error(std::string("cannot load NCCL: ") + dlerror());
        return false;
    }
#define PP_SYM(field, name)                                              \
    g_nccl.field = reinterpret_cast<decltype(g_nccl.field)>(dlsym(h, name)); \
    if (!g_nccl.field) {                                                 \
        set_error(std::string("NCCL symbol missing: ") + name);          \
        return false;                                                    \
    }
    PP_SYM(GetUniqueId, "ncclGetUniqueId")
    PP_SYM(CommInitRank, "ncclCommInitRank")
    PP_SYM(CommDestroy, "ncclCommDestroy")
    PP_SYM(AllGather, "ncclAllGather")
    PP_SYM(Send, "ncclSend")
    PP_SYM(Recv, "ncclRecv")
    PP_SYM(GroupStart, "ncclGroupStart")
    PP_SYM(GroupEnd, "ncclGroupEnd")
    PP_SYM(GetErrorString, "ncclGetErrorString")
#undef PP_SYM
    g_nccl.lib = h;
    return true;
}

static pp_status nccl_fail(ncclResult_t r, const char* what) {
    set_error(std::string(what) + ": " + (g_nccl.GetErrorString ? g_nccl.GetErrorString(r) : "nccl error"));
    return PP_E_NCCL;
}

struct DistState {
    cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};  // start, local done, gathered, exchanged
    double last_local_ms = 0, last_gather_ms = 0, last_exchange_ms = 0;
    uint64_t last_bytes = 0;  // bytes this rank moved between GPUs in the last exchange
    ncclComm_t comm = nullptr;
    int nranks = 0, rank = 0, device = 0;
    void* staging = nullptr;
    size_t staging_bytes = 0;
    uint64_t* d_info = nullptr;  // [P][4] gathered (n, t, pivot, key_bytes)
    uint64_t* d_ag = nullptr;    // all-gather scratch (grown on demand, freed at finalize)
    size_t d_ag_words = 0;
    uint64_t staging_cap_bytes = 256ull << 20;
};
static DistState g_dist;

pp_status dist_unique_id(void* out128) {
    if (!out128) return PP_E_INVAL;
    if (!nccl_load()) return PP_E_NCCL;
    ncclUniqueId id;
    ncclResult_t r = g_nccl.GetUniqueId(&id);
    if (r != ncclSuccess) return nccl_fail(r, "ncclGetUniqueId");
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
    memcpy(out128, &id, 128);
    return PP_OK;
}

pp_status dist_init(const void* id128, int nranks, int rank, int device) {
    if (!id128 || nranks < 1 || rank < 0 || rank >= nranks) {
        set_error("pp_dist_init: bad arguments");
        return PP_E_INVAL;
    }
    if (!nccl_load()) return PP_E_NCCL;
    if (g_dist.comm) {
        set_error("pp_dist_init: already initialised (call pp_dist_finalize first)");
        return PP_E_INVAL;
    }
    cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
    ncclUniqueId id;
    memcpy(&id, id128, 128);
    ncclResult_t r = g_nccl.CommInitRank(&g_dist.comm, nranks, id, rank);
    if (r != ncclSuccess) {
        g_dist.comm = nullptr;
        return nccl_fail(r, "ncclCommInitRank");
    }
    g_dist.nranks = nranks;
    g_dist.rank = rank;
    g_dist.device = device;
    e = cudaMalloc(&g_dist.d_info, sizeof(uint64_t) * 4 * (nranks + 1));
    if (e != cudaSuccess) return cuda_fail(e, "dist info alloc");
    for (auto& ev : g_dist.ev)
        if (!ev) cudaEventCreate(&ev);
    return PP_OK;
}

pp_status dist_last_timing(double* out4) {
    if (!out4) return PP_E_INVAL;
    out4[0] = g_dist.last_local_ms;
    out4[1] = g_dist.last_gather_ms;
    out4[2] = g_dist.last_exchange_ms;
    out4[3] = (double)g_dist.last_bytes;
    return PP_OK;
}

// phase times of the call that just synchronised (events on its stream)
static void dist_read_timing(uint64_t bytes) {
    float a = 0, b = 0, c = 0;
    cudaEventElapsedTime(&a, g_dist.ev[0], g_dist.ev[1]);
    cudaEventElapsedTime(&b, g_dist.ev[1], g_dist.ev[2]);
    cudaEventElapsedTime(&c, g_dist.ev[2], g_dist.ev[3]);
    g_dist.last_local_ms = a;
    g_dist.last_gather_ms = b;
    g_dist.last_exchange_ms = c;
    g_dist.last_bytes = bytes;
}

pp_status dist_finalize() {
    ipc_close_all();
    for (auto& ev : g_dist.ev)
        if (ev) {
            cudaEventDestroy(ev);
            ev = nullptr;
        }
    if (g_dist.comm) g_nccl.CommDestroy(g_dist.comm);
    g_dist.comm = nullptr;
    if (g_dist.staging) cudaFree(g_dist.staging);
    if (g_dist.d_info) cudaFree(g_dist.d_info);
    if (g_dist.d_ag) cudaFree(g_dist.d_ag);
    g_dist.staging = nullptr;
    g_dist.d_info = nullptr;
    g_dist.d_ag = nullptr;
    g_dist.d_ag_words = 0;
    g_dist.staging_bytes = 0;
    return PP_OK;
}

void dist_set_staging(uint64_t bytes) { g_dist.staging_cap_bytes = bytes < 16 ? 16 : bytes; }

static pp_status allgather_u64(const uint64_t* host_in, uint64_t count, std::vector<uint64_t>& host_out,
                               cudaStream_t st);
template <typename K>
static pp_status swap_ranges_impl(const uint64_t* host_tri, uint64_t np, cudaStream_t st, bool sys_fence);

// The exchange one-sidedly over CUDA-IPC peer mappings (param dist_p2p):
// every rank's shard is mapped on every rank (handles + offsets gathered
// once per call, mappings cached), each rank swaps its share of the pairs
// (p2p_pieces) with swap_ranges_kernel directly between its shard and the
// peers' -- no staging buffer, no second copy -- and a final collective keeps
// any rank from returning while a peer may still be writing into its shard.
// Ordering: a rank's swaps are enqueued after the (n_r, t_r) all-gather, which
// completes only once every rank has contributed, i.e. after every rank's
// local partition finished (stream order).  Needs peer access between the
// GPUs (NVLink / NVSwitch); untested here beyond one GPU.
template <typename K>
static pp_status exchange_p2p(K* shard, uint64_t n_local, const std::vector<uint64_t>& ns,
                              const std::vector<uint64_t>& ts, cudaStream_t st, uint64_t* moved) {
    const int P = g_dist.nranks, me = g_dist.rank;
    std::vector<uint64_t> mine(9, 0), all;
    if (n_local > 0) {
        pp_status s = ipc_export(shard, mine.data(), &mine[8]);
        if (s != PP_OK) return s;
    }
    pp_status s = allgather_u64(mine.data(), 9, all, st);
    if (s != PP_OK) return s;
    std::vector<P2PPiece> pcs;
    p2p_pieces(ns.data(), ts.data(), P, me, pcs);
    std::vector<uint64_t> bases(P, 0);
    for (int q = 1; q < P; ++q) bases[q] = bases[q - 1] + ns[q - 1];
    std::vector<K*> ptr(P, nullptr);
    ptr[me] = shard;
    for (const P2PPiece& p : pcs) {
        for (uint64_t q : {p.rank_a, p.rank_b}) {
            if (ptr[q]) continue;
            void* d = nullptr;
            s = ipc_import(&all[9 * q], all[9 * q + 8], &d);
            if (s != PP_OK) return s;
            ptr[q] = static_cast<K*>(d);
        }
    }
    std::vector<uint64_t> tri;
    *moved = 0;  // remote bytes read + written by this rank's swaps
    for (const P2PPiece& p : pcs) {
        *moved += 2 * p.len * sizeof(K);
        tri.push_back(reinterpret_cast<uint64_t>(ptr[p.rank_a] + (p.a - bases[p.rank_a])));
        tri.push_back(reinterpret_cast<uint64_t>(ptr[p.rank_b] + (p.b - bases[p.rank_b])));
        tri.push_back(p.len);
    }
    s = swap_ranges_impl<K>(tri.data(), pcs.size(), st, true);
    if (s != PP_OK) return s;
    std::vector<uint64_t> done;
    const uint64_t one = 1;
    return allgather_u64(&one, 1, done, st);  // no rank leaves before every peer's swaps finished
}

template <typename K>
pp_status partition_dist(K* shard, uint64_t n_local, K pivot, cudaStream_t st, uint64_t* global_split) {
    if (!g_dist.comm) {
        set_error("pp_partition_dist: call pp_dist_init first");
        return PP_E_INVAL;
    }
    const int P = g_dist.nranks, me = g_dist.rank;
    cudaEventRecord(g_dist.ev[0], st);
    // 1. local partition (library kernels), split left in device memory
    uint64_t* d_mine = g_dist.d_info + 4 * P;
    pp_status s = PP_OK;
    if (n_local > 0) {
        s = partition_device<K>(shard, n_local, pivot, st, d_mine + 1, nullptr);
    } else {
        cudaMemsetAsync(d_mine + 1, 0, 8, st);
    }
    if (s != PP_OK) return s;
    cudaEventRecord(g_dist.ev[1], st);
    uint64_t info[3] = {n_local, (uint64_t)pivot, (uint64_t)sizeof(K)};
    cudaError_t e = cudaMemcpyAsync(d_mine, &info[0], 8, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(d_mine + 2, &info[1], 16, cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) return cuda_fail(e, "dist info H2D");
    // 2. allgather (n_r, t_r, pivot, key bytes)
    ncclResult_t r = g_nccl.AllGather(d_mine, g_dist.d_info, 4, ncclUint64, g_dist.comm, st);
    if (r != ncclSuccess) return nccl_fail(r, "ncclAllGather");
    cudaEventRecord(g_dist.ev[2], st);
    std::vector<uint64_t> all(4 * P);
    e = cudaMemcpyAsync(all.data(), g_dist.d_info, 8 * 4 * P, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return cuda_fail(e, "dist gather");
    std::vector<uint64_t> ns(P), ts(P);
    for (int q = 0; q < P; ++q) {
        ns[q] = all[4 * q];
        ts[q] = all[4 * q + 1];
        if (all[4 * q + 2] != (uint64_t)pivot || all[4 * q + 3] != sizeof(K)) {
            set_error("pp_partition_dist: ranks passed different pivots or key types");
            return PP_E_INVAL;
        }
    }
    if (params().dist_p2p && P > 1) {  // one-sided over peer mappings, no staging
        uint64_t Kg = 0;
        for (int q = 0; q < P; ++q) Kg += ts[q];
        uint64_t moved = 0;
        pp_status s2 = exchange_p2p<K>(shard, n_local, ns, ts, st, &moved);
        if (s2 != PP_OK) return s2;
        cudaEventRecord(g_dist.ev[3], st);
        cudaEventSynchronize(g_dist.ev[3]);
        dist_read_timing(moved);
        if (global_split) *global_split = Kg;
        return PP_OK;
    }
    // 3. the same plan on every rank
    const uint64_t cap = std::max<uint64_t>(1, g_dist.staging_cap_bytes / sizeof(K));
    std::vector<Piece> pcs;
    const uint64_t K_global = plan_pieces(ns.data(), ts.data(), P, cap, pcs);
    uint64_t base = 0;
    for (int q = 0; q < me; ++q) base += ns[q];
    // staging: the most this rank receives in one round
    uint64_t need = 0, cur = 0, rnd = ~0ull;
    for (const Piece& p : pcs) {
        if (p.round != rnd) {
            rnd = p.round;
            cur = 0;
        }
        if ((int)p.rank_f == me || (int)p.rank_t == me) cur += p.len;
        need = std::max(need, cur);
    }
    if (need * sizeof(K) > g_dist.staging_bytes) {
        if (g_dist.staging) cudaFree(g_dist.staging);
        g_dist.staging = nullptr;
        g_dist.staging_bytes = 0;
        e = cudaMalloc(&g_dist.staging, need * sizeof(K));
        if (e != cudaSuccess) return cuda_fail(e, "dist staging alloc");
        g_dist.staging_bytes = need * sizeof(K);
    }
    K* staging = static_cast<K*>(g_dist.staging);
    const ncclDataType_t dt = sizeof(K) == 8 ? ncclUint64 : ncclUint32;
    // 4. rounds: send my range, receive the partner's into staging, copy back
    size_t i = 0;
    while (i < pcs.size()) {
        const uint64_t round = pcs[i].round;
        size_t j = i;
        while (j < pcs.size() && pcs[j].round == round) ++j;
        std::vector<uint64_t> offs, soffs, lens;
        uint64_t soff = 0;
        r = g_nccl.GroupStart();
        if (r != ncclSuccess) return nccl_fail(r, "ncclGroupStart");
        for (size_t k = i; k < j; ++k) {
            const Piece& p = pcs[k];
            int peer = -1;
            uint64_t off = 0;
            if ((int)p.rank_f == me) {
                peer = (int)p.rank_t;
                off = p.f - base;
            } else if ((int)p.rank_t == me) {
                peer = (int)p.rank_f;
                off = p.t - base;
            }
            if (peer < 0) continue;
            r = g_nccl.Send(shard + off, p.len, dt, peer, g_dist.comm, st);
            if (r == ncclSuccess) r = g_nccl.Recv(staging + soff, p.len, dt, peer, g_dist.comm, st);
            if (r != ncclSuccess) {
                g_nccl.GroupEnd();
                return nccl_fail(r, "ncclSend/Recv");
            }
            offs.push_back(off);
            soffs.push_back(soff);
            lens.push_back(p.len);
            soff += p.len;
        }
        r = g_nccl.GroupEnd();
        if (r != ncclSuccess) return nccl_fail(r, "ncclGroupEnd");
        for (size_t k = 0; k < offs.size(); ++k) {
            e = cudaMemcpyAsync(shard + offs[k], staging + soffs[k], lens[k] * sizeof(K), cudaMemcpyDeviceToDevice,
                                st);
            if (e != cudaSuccess) return cuda_fail(e, "dist place");
        }
        i = j;
    }
    cudaEventRecord(g_dist.ev[3], st);
    e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return cuda_fail(e, "dist exchange");
    uint64_t sent = 0;  // keys this rank sent (it receives as many)
    for (const Piece& p : pcs)
        if ((int)p.rank_f == me || (int)p.rank_t == me) sent += p.len;
    dist_read_timing(sent * sizeof(K));
    if (global_split) *global_split = K_global;
    return PP_OK;
}

template pp_status partition_dist<uint64_t>(uint64_t*, uint64_t, uint64_t, cudaStream_t, uint64_t*);
template pp_status partition_dist<uint32_t>(uint32_t*, uint64_t, uint32_t, cudaStream_t, uint64_t*);

// ---------------------------------------------------------------------------
// Distributed quicksort (BASELINE config 5 at P GPUs): segments spanning
// several ranks are split by partition_dist (median-of-3 pivot gathered from
// the owning ranks; "x <= p" step when the pivot is the minimum -- DESIGN.md
// R14); spanning segments of <= `small` keys are all-gathered, sorted on
// every participating rank, and each keeps its part.  When no segment spans
// two ranks each shard is a concatenation of whole segments in key order:
// one local quicksort per rank finishes.  Mirrors Partitioner.sort in
// paper_2004_12532_b200/dist.py (tested there over gloo with P = 2..4).
// ---------------------------------------------------------------------------
static pp_status allgather_u64(const uint64_t* host_in, uint64_t count, std::vector<uint64_t>& host_out,
                               cudaStream_t st) {
    const int P = g_dist.nranks;
    const size_t words = count * (P + 1);
    cudaError_t e = cudaSuccess;
    if (words > g_dist.d_ag_words) {  // grow (the previous user synchronised its stream)
        if (g_dist.d_ag) cudaFree(g_dist.d_ag);
        g_dist.d_ag = nullptr;
        g_dist.d_ag_words = 0;
        e = cudaMalloc(&g_dist.d_ag, 8 * words);
        if (e != cudaSuccess) return cuda_fail(e, "allgather buffer");
        g_dist.d_ag_words = words;
    }
    uint64_t* d = g_dist.d_ag;
    e = cudaMemcpyAsync(d + count * P, host_in, 8 * count, cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) return cuda_fail(e, "allgather H2D");
    ncclResult_t r = g_nccl.AllGather(d + count * P, d, count, ncclUint64, g_dist.comm, st);
    if (r != ncclSuccess) return nccl_fail(r, "ncclAllGather");
    host_out.assign(count * P, 0);
    e = cudaMemcpyAsync(host_out.data(), d, 8 * count * P, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);  // also: the buffer is free for the next call
    return e == cudaSuccess ? PP_OK : cuda_fail(e, "allgather D2H");
}

template <typename K>
pp_status quicksort_dist(K* shard, uint64_t n_local, cudaStream_t st, uint64_t small) {
    if (!g_dist.comm) {
        set_error("pp_quicksort_dist: call pp_dist_init first");
        return PP_E_INVAL;
    }
    const int P = g_dist.nranks, me = g_dist.rank;
    const uint64_t KMAXU = (uint64_t)(K)~(K)0;
    std::vector<uint64_t> all;
    pp_status s = allgather_u64(&n_local, 1, all, st);
    if (s != PP_OK) return s;
    std::vector<uint64_t> ns(all), base(P, 0);
    for (int r = 1; r < P; ++r) base[r] = base[r - 1] + ns[r - 1];
    const uint64_t N = base[P - 1] + ns[P - 1], b0 = base[me];
    auto owner = [&](uint64_t x) {
        int r = 0;
        while (r + 1 < P && base[r + 1] <= x) ++r;
        return r;
    };
    auto piece = [&](uint64_t lo, uint64_t hi, uint64_t& pa, uint64_t& pb) {
        const uint64_t a = std::max(lo, b0), b = std::min(hi, b0 + ns[me]);
        if (a < b) { pa = a - b0; pb = b - b0; } else { pa = pb = 0; }
    };
    struct Seg {
        uint64_t lo, hi;
    };
    std::vector<Seg> segs;
    if (N > 1) segs.push_back({0, N});
    cudaError_t e;
    for (;;) {
        std::vector<Seg> span, nxt;
        for (const Seg& sg : segs)
            if (sg.hi - sg.lo > 1 && owner(sg.lo) != owner(sg.hi - 1)) span.push_back(sg);
        if (span.empty()) break;
        for (const Seg& sg : span) {
            const uint64_t lo = sg.lo, hi = sg.hi;
            uint64_t pa, pb;
            piece(lo, hi, pa, pb);
            if (hi - lo <= small) {
                // all-gather the segment, sort it everywhere, keep my part
                std::vector<uint64_t> lens(P);
                uint64_t mx = 0, off = 0;
                for (int r = 0; r < P; ++r) {
                    const uint64_t a = std::max(lo, base[r]), b = std::min(hi, base[r] + ns[r]);
                    lens[r] = a < b ? b - a : 0;
                    mx = std::max(mx, lens[r]);
                    if (r < me) off += lens[r];
                }
                K* d = nullptr;
                e = cudaMalloc(&d, sizeof(K) * (mx * (P + 1) + (hi - lo)));
                if (e != cudaSuccess) return cuda_fail(e, "gather-sort buffer");
                K* mine = d + mx * P;
                K* full = mine + mx;
                if (pb > pa) e = cudaMemcpyAsync(mine, shard + pa, sizeof(K) * (pb - pa), cudaMemcpyDeviceToDevice, st);
                ncclResult_t r = g_nccl.AllGather(mine, d, mx, sizeof(K) == 8 ? ncclUint64 : ncclUint32, g_dist.comm,
                                                  st);
                if (r != ncclSuccess) {
                    cudaFree(d);
                    return nccl_fail(r, "ncclAllGather");
                }
                uint64_t at = 0;
                for (int q = 0; q < P; ++q) {
                    if (lens[q]) cudaMemcpyAsync(full + at, d + mx * q, sizeof(K) * lens[q], cudaMemcpyDeviceToDevice, st);
                    at += lens[q];
                }
                s = quicksort_device<K>(full, hi - lo, st);
                if (s == PP_OK && pb > pa)
                    e = cudaMemcpyAsync(shard + pa, full + off, sizeof(K) * (pb - pa), cudaMemcpyDeviceToDevice, st);
                if (s == PP_OK) e = cudaStreamSynchronize(st);
                cudaFree(d);
                if (s != PP_OK) return s;
                if (e != cudaSuccess) return cuda_fail(e, "gather-sort");
                continue;
            }
            // median of 3 from the owning ranks
            const uint64_t pos[3] = {lo, lo + (hi - lo - 1) / 2, hi - 1};
            uint64_t mv[6] = {0, 0, 0, 0, 0, 0};
            for (int i = 0; i < 3; ++i) {
                if (pos[i] >= b0 && pos[i] < b0 + ns[me]) {
                    K v;
                    e = cudaMemcpy(&v, shard + (pos[i] - b0), sizeof(K), cudaMemcpyDeviceToHost);
                    if (e != cudaSuccess) return cuda_fail(e, "pivot read");
                    mv[2 * i] = 1;
                    mv[2 * i + 1] = (uint64_t)v;
                }
            }
            s = allgather_u64(mv, 6, all, st);
            if (s != PP_OK) return s;
            uint64_t v3[3] = {0, 0, 0};
            for (int i = 0; i < 3; ++i)
                for (int q = 0; q < P; ++q)
                    if (all[6 * q + 2 * i]) {
                        v3[i] = all[6 * q + 2 * i + 1];
                        break;
                    }
            std::sort(v3, v3 + 3);
            const uint64_t p = v3[1];
            uint64_t k = 0;
            s = partition_dist<K>(shard + pa, pb - pa, (K)p, st, &k);
            if (s != PP_OK) return s;
            if (k == 0) {
                if (p == KMAXU) continue;  // all keys equal the maximum
                s = partition_dist<K>(shard + pa, pb - pa, (K)(p + 1), st, &k);
                if (s != PP_OK) return s;
                nxt.push_back({lo + k, hi});  // [lo, lo+k) all equal p
            } else {
                nxt.push_back({lo, lo + k});
                nxt.push_back({lo + k, hi});
            }
        }
        segs.clear();
        for (const Seg& sg : nxt)
            if (sg.hi - sg.lo > 1) segs.push_back(sg);
    }
    if (n_local > 1) {
        s = quicksort_device<K>(shard, n_local, st);
        if (s != PP_OK) return s;
    }
    e = cudaStreamSynchronize(st);
    return e == cudaSuccess ? PP_OK : cuda_fail(e, "quicksort_dist");
}

template pp_status quicksort_dist<uint64_t>(uint64_t*, uint64_t, cudaStream_t, uint64_t);
template pp_status quicksort_dist<uint32_t>(uint32_t*, uint64_t, cudaStream_t, uint64_t);

// ---------------------------------------------------------------------------
// Staging-free exchange primitive: swap ranges [a, a+len)
// <-> [b, b+len) elementwise for every piece, one thread per element pair
// (EREW), grid-stride over all pieces' elements; the piece of an element is
// found by binary search over the length prefix.  a and b are device
// pointers -- with peer-mapped b (CUDA IPC / symmetric memory) one rank
// performs its exchange pieces one-sidedly over NVLink with no staging
// buffer and no second copy; on one GPU it executes a whole plan of emulated
// ranks (tests).  The caller guarantees that no two ranges overlap.
// ---------------------------------------------------------------------------
template <typename K>
__global__ void __launch_bounds__(256) swap_ranges_kernel(const uint64_t* __restrict__ tri,
                                                          const uint64_t* __restrict__ pre, uint64_t np,
                                                          uint64_t total, int sys_fence) {
    for (uint64_t e = (uint64_t)blockIdx.x * 256 + threadIdx.x; e < total; e += (uint64_t)gridDim.x * 256) {
        uint64_t lo = 0, hi = np;  // last piece with pre <= e
        while (hi - lo > 1) {
            const uint64_t mid = (lo + hi) >> 1;
            if (pre[mid] <= e) lo = mid; else hi = mid;
        }
        const uint64_t i = e - pre[lo];
        K* a = reinterpret_cast<K*>(tri[3 * lo]) + i;
        K* b = reinterpret_cast<K*>(tri[3 * lo + 1]) + i;
        const K x = *a, y = *b;
        *a = y;
        *b = x;
    }
    if (sys_fence) __threadfence_system();  // peer writes ordered before the closing collective
}

static uint64_t* g_swap_buf = nullptr;
static size_t g_swap_cap = 0;

template <typename K>
static pp_status swap_ranges_impl(const uint64_t* host_tri, uint64_t np, cudaStream_t st, bool sys_fence) {
    if (np == 0) return PP_OK;
    if (!host_tri) return PP_E_INVAL;
    std::vector<uint64_t> buf(4 * np);  // [3 np triples][np prefix]
    uint64_t total = 0;
    for (uint64_t k = 0; k < np; ++k) {
        buf[3 * k] = host_tri[3 * k];
        buf[3 * k + 1] = host_tri[3 * k + 1];
        buf[3 * k + 2] = host_tri[3 * k + 2];
        if ((host_tri[3 * k] | host_tri[3 * k + 1]) % sizeof(K)) {
            set_error("pp_swap_ranges: unaligned range");
            return PP_E_INVAL;
        }
        buf[3 * np + k] = total;
        total += host_tri[3 * k + 2];
    }
    if (total == 0) return PP_OK;
    if (4 * np > g_swap_cap) {
        cudaStreamSynchronize(st);
        if (g_swap_buf) cudaFree(g_swap_buf);
        g_swap_buf = nullptr;
        g_swap_cap = 0;
        if (cudaMalloc(&g_swap_buf, 8 * 4 * np) != cudaSuccess) {
            cudaGetLastError();
            set_error("pp_swap_ranges: piece buffer allocation failed");
            return PP_E_NOMEM;
        }
        g_swap_cap = 4 * np;
    }
    cudaError_t e = cudaMemcpyAsync(g_swap_buf, buf.data(), 8 * 4 * np, cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) return cuda_fail(e, "pp_swap_ranges H2D");
    const uint64_t blocks = std::min<uint64_t>((total + 255) / 256, (uint64_t)sm_count() * 16);
    swap_ranges_kernel<K><<<(unsigned)blocks, 256, 0, st>>>(g_swap_buf, g_swap_buf + 3 * np, np, total,
                                                            sys_fence ? 1 : 0);
    note_launches(1);
    // the host triples were staged by the (pageable) copy; wait before the
    // vector goes away only if the copy could still read it
    e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    return e == cudaSuccess ? PP_OK : cuda_fail(e, "pp_swap_ranges");
}
template <typename K>
pp_status swap_ranges(const uint64_t* host_tri, uint64_t np, cudaStream_t st) {
    return swap_ranges_impl<K>(host_tri, np, st, false);
}
template pp_status swap_ranges<uint64_t>(const uint64_t*, uint64_t, cudaStream_t);
template pp_status swap_ranges<uint32_t>(const uint64_t*, uint64_t, cudaStream_t);

pp_status dist_p2p_pieces(const uint64_t* ns, const uint64_t* ts, int P, int rank, uint64_t* out, uint64_t out_cap,
                          uint64_t* n_out) {
    if (!ns || !ts || P < 1 || rank < 0 || rank >= P || !n_out) return PP_E_INVAL;
    for (int r = 0; r < P; ++r)
        if (ts[r] > ns[r]) return PP_E_INVAL;
    std::vector<P2PPiece> pcs;
    p2p_pieces(ns, ts, P, rank, pcs);
    *n_out = pcs.size();
    if (out) {
        for (size_t k = 0; k < pcs.size() && k < out_cap; ++k) {
            uint64_t* o = out + 5 * k;
            o[0] = pcs[k].rank_a;
            o[1] = pcs[k].a;
            o[2] = pcs[k].rank_b;
            o[3] = pcs[k].b;
            o[4] = pcs[k].len;
        }
    }
    return pcs.size() <= out_cap || !out ? PP_OK : PP_E_INVAL;
}

pp_status dist_plan(const uint64_t* ns, const uint64_t* ts, int P, uint64_t cap, uint64_t* out, uint64_t out_cap,
                    uint64_t* n_out, uint64_t* K_out) {
    if (!ns || !ts || P < 1 || cap < 1 || !n_out) return PP_E_INVAL;
    for (int r = 0; r < P; ++r)
        if (ts[r] > ns[r]) return PP_E_INVAL;
    std::vector<Piece> pcs;
    const uint64_t K = plan_pieces(ns, ts, P, cap, pcs);
    *n_out = pcs.size();
    if (K_out) *K_out = K;
    if (out) {
        for (size_t k = 0; k < pcs.size() && k < out_cap; ++k) {
            const Piece& p = pcs[k];
            uint64_t* o = out + 6 * k;
            o[0] = p.round;
            o[1] = p.rank_f;
            o[2] = p.f;
            o[3] = p.rank_t;
            o[4] = p.t;
            o[5] = p.len;
        }
    }
    return pcs.size() <= out_cap || !out ? PP_OK : PP_E_INVAL;
}

}  // namespace pp
