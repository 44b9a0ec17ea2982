// pp_dist.cu -- multi-GPU partition and quicksort of one array sharded
// contiguously over ranks (BASELINE config 3 / config 5 at P GPUs; SURVEY
// §8(a) a8, §8(e)).  A rank partitions its shard(s) locally with the
// single-GPU kernels, all-gathers (status, n_r, t_r, pivot) once, computes the
// exchange plan identically on every rank (a merge of the misplaced-successor
// ranges left of K with the misplaced-predecessor ranges right of K), and
// moves the matched ranges either through bounded staging (grouped
// send/recv rounds) or one-sidedly through peer mappings (param dist_p2p).
//
// The algorithm is written once against a Transport:
//   * NcclTransport -- the product path: NCCL (loaded at run time, the copy
//     PyTorch already loaded) with a NON-BLOCKING communicator; every wait
//     polls the stream and ncclCommGetAsyncError with a timeout and aborts the
//     communicator on failure, so a dead peer turns into PP_E_NCCL instead of
//     a hang.  Peer mappings through CUDA IPC.
//   * LoopTransport -- P emulated ranks as host threads of one process on one
//     GPU (disjoint slices of one device array): collectives rendezvous on a
//     host barrier and every received piece is ONE plain cudaMemcpyAsync from
//     the sender's range.  This runs the same plan -> rounds -> staging ->
//     place code (and the one-sided share rule) at P > 1 on a single GPU
//     (pp_*_dist_loopback_*; tests/test_gpu_dist.py).
// Every collective call agrees on a status before it returns: a rank that
// fails locally still takes part in the next all-gather with its status set,
// and every rank returns the same error.
#include <dlfcn.h>

#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <cstring>
#include <deque>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include <cuda.h>  // driver types only (cuMemGetAddressRange is fetched through the runtime)
#include <nccl.h>

#include "pp_device.cuh"
#include "pp_internal.h"

namespace pp {

void note_launches(uint64_t k);

// ---------------------------------------------------------------------------
// The exchange plan (host arithmetic; mirrored independently in Python by
// tests/dist_mirror.py and cross-checked by tests/test_dist.py).
// ---------------------------------------------------------------------------
struct Run {  // swap [a, a+len) on rank ra (misplaced successors) with [b, b+len) on rank rb (predecessors)
    uint64_t ra, a, rb, b, len;
};
struct Piece {
    uint64_t round, rank_f, f, rank_t, t, len;
};

// Pairs the i-th misplaced successor (global order, left of K) with the i-th
// misplaced predecessor (right of K): one run per maximal matched stretch.
// Positions are global (shard base of rank r = sum of ns[<r]).
static uint64_t match_runs(const uint64_t* ns, const uint64_t* ts, int P, std::vector<Run>& out) {
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
    size_t i = 0, j = 0;
    while (i < F.size() && j < T.size()) {
        const uint64_t m = std::min(F[i].e - F[i].s, T[j].e - T[j].s);
        out.push_back({F[i].rank, F[i].s, T[j].rank, T[j].s, m});
        F[i].s += m;
        T[j].s += m;
        if (F[i].s == F[i].e) ++i;
        if (T[j].s == T[j].e) ++j;
    }
    return K;
}

// Splits runs into pieces of <= cap keys and groups them into rounds in which
// no rank moves more than cap keys (a piece opens a new round when either of
// its ranks would exceed cap).  Identical on every rank.
static void schedule_rounds(const std::vector<Run>& runs, int P, uint64_t cap, std::vector<Piece>& out) {
    out.clear();
    std::vector<uint64_t> used(P, 0);
    uint64_t round = 0;
    for (const Run& r : runs) {
        for (uint64_t s = 0; s < r.len;) {
            const uint64_t len = std::min(cap, r.len - s);
            if (used[r.ra] + len > cap || used[r.rb] + len > cap) {
                ++round;
                std::fill(used.begin(), used.end(), 0);
            }
            out.push_back({round, r.ra, r.a + s, r.rb, r.b + s, len});
            used[r.ra] += len;
            used[r.rb] += len;
            s += len;
        }
    }
}

static uint64_t plan_pieces(const uint64_t* ns, const uint64_t* ts, int P, uint64_t cap, std::vector<Piece>& out) {
    std::vector<Run> runs;
    const uint64_t K = match_runs(ns, ts, P, runs);
    schedule_rounds(runs, P, cap, out);
    return K;
}

// One-sided (staging-free) exchange: who executes which pairs.  Every run
// has its two ranks distinct (a shard's misplaced keys are all successors --
// it ends left of K -- or all predecessors).  The left rank swaps the first
// ceil(len/2) pairs, the right rank the rest, each reading and writing its
// partner's keys through the peer mapping, so both directions of every link
// carry traffic.  Mirrored by tests/dist_mirror.py p2p_pieces.
static void p2p_share(const std::vector<Run>& runs, int me, std::vector<Run>& out) {
    out.clear();
    for (const Run& p : runs) {
        const uint64_t h = (p.len + 1) / 2;
        if ((int)p.ra == me) out.push_back({p.ra, p.a, p.rb, p.b, h});
        if ((int)p.rb == me && p.len > h) out.push_back({p.ra, p.a + h, p.rb, p.b + h, p.len - h});
    }
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
// Transport interface.
// ---------------------------------------------------------------------------
static constexpr int kPeerWords = 9;  // exported peer record (after the status word)

struct Transport {
    int P = 1, me = 0;
    virtual ~Transport() = default;
    // all-gather `bytes` per rank: device d_send -> device d_recv[P * bytes]
    virtual pp_status allgather(const void* d_send, void* d_recv, size_t bytes, cudaStream_t st) = 0;
    // grouped point-to-point; matched per (src, dst) pair in issue order
    virtual pp_status group_start() = 0;
    virtual pp_status send(const void* d, size_t bytes, int peer, cudaStream_t st) = 0;
    virtual pp_status recv(void* d, size_t bytes, int peer, cudaStream_t st) = 0;
    virtual pp_status group_end(cudaStream_t st) = 0;
    // wait for everything enqueued on st, detecting peer failures
    virtual pp_status wait(cudaStream_t st) = 0;
    // one-sided exchange: describe a local device range / map a peer's
    virtual pp_status export_range(void* d, uint64_t* rec) = 0;
    virtual pp_status import_range(const uint64_t* rec, void** d) = 0;
    // local library calls (the loopback serialises them: one process-wide workspace)
    virtual void local_begin() {}
    virtual pp_status local_end(cudaStream_t) { return PP_OK; }
    // test hooks (loopback only): a rank that never arrives
    virtual bool absent() const { return false; }
};

// ---------------------------------------------------------------------------
// NCCL, loaded at run time.
// ---------------------------------------------------------------------------
struct NcclApi {
    void* lib = nullptr;
    decltype(&ncclGetUniqueId) GetUniqueId = nullptr;
    decltype(&ncclCommInitRankConfig) CommInitRankConfig = nullptr;
    decltype(&ncclCommDestroy) CommDestroy = nullptr;
    decltype(&ncclCommAbort) CommAbort = nullptr;
    decltype(&ncclCommGetAsyncError) CommGetAsyncError = nullptr;
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
    PP_SYM(CommInitRankConfig, "ncclCommInitRankConfig")
    PP_SYM(CommDestroy, "ncclCommDestroy")
    PP_SYM(CommAbort, "ncclCommAbort")
    PP_SYM(CommGetAsyncError, "ncclCommGetAsyncError")
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

static double now_ms() {
    using namespace std::chrono;
    return duration<double, std::milli>(steady_clock::now().time_since_epoch()).count();
}

struct NcclTransport : Transport {
    ncclComm_t comm = nullptr;
    bool dead = false;

    pp_status fail(const std::string& what) {
        if (comm && !dead) g_nccl.CommAbort(comm);  // unblocks kernels waiting on a dead peer
        dead = true;
        set_error(what);
        return PP_E_NCCL;
    }
    // Non-blocking communicator: a call may return ncclInProgress; poll the
    // communicator's async state until it settles, with a timeout.
    pp_status settle(ncclResult_t r, const char* what) {
        if (dead) return fail(std::string(what) + ": communicator aborted earlier");
        const double t0 = now_ms(), lim = (double)params().dist_timeout_ms;
        while (r == ncclInProgress) {
            if (now_ms() - t0 > lim) return fail(std::string(what) + ": timed out (dist_timeout_ms)");
            std::this_thread::yield();
            ncclResult_t a = ncclSuccess;
            g_nccl.CommGetAsyncError(comm, &a);
            r = a;
        }
        if (r != ncclSuccess) return fail(std::string(what) + ": " + g_nccl.GetErrorString(r));
        return PP_OK;
    }
    pp_status allgather(const void* d_send, void* d_recv, size_t bytes, cudaStream_t st) override {
        return settle(g_nccl.AllGather(d_send, d_recv, bytes, ncclUint8, comm, st), "ncclAllGather");
    }
    pp_status group_start() override { return settle(g_nccl.GroupStart(), "ncclGroupStart"); }
    pp_status send(const void* d, size_t bytes, int peer, cudaStream_t st) override {
        return settle(g_nccl.Send(d, bytes, ncclUint8, peer, comm, st), "ncclSend");
    }
    pp_status recv(void* d, size_t bytes, int peer, cudaStream_t st) override {
        return settle(g_nccl.Recv(d, bytes, ncclUint8, peer, comm, st), "ncclRecv");
    }
    pp_status group_end(cudaStream_t) override { return settle(g_nccl.GroupEnd(), "ncclGroupEnd"); }
    // stream completion polled together with the communicator's async error
    // (a failed or vanished peer), bounded by dist_timeout_ms
    pp_status wait(cudaStream_t st) override {
        if (dead) return fail("communicator aborted earlier");
        const double t0 = now_ms(), lim = (double)params().dist_timeout_ms;
        for (;;) {
            cudaError_t e = cudaStreamQuery(st);
            if (e == cudaSuccess) return PP_OK;
            if (e != cudaErrorNotReady) return cuda_fail(e, "dist stream");
            ncclResult_t a = ncclSuccess;
            g_nccl.CommGetAsyncError(comm, &a);
            if (a != ncclSuccess && a != ncclInProgress)
                return fail(std::string("NCCL async error: ") + g_nccl.GetErrorString(a));
            const double el = now_ms() - t0;
            if (el > lim) return fail("dist wait timed out (dist_timeout_ms); communicator aborted");
            if (el > 1.0) std::this_thread::sleep_for(std::chrono::microseconds(20));  // spin the first ms
            else std::this_thread::yield();
        }
    }
    pp_status export_range(void* d, uint64_t* rec) override {
        std::memset(rec, 0, 8 * kPeerWords);
        return d ? ipc_export(d, rec, &rec[8]) : PP_OK;
    }
    pp_status import_range(const uint64_t* rec, void** d) override { return ipc_import(rec, rec[8], d); }
};

// ---------------------------------------------------------------------------
// Loopback: P emulated ranks = P host threads of this process, one GPU.
// ---------------------------------------------------------------------------
struct LoopHub {
    int P = 1;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    uint64_t gen = 0;
    bool broken = false;
    std::vector<const void*> slot;                               // per rank: all-gather source
    std::vector<std::deque<std::pair<const void*, size_t>>> box;  // [src * P + dst]: posted sends, FIFO
    std::mutex local_mu;                                         // serialises local library calls

    explicit LoopHub(int p) : P(p), slot(p, nullptr), box((size_t)p * p) {}

    pp_status barrier() {
        std::unique_lock<std::mutex> lk(mu);
        if (broken) return PP_E_NCCL;
        const uint64_t g = gen;
        if (++arrived == P) {
            arrived = 0;
            ++gen;
            cv.notify_all();
            return PP_OK;
        }
        const auto lim = std::chrono::milliseconds(params().dist_timeout_ms);
        if (!cv.wait_for(lk, lim, [&] { return gen != g || broken; })) {
            broken = true;  // a rank never arrived: every waiting and later rank fails
            cv.notify_all();
        }
        if (gen != g) return PP_OK;
        set_error("loopback rendezvous timed out (a rank did not arrive; dist_timeout_ms)");
        return PP_E_NCCL;
    }
};

struct LoopTransport : Transport {
    LoopHub* hub = nullptr;
    bool absent_ = false;
    struct Pend {
        int peer;
        const void* src;
        void* dst;
        size_t bytes;
    };
    std::vector<Pend> sends, recvs;

    pp_status allgather(const void* d_send, void* d_recv, size_t bytes, cudaStream_t st) override {
        pp_status s = wait(st);  // the source is ready
        if (s != PP_OK) return s;
        {
            std::lock_guard<std::mutex> lk(hub->mu);
            hub->slot[me] = d_send;
        }
        if ((s = hub->barrier()) != PP_OK) return s;
        for (int q = 0; q < P; ++q) {
            const void* src;
            {
                std::lock_guard<std::mutex> lk(hub->mu);
                src = hub->slot[q];
            }
            cudaError_t e = cudaMemcpyAsync(static_cast<char*>(d_recv) + bytes * q, src, bytes,
                                            cudaMemcpyDeviceToDevice, st);
            if (e != cudaSuccess) return cuda_fail(e, "loopback all-gather copy");
        }
        if ((s = wait(st)) != PP_OK) return s;
        return hub->barrier();  // no rank reuses its source before every peer copied it
    }
    pp_status group_start() override {
        sends.clear();
        recvs.clear();
        return PP_OK;
    }
    pp_status send(const void* d, size_t bytes, int peer, cudaStream_t) override {
        sends.push_back({peer, d, nullptr, bytes});
        return PP_OK;
    }
    pp_status recv(void* d, size_t bytes, int peer, cudaStream_t) override {
        recvs.push_back({peer, nullptr, d, bytes});
        return PP_OK;
    }
    pp_status group_end(cudaStream_t st) override {
        pp_status s = wait(st);
        if (s != PP_OK) return s;
        {
            std::lock_guard<std::mutex> lk(hub->mu);
            for (const Pend& p : sends) hub->box[(size_t)me * P + p.peer].push_back({p.src, p.bytes});
        }
        if ((s = hub->barrier()) != PP_OK) return s;
        for (const Pend& p : recvs) {  // one plain copy per received piece, from the sender's range
            std::pair<const void*, size_t> m{nullptr, 0};
            {
                std::lock_guard<std::mutex> lk(hub->mu);
                auto& q = hub->box[(size_t)p.peer * P + me];
                if (!q.empty()) {
                    m = q.front();
                    q.pop_front();
                }
            }
            if (!m.first || m.second != p.bytes) {
                set_error("loopback: unmatched send/recv (plan differs between ranks)");
                return PP_E_INTERNAL;
            }
            cudaError_t e = cudaMemcpyAsync(p.dst, m.first, p.bytes, cudaMemcpyDeviceToDevice, st);
            if (e != cudaSuccess) return cuda_fail(e, "loopback piece copy");
        }
        sends.clear();
        recvs.clear();
        if ((s = wait(st)) != PP_OK) return s;
        return hub->barrier();  // senders keep their ranges until every receiver copied them
    }
    pp_status wait(cudaStream_t st) override {
        cudaError_t e = cudaStreamSynchronize(st);
        return e == cudaSuccess ? PP_OK : cuda_fail(e, "loopback stream");
    }
    pp_status export_range(void* d, uint64_t* rec) override {
        std::memset(rec, 0, 8 * kPeerWords);
        rec[0] = reinterpret_cast<uint64_t>(d);  // same process: the address itself
        return PP_OK;
    }
    pp_status import_range(const uint64_t* rec, void** d) override {
        *d = reinterpret_cast<void*>(rec[0]);
        return PP_OK;
    }
    void local_begin() override { hub->local_mu.lock(); }
    pp_status local_end(cudaStream_t st) override {
        pp_status s = wait(st);  // the shared workspace is free for the next emulated rank
        hub->local_mu.unlock();
        return s;
    }
    bool absent() const override { return absent_; }
};

// ---------------------------------------------------------------------------
// Per-rank context (one in the NCCL process; one per thread in the loopback).
// ---------------------------------------------------------------------------
struct DistCtx {
    Transport* tp = nullptr;
    int P = 1, me = 0, device = 0;
    void* staging = nullptr;
    size_t staging_bytes = 0;
    uint64_t* d_ag = nullptr;  // all-gather scratch (words)
    size_t d_ag_words = 0;
    void* gs = nullptr;  // gather-sort scratch
    size_t gs_bytes = 0;
    uint64_t* d_swap = nullptr;  // one-sided swap piece table
    size_t d_swap_words = 0;
    cudaEvent_t ev[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};  // start, local done, gathered, exchanged, join
    // staged exchange: the copies staging -> shard of round r run on pst while
    // round r+1 transfers into the other staging half
    cudaStream_t pst = nullptr;
    cudaEvent_t ev_recv[2] = {nullptr, nullptr}, ev_place[2] = {nullptr, nullptr};
    // count-first overlapped exchange (dist_overlap): exchange stream, one
    // event per chunk, per-chunk count partials + the local splits' check words
    cudaStream_t xst = nullptr;
    std::vector<cudaEvent_t> ev_chunk;
    uint64_t* d_cnt = nullptr;
    size_t d_cnt_words = 0;
    double last_local_ms = 0, last_gather_ms = 0, last_exchange_ms = 0;
    uint64_t last_bytes = 0;

    pp_status init_overlap(size_t chunks, size_t cnt_words) {
        if (!xst && cudaStreamCreateWithFlags(&xst, cudaStreamNonBlocking) != cudaSuccess)
            return cuda_fail(cudaGetLastError(), "stream");
        while (ev_chunk.size() < chunks) {
            cudaEvent_t e = nullptr;
            if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess)
                return cuda_fail(cudaGetLastError(), "event");
            ev_chunk.push_back(e);
        }
        if (cnt_words > d_cnt_words) {
            if (d_cnt) cudaFree(d_cnt);
            d_cnt = nullptr;
            d_cnt_words = 0;
            if (cudaMalloc(&d_cnt, 8 * cnt_words) != cudaSuccess) {
                cudaGetLastError();
                set_error("dist overlap scratch cudaMalloc failed");
                return PP_E_NOMEM;
            }
            d_cnt_words = cnt_words;
        }
        return PP_OK;
    }

    pp_status init_events() {
        for (auto& e : ev)
            if (!e && cudaEventCreate(&e) != cudaSuccess) return cuda_fail(cudaGetLastError(), "event");
        for (int h = 0; h < 2; ++h) {
            if (!ev_recv[h] && cudaEventCreateWithFlags(&ev_recv[h], cudaEventDisableTiming) != cudaSuccess)
                return cuda_fail(cudaGetLastError(), "event");
            if (!ev_place[h] && cudaEventCreateWithFlags(&ev_place[h], cudaEventDisableTiming) != cudaSuccess)
                return cuda_fail(cudaGetLastError(), "event");
        }
        if (!pst && cudaStreamCreateWithFlags(&pst, cudaStreamNonBlocking) != cudaSuccess)
            return cuda_fail(cudaGetLastError(), "stream");
        return PP_OK;
    }
    void release() {
        if (pst) cudaStreamSynchronize(pst);
        if (xst) cudaStreamSynchronize(xst);
        for (cudaEvent_t e : ev_chunk) cudaEventDestroy(e);
        ev_chunk.clear();
        if (xst) cudaStreamDestroy(xst);
        xst = nullptr;
        if (d_cnt) cudaFree(d_cnt);
        d_cnt = nullptr;
        d_cnt_words = 0;
        for (auto& e : ev)
            if (e) {
                cudaEventDestroy(e);
                e = nullptr;
            }
        for (int h = 0; h < 2; ++h) {
            if (ev_recv[h]) cudaEventDestroy(ev_recv[h]);
            if (ev_place[h]) cudaEventDestroy(ev_place[h]);
            ev_recv[h] = ev_place[h] = nullptr;
        }
        if (pst) cudaStreamDestroy(pst);
        pst = nullptr;
        if (staging) cudaFree(staging);
        if (d_ag) cudaFree(d_ag);
        if (gs) cudaFree(gs);
        if (d_swap) cudaFree(d_swap);
        staging = gs = nullptr;
        d_ag = d_swap = nullptr;
        staging_bytes = gs_bytes = d_ag_words = d_swap_words = 0;
    }
};

static NcclTransport g_nccl_tp;
static DistCtx g_ctx;
static uint64_t g_staging_cap_bytes = 256ull << 20;

pp_status dist_unique_id(void* out128) {
    if (!out128) return PP_E_INVAL;
    if (!nccl_load()) return PP_E_NCCL;
    ncclUniqueId id;
    ncclResult_t r = g_nccl.GetUniqueId(&id);
    if (r != ncclSuccess) {
        set_error(std::string("ncclGetUniqueId: ") + g_nccl.GetErrorString(r));
        return PP_E_NCCL;
    }
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
    if (g_ctx.tp) {
        set_error("pp_dist_init: already initialised (call pp_dist_finalize first)");
        return PP_E_INVAL;
    }
    cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
    ncclUniqueId id;
    memcpy(&id, id128, 128);
    ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
    cfg.blocking = 0;  // every call returns; waits poll with a timeout (NcclTransport::settle / wait)
    g_nccl_tp = NcclTransport();
    ncclResult_t r = g_nccl.CommInitRankConfig(&g_nccl_tp.comm, nranks, id, rank, &cfg);
    if (r != ncclSuccess && r != ncclInProgress) {
        g_nccl_tp.comm = nullptr;
        set_error(std::string("ncclCommInitRankConfig: ") + g_nccl.GetErrorString(r));
        return PP_E_NCCL;
    }
    if (g_nccl_tp.settle(r, "ncclCommInitRankConfig") != PP_OK) {
        g_nccl_tp.comm = nullptr;
        return PP_E_NCCL;
    }
    g_nccl_tp.P = nranks;
    g_nccl_tp.me = rank;
    g_ctx = DistCtx();
    g_ctx.tp = &g_nccl_tp;
    g_ctx.P = nranks;
    g_ctx.me = rank;
    g_ctx.device = device;
    return g_ctx.init_events();
}

pp_status dist_last_timing(double* out4) {
    if (!out4) return PP_E_INVAL;
    out4[0] = g_ctx.last_local_ms;
    out4[1] = g_ctx.last_gather_ms;
    out4[2] = g_ctx.last_exchange_ms;
    out4[3] = (double)g_ctx.last_bytes;
    return PP_OK;
}

pp_status dist_finalize() {
    ipc_close_all();
    g_ctx.release();
    if (g_nccl_tp.comm) {
        if (g_nccl_tp.dead)
            ;  // aborted already (CommAbort frees it)
        else
            g_nccl.CommDestroy(g_nccl_tp.comm);
    }
    g_nccl_tp = NcclTransport();
    g_ctx = DistCtx();
    return PP_OK;
}

void dist_set_staging(uint64_t bytes) { g_staging_cap_bytes = bytes < 16 ? 16 : bytes; }

// ---------------------------------------------------------------------------
// Collective helpers on a context.
// ---------------------------------------------------------------------------
// all-gather scratch of >= words (grown identically on every rank: same call
// sequence; every collective call ends with a wait, so nothing uses it)
static pp_status ensure_ag(DistCtx& c, size_t words) {
    if (words <= c.d_ag_words) return PP_OK;
    if (c.d_ag) cudaFree(c.d_ag);
    c.d_ag = nullptr;
    c.d_ag_words = 0;
    words = std::max<size_t>(words, 256);
    cudaError_t e = cudaMalloc(&c.d_ag, 8 * words);
    if (e != cudaSuccess) return cuda_fail(e, "all-gather scratch");
    c.d_ag_words = words;
    return PP_OK;
}

// host words -> all ranks' words (count per rank), through the device scratch
static pp_status ag_host(DistCtx& c, const uint64_t* in, uint64_t count, std::vector<uint64_t>& out, cudaStream_t st) {
    pp_status s = ensure_ag(c, count * (c.P + 1));
    if (s != PP_OK) return s;
    uint64_t* d = c.d_ag;
    cudaError_t e = cudaMemcpyAsync(d + count * c.P, in, 8 * count, cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) return cuda_fail(e, "all-gather H2D");
    s = c.tp->allgather(d + count * c.P, d, 8 * count, st);
    if (s != PP_OK) return s;
    out.assign(count * c.P, 0);
    e = cudaMemcpyAsync(out.data(), d, 8 * count * c.P, cudaMemcpyDeviceToHost, st);
    if (e != cudaSuccess) return cuda_fail(e, "all-gather D2H");
    return c.tp->wait(st);
}

// Every rank contributes its status; all return the lowest-ranked failure.
static pp_status agree(DistCtx& c, pp_status mine, cudaStream_t st) {
    const uint64_t w = (uint64_t)mine;
    std::vector<uint64_t> all;
    pp_status s = ag_host(c, &w, 1, all, st);
    if (s != PP_OK) return s;
    for (int q = 0; q < c.P; ++q)
        if (all[q] != PP_OK) {
            if (q != c.me) set_error("peer rank " + std::to_string(q) + " failed with status " + std::to_string(all[q]));
            return (pp_status)all[q];
        }
    return PP_OK;
}

static pp_status grow(void** p, size_t* have, size_t want) {
    if (want <= *have) return PP_OK;
    if (*p) cudaFree(*p);
    *p = nullptr;
    *have = 0;
    cudaError_t e = cudaMalloc(p, want);
    if (e != cudaSuccess) {
        cudaGetLastError();
        *p = nullptr;
        set_error("dist buffer cudaMalloc of " + std::to_string(want) + " bytes failed");
        return PP_E_NOMEM;
    }
    *have = want;
    return PP_OK;
}

// ---------------------------------------------------------------------------
// Staging-free exchange primitive: swap ranges [a, a+len)
// <-> [b, b+len) elementwise for every piece, one thread per element pair
// (EREW), grid-stride over all pieces' elements; the piece of an element is
// found by binary search over the length prefix.  a and b are device
// pointers -- with peer-mapped b (CUDA IPC) one rank performs its exchange
// pieces one-sidedly with no staging buffer and no second copy.  The caller
// guarantees that no two ranges overlap.
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

// Enqueues the swaps on st; the piece table is copied into *buf (grown; the
// previous user synchronised) from host memory that the call keeps alive
// until the copy is done (it waits for st before returning).
template <typename K>
static pp_status swap_ranges_impl(const uint64_t* host_tri, uint64_t np, cudaStream_t st, bool sys_fence,
                                  uint64_t** buf, size_t* cap_words) {
    if (np == 0) return PP_OK;
    if (!host_tri) return PP_E_INVAL;
    std::vector<uint64_t> tab(4 * np);  // [3 np triples][np prefix]
    uint64_t total = 0;
    for (uint64_t k = 0; k < np; ++k) {
        tab[3 * k] = host_tri[3 * k];
        tab[3 * k + 1] = host_tri[3 * k + 1];
        tab[3 * k + 2] = host_tri[3 * k + 2];
        if ((host_tri[3 * k] | host_tri[3 * k + 1]) % sizeof(K)) {
            set_error("pp_swap_ranges: unaligned range");
            return PP_E_INVAL;
        }
        tab[3 * np + k] = total;
        total += host_tri[3 * k + 2];
    }
    if (total == 0) return PP_OK;
    if (4 * np > *cap_words) {
        cudaStreamSynchronize(st);
        size_t have = *cap_words * 8;
        void* p = *buf;
        pp_status s = grow(&p, &have, 8 * 4 * np);
        *buf = static_cast<uint64_t*>(p);
        *cap_words = have / 8;
        if (s != PP_OK) return s;
    }
    cudaError_t e = cudaMemcpyAsync(*buf, tab.data(), 8 * 4 * np, cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) return cuda_fail(e, "pp_swap_ranges H2D");
    const uint64_t blocks = std::min<uint64_t>((total + 255) / 256, (uint64_t)sm_count() * 16);
    swap_ranges_kernel<K><<<(unsigned)blocks, 256, 0, st>>>(*buf, *buf + 3 * np, np, total, sys_fence ? 1 : 0);
    note_launches(1);
    e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);  // the host table stays alive until the copy ran
    return e == cudaSuccess ? PP_OK : cuda_fail(e, "pp_swap_ranges");
}

static uint64_t* g_swap_buf = nullptr;
static size_t g_swap_cap = 0;
template <typename K>
pp_status swap_ranges(const uint64_t* host_tri, uint64_t np, cudaStream_t st) {
    return swap_ranges_impl<K>(host_tri, np, st, false, &g_swap_buf, &g_swap_cap);
}
template pp_status swap_ranges<uint64_t>(const uint64_t*, uint64_t, cudaStream_t);
template pp_status swap_ranges<uint32_t>(const uint64_t*, uint64_t, cudaStream_t);

// ---------------------------------------------------------------------------
// Staged exchange: rounds of grouped send/recv into one half of a
// double-buffered staging buffer, then a copy into place on the side stream
// pst, which overlaps the next round's transfer into the other half.  Round
// r+1's sends read ranges disjoint from round r's place targets; a half is
// reused only after its previous place copies (ev_place).  The state carries
// across calls (the overlapped exchange runs one call per chunk step).
// ---------------------------------------------------------------------------
struct StagedState {
    uint64_t rno = 0;
    bool placed[2] = {false, false};
};

template <typename K>
static pp_status staged_rounds(DistCtx& c, K* shard, const std::vector<Piece>& pcs, uint64_t half, cudaStream_t xs,
                               StagedState& ss, uint64_t& moved) {
    Transport& tp = *c.tp;
    const int me = c.me;
    size_t i = 0;
    while (i < pcs.size()) {
        const uint64_t round = pcs[i].round;
        const int hf = (int)(ss.rno++ & 1);
        K* staging = static_cast<K*>(c.staging) + (size_t)hf * half;
        if (ss.placed[hf] && cudaStreamWaitEvent(xs, c.ev_place[hf], 0) != cudaSuccess)
            return cuda_fail(cudaGetLastError(), "dist staging order");
        size_t j = i;
        while (j < pcs.size() && pcs[j].round == round) ++j;
        std::vector<uint64_t> offs, soffs, lens;
        uint64_t soff = 0;
        pp_status sr = tp.group_start();
        for (size_t k = i; k < j && sr == PP_OK; ++k) {
            const Piece& p = pcs[k];
            int peer = -1;
            uint64_t off = 0;
            if ((int)p.rank_f == me) {
                peer = (int)p.rank_t;
                off = p.f;
            } else if ((int)p.rank_t == me) {
                peer = (int)p.rank_f;
                off = p.t;
            }
            if (peer < 0) continue;
            sr = tp.send(shard + off, p.len * sizeof(K), peer, xs);
            if (sr == PP_OK) sr = tp.recv(staging + soff, p.len * sizeof(K), peer, xs);
            offs.push_back(off);
            soffs.push_back(soff);
            lens.push_back(p.len);
            soff += p.len;
            moved += p.len * sizeof(K);
        }
        const pp_status se = tp.group_end(xs);
        if (sr == PP_OK) sr = se;
        if (sr != PP_OK) return sr;
        if (!offs.empty()) {
            cudaError_t e = cudaEventRecord(c.ev_recv[hf], xs);
            if (e == cudaSuccess) e = cudaStreamWaitEvent(c.pst, c.ev_recv[hf], 0);
            for (size_t k = 0; k < offs.size() && e == cudaSuccess; ++k)
                e = cudaMemcpyAsync(shard + offs[k], staging + soffs[k], lens[k] * sizeof(K), cudaMemcpyDeviceToDevice,
                                    c.pst);
            if (e == cudaSuccess) e = cudaEventRecord(c.ev_place[hf], c.pst);
            if (e != cudaSuccess) return cuda_fail(e, "dist place");
            ss.placed[hf] = true;
        }
        i = j;
    }
    return PP_OK;
}

// the exchange on xs ends when every place copy has
static pp_status staged_join(DistCtx& c, cudaStream_t xs, const StagedState& ss) {
    for (int h = 0; h < 2; ++h)
        if (ss.placed[h] && cudaStreamWaitEvent(xs, c.ev_place[h], 0) != cudaSuccess)
            return cuda_fail(cudaGetLastError(), "dist place join");
    return PP_OK;
}

// ---------------------------------------------------------------------------
// Batched distributed partition: S segments, each a contiguous range of the
// global array cut into per-rank pieces (a piece may be empty); every
// segment is partitioned by its own pivot.  One record all-gather for all
// segments, one exchange (all segments' runs in one round schedule).
// ---------------------------------------------------------------------------
struct SegPiece {
    uint64_t off, len;  // this rank's piece: shard[off, off + len)
    uint64_t pivot;
};

template <typename K>
static pp_status partition_multi(DistCtx& c, K* shard, const std::vector<SegPiece>& mine, cudaStream_t st,
                                 std::vector<uint64_t>& K_out, bool timing) {
    Transport& tp = *c.tp;
    const int P = c.P, me = c.me;
    const size_t S = mine.size();
    if (tp.absent()) {  // test hook: this rank never takes part
        set_error("rank absent (dist_fault = 2)");
        return PP_E_INTERNAL;
    }
    const size_t RW = 2 + 4 * S;  // record: [status, key bytes, n[S], pivot[S], off[S], t[S]]
    if (timing) cudaEventRecord(c.ev[0], st);
    pp_status s = PP_OK;
    uint64_t my_total = 0;
    for (const SegPiece& p : mine) my_total += p.len;
    // staging: a rank moves <= min(cap, its misplaced keys) per round
    const uint64_t cap = std::max<uint64_t>(1, g_staging_cap_bytes / sizeof(K));
    // two staging halves of min(cap, my misplaced keys) each (double-buffered rounds)
    const uint64_t half = std::max<uint64_t>(1, std::min(cap, my_total));
    if (!params().dist_p2p && P > 1) s = grow(&c.staging, &c.staging_bytes, 2 * sizeof(K) * half);
    {  // record scratch: [P gathered records][my record]; without it this rank cannot take part
        const pp_status sa = ensure_ag(c, RW * (P + 1));
        if (sa != PP_OK) return sa;
    }
    if (s == PP_OK && params().dist_fault == 1 && params().dist_fault_rank == me) {
        set_error("injected local failure (dist_fault = 1)");
        s = PP_E_INTERNAL;
    }
    uint64_t* rec = c.d_ag + RW * P;  // my record (device); t[] is written by the local partitions
    // 1. local partitions (library kernels)
    if (s == PP_OK) {
        tp.local_begin();
        for (size_t k = 0; k < S && s == PP_OK; ++k) {
            uint64_t* t_slot = rec + 2 + 3 * S + k;
            if (mine[k].len > 0)
                s = partition_device<K>(shard + mine[k].off, mine[k].len, (K)mine[k].pivot, st, t_slot, nullptr);
            else if (cudaMemsetAsync(t_slot, 0, 8, st) != cudaSuccess)
                s = cuda_fail(cudaGetLastError(), "memset");
        }
        const pp_status s2 = tp.local_end(st);
        if (s == PP_OK) s = s2;
    }
    if (timing) cudaEventRecord(c.ev[1], st);
    std::vector<uint64_t> head(2 + 3 * S);
    head[0] = (uint64_t)s;
    head[1] = sizeof(K);
    for (size_t k = 0; k < S; ++k) {
        head[2 + k] = mine[k].len;
        head[2 + S + k] = mine[k].pivot;
        head[2 + 2 * S + k] = mine[k].off;
    }
    cudaError_t e = cudaMemcpyAsync(rec, head.data(), 8 * head.size(), cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) return cuda_fail(e, "dist record H2D");
    // 2. all-gather the records (status agreement included)
    pp_status sg = tp.allgather(rec, c.d_ag, 8 * RW, st);
    if (sg != PP_OK) return sg;
    if (timing) cudaEventRecord(c.ev[2], st);
    std::vector<uint64_t> all(RW * P);
    e = cudaMemcpyAsync(all.data(), c.d_ag, 8 * RW * P, cudaMemcpyDeviceToHost, st);
    if (e != cudaSuccess) return cuda_fail(e, "dist record D2H");
    if ((sg = tp.wait(st)) != PP_OK) return sg;
    for (int q = 0; q < P; ++q)
        if (all[RW * q] != PP_OK) {
            if (q != me) set_error("peer rank " + std::to_string(q) + " failed with status " + std::to_string(all[RW * q]));
            return (pp_status)all[RW * q];
        }
    for (int q = 0; q < P; ++q) {
        bool bad = all[RW * q + 1] != sizeof(K);
        for (size_t k = 0; k < S; ++k) bad |= all[RW * q + 2 + S + k] != mine[k].pivot;
        if (bad) {
            set_error("pp_partition_dist: ranks passed different pivots or key types");
            return PP_E_INVAL;
        }
    }
    // 3. the same plan on every rank: runs per segment in shard-local offsets
    std::vector<Run> runs;
    K_out.assign(S, 0);
    {
        std::vector<uint64_t> ns(P), ts(P), base(P);
        std::vector<Run> rs;
        for (size_t k = 0; k < S; ++k) {
            uint64_t b = 0;
            for (int q = 0; q < P; ++q) {
                ns[q] = all[RW * q + 2 + k];
                ts[q] = all[RW * q + 2 + 3 * S + k];
                base[q] = b;
                b += ns[q];
                if (ts[q] > ns[q]) {
                    set_error("pp_partition_dist: corrupt local split");
                    return PP_E_INTERNAL;
                }
            }
            K_out[k] = match_runs(ns.data(), ts.data(), P, rs);
            for (const Run& r : rs)
                runs.push_back({r.ra, all[RW * r.ra + 2 + 2 * S + k] + (r.a - base[r.ra]), r.rb,
                                all[RW * r.rb + 2 + 2 * S + k] + (r.b - base[r.rb]), r.len});
        }
    }
    uint64_t moved = 0;
    if (params().dist_p2p && P > 1) {
        // 4a. one-sided: map the peers' shards, swap my share, then agree
        std::vector<uint64_t> prec(1 + kPeerWords), allp;
        pp_status se = tp.export_range(shard, prec.data() + 1);
        prec[0] = (uint64_t)se;
        pp_status sa = ag_host(c, prec.data(), 1 + kPeerWords, allp, st);
        if (sa != PP_OK) return sa;
        for (int q = 0; q < P; ++q)
            if (allp[(1 + kPeerWords) * q] != PP_OK) return agree(c, (pp_status)allp[(1 + kPeerWords) * q], st);
        std::vector<Run> share;
        p2p_share(runs, me, share);
        std::vector<K*> ptr(P, nullptr);
        ptr[me] = shard;
        pp_status sl = PP_OK;
        for (const Run& p : share)
            for (uint64_t q : {p.ra, p.rb}) {
                if (ptr[q] || sl != PP_OK) continue;
                void* d = nullptr;
                sl = tp.import_range(&allp[(1 + kPeerWords) * q + 1], &d);
                ptr[q] = static_cast<K*>(d);
            }
        if (sl == PP_OK && !share.empty()) {
            std::vector<uint64_t> tri;
            for (const Run& p : share) {
                moved += 2 * p.len * sizeof(K);
                tri.push_back(reinterpret_cast<uint64_t>(ptr[p.ra] + p.a));
                tri.push_back(reinterpret_cast<uint64_t>(ptr[p.rb] + p.b));
                tri.push_back(p.len);
            }
            tp.local_begin();
            sl = swap_ranges_impl<K>(tri.data(), share.size(), st, true, &c.d_swap, &c.d_swap_words);
            const pp_status s2 = tp.local_end(st);
            if (sl == PP_OK) sl = s2;
        }
        // no rank leaves (or reads its shard) before every peer's swaps finished
        if ((sl = agree(c, sl, st)) != PP_OK) return sl;
    } else if (P > 1) {
        // 4b. staged rounds (double-buffered staging halves, place copies on pst)
        std::vector<Piece> pcs;
        schedule_rounds(runs, P, cap, pcs);
        StagedState ss;
        pp_status sr = staged_rounds<K>(c, shard, pcs, half, st, ss, moved);
        if (sr == PP_OK) sr = staged_join(c, st, ss);
        if (sr != PP_OK) return sr;
    }
    if (timing) cudaEventRecord(c.ev[3], st);
    if ((s = tp.wait(st)) != PP_OK) return s;
    if (timing) {
        float a = 0, b = 0, d = 0;
        cudaEventElapsedTime(&a, c.ev[0], c.ev[1]);
        cudaEventElapsedTime(&b, c.ev[1], c.ev[2]);
        cudaEventElapsedTime(&d, c.ev[2], c.ev[3]);
        c.last_local_ms = a;
        c.last_gather_ms = b;
        c.last_exchange_ms = d;
        c.last_bytes = moved;
    }
    return PP_OK;
}


// ---------------------------------------------------------------------------
// Count-first overlapped exchange (param dist_overlap = 1).
// The shard is cut into C chunks (the same C on every rank).  (1) One read
// pass counts the predecessors of every chunk (chunk_count_kernel, fixed-order
// sums: no atomics).  (2) ONE all-gather of (status, key bytes, pivot, C, n,
// n_c[C], t_c[C]) fixes K and the plan BEFORE any key moves: every chunk
// acts as a unit of the same interval merge as the ranks of match_runs (a
// chunk partitioned in place holds its predecessors first, so its misplaced
// range is [β_u + t_u, min(K, β_u + n_u)) or [max(K, β_u), β_u + t_u) exactly
// as for a shard).  A matched run between chunk c of one rank and chunk c' of
// another can move once both are partitioned: it belongs to step max(c, c').
// (3) All C local partitions are enqueued on the caller's stream, an event
// after each; (4) the exchange of step k waits on chunk k's event on a second
// stream, so it overlaps the partition of chunks k+1.. (staged rounds through
// NCCL, or one-sided peer swaps after a per-step status barrier).  The local
// splits are checked against the counts at the end (PP_E_INTERNAL on every
// rank on a mismatch).  Unlike whole shards, two chunks of the rank holding K
// can be matched with each other: those runs are local swaps.  Cost: one extra read of the shard; gain: the
// NVLink-bound exchange runs under the local partition (§9).
// ---------------------------------------------------------------------------
template <typename K>
__global__ void __launch_bounds__(256) chunk_count_kernel(const K* __restrict__ keys, uint64_t n, uint64_t L,
                                                          K pivot, uint64_t* __restrict__ partial) {
    __shared__ uint64_t ws[8];
    const uint64_t lo = (uint64_t)blockIdx.y * L, hi = lo + L < n ? lo + L : n;
    const uint64_t S = (uint64_t)gridDim.x * 256;
    uint64_t cnt = 0;
    uint64_t x = lo + (uint64_t)blockIdx.x * 256 + threadIdx.x;
    for (; x + 3 * S < hi; x += 4 * S) {  // four independent loads in flight per thread
        const K a = keys[x], b = keys[x + S], d = keys[x + 2 * S], e = keys[x + 3 * S];
        cnt += (uint64_t)is_pred(a, pivot) + is_pred(b, pivot) + is_pred(d, pivot) + is_pred(e, pivot);
    }
    for (; x < hi; x += S) cnt += is_pred(keys[x], pivot) ? 1 : 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = cnt;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < 8; ++w) cnt += ws[w];
        partial[(uint64_t)blockIdx.y * gridDim.x + blockIdx.x] = cnt;
    }
}

// out[c] = sum of chunk c's B partials, in index order (thread c)
__global__ void chunk_count_reduce_kernel(const uint64_t* __restrict__ partial, uint32_t B, uint32_t C,
                                          uint64_t* __restrict__ out) {
    for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < C; c += gridDim.x * blockDim.x) {
        uint64_t t = 0;
        for (uint32_t b = 0; b < B; ++b) t += partial[(uint64_t)c * B + b];
        out[c] = t;
    }
}

template <typename K>
static pp_status partition_overlap(DistCtx& c, K* shard, uint64_t n_local, K pivot, cudaStream_t st,
                                   uint64_t* K_out) {
    Transport& tp = *c.tp;
    const int P = c.P, me = c.me;
    if (tp.absent()) {  // test hook: this rank never takes part
        set_error("rank absent (dist_fault = 2)");
        return PP_E_INTERNAL;
    }
    const uint64_t C = (uint64_t)std::max<int64_t>(1, params().dist_chunks);
    uint64_t L = (n_local + C - 1) / C;
    L = std::max<uint64_t>(64, (L + 63) / 64 * 64);  // chunk length (the last chunks may be short or empty)
    auto clo = [&](uint64_t k) { return std::min(n_local, k * L); };
    auto chi = [&](uint64_t k) { return std::min(n_local, (k + 1) * L); };
    const size_t RW = 5 + 2 * C;  // record: [status, key bytes, pivot, C, n, n_c[C], t_c[C]]
    const uint32_t B = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>(1024, (uint64_t)sm_count() * 8 / C));
    cudaEventRecord(c.ev[0], st);
    pp_status s = PP_OK;
    const uint64_t cap = std::max<uint64_t>(1, g_staging_cap_bytes / sizeof(K));
    const uint64_t half = std::max<uint64_t>(1, std::min(cap, n_local));
    if (!params().dist_p2p && P > 1) s = grow(&c.staging, &c.staging_bytes, 2 * sizeof(K) * half);
    {
        pp_status sa = ensure_ag(c, RW * (P + 1));
        if (sa == PP_OK) sa = c.init_overlap(C, C * B + C);
        if (sa != PP_OK) return sa;  // without them this rank cannot take part (as partition_multi)
    }
    if (s == PP_OK && params().dist_fault == 1 && params().dist_fault_rank == me) {
        set_error("injected local failure (dist_fault = 1)");
        s = PP_E_INTERNAL;
    }
    uint64_t* rec = c.d_ag + RW * P;
    uint64_t* d_tchk = c.d_cnt + C * B;  // the local partitions' splits
    // 1. per-chunk predecessor counts -> rec[5 + C ..]
    if (s == PP_OK && n_local > 0) {
        tp.local_begin();
        chunk_count_kernel<K><<<dim3(B, (unsigned)C), 256, 0, st>>>(shard, n_local, L, pivot, c.d_cnt);
        chunk_count_reduce_kernel<<<1, 256, 0, st>>>(c.d_cnt, B, (uint32_t)C, rec + 5 + C);
        note_launches(2);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) s = cuda_fail(e, "chunk count");
        const pp_status s2 = tp.local_end(st);
        if (s == PP_OK) s = s2;
    } else if (cudaMemsetAsync(rec + 5 + C, 0, 8 * C, st) != cudaSuccess) {
        s = cuda_fail(cudaGetLastError(), "memset");
    }
    cudaEventRecord(c.ev[1], st);
    std::vector<uint64_t> head(5 + C);
    head[0] = (uint64_t)s;
    head[1] = sizeof(K);
    head[2] = (uint64_t)pivot;
    head[3] = C;
    head[4] = n_local;
    for (uint64_t k = 0; k < C; ++k) head[5 + k] = chi(k) - clo(k);
    cudaError_t e = cudaMemcpyAsync(rec, head.data(), 8 * head.size(), cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) return cuda_fail(e, "dist record H2D");
    // 2. all-gather the records (status agreement included) -> K and the plan
    pp_status sg = tp.allgather(rec, c.d_ag, 8 * RW, st);
    if (sg != PP_OK) return sg;
    cudaEventRecord(c.ev[2], st);
    std::vector<uint64_t> all(RW * P);
    e = cudaMemcpyAsync(all.data(), c.d_ag, 8 * RW * P, cudaMemcpyDeviceToHost, st);
    if (e != cudaSuccess) return cuda_fail(e, "dist record D2H");
    if ((sg = tp.wait(st)) != PP_OK) return sg;
    for (int q = 0; q < P; ++q)
        if (all[RW * q] != PP_OK) {
            if (q != me) set_error("peer rank " + std::to_string(q) + " failed with status " + std::to_string(all[RW * q]));
            return (pp_status)all[RW * q];
        }
    for (int q = 0; q < P; ++q)
        if (all[RW * q + 1] != sizeof(K) || all[RW * q + 2] != (uint64_t)pivot || all[RW * q + 3] != C) {
            set_error("pp_partition_dist (dist_overlap): ranks passed different pivots, key types or dist_chunks");
            return PP_E_INVAL;
        }
    const uint64_t U = (uint64_t)P * C;
    std::vector<uint64_t> ns(U), ts(U), rbase(P, 0);
    for (int q = 0; q < P; ++q) {
        if (q > 0) rbase[q] = rbase[q - 1] + all[RW * (q - 1) + 4];
        for (uint64_t k = 0; k < C; ++k) {
            ns[q * C + k] = all[RW * q + 5 + k];
            ts[q * C + k] = all[RW * q + 5 + C + k];
            if (ts[q * C + k] > ns[q * C + k]) {
                set_error("pp_partition_dist: corrupt chunk count");
                return PP_E_INTERNAL;
            }
        }
    }
    std::vector<Run> uruns;
    const uint64_t Kg = match_runs(ns.data(), ts.data(), (int)U, uruns);
    std::vector<std::vector<Run>> by_step(C);  // runs in rank-local offsets, by the step that frees them
    for (const Run& r : uruns) {
        const uint64_t qa = r.ra / C, qb = r.rb / C;
        const uint64_t step = std::max(r.ra % C, r.rb % C);
        by_step[step].push_back({qa, r.a - rbase[qa], qb, r.b - rbase[qb], r.len});
    }
    // 3. every chunk's local partition, enqueued up front on st (an event after each)
    pp_status sl = PP_OK;
    tp.local_begin();
    for (uint64_t k = 0; k < C && sl == PP_OK; ++k) {
        const uint64_t lo = clo(k), len = chi(k) - lo;
        if (len > 0) sl = partition_device<K>(shard + lo, len, pivot, st, d_tchk + k, nullptr);
        else if (cudaMemsetAsync(d_tchk + k, 0, 8, st) != cudaSuccess) sl = cuda_fail(cudaGetLastError(), "memset");
        if (sl == PP_OK && cudaEventRecord(c.ev_chunk[k], st) != cudaSuccess) sl = cuda_fail(cudaGetLastError(), "event");
    }
    {
        const pp_status s2 = tp.local_end(st);  // loopback: waits; NCCL: no-op
        if (sl == PP_OK) sl = s2;
    }
    // enqueue failures are agreed on before any exchange (kernels keep running)
    if ((sl = agree(c, sl, c.xst)) != PP_OK) {
        cudaStreamSynchronize(st);
        return sl;
    }
    // 4. the exchange, step by step on xst
    uint64_t moved = 0;
    pp_status sx = PP_OK;
    if (params().dist_p2p && P > 1) {
        std::vector<uint64_t> prec(1 + kPeerWords), allp;
        pp_status se = tp.export_range(shard, prec.data() + 1);
        prec[0] = (uint64_t)se;
        sx = ag_host(c, prec.data(), 1 + kPeerWords, allp, c.xst);
        for (int q = 0; q < P && sx == PP_OK; ++q)
            if (allp[(1 + kPeerWords) * q] != PP_OK) sx = (pp_status)allp[(1 + kPeerWords) * q];
        std::vector<K*> ptr(P, nullptr);
        ptr[me] = shard;
        for (uint64_t k = 0; k < C && sx == PP_OK; ++k) {
            if (by_step[k].empty()) continue;  // the same on every rank
            std::vector<Run> share;
            p2p_share(by_step[k], me, share);
            pp_status sk = PP_OK;
            for (const Run& p : share)
                for (uint64_t q : {p.ra, p.rb}) {
                    if (ptr[q] || sk != PP_OK) continue;
                    void* d = nullptr;
                    sk = tp.import_range(&allp[(1 + kPeerWords) * q + 1], &d);
                    ptr[q] = static_cast<K*>(d);
                }
            if (sk == PP_OK && cudaEventSynchronize(c.ev_chunk[k]) != cudaSuccess)
                sk = cuda_fail(cudaGetLastError(), "chunk event");
            // every rank's chunks <= k are final before anyone swaps into them
            if ((sk = agree(c, sk, c.xst)) != PP_OK) {
                sx = sk;
                break;
            }
            if (!share.empty()) {
                std::vector<uint64_t> tri;
                for (const Run& p : share) {
                    moved += 2 * p.len * sizeof(K);
                    tri.push_back(reinterpret_cast<uint64_t>(ptr[p.ra] + p.a));
                    tri.push_back(reinterpret_cast<uint64_t>(ptr[p.rb] + p.b));
                    tri.push_back(p.len);
                }
                tp.local_begin();
                sx = swap_ranges_impl<K>(tri.data(), share.size(), c.xst, true, &c.d_swap, &c.d_swap_words);
                const pp_status s2 = tp.local_end(c.xst);
                if (sx == PP_OK) sx = s2;
            }
        }
    } else {  // P = 1 too: the rank's own chunks trade by local swaps
        StagedState ss;
        for (uint64_t k = 0; k < C && sx == PP_OK; ++k) {
            if (by_step[k].empty()) continue;
            if (cudaStreamWaitEvent(c.xst, c.ev_chunk[k], 0) != cudaSuccess) {
                sx = cuda_fail(cudaGetLastError(), "chunk order");
                break;
            }
            // runs between two chunks of this rank (only the rank holding K has
            // them) are local swaps; the others go through the staged rounds
            std::vector<Run> cross;
            std::vector<uint64_t> tri;
            for (const Run& r : by_step[k]) {
                if (r.ra != r.rb) {
                    cross.push_back(r);
                } else if ((int)r.ra == me) {
                    tri.push_back(reinterpret_cast<uint64_t>(shard + r.a));
                    tri.push_back(reinterpret_cast<uint64_t>(shard + r.b));
                    tri.push_back(r.len);
                }
            }
            if (!tri.empty()) {
                tp.local_begin();
                sx = swap_ranges_impl<K>(tri.data(), tri.size() / 3, c.xst, false, &c.d_swap, &c.d_swap_words);
                const pp_status s2 = tp.local_end(c.xst);
                if (sx == PP_OK) sx = s2;
                if (sx != PP_OK) break;
            }
            std::vector<Piece> pcs;
            schedule_rounds(cross, P, cap, pcs);
            sx = staged_rounds<K>(c, shard, pcs, half, c.xst, ss, moved);
        }
        if (sx == PP_OK) sx = staged_join(c, c.xst, ss);
    }
    // 5. join, check the local splits against the counts, agree
    if (cudaEventRecord(c.ev[4], c.xst) != cudaSuccess || cudaStreamWaitEvent(st, c.ev[4], 0) != cudaSuccess ||
        cudaEventRecord(c.ev[3], st) != cudaSuccess) {
        if (sx == PP_OK) sx = cuda_fail(cudaGetLastError(), "dist join");
    }
    if (sx == PP_OK) sx = tp.wait(c.xst);
    std::vector<uint64_t> tchk(C, 0);
    if (cudaMemcpyAsync(tchk.data(), d_tchk, 8 * C, cudaMemcpyDeviceToHost, st) != cudaSuccess && sx == PP_OK)
        sx = cuda_fail(cudaGetLastError(), "split check D2H");
    if (cudaStreamSynchronize(st) != cudaSuccess && sx == PP_OK) sx = cuda_fail(cudaGetLastError(), "dist stream");
    for (uint64_t k = 0; k < C && sx == PP_OK; ++k)
        if (tchk[k] != all[RW * me + 5 + C + k]) {
            set_error("pp_partition_dist (dist_overlap): a chunk's split differs from its count");
            sx = PP_E_INTERNAL;
        }
    // no rank returns (or reads its shard) while a peer may still write into it
    if ((sx = agree(c, sx, st)) != PP_OK) return sx;
    float a = 0, b = 0, d = 0;
    cudaEventElapsedTime(&a, c.ev[0], c.ev[1]);
    cudaEventElapsedTime(&b, c.ev[1], c.ev[2]);
    cudaEventElapsedTime(&d, c.ev[2], c.ev[3]);
    c.last_local_ms = a;   // the count pass
    c.last_gather_ms = b;
    c.last_exchange_ms = d;  // local partitions + the overlapped exchange
    c.last_bytes = moved;
    if (K_out) *K_out = Kg;
    return PP_OK;
}

template <typename K>
static pp_status partition_dist_ctx(DistCtx& c, K* shard, uint64_t n_local, K pivot, cudaStream_t st,
                                    uint64_t* global_split) {
    if (params().dist_overlap) return partition_overlap<K>(c, shard, n_local, pivot, st, global_split);
    std::vector<uint64_t> Ks;
    pp_status s = partition_multi<K>(c, shard, {SegPiece{0, n_local, (uint64_t)pivot}}, st, Ks, true);
    if (s == PP_OK && global_split) *global_split = Ks[0];
    return s;
}

template <typename K>
pp_status partition_dist(K* shard, uint64_t n_local, K pivot, cudaStream_t st, uint64_t* global_split) {
    if (!g_ctx.tp) {
        set_error("pp_partition_dist: call pp_dist_init first");
        return PP_E_INVAL;
    }
    return partition_dist_ctx<K>(g_ctx, shard, n_local, pivot, st, global_split);
}
template pp_status partition_dist<uint64_t>(uint64_t*, uint64_t, uint64_t, cudaStream_t, uint64_t*);
template pp_status partition_dist<uint32_t>(uint32_t*, uint64_t, uint32_t, cudaStream_t, uint64_t*);

// ---------------------------------------------------------------------------
// Distributed quicksort (BASELINE config 5 at P GPUs; PAPER.md:1701-1732 with
// the parallel partition at the top levels).  Level by level over the
// segments that span ranks, all identical on every rank:
//   * pivots: the median-of-3 sample keys (R14) of every spanning
//     segment are copied device-to-device into one sample array, ONE
//     all-gather per level, each taken from its owner's slot;
//   * segments > `small` keys: ONE batched partition_multi for all of them
//     (one record all-gather, one exchange); a segment whose pivot is its
//     minimum (split 0) is re-partitioned next level by "x <= p" (pivot p+1),
//     whose left part (all == p) is final; every segment carries the bounds
//     its ancestors' pivots imply: bounds of one value = all equal, final; a
//     pivot equal to the lower bound splits by x < kmin + 1 at once;
//   * segments <= `small`: ONE all-gather of every rank's pieces of all of
//     them; each participating rank sorts the whole segment locally and keeps
//     its part.
// When no segment spans ranks each shard is a concatenation of whole
// segments in key order: one local quicksort per rank finishes.
// ---------------------------------------------------------------------------
template <typename K>
static pp_status quicksort_dist_ctx(DistCtx& c, K* shard, uint64_t n_local, cudaStream_t st, uint64_t small) {
    Transport& tp = *c.tp;
    const int P = c.P, me = c.me;
    const uint64_t KMAXU = (uint64_t)(K)~(K)0;
    if (tp.absent()) {
        set_error("rank absent (dist_fault = 2)");
        return PP_E_INTERNAL;
    }
    std::vector<uint64_t> all;
    const uint64_t hdr[2] = {PP_OK, n_local};
    pp_status s = ag_host(c, hdr, 2, all, st);
    if (s != PP_OK) return s;
    std::vector<uint64_t> ns(P), base(P, 0);
    for (int r = 0; r < P; ++r) ns[r] = all[2 * r + 1];
    for (int r = 1; r < P; ++r) base[r] = base[r - 1] + ns[r - 1];
    const uint64_t N = base[P - 1] + ns[P - 1], b0 = base[me];
    auto owner = [&](uint64_t x) {
        int r = 0;
        while (r + 1 < P && base[r + 1] <= x) ++r;
        return r;
    };
    auto inter = [&](uint64_t lo, uint64_t hi, int r, uint64_t& a, uint64_t& b) {  // piece of rank r (global)
        a = std::max(lo, base[r]);
        b = std::min(hi, base[r] + ns[r]);
        if (a >= b) a = b = 0;
    };
    struct Seg {
        uint64_t lo, hi;
        bool leq;  // re-partition by x <= pivot (the pivot was the minimum)
        uint64_t pivot;
        uint64_t kmin, kmax;  // every key of the segment is in [kmin, kmax] (the pivots above it)
    };
    std::vector<Seg> segs;
    if (N > 1) segs.push_back({0, N, false, 0, 0, KMAXU});
    cudaError_t e;
    while (true) {
        std::vector<Seg> big, sm, nxt;
        // (a segment whose bounds are one value is all equal keys: final, no round)
        for (const Seg& sg : segs)
            if (sg.hi - sg.lo > 1 && sg.kmin != sg.kmax && owner(sg.lo) != owner(sg.hi - 1))
                (sg.hi - sg.lo <= small ? sm : big).push_back(sg);
        if (big.empty() && sm.empty()) break;
        static const bool dprof = getenv("PP_QS_DIST_PROF") != nullptr;  // measurement: rounds per sort
        if (dprof && me == 0) {
            uint64_t kb = 0;
            for (const Seg& sg : big) kb += sg.hi - sg.lo;
            fprintf(stderr, "qs dist round: big=%zu (%llu keys) small=%zu\n", big.size(), (unsigned long long)kb, sm.size());
        }
        // ---- pivots: one all-gather of the sample keys of this level ----
        // median of 3 (A[lo], A[mid], A[hi-1]; R14), or of 31 evenly spaced keys
        // with qs_pivot = 2 (the single-GPU level loop's rule)
        // (param dist_split = 1: 63 evenly spaced keys, and the pivot is the sample
        // quantile of the rank boundary inside the segment -- see below)
        const bool bsplit = params().dist_split != 0;
        const int NSMP = bsplit ? 63 : params().qs_pivot == 2 ? 31 : 3;
        std::vector<uint64_t> spos;  // NSMP per segment needing a sample
        for (const Seg& sg : big)
            if (!sg.leq) {
                const uint64_t len = sg.hi - sg.lo;
                if (NSMP == 3) {
                    spos.push_back(sg.lo);
                    spos.push_back(sg.lo + (len - 1) / 2);
                    spos.push_back(sg.hi - 1);
                } else {
                    const uint64_t d = (uint64_t)NSMP - 1;
                    for (uint64_t j = 0; j < (uint64_t)NSMP; ++j)
                        spos.push_back(sg.lo + (len - 1) / d * j + ((len - 1) % d) * j / d);
                }
            }
        std::vector<uint64_t> sval;
        if (!spos.empty()) {
            const size_t m = spos.size();
            // every rank takes part in the agreement (a failed allocation on one rank must not
            // leave the others in a different collective)
            if ((s = agree(c, grow(&c.gs, &c.gs_bytes, 8 * m * (P + 1)), st)) != PP_OK) return s;
            uint64_t* d_samp = static_cast<uint64_t*>(c.gs) + m * P;
            e = cudaMemsetAsync(d_samp, 0, 8 * m, st);
            for (size_t i = 0; i < m && e == cudaSuccess; ++i)
                if (owner(spos[i]) == me)  // little-endian: a u32 key lands in the low half of its word
                    e = cudaMemcpyAsync(d_samp + i, shard + (spos[i] - b0), sizeof(K), cudaMemcpyDeviceToDevice, st);
            if (e != cudaSuccess) return cuda_fail(e, "pivot samples");
            if ((s = tp.allgather(d_samp, c.gs, 8 * m, st)) != PP_OK) return s;
            std::vector<uint64_t> got(m * P);
            e = cudaMemcpyAsync(got.data(), c.gs, 8 * m * P, cudaMemcpyDeviceToHost, st);
            if (e != cudaSuccess) return cuda_fail(e, "pivot samples D2H");
            if ((s = tp.wait(st)) != PP_OK) return s;
            for (size_t i = 0; i < m; ++i) sval.push_back(got[m * owner(spos[i]) + i]);
        }
        // ---- big spanning segments: one batched distributed partition ----
        if (!big.empty()) {
            std::vector<SegPiece> mine;
            std::vector<uint64_t> piv(big.size());
            for (size_t k = 0, si = 0; k < big.size(); ++k) {
                const Seg& sg = big[k];
                uint64_t p = sg.pivot;
                if (!sg.leq) {
                    std::vector<uint64_t> v(sval.begin() + si, sval.begin() + si + NSMP);
                    si += NSMP;
                    std::sort(v.begin(), v.end());
                    p = v[NSMP / 2];
                    if (bsplit) {
                        // the rank boundary inside the segment nearest its middle; the
                        // pivot is the sample quantile of its position, so the split
                        // lands near the boundary and the spanning part shrinks by
                        // ~1/NSMP per round instead of ~1/2
                        const uint64_t mid = sg.lo + (sg.hi - sg.lo) / 2;
                        uint64_t bnd = 0, best = ~0ull;
                        for (int r = 1; r < P; ++r)
                            if (base[r] > sg.lo && base[r] < sg.hi) {
                                const uint64_t dd = base[r] > mid ? base[r] - mid : mid - base[r];
                                if (dd < best) { best = dd; bnd = base[r]; }
                            }
                        const double f = (double)(bnd - sg.lo) / (double)(sg.hi - sg.lo);
                        p = v[std::min<size_t>((size_t)(f * (NSMP - 1) + 0.5), (size_t)NSMP - 1)];
                    }
                    // at the lower bound the x < p split is empty: split by x < kmin + 1 now
                    if (p == sg.kmin) p = (uint64_t)(K)(p + 1);
                }
                piv[k] = p;
                uint64_t a, b;
                inter(sg.lo, sg.hi, me, a, b);
                // x <= p is x < p + 1 (p < KMAX here: see below)
                mine.push_back({a < b ? a - b0 : 0, b - a, sg.leq ? p + 1 : p});
            }
            std::vector<uint64_t> Ks;
            if ((s = partition_multi<K>(c, shard, mine, st, Ks, false)) != PP_OK) return s;
            for (size_t k = 0; k < big.size(); ++k) {
                const Seg& sg = big[k];
                const uint64_t kk = Ks[k], p = piv[k];
                if (sg.leq) {
                    nxt.push_back({sg.lo + kk, sg.hi, false, 0, p + 1, sg.kmax});  // [lo, lo+kk) all == p: final
                } else if (kk == 0) {
                    // every key >= p; p == kmax (e.g. all == MAX): all equal, final
                    if (p != sg.kmax) nxt.push_back({sg.lo, sg.hi, true, p, p, sg.kmax});
                } else {
                    nxt.push_back({sg.lo, sg.lo + kk, false, 0, sg.kmin, p - 1});
                    nxt.push_back({sg.lo + kk, sg.hi, false, 0, p, sg.kmax});
                }
            }
        }
        // ---- small spanning segments: one gather, sort locally, keep my part ----
        if (!sm.empty()) {
            std::vector<uint64_t> contrib(P, 0);
            uint64_t tot = 0;
            for (const Seg& sg : sm) {
                tot += sg.hi - sg.lo;
                for (int r = 0; r < P; ++r) {
                    uint64_t a, b;
                    inter(sg.lo, sg.hi, r, a, b);
                    contrib[r] += b - a;
                }
            }
            const uint64_t mx = *std::max_element(contrib.begin(), contrib.end());
            // layout: gathered [P][mx] | mine [mx] | assembled segments [tot]
            s = grow(&c.gs, &c.gs_bytes, sizeof(K) * (mx * (P + 1) + tot));
            if ((s = agree(c, s, st)) != PP_OK) return s;
            K* g = static_cast<K*>(c.gs);
            K* snd = g + mx * P;
            K* asm_ = snd + mx;
            uint64_t at = 0;
            e = cudaSuccess;
            for (const Seg& sg : sm) {
                uint64_t a, b;
                inter(sg.lo, sg.hi, me, a, b);
                if (b > a) e = cudaMemcpyAsync(snd + at, shard + (a - b0), sizeof(K) * (b - a), cudaMemcpyDeviceToDevice, st);
                at += b - a;
                if (e != cudaSuccess) return cuda_fail(e, "gather-sort pack");
            }
            if ((s = tp.allgather(snd, g, sizeof(K) * mx, st)) != PP_OK) return s;
            std::vector<uint64_t> rat(P, 0);  // read cursor per rank in the gathered rows
            uint64_t seg_at = 0;
            pp_status sl = PP_OK;
            tp.local_begin();
            for (const Seg& sg : sm) {
                const uint64_t len = sg.hi - sg.lo;
                K* full = asm_ + seg_at;
                uint64_t w = 0, my_off = 0, my_len = 0;
                for (int r = 0; r < P && e == cudaSuccess; ++r) {
                    uint64_t a, b;
                    inter(sg.lo, sg.hi, r, a, b);
                    if (r == me) {
                        my_off = w;
                        my_len = b - a;
                    }
                    if (b > a) e = cudaMemcpyAsync(full + w, g + mx * r + rat[r], sizeof(K) * (b - a), cudaMemcpyDeviceToDevice, st);
                    rat[r] += b - a;
                    w += b - a;
                }
                if (e != cudaSuccess) break;
                if (my_len > 0 && sl == PP_OK) {  // only participating ranks sort
                    sl = quicksort_device<K>(full, len, st);
                    if (sl == PP_OK)
                        e = cudaMemcpyAsync(shard + (std::max(sg.lo, b0) - b0), full + my_off, sizeof(K) * my_len,
                                            cudaMemcpyDeviceToDevice, st);
                }
                seg_at += len;
            }
            const pp_status s2 = tp.local_end(st);
            if (sl == PP_OK && e != cudaSuccess) sl = cuda_fail(e, "gather-sort");
            if (sl == PP_OK) sl = s2;
            if ((s = agree(c, sl, st)) != PP_OK) return s;  // also: every rank read the gather before reuse
        }
        segs.clear();
        for (const Seg& sg : nxt)
            if (sg.hi - sg.lo > 1) segs.push_back(sg);
    }
    pp_status sl = PP_OK;
    if (n_local > 1) {
        tp.local_begin();
        sl = quicksort_device<K>(shard, n_local, st);
        const pp_status s2 = tp.local_end(st);
        if (sl == PP_OK) sl = s2;
    }
    if (sl == PP_OK) sl = tp.wait(st);
    return agree(c, sl, st);
}

template <typename K>
pp_status quicksort_dist(K* shard, uint64_t n_local, cudaStream_t st, uint64_t small) {
    if (!g_ctx.tp) {
        set_error("pp_quicksort_dist: call pp_dist_init first");
        return PP_E_INVAL;
    }
    return quicksort_dist_ctx<K>(g_ctx, shard, n_local, st, small);
}
template pp_status quicksort_dist<uint64_t>(uint64_t*, uint64_t, cudaStream_t, uint64_t);
template pp_status quicksort_dist<uint32_t>(uint32_t*, uint64_t, cudaStream_t, uint64_t);

// ---------------------------------------------------------------------------
// Loopback drivers: P emulated ranks on this GPU, rank r = keys[sum ns[<r],
// + ns[r]); each runs the collective call on its own thread and stream.
// ---------------------------------------------------------------------------
template <typename K, typename F>
static pp_status loopback_run(K* keys, const uint64_t* ns, int P, F&& body) {
    if (P < 1 || P > 64 || !ns) {
        set_error("loopback: 1 <= nranks <= 64 and ns != NULL required");
        return PP_E_INVAL;
    }
    int dev = 0;
    cudaGetDevice(&dev);
    LoopHub hub(P);
    std::vector<LoopTransport> tps(P);
    std::vector<DistCtx> ctx(P);
    std::vector<cudaStream_t> sts(P, nullptr);
    std::vector<pp_status> res(P, PP_OK);
    std::vector<std::string> errs(P);
    std::vector<uint64_t> off(P, 0);
    for (int r = 1; r < P; ++r) off[r] = off[r - 1] + ns[r - 1];
    for (int r = 0; r < P; ++r) {
        tps[r].P = P;
        tps[r].me = r;
        tps[r].hub = &hub;
        tps[r].absent_ = params().dist_fault == 2 && params().dist_fault_rank == r;
        ctx[r].tp = &tps[r];
        ctx[r].P = P;
        ctx[r].me = r;
        ctx[r].device = dev;
        if (ctx[r].init_events() != PP_OK || cudaStreamCreateWithFlags(&sts[r], cudaStreamNonBlocking) != cudaSuccess) {
            for (int q = 0; q <= r; ++q) {
                ctx[q].release();
                if (sts[q]) cudaStreamDestroy(sts[q]);
            }
            return cuda_fail(cudaGetLastError(), "loopback setup");
        }
    }
    cudaDeviceSynchronize();  // the caller's prior work on keys is complete
    std::vector<std::thread> th;
    for (int r = 0; r < P; ++r)
        th.emplace_back([&, r] {
            cudaSetDevice(dev);
            res[r] = body(ctx[r], keys + off[r], ns[r], sts[r], r);
        });
    for (auto& t : th) t.join();
    for (int r = 0; r < P; ++r) {
        ctx[r].release();
        cudaStreamDestroy(sts[r]);
    }
    for (int r = 0; r < P; ++r)
        if (res[r] != PP_OK) return res[r];
    return PP_OK;
}

template <typename K>
pp_status partition_dist_loopback(K* keys, const uint64_t* ns, int P, K pivot, uint64_t* split_out) {
    std::vector<uint64_t> Ks(P > 0 ? P : 1, 0);
    pp_status s = loopback_run<K>(keys, ns, P, [&](DistCtx& c, K* shard, uint64_t n, cudaStream_t st, int r) {
        return partition_dist_ctx<K>(c, shard, n, pivot, st, &Ks[r]);
    });
    if (s != PP_OK) return s;
    for (int r = 1; r < P; ++r)
        if (Ks[r] != Ks[0]) {
            set_error("loopback: ranks disagree on the global split");
            return PP_E_INTERNAL;
        }
    if (split_out) *split_out = Ks[0];
    return PP_OK;
}
template pp_status partition_dist_loopback<uint64_t>(uint64_t*, const uint64_t*, int, uint64_t, uint64_t*);
template pp_status partition_dist_loopback<uint32_t>(uint32_t*, const uint64_t*, int, uint32_t, uint64_t*);

template <typename K>
pp_status quicksort_dist_loopback(K* keys, const uint64_t* ns, int P, uint64_t small) {
    return loopback_run<K>(keys, ns, P, [&](DistCtx& c, K* shard, uint64_t n, cudaStream_t st, int) {
        return quicksort_dist_ctx<K>(c, shard, n, st, small);
    });
}
template pp_status quicksort_dist_loopback<uint64_t>(uint64_t*, const uint64_t*, int, uint64_t);
template pp_status quicksort_dist_loopback<uint32_t>(uint32_t*, const uint64_t*, int, uint64_t);

// ---------------------------------------------------------------------------
// Host arithmetic exported for tests.
// ---------------------------------------------------------------------------
pp_status dist_p2p_pieces(const uint64_t* ns, const uint64_t* ts, int P, int rank, uint64_t* out, uint64_t out_cap,
                          uint64_t* n_out) {
    if (!ns || !ts || P < 1 || rank < 0 || rank >= P || !n_out) return PP_E_INVAL;
    for (int r = 0; r < P; ++r)
        if (ts[r] > ns[r]) return PP_E_INVAL;
    std::vector<Run> runs, pcs;
    match_runs(ns, ts, P, runs);
    p2p_share(runs, rank, pcs);
    *n_out = pcs.size();
    if (out) {
        for (size_t k = 0; k < pcs.size() && k < out_cap; ++k) {
            uint64_t* o = out + 5 * k;
            o[0] = pcs[k].ra;
            o[1] = pcs[k].a;
            o[2] = pcs[k].rb;
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
