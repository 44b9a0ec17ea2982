// pp_api.cu -- the C ABI (include/pp.h): argument checks, workspace, error
// reporting, host-buffer variants.  Every compute step runs in the kernels of
// pp_partition.cu / pp_quicksort.cu; there is no CPU fallback.
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>
#include <algorithm>

#include "pp_internal.h"

namespace pp {

uint64_t launch_count(int reset);
uint64_t max_groups();
void timing_enable(int on);
int timing_read(double* out);

static std::mutex g_mu;
static std::mutex g_err_mu;  // set_error may run on the loopback's rank threads
static std::string g_err;
static Params g_params;
static LastStats g_stats;
static Ctl* g_last_ctl = nullptr;          // Ctl of the last partition (in the workspace), for pp_last_stats
static cudaStream_t g_last_ctl_st = nullptr; // the stream that call ran on

Params& params() { return g_params; }
LastStats& last_stats() { return g_stats; }

void set_error(const std::string& msg) {
    std::lock_guard<std::mutex> lk(g_err_mu);
    g_err = msg;
}
pp_status cuda_fail(cudaError_t e, const char* what) {
    set_error(std::string(what) + ": " + cudaGetErrorString(e));
    return PP_E_CUDA;
}

int sm_count() {
    static int n = 0;
    if (n == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}

// One growing device workspace.  Growth synchronises the stream first so an
// in-flight call never loses its buffer.
static void* g_ws = nullptr;
static size_t g_ws_bytes = 0;
// Caller-owned workspace (pp_set_workspace); when set, it replaces the
// internal one and is never grown or freed by the library.
static void* g_user_ws = nullptr;
static size_t g_user_ws_bytes = 0;
bool user_workspace(void** p, size_t* bytes) {
    if (!g_user_ws) return false;
    *p = g_user_ws;
    *bytes = g_user_ws_bytes;
    return true;
}
void* workspace(size_t bytes, cudaStream_t st) {
    if (g_user_ws) {
        if (bytes <= g_user_ws_bytes) return g_user_ws;
        set_error("caller workspace too small: need " + std::to_string(bytes) + " bytes, have " +
                  std::to_string(g_user_ws_bytes) + " (pp_workspace_bytes)");
        return nullptr;
    }
    if (bytes <= g_ws_bytes) return g_ws;
    if (g_ws) {
        cudaStreamSynchronize(st);
        cudaDeviceSynchronize();
        g_last_ctl = nullptr;  // pointed into the old workspace
        cudaFree(g_ws);
        g_ws = nullptr;
        g_ws_bytes = 0;
    }
    size_t want = bytes + (bytes >> 2);
    if (cudaMalloc(&g_ws, want) != cudaSuccess) {
        cudaGetLastError();
        set_error("workspace cudaMalloc failed");
        return nullptr;
    }
    g_ws_bytes = want;
    return g_ws;
}

// one device word for the split of synchronous calls that need it
static void* host_split_slot() {
    static void* p = nullptr;
    if (!p && cudaMalloc(&p, 256) != cudaSuccess) {
        cudaGetLastError();
        p = nullptr;
    }
    return p;
}

// pinned host word for split readback
static uint64_t* pinned_word() {
    static uint64_t* p = nullptr;
    if (!p && cudaMallocHost(&p, 64) != cudaSuccess) {
        cudaGetLastError();
        p = nullptr;
    }
    return p;
}

// Ordering of the shared workspace across streams: every call
// that may use it waits for the last such call when that one ran on another
// stream (an event recorded on its stream once it had enqueued its work),
// and records the event on its own stream when it has enqueued its work.
// Async calls stay async; calls on one stream pay nothing but the record.
static cudaEvent_t g_ws_ev = nullptr;
static cudaStream_t g_ws_st = nullptr;
static bool g_ws_pending = false;
struct WsOrder {
    cudaStream_t st;
    explicit WsOrder(cudaStream_t s) : st(s) {
        if (!g_ws_ev && cudaEventCreateWithFlags(&g_ws_ev, cudaEventDisableTiming) != cudaSuccess) {
            cudaGetLastError();
            g_ws_ev = nullptr;
        }
        if (g_ws_ev && g_ws_pending && g_ws_st != st) cudaStreamWaitEvent(st, g_ws_ev, 0);
    }
    ~WsOrder() {
        if (!g_ws_ev) return;
        if (cudaEventRecord(g_ws_ev, st) == cudaSuccess) {
            g_ws_st = st;
            g_ws_pending = true;
        } else {
            cudaGetLastError();
        }
    }
};

// The library binds to the device of its first call (workspace, streams,
// pinned buffers and the SM count are per device); keys on another device,
// or a current device that is not the keys' device, are rejected.
static int g_dev = -1;

template <typename K>
static pp_status check_device_keys(const K* keys, uint64_t n) {
    if (n == 0) return PP_OK;
    if (!keys) {
        set_error("keys is NULL with n > 0");
        return PP_E_INVAL;
    }
    if ((uintptr_t)keys % sizeof(K)) {
        set_error("keys not aligned to the key size");
        return PP_E_INVAL;
    }
    cudaPointerAttributes a;
    cudaError_t e = cudaPointerGetAttributes(&a, keys);
    if (e != cudaSuccess) {
        cudaGetLastError();
        set_error("keys is not a CUDA-visible pointer");
        return PP_E_INVAL;
    }
    if (a.type != cudaMemoryTypeDevice && a.type != cudaMemoryTypeManaged) {
        set_error("keys must be a device pointer (use the *_host variants for host memory)");
        return PP_E_INVAL;
    }
    int cur = 0;
    cudaGetDevice(&cur);
    if (a.type == cudaMemoryTypeDevice && a.device != cur) {
        set_error("keys are on device " + std::to_string(a.device) + " but the current device is " +
                  std::to_string(cur));
        return PP_E_INVAL;
    }
    if (g_dev < 0) g_dev = cur;
    if (cur != g_dev) {
        set_error("the library is bound to device " + std::to_string(g_dev) + " (its first call); got device " +
                  std::to_string(cur));
        return PP_E_INVAL;
    }
    return PP_OK;
}

template <typename K>
static pp_status partition_sync(K* keys, uint64_t n, K pivot, void* stream, uint64_t* split_out) {
    std::lock_guard<std::mutex> lk(g_mu);
    if (!split_out) {
        set_error("split_out is NULL");
        return PP_E_INVAL;
    }
    pp_status s = check_device_keys(keys, n);
    if (s != PP_OK) return s;
    if (n == 0) {
        *split_out = 0;
        g_stats = LastStats();
        return PP_OK;
    }
    cudaStream_t st = (cudaStream_t)stream;
    uint64_t* pw = pinned_word();
    if (!pw) {
        set_error("cudaMallocHost failed");
        return PP_E_NOMEM;
    }
    Ctl* ctl = nullptr;
    {
        WsOrder ws_order(st);
        s = partition_device<K>(keys, n, pivot, st, nullptr, &ctl);
    }
    if (s != PP_OK) return s;
    g_last_ctl = ctl;
    g_last_ctl_st = st;
    cudaError_t e = cudaMemcpyAsync(pw, &ctl->K, sizeof(uint64_t), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return cuda_fail(e, "partition");
    *split_out = *pw;
    return PP_OK;
}

template <typename K>
static pp_status partition_async(K* keys, uint64_t n, K pivot, void* stream, uint64_t* d_split) {
    std::lock_guard<std::mutex> lk(g_mu);
    pp_status s = check_device_keys(keys, n);
    if (s != PP_OK) return s;
    if (!d_split) {
        set_error("d_split is NULL");
        return PP_E_INVAL;
    }
    cudaStream_t st = (cudaStream_t)stream;
    if (n == 0) {
        cudaError_t e = cudaMemsetAsync(d_split, 0, sizeof(uint64_t), st);
        return e == cudaSuccess ? PP_OK : cuda_fail(e, "memset");
    }
    Ctl* ctl = nullptr;
    {
        WsOrder ws_order(st);
        s = partition_device<K>(keys, n, pivot, st, d_split, &ctl);
    }
    g_last_ctl = s == PP_OK ? ctl : nullptr;
    g_last_ctl_st = st;
    return s;
}

// Standard Algorithm (stable, out-of-place; pp_stable.cu): in and out are
// distinct device arrays of n keys; the split goes to split_out (host, sync)
// or d_split (device, async).
template <typename K>
static pp_status partition_stable(const K* in, K* out, uint64_t n, K pivot, void* stream, uint64_t* split_out,
                                  uint64_t* d_split) {
    std::lock_guard<std::mutex> lk(g_mu);
    if (!split_out && !d_split) {
        set_error("split_out / d_split is NULL");
        return PP_E_INVAL;
    }
    pp_status s = check_device_keys(in, n);
    if (s == PP_OK) s = check_device_keys(out, n);
    if (s != PP_OK) return s;
    if (n > 0 && in < out + n && out < in + n) {
        set_error("in and out overlap (the Standard Algorithm is out of place)");
        return PP_E_INVAL;
    }
    cudaStream_t st = (cudaStream_t)stream;
    g_last_ctl = nullptr;
    if (n == 0) {
        g_stats = LastStats();
        if (split_out) *split_out = 0;
        if (d_split) {
            const cudaError_t e = cudaMemsetAsync(d_split, 0, sizeof(uint64_t), st);
            if (e != cudaSuccess) return cuda_fail(e, "memset");
        }
        return PP_OK;
    }
    WsOrder ws_order(st);
    if (d_split) return partition_stable_device<K>(in, out, n, pivot, st, d_split, nullptr);
    uint64_t* pw = pinned_word();
    if (!pw) {
        set_error("cudaMallocHost failed");
        return PP_E_NOMEM;
    }
    uint64_t* total = nullptr;
    s = partition_stable_device<K>(in, out, n, pivot, st, nullptr, &total);
    if (s != PP_OK) return s;
    cudaError_t e = cudaMemcpyAsync(pw, total, 8, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return cuda_fail(e, "stable partition");
    *split_out = *pw;
    return PP_OK;
}

// Blocked-Prefix-Sum partition (pp_bps.cu), in place; sync (split_out) or
// async (d_split).
template <typename K>
static pp_status partition_bps(K* keys, uint64_t n, K pivot, void* stream, uint64_t* split_out, uint64_t* d_split) {
    std::lock_guard<std::mutex> lk(g_mu);
    if (!split_out && !d_split) {
        set_error("split_out / d_split is NULL");
        return PP_E_INVAL;
    }
    pp_status s = check_device_keys(keys, n);
    if (s != PP_OK) return s;
    cudaStream_t st = (cudaStream_t)stream;
    g_last_ctl = nullptr;
    if (n == 0) {
        g_stats = LastStats();
        if (split_out) *split_out = 0;
        if (d_split) {
            const cudaError_t e = cudaMemsetAsync(d_split, 0, sizeof(uint64_t), st);
            if (e != cudaSuccess) return cuda_fail(e, "memset");
        }
        return PP_OK;
    }
    WsOrder ws_order(st);
    if (d_split) return partition_bps_device<K>(keys, n, pivot, st, d_split);
    uint64_t* pw = pinned_word();
    uint64_t* dk = static_cast<uint64_t*>(host_split_slot());
    if (!pw || !dk) {
        set_error("split buffers unavailable");
        return PP_E_NOMEM;
    }
    s = partition_bps_device<K>(keys, n, pivot, st, dk);
    if (s != PP_OK) return s;
    cudaError_t e = cudaMemcpyAsync(pw, dk, 8, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return cuda_fail(e, "bps partition");
    *split_out = *pw;
    return PP_OK;
}

// In-place stable partition (pp_stable.cu): synchronous, split to the host.
template <typename K>
static pp_status partition_stable_inplace(K* keys, uint64_t n, K pivot, void* stream, uint64_t* split_out) {
    std::lock_guard<std::mutex> lk(g_mu);
    if (!split_out) {
        set_error("split_out is NULL");
        return PP_E_INVAL;
    }
    pp_status s = check_device_keys(keys, n);
    if (s != PP_OK) return s;
    g_last_ctl = nullptr;
    if (n == 0) {
        g_stats = LastStats();
        *split_out = 0;
        return PP_OK;
    }
    cudaStream_t st = (cudaStream_t)stream;
    uint64_t* pw = pinned_word();
    uint64_t* dk = static_cast<uint64_t*>(host_split_slot());
    if (!pw || !dk) {
        set_error("split buffers unavailable");
        return PP_E_NOMEM;
    }
    {
        WsOrder ws_order(st);
        s = partition_stable_inplace_device<K>(keys, n, pivot, st, dk);
    }
    if (s != PP_OK) return s;
    cudaError_t e = cudaMemcpyAsync(pw, dk, 8, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return cuda_fail(e, "stable in-place partition");
    *split_out = *pw;
    return PP_OK;
}

template <typename K>
static pp_status quicksort_sync(K* keys, uint64_t n, void* stream) {
    std::lock_guard<std::mutex> lk(g_mu);
    pp_status s = check_device_keys(keys, n);
    if (s != PP_OK) return s;
    if (n <= 1) return PP_OK;
    cudaStream_t st = (cudaStream_t)stream;
    g_last_ctl = nullptr;
    {
        WsOrder ws_order(st);
        s = quicksort_device<K>(keys, n, st);
    }
    if (s != PP_OK) return s;
    cudaError_t e = cudaStreamSynchronize(st);
    return e == cudaSuccess ? PP_OK : cuda_fail(e, "quicksort");
}

// host-buffer variants: library-owned device buffer, H2D, work, D2H
static void* g_hbuf = nullptr;
static size_t g_hbuf_bytes = 0;
static cudaStream_t g_hstream = nullptr;
static void* host_device_buffer(size_t bytes) {
    if (!g_hstream) cudaStreamCreateWithFlags(&g_hstream, cudaStreamNonBlocking);
    if (bytes <= g_hbuf_bytes) return g_hbuf;
    if (g_hbuf) cudaFree(g_hbuf);
    g_hbuf = nullptr;
    g_hbuf_bytes = 0;
    if (cudaMalloc(&g_hbuf, bytes) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    g_hbuf_bytes = bytes;
    return g_hbuf;
}

// Host-buffer partition with the transfers streamed.  A
// partition's arrangement within each side is free, so the
// host result is built chunk by chunk: chunks of C keys are uploaded
// alternately from the front and the back of the array (copy engine 1), each
// is partitioned in place on the device as soon as it lands (the full GPU
// partition, one launch chain per chunk), and its predecessors are written
// back to the host front [T, T + t_c), its successors to the host back
// [n - F - f_c, n - F) (copy engine 2), each as soon as every host position
// of its destination has been uploaded (its original key is on the device).
// Uploading from both ends keeps both destination frontiers covered, so the
// downloads overlap the uploads on the full-duplex link.  Result: keys < pivot
// in [0, K), the rest in [K, n); the split K is returned.
static cudaStream_t g_hs_up = nullptr, g_hs_dn = nullptr;
static std::vector<cudaEvent_t> g_hs_ev_up, g_hs_ev_part;
static uint64_t* g_hs_splits = nullptr;  // pinned, one per chunk
static size_t g_hs_nsplit = 0;
static uint64_t* g_hs_dsplit = nullptr;  // device, one per chunk
static size_t g_hs_ndsplit = 0;

template <typename K>
static pp_status partition_host(K* host_keys, uint64_t n, K pivot, uint64_t* split_out) {
    if (!split_out || (n > 0 && !host_keys)) {
        set_error("NULL argument");
        return PP_E_INVAL;
    }
    if (n == 0) {
        *split_out = 0;
        return PP_OK;
    }
    std::lock_guard<std::mutex> lk(g_mu);
    K* d = static_cast<K*>(host_device_buffer(n * sizeof(K)));
    if (!d) {
        set_error("device buffer allocation failed");
        return PP_E_NOMEM;
    }
    g_last_ctl = nullptr;
    WsOrder ws_order(g_hstream);
    if (!g_hs_up) {
        cudaStreamCreateWithFlags(&g_hs_up, cudaStreamNonBlocking);
        cudaStreamCreateWithFlags(&g_hs_dn, cudaStreamNonBlocking);
    }
    const uint64_t C = (uint64_t)std::max<int64_t>(g_params.host_chunk, 1 << 12);
    const uint64_t nch = (n + C - 1) / C;
    auto clen = [&](uint64_t c) { return std::min<uint64_t>(C, n - c * C); };
    while (g_hs_ev_up.size() < nch) {
        cudaEvent_t a, b;
        cudaEventCreateWithFlags(&a, cudaEventDisableTiming);
        cudaEventCreateWithFlags(&b, cudaEventDisableTiming);
        g_hs_ev_up.push_back(a);
        g_hs_ev_part.push_back(b);
    }
    if (g_hs_nsplit < nch) {
        if (g_hs_splits) cudaFreeHost(g_hs_splits);
        g_hs_splits = nullptr;
        g_hs_nsplit = 0;
        if (cudaMallocHost(&g_hs_splits, 8 * nch) != cudaSuccess) {
            cudaGetLastError();
            set_error("pinned split buffer allocation failed");
            return PP_E_NOMEM;
        }
        g_hs_nsplit = nch;
    }
    if (g_hs_ndsplit < nch) {
        cudaStreamSynchronize(g_hstream);
        if (g_hs_dsplit) cudaFree(g_hs_dsplit);
        g_hs_dsplit = nullptr;
        g_hs_ndsplit = 0;
        if (cudaMalloc(&g_hs_dsplit, 8 * nch) != cudaSuccess) {
            cudaGetLastError();
            set_error("device split buffer allocation failed");
            return PP_E_NOMEM;
        }
        g_hs_ndsplit = nch;
    }
    // upload order: front, back, front, back, ...; seq[c] = position in it
    std::vector<uint64_t> order(nch), seq(nch);
    for (uint64_t k = 0, f = 0, b = nch; k < nch; ++k) {
        const uint64_t c = (k % 2 == 0) ? f++ : --b;
        order[k] = c;
        seq[c] = k;
    }
    cudaError_t e = cudaSuccess;
    for (uint64_t k = 0; k < nch && e == cudaSuccess; ++k) {
        const uint64_t c = order[k];
        e = cudaMemcpyAsync(d + c * C, host_keys + c * C, clen(c) * sizeof(K), cudaMemcpyHostToDevice, g_hs_up);
        if (e == cudaSuccess) e = cudaEventRecord(g_hs_ev_up[c], g_hs_up);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(g_hstream, g_hs_ev_up[c], 0);
        if (e != cudaSuccess) break;
        const pp_status ps = partition_device<K>(d + c * C, clen(c), pivot, g_hstream, g_hs_dsplit + c, nullptr);
        if (ps != PP_OK) return ps;
        e = cudaMemcpyAsync(g_hs_splits + c, g_hs_dsplit + c, 8, cudaMemcpyDeviceToHost, g_hstream);
        if (e == cudaSuccess) e = cudaEventRecord(g_hs_ev_part[c], g_hstream);
    }
    if (e != cudaSuccess) return cuda_fail(e, "streamed partition enqueue");
    // downloads, in upload order; a destination range waits for the upload
    // of every chunk it overlaps (uploads complete in order: the latest one)
    uint64_t T = 0, F = 0;
    auto download = [&](uint64_t c, uint64_t src_off, uint64_t len, uint64_t dst) -> cudaError_t {
        if (len == 0) return cudaSuccess;
        uint64_t last = 0;
        for (uint64_t j = dst / C; j <= (dst + len - 1) / C; ++j) last = std::max(last, seq[j]);
        cudaError_t r = cudaStreamWaitEvent(g_hs_dn, g_hs_ev_up[order[last]], 0);
        if (r == cudaSuccess) r = cudaStreamWaitEvent(g_hs_dn, g_hs_ev_part[c], 0);
        if (r == cudaSuccess)
            r = cudaMemcpyAsync(host_keys + dst, d + c * C + src_off, len * sizeof(K), cudaMemcpyDeviceToHost,
                                g_hs_dn);
        return r;
    };
    for (uint64_t k = 0; k < nch && e == cudaSuccess; ++k) {
        const uint64_t c = order[k];
        e = cudaEventSynchronize(g_hs_ev_part[c]);
        if (e != cudaSuccess) break;
        const uint64_t t = g_hs_splits[c], f = clen(c) - t;
        e = download(c, 0, t, T);
        if (e == cudaSuccess) e = download(c, t, f, n - F - f);
        T += t;
        F += f;
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(g_hs_dn);
    if (e != cudaSuccess) return cuda_fail(e, "streamed partition");
    *split_out = T;
    return PP_OK;
}

template <typename K>
static pp_status quicksort_host(K* host_keys, uint64_t n) {
    if (n > 0 && !host_keys) {
        set_error("NULL argument");
        return PP_E_INVAL;
    }
    if (n <= 1) return PP_OK;
    K* d;
    {
        std::lock_guard<std::mutex> lk(g_mu);
        d = static_cast<K*>(host_device_buffer(n * sizeof(K)));
        if (!d) {
            set_error("device buffer allocation failed");
            return PP_E_NOMEM;
        }
        cudaError_t e = cudaMemcpyAsync(d, host_keys, n * sizeof(K), cudaMemcpyHostToDevice, g_hstream);
        if (e != cudaSuccess) return cuda_fail(e, "H2D");
    }
    pp_status s = quicksort_sync<K>(d, n, g_hstream);
    if (s != PP_OK) return s;
    std::lock_guard<std::mutex> lk(g_mu);
    cudaError_t e = cudaMemcpyAsync(host_keys, d, n * sizeof(K), cudaMemcpyDeviceToHost, g_hstream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(g_hstream);
    if (e != cudaSuccess) return cuda_fail(e, "D2H");
    return PP_OK;
}

template <typename K>
static pp_status ss_groups(K* keys, uint64_t n, K pivot, uint64_t g, void* stream, uint64_t* T, uint64_t* vlo,
                           uint64_t* vhi, uint64_t* info) {
    std::lock_guard<std::mutex> lk(g_mu);
    pp_status s = check_device_keys(keys, n);
    if (s != PP_OK) return s;
    if (!T || !vlo || !vhi || !info) {
        set_error("NULL output array");
        return PP_E_INVAL;
    }
    WsOrder ws_order((cudaStream_t)stream);
    return ss_groups_device<K>(keys, n, pivot, g, (cudaStream_t)stream, T, vlo, vhi, info);
}

}  // namespace pp

using namespace pp;

extern "C" {

pp_status pp_partition_u64(uint64_t* keys, uint64_t n, uint64_t pivot, void* stream, uint64_t* split_out) {
    return partition_sync<uint64_t>(keys, n, pivot, stream, split_out);
}
pp_status pp_partition_u32(uint32_t* keys, uint64_t n, uint32_t pivot, void* stream, uint64_t* split_out) {
    return partition_sync<uint32_t>(keys, n, pivot, stream, split_out);
}
pp_status pp_partition_async_u64(uint64_t* keys, uint64_t n, uint64_t pivot, void* stream, uint64_t* d_split) {
    return partition_async<uint64_t>(keys, n, pivot, stream, d_split);
}
pp_status pp_partition_async_u32(uint32_t* keys, uint64_t n, uint32_t pivot, void* stream, uint64_t* d_split) {
    return partition_async<uint32_t>(keys, n, pivot, stream, d_split);
}
pp_status pp_quicksort_u64(uint64_t* keys, uint64_t n, void* stream) {
    return quicksort_sync<uint64_t>(keys, n, stream);
}
pp_status pp_partition_stable_u64(const uint64_t* in, uint64_t* out, uint64_t n, uint64_t pivot, void* stream,
                                  uint64_t* split_out) {
    return partition_stable<uint64_t>(in, out, n, pivot, stream, split_out, nullptr);
}
pp_status pp_partition_stable_u32(const uint32_t* in, uint32_t* out, uint64_t n, uint32_t pivot, void* stream,
                                  uint64_t* split_out) {
    return partition_stable<uint32_t>(in, out, n, pivot, stream, split_out, nullptr);
}
pp_status pp_partition_stable_inplace_u64(uint64_t* keys, uint64_t n, uint64_t pivot, void* stream,
                                          uint64_t* split_out) {
    return partition_stable_inplace<uint64_t>(keys, n, pivot, stream, split_out);
}
pp_status pp_partition_stable_inplace_u32(uint32_t* keys, uint64_t n, uint32_t pivot, void* stream,
                                          uint64_t* split_out) {
    return partition_stable_inplace<uint32_t>(keys, n, pivot, stream, split_out);
}
pp_status pp_partition_bps_u64(uint64_t* keys, uint64_t n, uint64_t pivot, void* stream, uint64_t* split_out) {
    return partition_bps<uint64_t>(keys, n, pivot, stream, split_out, nullptr);
}
pp_status pp_partition_bps_u32(uint32_t* keys, uint64_t n, uint32_t pivot, void* stream, uint64_t* split_out) {
    return partition_bps<uint32_t>(keys, n, pivot, stream, split_out, nullptr);
}
pp_status pp_partition_bps_async_u64(uint64_t* keys, uint64_t n, uint64_t pivot, void* stream, uint64_t* d_split) {
    return partition_bps<uint64_t>(keys, n, pivot, stream, nullptr, d_split);
}
pp_status pp_swap_ranges_u64(const uint64_t* triples, uint64_t n_pieces, void* stream) {
    std::lock_guard<std::mutex> lk(g_mu);
    return swap_ranges<uint64_t>(triples, n_pieces, (cudaStream_t)stream);
}
pp_status pp_swap_ranges_u32(const uint64_t* triples, uint64_t n_pieces, void* stream) {
    std::lock_guard<std::mutex> lk(g_mu);
    return swap_ranges<uint32_t>(triples, n_pieces, (cudaStream_t)stream);
}
pp_status pp_partition_stable_async_u64(const uint64_t* in, uint64_t* out, uint64_t n, uint64_t pivot,
                                        void* stream, uint64_t* d_split) {
    return partition_stable<uint64_t>(in, out, n, pivot, stream, nullptr, d_split);
}
pp_status pp_quicksort_u32(uint32_t* keys, uint64_t n, void* stream) {
    return quicksort_sync<uint32_t>(keys, n, stream);
}
pp_status pp_partition_host_u64(uint64_t* host_keys, uint64_t n, uint64_t pivot, uint64_t* split_out) {
    return partition_host<uint64_t>(host_keys, n, pivot, split_out);
}
pp_status pp_partition_host_u32(uint32_t* host_keys, uint64_t n, uint32_t pivot, uint64_t* split_out) {
    return partition_host<uint32_t>(host_keys, n, pivot, split_out);
}
pp_status pp_quicksort_host_u64(uint64_t* host_keys, uint64_t n) { return quicksort_host<uint64_t>(host_keys, n); }

uint64_t pp_partition(uint64_t* keys, uint64_t n, uint64_t pivot) {
    uint64_t k = 0;
    return pp_partition_u64(keys, n, pivot, nullptr, &k) == PP_OK ? k : UINT64_MAX;
}
pp_status pp_quicksort(uint64_t* keys, uint64_t n) { return pp_quicksort_u64(keys, n, nullptr); }

pp_status pp_ss_groups_u64(uint64_t* keys, uint64_t n, uint64_t pivot, uint64_t g, void* stream, uint64_t* T,
                           uint64_t* vlo, uint64_t* vhi, uint64_t* info) {
    return ss_groups<uint64_t>(keys, n, pivot, g, stream, T, vlo, vhi, info);
}
pp_status pp_ss_groups_u32(uint32_t* keys, uint64_t n, uint32_t pivot, uint64_t g, void* stream, uint64_t* T,
                           uint64_t* vlo, uint64_t* vhi, uint64_t* info) {
    return ss_groups<uint32_t>(keys, n, pivot, g, stream, T, vlo, vhi, info);
}
uint64_t pp_max_groups(void) { return max_groups(); }

pp_status pp_dist_unique_id(void* out128) {
    std::lock_guard<std::mutex> lk(g_mu);
    return dist_unique_id(out128);
}
pp_status pp_dist_init(const void* id128, int nranks, int rank, int device) {
    std::lock_guard<std::mutex> lk(g_mu);
    return dist_init(id128, nranks, rank, device);
}
pp_status pp_dist_finalize(void) {
    std::lock_guard<std::mutex> lk(g_mu);
    return dist_finalize();
}
pp_status pp_dist_set_staging(uint64_t bytes) {
    std::lock_guard<std::mutex> lk(g_mu);
    dist_set_staging(bytes);
    return PP_OK;
}
pp_status pp_partition_dist_u64(uint64_t* shard, uint64_t n_local, uint64_t pivot, void* stream,
                                uint64_t* global_split_out) {
    std::lock_guard<std::mutex> lk(g_mu);
    pp_status s = check_device_keys(shard, n_local);
    if (s != PP_OK) return s;
    WsOrder ws_order((cudaStream_t)stream);
    return partition_dist<uint64_t>(shard, n_local, pivot, (cudaStream_t)stream, global_split_out);
}
pp_status pp_partition_dist_u32(uint32_t* shard, uint64_t n_local, uint32_t pivot, void* stream,
                                uint64_t* global_split_out) {
    std::lock_guard<std::mutex> lk(g_mu);
    pp_status s = check_device_keys(shard, n_local);
    if (s != PP_OK) return s;
    WsOrder ws_order((cudaStream_t)stream);
    return partition_dist<uint32_t>(shard, n_local, pivot, (cudaStream_t)stream, global_split_out);
}
pp_status pp_quicksort_dist_u64(uint64_t* shard, uint64_t n_local, void* stream) {
    std::lock_guard<std::mutex> lk(g_mu);
    pp_status s = check_device_keys(shard, n_local);
    if (s != PP_OK) return s;
    WsOrder ws_order((cudaStream_t)stream);
    return quicksort_dist<uint64_t>(shard, n_local, (cudaStream_t)stream, (uint64_t)g_params.dist_small);
}
pp_status pp_quicksort_dist_u32(uint32_t* shard, uint64_t n_local, void* stream) {
    std::lock_guard<std::mutex> lk(g_mu);
    pp_status s = check_device_keys(shard, n_local);
    if (s != PP_OK) return s;
    WsOrder ws_order((cudaStream_t)stream);
    return quicksort_dist<uint32_t>(shard, n_local, (cudaStream_t)stream, (uint64_t)g_params.dist_small);
}
pp_status pp_partition_dist_loopback_u64(uint64_t* keys, const uint64_t* ns, int nranks, uint64_t pivot,
                                         uint64_t* global_split_out) {
    std::lock_guard<std::mutex> lk(g_mu);
    uint64_t n = 0;
    for (int r = 0; ns && r < nranks; ++r) n += ns[r];
    pp_status s = check_device_keys(keys, n);
    if (s != PP_OK) return s;
    return partition_dist_loopback<uint64_t>(keys, ns, nranks, pivot, global_split_out);
}
pp_status pp_partition_dist_loopback_u32(uint32_t* keys, const uint64_t* ns, int nranks, uint32_t pivot,
                                         uint64_t* global_split_out) {
    std::lock_guard<std::mutex> lk(g_mu);
    uint64_t n = 0;
    for (int r = 0; ns && r < nranks; ++r) n += ns[r];
    pp_status s = check_device_keys(keys, n);
    if (s != PP_OK) return s;
    return partition_dist_loopback<uint32_t>(keys, ns, nranks, pivot, global_split_out);
}
pp_status pp_quicksort_dist_loopback_u64(uint64_t* keys, const uint64_t* ns, int nranks) {
    std::lock_guard<std::mutex> lk(g_mu);
    uint64_t n = 0;
    for (int r = 0; ns && r < nranks; ++r) n += ns[r];
    pp_status s = check_device_keys(keys, n);
    if (s != PP_OK) return s;
    return quicksort_dist_loopback<uint64_t>(keys, ns, nranks, (uint64_t)g_params.dist_small);
}
pp_status pp_quicksort_dist_loopback_u32(uint32_t* keys, const uint64_t* ns, int nranks) {
    std::lock_guard<std::mutex> lk(g_mu);
    uint64_t n = 0;
    for (int r = 0; ns && r < nranks; ++r) n += ns[r];
    pp_status s = check_device_keys(keys, n);
    if (s != PP_OK) return s;
    return quicksort_dist_loopback<uint32_t>(keys, ns, nranks, (uint64_t)g_params.dist_small);
}
pp_status pp_dist_plan(const uint64_t* ns, const uint64_t* ts, int nranks, uint64_t cap, uint64_t* out,
                       uint64_t out_cap, uint64_t* n_out, uint64_t* K_out) {
    return dist_plan(ns, ts, nranks, cap, out, out_cap, n_out, K_out);
}
pp_status pp_dist_p2p_pieces(const uint64_t* ns, const uint64_t* ts, int nranks, int rank, uint64_t* out,
                             uint64_t out_cap, uint64_t* n_out) {
    return dist_p2p_pieces(ns, ts, nranks, rank, out, out_cap, n_out);
}
pp_status pp_ipc_export(const void* d_ptr, void* handle_out, uint64_t* offset_out) {
    std::lock_guard<std::mutex> lk(g_mu);
    return ipc_export(d_ptr, handle_out, offset_out);
}
pp_status pp_ipc_import(const void* handle, uint64_t offset, void** d_ptr_out) {
    std::lock_guard<std::mutex> lk(g_mu);
    return ipc_import(handle, offset, d_ptr_out);
}
pp_status pp_dist_last_timing(double* out4) {
    std::lock_guard<std::mutex> lk(g_mu);
    return dist_last_timing(out4);
}
pp_status pp_ipc_close_all(void) {
    std::lock_guard<std::mutex> lk(g_mu);
    return ipc_close_all();
}

uint64_t pp_workspace_bytes(uint64_t n, int key_bytes, int op) {
    std::lock_guard<std::mutex> lk(g_mu);
    const uint64_t part = (partition_workspace_bound(n) + 255) & ~uint64_t(255);
    if (op != 1) return part;
    return part + (key_bytes == 4 ? quicksort_workspace_bound<uint32_t>(n) : quicksort_workspace_bound<uint64_t>(n));
}
pp_status pp_set_workspace(void* d_ws, uint64_t bytes) {
    std::lock_guard<std::mutex> lk(g_mu);
    if (!d_ws) {
        g_user_ws = nullptr;
        g_user_ws_bytes = 0;
        return PP_OK;
    }
    if (bytes == 0 || (uintptr_t)d_ws % 256) {
        set_error("pp_set_workspace: workspace must be non-empty and 256-byte aligned");
        return PP_E_INVAL;
    }
    cudaPointerAttributes a;
    cudaError_t e = cudaPointerGetAttributes(&a, d_ws);
    if (e != cudaSuccess || (a.type != cudaMemoryTypeDevice && a.type != cudaMemoryTypeManaged)) {
        cudaGetLastError();
        set_error("pp_set_workspace: not a device pointer");
        return PP_E_INVAL;
    }
    g_user_ws = d_ws;
    g_user_ws_bytes = bytes;
    return PP_OK;
}
uint64_t pp_last_aux_bytes(void) { return g_stats.aux_bytes; }

pp_status pp_last_stats(uint64_t* out) {
    std::lock_guard<std::mutex> lk(g_mu);
    if (!out) return PP_E_INVAL;
    Ctl c;
    memset(&c, 0, sizeof(c));
    if (g_last_ctl) {  // read on the stream of the call that wrote it
        cudaError_t e = cudaMemcpyAsync(&c, g_last_ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, g_last_ctl_st);
        if (e == cudaSuccess) e = cudaStreamSynchronize(g_last_ctl_st);
        if (e != cudaSuccess) return cuda_fail(e, "stats");
    }
    const LastStats& S = g_stats;
    uint64_t v[13] = {S.n, c.K, c.W, c.vmin, c.vmax, c.ML, S.g, S.line_keys, S.n_lines, S.head,
                      S.aux_bytes, S.path, c.nTasks};
    memcpy(out, v, sizeof(v));
    if (c.err) {
        set_error("device invariant check failed (misplaced counts differ)");
        return PP_E_INTERNAL;
    }
    return PP_OK;
}

pp_status pp_audit_set(uint32_t* d_shadow, const void* keys, uint64_t n, int key_bytes) {
    std::lock_guard<std::mutex> lk(g_mu);
    if (d_shadow != nullptr && (keys == nullptr || (key_bytes != 4 && key_bytes != 8))) {
        set_error("pp_audit_set: keys and key_bytes (4 or 8) required with a shadow array");
        return PP_E_INVAL;
    }
    return audit_set_partition(d_shadow, keys, d_shadow ? n : 0, (uint32_t)(key_bytes > 0 ? key_bytes : 8));
}

pp_status pp_quicksort_last_stats(uint64_t* out6) {
    std::lock_guard<std::mutex> lk(g_mu);
    return quicksort_last_stats(out6);
}

void pp_reset_params(void) {
    std::lock_guard<std::mutex> lk(g_mu);
    g_params = Params();
}

pp_status pp_set_param(const char* name, int64_t value) {
    std::lock_guard<std::mutex> lk(g_mu);
    if (!name) return PP_E_INVAL;
    Params& P = g_params;
    std::string k(name);
    if (k == "g") P.g = value;
    else if (k == "min_lines_per_group") P.min_lines_per_group = value;
    else if (k == "small_n") P.small_n = value;
    else if (k == "path") P.path = value;
    else if (k == "tile") P.tile = value;
    else if (k == "ranks") P.ranks = value;
    else if (k == "seed") P.seed = (uint64_t)value;
    else if (k == "strided") P.seed = value ? 0 : Params().seed;
    else if (k == "leaf") P.leaf = value;
    else if (k == "qs_cta_max") P.qs_cta_max = value;
    else if (k == "qs_small") P.qs_small = value;
    else if (k == "qs_waves") P.qs_waves = value;
    else if (k == "qs_heavy") P.qs_heavy = value;
    else if (k == "qs_prio") P.qs_prio = value;
    else if (k == "qs_dev") P.qs_dev = value;
    else if (k == "dist_split") P.dist_split = value ? 1 : 0;
    else if (k == "qs_dev_check") P.qs_dev_check = value;
    else if (k == "host_chunk") P.host_chunk = value;
    else if (k == "dist_p2p") P.dist_p2p = value ? 1 : 0;
    else if (k == "dist_timeout_ms") P.dist_timeout_ms = value < 1 ? 1 : value;
    else if (k == "dist_fault") P.dist_fault = value;
    else if (k == "dist_fault_rank") P.dist_fault_rank = value;
    else if (k == "dist_small") P.dist_small = value < 1 ? 1 : value;
    else if (k == "dist_overlap") P.dist_overlap = value ? 1 : 0;
    else if (k == "dist_chunks") P.dist_chunks = value < 1 ? 1 : value > 1024 ? 1024 : value;
    else if (k == "qs_lanes") P.qs_lanes = value;
    else if (k == "qs_deep") P.qs_deep = value;
    else if (k == "qs_pivot") P.qs_pivot = value < 0 || value > 2 ? 0 : value;
    else if (k == "qs_early") P.qs_early = value;
    else if (k == "qs_early_min") P.qs_early_min = value;
    else if (k == "qs_minl") P.qs_minl = value;
    else if (k == "bps_nt") P.bps_nt = value;
    else if (k == "cleanup_chain") P.cleanup_chain = value;
    else if (k == "cleanup_bitmap") P.cleanup_bitmap = value;
    else {
        set_error("unknown parameter " + k);
        return PP_E_INVAL;
    }
    return PP_OK;
}
int64_t pp_get_param(const char* name) {
    std::lock_guard<std::mutex> lk(g_mu);
    if (!name) return INT64_MIN;
    const Params& P = g_params;
    std::string k(name);
    if (k == "g") return P.g;
    if (k == "min_lines_per_group") return P.min_lines_per_group;
    if (k == "small_n") return P.small_n;
    if (k == "path") return P.path;
    if (k == "tile") return P.tile;
    if (k == "ranks") return P.ranks;
    if (k == "seed") return (int64_t)P.seed;
    if (k == "strided") return P.seed == 0 ? 1 : 0;
    if (k == "leaf") return P.leaf;
    if (k == "qs_cta_max") return P.qs_cta_max;
    if (k == "qs_small") return P.qs_small;
    if (k == "qs_waves") return P.qs_waves;
    if (k == "qs_heavy") return P.qs_heavy;
    if (k == "qs_prio") return P.qs_prio;
    if (k == "qs_dev") return P.qs_dev;
    if (k == "dist_split") return P.dist_split;
    if (k == "qs_dev_check") return P.qs_dev_check;
    if (k == "host_chunk") return P.host_chunk;
    if (k == "dist_p2p") return P.dist_p2p;
    if (k == "dist_timeout_ms") return P.dist_timeout_ms;
    if (k == "dist_fault") return P.dist_fault;
    if (k == "dist_fault_rank") return P.dist_fault_rank;
    if (k == "dist_small") return P.dist_small;
    if (k == "dist_overlap") return P.dist_overlap;
    if (k == "dist_chunks") return P.dist_chunks;
    if (k == "qs_lanes") return P.qs_lanes;
    if (k == "qs_deep") return P.qs_deep;
    if (k == "qs_pivot") return P.qs_pivot;
    if (k == "qs_early") return P.qs_early;
    if (k == "qs_early_min") return P.qs_early_min;
    if (k == "qs_minl") return P.qs_minl;
    if (k == "bps_nt") return P.bps_nt;
    if (k == "cleanup_chain") return P.cleanup_chain;
    if (k == "cleanup_bitmap") return P.cleanup_bitmap;
    return INT64_MIN;
}

const char* pp_status_string(pp_status s) {
    switch (s) {
        case PP_OK: return "PP_OK";
        case PP_E_INVAL: return "PP_E_INVAL";
        case PP_E_CUDA: return "PP_E_CUDA";
        case PP_E_NOMEM: return "PP_E_NOMEM";
        case PP_E_NCCL: return "PP_E_NCCL";
        case PP_E_INTERNAL: return "PP_E_INTERNAL";
    }
    return "PP_E_UNKNOWN";
}
const char* pp_last_error(void) { return g_err.c_str(); }
uint64_t pp_launch_count(int reset) { return launch_count(reset); }
void pp_timing(int enable) {
    std::lock_guard<std::mutex> lk(g_mu);
    timing_enable(enable);
}
pp_status pp_timing_read(double* out4) {
    std::lock_guard<std::mutex> lk(g_mu);
    if (!out4) return PP_E_INVAL;
    int r = timing_read(out4);
    if (r) {
        set_error("timing events incomplete or failed");
        return r == 1 ? PP_E_INVAL : PP_E_CUDA;
    }
    return PP_OK;
}

}  // extern "C"
