// bwprobe.cu -- HBM bandwidth probe (diagnostic tool, not part of the
// library): read+write copy, read-only and write-only streams with 16-byte
// vector accesses, grid-stride, several grid sizes; CUDA-event timed.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__global__ void copy_kernel(const uint4* __restrict__ a, uint4* __restrict__ b, size_t n) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        b[i] = __ldcs(a + i);
}
__global__ void copy4_kernel(const uint4* __restrict__ a, uint4* __restrict__ b, size_t n) {
    // 4 independent 16-B loads in flight per thread
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + 3 * stride < n; i += 4 * stride) {
        uint4 x0 = __ldcs(a + i), x1 = __ldcs(a + i + stride), x2 = __ldcs(a + i + 2 * stride),
              x3 = __ldcs(a + i + 3 * stride);
        __stcs(b + i, x0);
        __stcs(b + i + stride, x1);
        __stcs(b + i + 2 * stride, x2);
        __stcs(b + i + 3 * stride, x3);
    }
    for (; i < n; i += stride) b[i] = __ldcs(a + i);
}
__global__ void read_kernel(const uint4* __restrict__ a, size_t n, unsigned* out) {
    unsigned acc = 0;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        const uint4 x = __ldcs(a + i);
        acc ^= x.x ^ x.y ^ x.z ^ x.w;
    }
    if (acc == 0x12345678u) out[0] = acc;
}
__global__ void write_kernel(uint4* __restrict__ b, size_t n) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        __stcs(b + i, make_uint4((unsigned)i, 1, 2, 3));
}

extern "C" int bw_probe(size_t bytes, int reps) {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const size_t n = bytes / 16;
    uint4 *a, *b;
    unsigned* o;
    if (cudaMalloc(&a, bytes) || cudaMalloc(&b, bytes) || cudaMalloc(&o, 64)) return 1;
    cudaMemset(a, 1, bytes);
    cudaMemset(b, 2, bytes);
    cudaEvent_t s, e;
    cudaEventCreate(&s);
    cudaEventCreate(&e);
    for (int kind = 0; kind < 4; ++kind) {
        for (int mult : {2, 4, 8, 16, 32}) {
            const int grid = sms * mult, block = 256;
            float best = 1e30f;
            for (int r = 0; r < reps + 1; ++r) {
                cudaEventRecord(s);
                if (kind == 0) copy_kernel<<<grid, block>>>(a, b, n);
                else if (kind == 1) copy4_kernel<<<grid, block>>>(a, b, n);
                else if (kind == 2) read_kernel<<<grid, block>>>(a, n, o);
                else write_kernel<<<grid, block>>>(b, n);
                cudaEventRecord(e);
                cudaEventSynchronize(e);
                float ms = 0;
                cudaEventElapsedTime(&ms, s, e);
                if (r > 0 && ms < best) best = ms;
            }
            const double moved = (kind <= 1 ? 2.0 : 1.0) * (double)bytes;
            printf("%s grid=%d x256: %.1f GB/s\n", kind == 0 ? "copy" : kind == 1 ? "copy4" : kind == 2 ? "read" : "write",
                   grid, moved / (best * 1e-3) / 1e9);
        }
    }
    fflush(stdout);
    cudaFree(a);
    cudaFree(b);
    cudaFree(o);
    return 0;
}
