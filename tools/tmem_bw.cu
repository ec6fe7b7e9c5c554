// TMEM read bandwidth on the box (the kNN epilogue's ceiling):
// every SM allocates 512 TMEM columns; W warps (4 per lane quadrant) loop
// tcgen05.ld.32x32b.x16 (+ wait::ld) over their quadrant's columns and fold the
// values into a register.  Bytes per SM-cycle = loads x 2 KB / (kernel time x clock).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/tmem_bw tools/tmem_bw.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__device__ __forceinline__ uint32_t su32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <int X>
__global__ void __launch_bounds__(512, 1) tmem_read(int iters, unsigned* sink) {
    __shared__ uint32_t tbase;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tbase)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t quad = warp & 3, slice = warp >> 2;            // 4 slices of 128 columns
    const uint32_t t0 = tbase + (quad * 32 << 16) + slice * 128;
    unsigned acc = 0;
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int c = 0; c < 128; c += 16 * X) {
            uint32_t r[16 * X];
            if (X == 1) {
                asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                             : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                               "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                             : "r"(t0 + c));
            }
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int k = 0; k < 16 * X; k++) acc ^= r[k];
        }
    }
    if (acc == 0x12345678u) sink[0] = acc;
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
    }
}

int main() {
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);   // kHz
    unsigned* sink;
    cudaMalloc(&sink, 4);
    const int iters = 20000;
    tmem_read<1><<<nsm, 512>>>(100, sink);
    cudaDeviceSynchronize();
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int rep = 0; rep < 5; rep++) {
        cudaEventRecord(e0);
        tmem_read<1><<<nsm, 512>>>(iters, sink);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    const double bytes_per_sm = (double)iters * 16 /*warps*/ * 8 /*loads*/ * 2048.0;
    const double sec = best * 1e-3;
    const double per_sm_per_s = bytes_per_sm / sec;
    printf("{\"tmem_read_bytes_per_sm_cycle_at_max_clock\": %.1f, \"tmem_read_TBps_chip\": %.2f, \"ms\": %.3f, "
           "\"max_clock_mhz\": %d, \"status\": \"%s\", \"how\": \"16 warps/SM x tcgen05.ld.32x32b.x16 + wait::ld, 512 TMEM columns, best of 5\"}\n",
           per_sm_per_s / (clk * 1e3), per_sm_per_s * nsm / 1e12, best, clk / 1000,
           cudaGetErrorString(cudaGetLastError()));
    return 0;
}
