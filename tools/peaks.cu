// Measured device peaks for the roofline denominators MEASURED_PEAKS.json lacks
// (VERDICT r1 item 9 / SURVEY.md §8d):
//   * dense int8 tensor throughput: tcgen05.mma.cta_group::1.kind::i8, M=128 N=256
//     K=32 per instruction, operands resident in shared memory (SWIZZLE_128B
//     K-major), accumulating in TMEM — one issuing thread per SM, all 148 SMs;
//   * FP64 FMA throughput: independent DFMA chains on every SM.
// Timed with CUDA events after a warm-up launch; prints one JSON line.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/peaks tools/peaks.cu && /tmp/peaks
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

constexpr int TM = 128, TN = 256, KB = 128;   // bytes of K per smem tile
constexpr uint32_t IDESC = (2u << 4) | ((uint32_t)(TN >> 3) << 17) | ((uint32_t)(TM >> 4) << 24);

__device__ __forceinline__ uint32_t su32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)1 << 16;
    d |= (uint64_t)(1024 >> 4) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)2 << 61;
    return d;
}

__global__ void __launch_bounds__(128, 1) i8_kernel(int iters, int* sink) {
    extern __shared__ __align__(1024) uint8_t raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    uint8_t* A = sm;                      // 128 x 128 B
    uint8_t* B = sm + TM * KB;            // 256 x 128 B
    __shared__ uint32_t tbase;
    __shared__ __align__(8) uint64_t bar;
    for (int i = threadIdx.x; i < (TM + TN) * KB; i += blockDim.x) sm[i] = (uint8_t)(i * 37 + 11);
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(su32(&tbase)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (threadIdx.x == 0) {
        const uint32_t a0 = su32(A), b0 = su32(B);
        for (int it = 0; it < iters; it++) {
#pragma unroll
            for (int k = 0; k < KB / 32; k++) {
                const uint64_t ad = desc_sw128(a0 + 32 * k), bd = desc_sw128(b0 + 32 * k);
                const uint32_t acc = (it | k) ? 1u : 0u;
                asm volatile(
                    "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
                    " tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tbase),
                    "l"(ad), "l"(bd), "r"(IDESC), "r"(acc));
            }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
            su32(&bar)) : "memory");
        uint32_t done = 0;
        while (!done) {
            asm volatile(
                "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n"
                " selp.u32 %0, 1, 0, p;\n}\n" : "=r"(done) : "r"(su32(&bar)) : "memory");
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (threadIdx.x < 32) {
        uint32_t v;
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v) : "r"(tbase));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (v == 0x12345678u) sink[0] = 1;
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tbase));
    }
}

__global__ void fp64_kernel(int iters, double* out) {
    double a[8];
#pragma unroll
    for (int j = 0; j < 8; j++) a[j] = threadIdx.x * 1e-9 + j;
    const double m = 0.999999, c = 1e-7;
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int j = 0; j < 8; j++) a[j] = fma(a[j], m, c);
    }
    double s = 0;
#pragma unroll
    for (int j = 0; j < 8; j++) s += a[j];
    if (s == 12345.678) out[0] = s;
}

int main() {
    int dev = 0, nsm = 0, clk = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    int* sink;
    double* dout;
    cudaMalloc(&sink, 4);
    cudaMalloc(&dout, 8);
    const size_t smem = (TM + TN) * KB + 1024;
    cudaFuncSetAttribute(i8_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    // int8: ops per MMA = 2 * M * N * K(32)
    const int iters = 20000;
    i8_kernel<<<nsm, 128, smem>>>(200, sink);
    cudaDeviceSynchronize();
    float best_i8 = 1e30f;
    for (int r = 0; r < 5; r++) {
        cudaEventRecord(e0);
        i8_kernel<<<nsm, 128, smem>>>(iters, sink);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best_i8) best_i8 = ms;
    }
    const double i8_ops = 2.0 * TM * TN * 32 * (KB / 32) * (double)iters * nsm;
    // fp64: 8 chains x iters DFMA per thread, 2 flops each
    const int fiters = 20000, fthreads = 1024, fblocks = nsm * 2;
    fp64_kernel<<<fblocks, fthreads>>>(100, dout);
    cudaDeviceSynchronize();
    float best_f = 1e30f;
    for (int r = 0; r < 5; r++) {
        cudaEventRecord(e0);
        fp64_kernel<<<fblocks, fthreads>>>(fiters, dout);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best_f) best_f = ms;
    }
    const double f_flops = 2.0 * 8 * (double)fiters * fthreads * fblocks;
    cudaError_t err = cudaGetLastError();
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
    printf("{\"int8_dense_tops\": %.1f, \"int8_how\": \"tcgen05.mma kind::i8 M=128 N=256 K=32 from smem, "
           "1 issuing thread x %d SMs, %d x 4 MMAs, best of 5 (CUDA events)\", "
           "\"fp64_tflops\": %.2f, \"fp64_how\": \"8 independent DFMA chains x %d threads x %d blocks, "
           "best of 5\", \"int8_ms\": %.3f, \"fp64_ms\": %.3f, \"sm_count\": %d, \"status\": \"%s\"}\n",
           i8_ops / (best_i8 * 1e-3) / 1e12, nsm, iters, f_flops / (best_f * 1e-3) / 1e12, fthreads,
           fblocks, best_i8, best_f, nsm, cudaGetErrorString(err));
    return err == cudaSuccess ? 0 : 1;
}
