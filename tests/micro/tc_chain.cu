// Microbenchmark: latency and throughput of the split-BF16 MMA chains
// k_evaluate_tc issues (6 accumulating tcgen05.mma kind::f16, M = 128, K = 16,
// N columns, then one commit), alone and with several CTAs per SM. Not part of
// the product; informs k_evaluate_tc's unit size and pipelining.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tc_chain tc_chain.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((128u >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((256u >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;
    return d;
}
__device__ __forceinline__ uint32_t idesc(int n) {
    return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | (8u << 24);
}
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
        "l"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void wait_bar(uint64_t* bar, uint32_t ph) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tW_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"(su32(bar)),
        "r"(ph)
        : "memory");
}

// mode 0: latency (commit + wait after each 6-MMA set); mode 1: throughput (one commit
// and wait at the end)
__global__ void k_chain(int n, int chains, int ncols, int reps, int mode, unsigned long long* out) {
    extern __shared__ __align__(1024) char sm[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    const int tid = threadIdx.x;
    for (int i = tid; i < 3 * 4096 + 3 * n * chains * 32; i += blockDim.x) sm[i] = 0;
    if (tid < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tbase)),
                     "r"((uint32_t)ncols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tm = tbase;
    if (tid == 0) {
        const uint32_t sA = su32(sm), sB = su32(sm + 3 * 4096);
        const uint32_t id = idesc(n);
        constexpr int pa[6] = {0, 1, 2, 0, 1, 0};
        constexpr int pb[6] = {2, 1, 0, 1, 0, 0};
        uint32_t ph = 0;
        unsigned long long t0 = clock64();
        for (int r = 0; r < reps; ++r) {
            for (int q = 0; q < 6; ++q)
                for (int c = 0; c < chains; ++c)
                    mma(tm + (uint32_t)(c * n), sdesc(sA + pa[q] * 4096u),
                        sdesc(sB + pb[q] * (uint32_t)(n * 32 * chains) + (uint32_t)(c * n / 8) * 256u), id,
                        q ? 1u : 0u);
            if (mode == 0 || r == reps - 1) {
                asm volatile(
                    "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                        su32(&bar))
                    : "memory");
                wait_bar(&bar, ph);
                ph ^= 1;
            }
        }
        unsigned long long t1 = clock64();
        out[blockIdx.x] = (t1 - t0) / reps;
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (tid < 32)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"((uint32_t)ncols));
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    unsigned long long* d;
    cudaMalloc(&d, sizeof(unsigned long long) * sms * 16);
    cudaFuncSetAttribute(k_chain, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    static unsigned long long h[148 * 16];
    const int Ns[] = {32, 64, 96, 128, 160, 192, 256};
    for (int mode = 0; mode < 2; ++mode)
        for (int per_sm : {1, 2, 4})
            for (int n : Ns)
                for (int chains : {1, 2}) {
                    if (n * chains > 256) continue;
                    int ncols = 32;
                    while (ncols < n * chains) ncols <<= 1;
                    if (ncols * per_sm > 512) continue;
                    const size_t smem = (size_t)(220 * 1024) / per_sm - 4096;
                    const size_t need = 3 * 4096 + 3 * (size_t)n * chains * 32;
                    if (need > smem) continue;
                    const int reps = mode == 0 ? 200 : 2000;
                    k_chain<<<sms * per_sm, 128, smem>>>(n, chains, ncols, reps, mode, d);
                    cudaError_t e = cudaGetLastError();
                    if (e == cudaSuccess) e = cudaDeviceSynchronize();
                    if (e != cudaSuccess) {
                        printf("error %s\n", cudaGetErrorString(e));
                        return 1;
                    }
                    cudaMemcpy(h, d, sizeof(unsigned long long) * sms * per_sm, cudaMemcpyDeviceToHost);
                    double avg = 0;
                    for (int i = 0; i < sms * per_sm; ++i) avg += (double)h[i];
                    avg /= sms * per_sm;
                    const double flop = 6.0 * 2 * 128 * n * chains * 16;
                    printf("%s ctas/SM %d  N %3d x %d chains: %7.1f cycles per 6-MMA set  (%.0f flop/clk/SM)\n",
                           mode ? "thru" : "lat ", per_sm, n, chains, avg, flop * per_sm / avg);
                }
    return 0;
}
