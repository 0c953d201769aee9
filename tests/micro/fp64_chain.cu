// Microbenchmark: cycles per step of the exact re-rank's two serial FP64 chains
// (k_rerank_cta: phasor recurrence ph *= rot, and acc += p_k ph_k), single lane.
// Not part of the product; informs the C1 re-rank design.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64_chain fp64_chain.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_lat(int n, double a, double b, double* out, long long* cyc) {
    // dependent DADD chain
    double x = a;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) x = __dadd_rn(x, b);
    long long t1 = clock64();
    double y = a;
    for (int i = 0; i < n; ++i) y = __dmul_rn(y, b);
    long long t2 = clock64();
    double z = a;
    for (int i = 0; i < n; ++i) z = __fma_rn(z, b, a);
    long long t3 = clock64();
    // phasor recurrence as in exact_chain_cta
    double pr = a, pi = b, rr = 0.9999999, ri = 0.0001;
    for (int i = 0; i < n; ++i) {
        const double nr = __dsub_rn(__dmul_rn(pr, rr), __dmul_rn(pi, ri));
        pi = __dadd_rn(__dmul_rn(pr, ri), __dmul_rn(pi, rr));
        pr = nr;
    }
    long long t4 = clock64();
    out[0] = x + y + z + pr + pi;
    cyc[0] = (t1 - t0) / n;
    cyc[1] = (t2 - t1) / n;
    cyc[2] = (t3 - t2) / n;
    cyc[3] = (t4 - t3) / n;
}

int main() {
    double* o;
    long long* c;
    cudaMalloc(&o, 64);
    cudaMalloc(&c, 64);
    k_lat<<<1, 1>>>(1 << 16, 1.0, 1.0000001, o, c);
    k_lat<<<1, 1>>>(1 << 16, 1.0, 1.0000001, o, c);
    long long h[4];
    cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
    printf("cycles/step: dadd %lld  dmul %lld  dfma %lld  phasor %lld\n", h[0], h[1], h[2], h[3]);
    return 0;
}
