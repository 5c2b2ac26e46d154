// Throughput probe: integer (IMAD-pipe) Harvey/Shoup butterfly vs an FP64-pipe modular
// butterfly for primes q < 2^50 (values are exact integers held in doubles).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_probe tools/fp64_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mulhi(uint64_t a, uint64_t b) { return __umul64hi(a, b); }

__global__ void k_int(uint64_t q, uint64_t w, uint64_t wsh, int iters, uint64_t *sink) {
    uint64_t x[8], y[8];
    const uint64_t q2 = 2 * q;
    for (int e = 0; e < 8; e++) {
        x[e] = (threadIdx.x * 977u + e * 131u) % q;
        y[e] = (blockIdx.x * 613u + e * 71u) % q;
    }
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int e = 0; e < 8; e++) {
            const uint64_t xx = x[e] >= q2 ? x[e] - q2 : x[e];
            const uint64_t t = y[e] * w - mulhi(y[e], wsh) * q;
            x[e] = xx + t;
            y[e] = xx - t + q2;
        }
    }
    uint64_t acc = 0;
    for (int e = 0; e < 8; e++) acc ^= x[e] ^ y[e];
    if (acc == 0x12345) sink[0] = acc;
}

// t = Y*W mod q (result in (-2q, 3q)), exact for |Y| < 2^53, W < q < 2^50
__device__ __forceinline__ double modmul_f64(double y, double w, double q, double qinv) {
    const double MAGIC = 6755399441055744.0;  // 1.5 * 2^52: rint via add/sub
    const double h = __dmul_rn(y, w);
    const double l = __fma_rn(y, w, -h);
    const double qt = __dadd_rn(__fma_rn(h, qinv, MAGIC), -MAGIC);
    return __dadd_rn(__fma_rn(-qt, q, h), l);
}

__global__ void k_f64(double q, double w, double qinv, int iters, double *sink) {
    double x[8], y[8];
    for (int e = 0; e < 8; e++) {
        x[e] = (double)((threadIdx.x * 977u + e * 131u) % 1000003u);
        y[e] = (double)((blockIdx.x * 613u + e * 71u) % 1000003u);
    }
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int e = 0; e < 8; e++) {
            const double t = modmul_f64(y[e], w, q, qinv);
            const double xn = __dadd_rn(x[e], t);
            y[e] = __dadd_rn(x[e], -t);
            // keep x bounded: one symmetric fold every butterfly (rint(x / q) * q)
            x[e] = __fma_rn(-__dadd_rn(__fma_rn(xn, qinv, 6755399441055744.0), -6755399441055744.0), q, xn);
        }
    }
    double acc = 0;
    for (int e = 0; e < 8; e++) acc += x[e] + y[e];
    if (acc == 12345.0) sink[0] = acc;
}

// mixed: half the chains on each pipe (does the SM overlap IMAD and FP64?)
__global__ void k_mix(uint64_t q, uint64_t w, uint64_t wsh, double qd, double wd, double qinv, int iters, uint64_t *sink) {
    uint64_t x[4], y[4];
    double a[4], b[4];
    const uint64_t q2 = 2 * q;
    for (int e = 0; e < 4; e++) {
        x[e] = (threadIdx.x * 977u + e * 131u) % q;
        y[e] = (blockIdx.x * 613u + e * 71u) % q;
        a[e] = (double)((threadIdx.x * 977u + e * 131u) % 1000003u);
        b[e] = (double)((blockIdx.x * 613u + e * 71u) % 1000003u);
    }
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int e = 0; e < 4; e++) {
            const uint64_t xx = x[e] >= q2 ? x[e] - q2 : x[e];
            const uint64_t t = y[e] * w - mulhi(y[e], wsh) * q;
            x[e] = xx + t;
            y[e] = xx - t + q2;
            const double u = modmul_f64(b[e], wd, qd, qinv);
            const double an = __dadd_rn(a[e], u);
            b[e] = __dadd_rn(a[e], -u);
            a[e] = __fma_rn(-__dadd_rn(__fma_rn(an, qinv, 6755399441055744.0), -6755399441055744.0), qd, an);
        }
    }
    uint64_t acc = 0;
    for (int e = 0; e < 4; e++) acc ^= x[e] ^ y[e] ^ (uint64_t)(a[e] + b[e]);
    if (acc == 0x12345) sink[0] = acc;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const uint64_t q = 1099511480321ull;  // 40-bit NTT prime (== 1 mod 2^15)
    const uint64_t w = 123456789ull % q, wsh = (uint64_t)(((unsigned __int128)w << 64) / q);
    uint64_t *sink;
    cudaMalloc(&sink, 64);
    const int blocks = sms * 8, threads = 256, iters = 4096;
    cudaEvent_t s, e;
    cudaEventCreate(&s);
    cudaEventCreate(&e);
    const double bf = (double)blocks * threads * 8 * iters;
    for (int rep = 0; rep < 2; rep++) {
        float ms;
        cudaEventRecord(s);
        k_int<<<blocks, threads>>>(q, w, wsh, iters, sink);
        cudaEventRecord(e);
        cudaEventSynchronize(e);
        cudaEventElapsedTime(&ms, s, e);
        printf("int64 Harvey/Shoup : %8.1f G butterflies/s\n", bf / (ms * 1e6));
        cudaEventRecord(s);
        k_f64<<<blocks, threads>>>((double)q, (double)w, 1.0 / (double)q, iters, (double *)sink);
        cudaEventRecord(e);
        cudaEventSynchronize(e);
        cudaEventElapsedTime(&ms, s, e);
        printf("fp64 exact modmul  : %8.1f G butterflies/s (incl. one fold per butterfly)\n", bf / (ms * 1e6));
        cudaEventRecord(s);
        k_mix<<<blocks, threads>>>(q, w, wsh, (double)q, (double)w, 1.0 / (double)q, iters, sink);
        cudaEventRecord(e);
        cudaEventSynchronize(e);
        cudaEventElapsedTime(&ms, s, e);
        printf("mixed (4 int + 4 fp64 chains): %8.1f G butterflies/s\n", bf / (ms * 1e6));
    }
    printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
