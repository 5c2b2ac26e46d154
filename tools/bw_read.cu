// Read-only HBM bandwidth probe (what a streaming reduction like k_tensor_sum can reach):
// grid-stride 16-byte loads summed into a register, one store per thread.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bw_read tools/bw_read.cu && tools/bw_read
#include <cstdio>
#include <cuda_runtime.h>

__global__ void rd(const ulonglong2 *__restrict__ p, size_t n, unsigned long long *out) {
    unsigned long long s = 0;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        ulonglong2 v = __ldcs(p + i);
        s += v.x ^ v.y;
    }
    if (s == 42) out[0] = s;
}

int main() {
    const size_t bytes = size_t(1) << 30, n = bytes / 16;
    ulonglong2 *p;
    unsigned long long *o;
    cudaMalloc(&p, bytes);
    cudaMalloc(&o, 8);
    cudaMemset(p, 1, bytes);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int bpsm : {4, 8, 16, 32}) {
        for (int t : {256, 512}) {
            rd<<<sms * bpsm, t>>>(p, n, o);
            cudaEventRecord(a);
            for (int r = 0; r < 10; r++) rd<<<sms * bpsm, t>>>(p, n, o);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            printf("blocks/SM %2d threads %3d: %.0f GB/s read-only\n", bpsm, t, 10.0 * bytes / (ms * 1e-3) / 1e9);
        }
    }
    return 0;
}
