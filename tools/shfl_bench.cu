// Throughput of warp-uniform LDS.128 broadcasts vs SHFL.IDX on one B200 (which unit limits a
// table broadcast in the lookup): nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/sb tools/shfl_bench.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void lds_bcast(int iters, float* out) {
    __shared__ uint4 buf[256];
    for (int i = threadIdx.x; i < 256; i += blockDim.x) buf[i] = make_uint4(i, i + 1, i + 2, i + 3);
    __syncthreads();
    unsigned acc = 0;
    int j = 0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            uint4 v = buf[(j + u) & 255];  // uniform address
            acc += v.x ^ v.y ^ v.z ^ v.w;
        }
        j += 8;
    }
    if (acc == 0x12345) out[0] = acc;
}
__global__ void shfl_idx(int iters, float* out) {
    unsigned v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = threadIdx.x * 2654435761u + u;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = __shfl_sync(0xffffffffu, v[u], (it + u) & 31) + 1u;
    }
    unsigned acc = 0;
#pragma unroll
    for (int u = 0; u < 8; ++u) acc ^= v[u];
    if (acc == 0x12345) out[0] = acc;
}
__global__ void lds_gather(int iters, float* out) {
    __shared__ float buf[8192];
    for (int i = threadIdx.x; i < 8192; i += blockDim.x) buf[i] = i;
    __syncthreads();
    float acc = 0;
    int j = threadIdx.x & 31;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 8; ++u) acc += buf[((it * 8 + u) * 32 + j) & 8191];
    }
    if (acc == 0.5f) out[0] = acc;
}
__global__ void mixed(int iters, float* out) {
    __shared__ float buf[8192];
    for (int i = threadIdx.x; i < 8192; i += blockDim.x) buf[i] = i;
    __syncthreads();
    float acc = 0;
    unsigned v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = threadIdx.x * 2654435761u + u;
    int j = threadIdx.x & 31;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            acc += buf[((it * 8 + u) * 32 + j) & 8191];
            v[u] = __shfl_sync(0xffffffffu, v[u], (it + u) & 31) + 1u;
        }
    }
    unsigned x = 0;
#pragma unroll
    for (int u = 0; u < 8; ++u) x ^= v[u];
    if (acc == 0.5f || x == 0x1234u) out[0] = acc;
}
__global__ void lds64_row(int iters, float* out) {
    // one LDS.64 per "row" with 8 active lanes (k = 8 entries of 8 B), the lookup's proposed table read
    __shared__ uint2 buf[4096];
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) buf[i] = make_uint2(i, i + 1);
    __syncthreads();
    unsigned acc = 0;
    const int lane = threadIdx.x & 31;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            if (lane < 8) { uint2 e = buf[((it * 8 + u) * 8 + lane) & 4095]; acc += e.x ^ e.y; }
        }
    }
    if (acc == 0x12345) out[0] = acc;
}
int main() {
    float* d; cudaMalloc(&d, 4);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const int iters = 20000, threads = 512, blocks = sms * 2;
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int k = 0; k < 5; ++k) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(a);
            if (k == 0) lds_bcast<<<blocks, threads>>>(iters, d);
            if (k == 1) shfl_idx<<<blocks, threads>>>(iters, d);
            if (k == 2) lds_gather<<<blocks, threads>>>(iters, d);
            if (k == 3) mixed<<<blocks, threads>>>(iters, d);
            if (k == 4) lds64_row<<<blocks, threads>>>(iters, d);
            cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            double warp_instr = (double)blocks * threads / 32 * iters * 8;
            double per_sm_clk = warp_instr / sms / (ms * 1e-3 * clk * 1e3);
            if (rep) printf("%s: %.3f ms, %.3f warp-instr/clk/SM (at %d MHz nominal)\n",
                            k == 0 ? "LDS.128 uniform" : k == 1 ? "SHFL.IDX" : k == 2 ? "LDS.32 gather" : k == 3 ? "gather+SHFL pairs" : "LDS.64 8 lanes", ms, per_sm_clk, clk / 1000);
        }
    }
    return 0;
}
