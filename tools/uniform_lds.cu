// Cost of warp-uniform shared-memory loads by width (LDS.32/64/128 with one address for all 32
// lanes): do they take pipe time proportional to the bytes delivered (32 lanes x width)?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ul tools/uniform_lds.cu && /tmp/ul
#include <cstdio>
#include <cuda_runtime.h>
template <int W>
__global__ void uni(int iters, unsigned* out, unsigned long long* clk) {
    __shared__ __align__(16) unsigned buf[4096];
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) buf[i] = i * 2654435761u;
    __syncthreads();
    const unsigned long long c0 = clock64();
    unsigned acc = 0;
    int j = (threadIdx.x >> 5) * 64;  // uniform per warp
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int a = (j + u * 4) & 4092;
            if (W == 1) acc += buf[a];
            if (W == 2) { uint2 v = *reinterpret_cast<const uint2*>(buf + a); acc += v.x ^ v.y; }
            if (W == 4) { uint4 v = *reinterpret_cast<const uint4*>(buf + a); acc += v.x ^ v.y ^ v.z ^ v.w; }
        }
        j += 32;
    }
    __syncthreads();
    const unsigned long long c1 = clock64();
    if (acc == 0x12345) out[0] = acc;
    if (threadIdx.x == 0) atomicMax(clk, c1 - c0);
}
int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    unsigned* out; unsigned long long* clk; cudaMalloc(&out, 4); cudaMalloc(&clk, 8);
    const int ctas = sms * 4, threads = 512, iters = 100000;
    auto run = [&](const char* n, void (*k)(int, unsigned*, unsigned long long*)) {
        k<<<ctas, threads>>>(1000, out, clk);
        cudaMemset(clk, 0, 8);
        k<<<ctas, threads>>>(iters, out, clk);
        cudaDeviceSynchronize();
        unsigned long long c; cudaMemcpy(&c, clk, 8, cudaMemcpyDeviceToHost);
        const double instr = 8.0 * iters * (threads / 32) * 4;  // warp-instructions per SM (4 CTAs/SM)
        printf("%-18s %.3f warp-instr/clk/SM  (%.2f clk each)\n", n, instr / c, c / instr);
    };
    run("LDS.32 uniform", uni<1>);
    run("LDS.64 uniform", uni<2>);
    run("LDS.128 uniform", uni<4>);
    return 0;
}
