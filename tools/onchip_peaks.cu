// Measured on-chip peaks of this B200 for the roofline denominators bench.py reports next to the
// derived ones (MEASURED_PEAKS.json holds only HBM and dense bf16):
//   * shared-memory load bandwidth: conflict-free LDS.32 / LDS.64 / LDS.128, bytes per clock per SM
//   * FP32 FFMA and FADD issue rate (lanes per clock per SM) -- the kNN sweep's pipe
//   * FP64 DFMA / DADD rate (lanes per clock per SM) -- the exact-key recomputation
// Every kernel runs 4 resident CTAs of 256 threads on every SM with long unrolled dependent-free
// streams; clocks are read with clock64() inside the kernel (SM clocks, not wall time), so the
// figures are per SM clock and scaled by the measured SM clock for GB/s.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/onchip tools/onchip_peaks.cu && /tmp/onchip
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e_)); return 1; } } while (0)

template <int VEC>
__global__ void lds_kernel(int iters, float* out, unsigned long long* clk) {
    __shared__ __align__(16) float buf[8192];  // 32 KB
    for (int i = threadIdx.x; i < 8192; i += blockDim.x) buf[i] = (float)i;
    __syncthreads();
    const unsigned long long c0 = clock64();
    float acc[VEC] = {};
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int base = w * 512;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            // lane-contiguous VEC-float accesses: conflict-free, 128 * VEC bytes per warp instruction
            const int off = ((base + u * 32 * VEC) & (8192 - 1) & ~(32 * VEC - 1)) + lane * VEC;
            if (VEC == 1) acc[0] += buf[off];
            if (VEC == 2) { const float2 v = *reinterpret_cast<const float2*>(buf + off); acc[0] += v.x; acc[1] += v.y; }
            if (VEC == 4) {
                const float4 v = *reinterpret_cast<const float4*>(buf + off);
                acc[0] += v.x; acc[1] += v.y; acc[2] += v.z; acc[3] += v.w;
            }
        }
        base += 8 * 32 * VEC;
    }
    __syncthreads();
    const unsigned long long c1 = clock64();
    float s = 0.f;
#pragma unroll
    for (int v = 0; v < VEC; ++v) s += acc[v];
    if (s == 0.123f) out[0] = s;
    if (threadIdx.x == 0) atomicMax(clk, c1 - c0);
}

template <typename T, bool FMA>
__global__ void alu_kernel(int iters, float* out, unsigned long long* clk) {
    T a[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) a[u] = (T)(threadIdx.x + u) * (T)1e-3;
    const T m = (T)0.999, c = (T)1e-7;
    __syncthreads();
    const unsigned long long c0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 16; ++u) a[u] = FMA ? a[u] * m + c : a[u] + c;
    }
    __syncthreads();
    const unsigned long long c1 = clock64();
    T s = 0;
#pragma unroll
    for (int u = 0; u < 16; ++u) s += a[u];
    if (s == (T)0.123) out[0] = (float)s;
    if (threadIdx.x == 0) atomicMax(clk, c1 - c0);
}

int main() {
    int sms = 0, clk_khz = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    CK(cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0));
    float* out;
    unsigned long long* clk;
    CK(cudaMalloc(&out, 4));
    CK(cudaMalloc(&clk, 8));
    const int ctas = sms * 4, threads = 256;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto run = [&](const char* name, void (*k)(int, float*, unsigned long long*), int iters, double per_thread_iter,
                   const char* unit) {
        k<<<ctas, threads>>>(iters / 10, out, clk);  // warm-up
        cudaMemset(clk, 0, 8);
        cudaEventRecord(e0);
        k<<<ctas, threads>>>(iters, out, clk);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        unsigned long long cyc = 0;
        cudaMemcpy(&cyc, clk, 8, cudaMemcpyDeviceToHost);
        const double total = per_thread_iter * iters * (double)threads * ctas;   // bytes or lane-ops
        const double per_clk_sm = total / sms / (double)cyc;                     // per SM clock (in-kernel)
        const double mhz = cyc / (ms * 1e3);                                     // effective SM clock
        printf("%-14s %10.3f ms  %8.1f %s/clk/SM  (SM clock %.0f MHz from clock64)  -> %.1f %s/s whole GPU\n", name, ms,
               per_clk_sm, unit, mhz, per_clk_sm * sms * mhz * 1e6 / 1e9, unit[0] == 'B' ? "GB" : "G-lane-op");
        return per_clk_sm;
    };
    printf("# B200 on-chip peaks (tools/onchip_peaks.cu), %d SMs, nominal max clock %d MHz\n", sms, clk_khz / 1000);
    const double l32 = run("LDS.32", lds_kernel<1>, 200000, 8 * 4.0, "B");
    const double l64 = run("LDS.64", lds_kernel<2>, 200000, 8 * 8.0, "B");
    const double l128 = run("LDS.128", lds_kernel<4>, 200000, 8 * 16.0, "B");
    const double f32f = run("FP32 FFMA", alu_kernel<float, true>, 200000, 16, "lane");
    const double f32a = run("FP32 FADD", alu_kernel<float, false>, 200000, 16, "lane");
    const double f64f = run("FP64 DFMA", alu_kernel<double, true>, 50000, 16, "lane");
    const double f64a = run("FP64 DADD", alu_kernel<double, false>, 50000, 16, "lane");
    const double smem = l32 > l64 ? (l32 > l128 ? l32 : l128) : (l64 > l128 ? l64 : l128);
    printf("{\"smem_bytes_per_clk_sm\": %.2f, \"lds32\": %.2f, \"lds64\": %.2f, \"lds128\": %.2f, "
           "\"fp32_ffma_lanes_per_clk_sm\": %.2f, \"fp32_fadd_lanes_per_clk_sm\": %.2f, "
           "\"fp64_dfma_lanes_per_clk_sm\": %.2f, \"fp64_dadd_lanes_per_clk_sm\": %.2f, \"sms\": %d}\n",
           smem, l32, l64, l128, f32f, f32a, f64f, f64a, sms);
    return 0;
}
