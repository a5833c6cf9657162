// Throughput microbenchmarks for design decisions (FP64 vs FP32 SIMT, F2F, SHFL).
#include <cstdio>
#include <cuda_runtime.h>
template <int OP>
__global__ void k(double* out, float* outf, int iters, double a, float af) {
  double x0 = threadIdx.x * 1e-3, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  float f0 = threadIdx.x * 1e-3f, f1 = f0 + 1, f2 = f0 + 2, f3 = f0 + 3, f4 = f0 + 4, f5 = f0 + 5, f6 = f0 + 6, f7 = f0 + 7;
  for (int i = 0; i < iters; ++i) {
    if (OP == 0) {  // DADD
      x0 = __dadd_rn(x0, a); x1 = __dadd_rn(x1, a); x2 = __dadd_rn(x2, a); x3 = __dadd_rn(x3, a);
      x4 = __dadd_rn(x4, a); x5 = __dadd_rn(x5, a); x6 = __dadd_rn(x6, a); x7 = __dadd_rn(x7, a);
    } else if (OP == 1) {  // FADD
      f0 = __fadd_rn(f0, af); f1 = __fadd_rn(f1, af); f2 = __fadd_rn(f2, af); f3 = __fadd_rn(f3, af);
      f4 = __fadd_rn(f4, af); f5 = __fadd_rn(f5, af); f6 = __fadd_rn(f6, af); f7 = __fadd_rn(f7, af);
    } else if (OP == 2) {  // DFMA
      x0 = fma(x0, a, a); x1 = fma(x1, a, a); x2 = fma(x2, a, a); x3 = fma(x3, a, a);
      x4 = fma(x4, a, a); x5 = fma(x5, a, a); x6 = fma(x6, a, a); x7 = fma(x7, a, a);
    } else if (OP == 3) {  // DSETP-ish compare+select
      x0 = x0 < a ? x0 + 1.0 : x0; x1 = x1 < a ? x1 + 1.0 : x1; x2 = x2 < a ? x2 + 1.0 : x2; x3 = x3 < a ? x3 + 1.0 : x3;
      x4 = x4 < a ? x4 + 1.0 : x4; x5 = x5 < a ? x5 + 1.0 : x5; x6 = x6 < a ? x6 + 1.0 : x6; x7 = x7 < a ? x7 + 1.0 : x7;
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
  outf[blockIdx.x * blockDim.x + threadIdx.x] = f0 + f1 + f2 + f3 + f4 + f5 + f6 + f7;
}
template <int OP>
void run(const char* name, int sms) {
  double* o; float* of;
  int blocks = sms * 4, threads = 512, iters = 20000;
  cudaMalloc(&o, blocks * threads * 8); cudaMalloc(&of, blocks * threads * 4);
  k<OP><<<blocks, threads>>>(o, of, 100, 1.0000001, 1.0000001f);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  k<OP><<<blocks, threads>>>(o, of, iters, 1.0000001, 1.0000001f);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  double ops = double(blocks) * threads * iters * 8;
  printf("%-6s %.3f Tops/s  (%.1f ops/clk/SM at 1.965GHz)\n", name, ops / ms / 1e9, ops / (ms * 1e-3) / sms / 1.965e9);
  cudaFree(o); cudaFree(of);
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  printf("device %s SMs %d smemPerBlockOptin %zu L2 %d regsPerSM %d\n", p.name, sms, p.sharedMemPerBlockOptin, p.l2CacheSize, p.regsPerMultiprocessor);
  run<0>("DADD", sms); run<1>("FADD", sms); run<2>("DFMA", sms); run<3>("DCMPSEL", sms);
  return 0;
}
