// peaks_fp64_alu.cu -- measured B200 compute ceilings for the encoder's
// non-tensor pipes: fp64 DADD / DMUL / DFMA and the
// integer ALU (LOP3, funnel shifts), as warp instructions per second over the
// whole GPU, plus the one-warp-instruction-per-cycle-per-SMSP issue ceiling.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -o peaks tools/peaks_fp64_alu.cu
//   ./peaks > profiles/peaks_fp64_alu.json
//
// Every kernel runs 8 independent dependency chains per thread at full
// occupancy (148 SMs x 8 CTAs x 256 threads), so each pipe is throughput-bound;
// cuobjdump -sass shows one DADD / DMUL / DFMA / LOP3 / SHF per asm statement
// (the loops unroll by 15 with a remainder, so every thread executes exactly
// iters x 16 x 8 of them).
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#define CK(x)                                                                       \
  do {                                                                              \
    cudaError_t e = (x);                                                            \
    if (e != cudaSuccess) {                                                         \
      fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e));                       \
      exit(1);                                                                      \
    }                                                                               \
  } while (0)

constexpr int kChains = 8;
constexpr int kUnroll = 16;

__global__ void k_dadd(double* out, int iters, double s) {
  double a[kChains];
  for (int c = 0; c < kChains; c++) a[c] = threadIdx.x * 1e-3 + c;
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int u = 0; u < kUnroll; u++)
#pragma unroll
      for (int c = 0; c < kChains; c++) asm volatile("add.rn.f64 %0, %0, %1;" : "+d"(a[c]) : "d"(s));
  }
  double t = 0;
  for (int c = 0; c < kChains; c++) t += a[c];
  if (t == 1234.5) out[0] = t;
}

__global__ void k_dmul(double* out, int iters, double s) {
  double a[kChains];
  for (int c = 0; c < kChains; c++) a[c] = threadIdx.x * 1e-3 + c;
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int u = 0; u < kUnroll; u++)
#pragma unroll
      for (int c = 0; c < kChains; c++) asm volatile("mul.rn.f64 %0, %0, %1;" : "+d"(a[c]) : "d"(s));
  }
  double t = 0;
  for (int c = 0; c < kChains; c++) t += a[c];
  if (t == 1234.5) out[0] = t;
}

__global__ void k_dfma(double* out, int iters, double s) {
  double a[kChains];
  for (int c = 0; c < kChains; c++) a[c] = threadIdx.x * 1e-3 + c;
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int u = 0; u < kUnroll; u++)
#pragma unroll
      for (int c = 0; c < kChains; c++) asm volatile("fma.rn.f64 %0, %0, %1, %1;" : "+d"(a[c]) : "d"(s));
  }
  double t = 0;
  for (int c = 0; c < kChains; c++) t += a[c];
  if (t == 1234.5) out[0] = t;
}

__global__ void k_lop3(unsigned* out, int iters, unsigned s) {
  unsigned a[kChains];
  for (int c = 0; c < kChains; c++) a[c] = threadIdx.x * 7u + c;
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int u = 0; u < kUnroll; u++)
#pragma unroll
      for (int c = 0; c < kChains; c++)
        asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(a[c]) : "r"(s), "r"(s + c));
  }
  unsigned t = 0;
  for (int c = 0; c < kChains; c++) t ^= a[c];
  if (t == 0x12345u) out[0] = t;
}

__global__ void k_shf(unsigned* out, int iters, unsigned s) {
  unsigned a[kChains];
  for (int c = 0; c < kChains; c++) a[c] = threadIdx.x * 7u + c;
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int u = 0; u < kUnroll; u++)
#pragma unroll
      for (int c = 0; c < kChains; c++)
        asm volatile("shf.l.wrap.b32 %0, %0, %1, %2;" : "+r"(a[c]) : "r"(s), "r"(c + 1));
  }
  unsigned t = 0;
  for (int c = 0; c < kChains; c++) t ^= a[c];
  if (t == 0x12345u) out[0] = t;
}

// issue ceiling: independent fp32 FFMA (fma pipe) and LOP3 (alu pipe)
// interleaved, so neither pipe is the limit and the dispatch of one warp
// instruction per cycle per SMSP is
__global__ void k_issue(float* out, int iters, float s, unsigned si) {
  float f[kChains];
  unsigned a[kChains];
  for (int c = 0; c < kChains; c++) {
    f[c] = threadIdx.x * 1e-3f + c;
    a[c] = threadIdx.x * 7u + c;
  }
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int u = 0; u < kUnroll; u++)
#pragma unroll
      for (int c = 0; c < kChains; c++) {
        asm volatile("fma.rn.f32 %0, %0, %1, %1;" : "+f"(f[c]) : "f"(s));
        asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(a[c]) : "r"(si), "r"(si + c));
      }
  }
  float t = 0;
  unsigned x = 0;
  for (int c = 0; c < kChains; c++) {
    t += f[c];
    x ^= a[c];
  }
  if (t == 1234.5f && x == 7u) out[0] = t;
}

template <class F>
double time_kernel(F launch, int reps) {
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  launch();  // warm-up
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < reps; r++) {
    CK(cudaEventRecord(e0));
    launch();
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    if (ms < best) best = ms;
  }
  return best / 1e3;
}

int main() {
  cudaDeviceProp p;
  CK(cudaGetDeviceProperties(&p, 0));
  const int sms = p.multiProcessorCount;
  const int blocks = sms * 8, threads = 256, iters = 2000;
  void* buf;
  CK(cudaMalloc(&buf, 64));
  const double warps = (double)blocks * threads / 32;
  const double per_warp = (double)iters * kUnroll * kChains;  // instructions of the measured kind
  struct R {
    const char* name;
    const char* pipe;
    double per_warp_mult;
    double secs;
  } rs[6];
  rs[0] = {"dadd", "fp64", 1, time_kernel([&] { k_dadd<<<blocks, threads>>>((double*)buf, iters, 1e-9); }, 5)};
  rs[1] = {"dmul", "fp64", 1, time_kernel([&] { k_dmul<<<blocks, threads>>>((double*)buf, iters, 1.0000001); }, 5)};
  rs[2] = {"dfma", "fp64", 1, time_kernel([&] { k_dfma<<<blocks, threads>>>((double*)buf, iters, 0.9999999); }, 5)};
  rs[3] = {"lop3", "alu", 1, time_kernel([&] { k_lop3<<<blocks, threads>>>((unsigned*)buf, iters, 0x9e3779b9u); }, 5)};
  rs[4] = {"shf", "alu", 1, time_kernel([&] { k_shf<<<blocks, threads>>>((unsigned*)buf, iters, 0x9e3779b9u); }, 5)};
  rs[5] = {"issue_ffma_lop3", "issue", 2,
           time_kernel([&] { k_issue<<<blocks, threads>>>((float*)buf, iters, 0.999f, 0x9e3779b9u); }, 5)};
  int clk_khz = 0;
  CK(cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0));
  printf("{\n \"gpu\": \"%s\", \"sms\": %d, \"clock_attr_mhz\": %.0f,\n", p.name, sms, clk_khz / 1e3);
  printf(" \"how\": \"tools/peaks_fp64_alu.cu: %d CTAs x %d threads, 8 independent chains per thread, %d x %d x 8 "
         "instructions per thread, best of 5 (CUDA events)\",\n",
         blocks, threads, iters, kUnroll);
  printf(" \"rates\": {\n");
  for (int k = 0; k < 6; k++) {
    const double inst = warps * per_warp * rs[k].per_warp_mult;
    const double wips = inst / rs[k].secs;  // warp instructions per second, whole GPU
    printf("  \"%s\": {\"pipe\": \"%s\", \"warp_inst_per_s\": %.6e, \"thread_ops_per_s\": %.6e, "
           "\"warp_inst_per_sm_per_clk_at_1965\": %.4f, \"ms\": %.4f}%s\n",
           rs[k].name, rs[k].pipe, wips, wips * 32, wips / sms / 1.965e9, rs[k].secs * 1e3, k < 5 ? "," : "");
  }
  printf(" }\n}\n");
  return 0;
}
