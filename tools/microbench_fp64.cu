// FP64 pipe microbenchmark for B200 (sm_100a): DFMA vs DMMA (mma.sync f64)
// throughput and streaming HBM read bandwidth. Standalone; informs the
// kernel choices in DESIGN.md. Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

template <int CH>
__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double acc[CH];
#pragma unroll
  for (int i = 0; i < CH; ++i) acc[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) acc[i] = fma(acc[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += acc[i];
  if (s == 12345.678) out[threadIdx.x] = s;
}

template <int CH>
__global__ void dmma884_kernel(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[CH][2];
#pragma unroll
  for (int i = 0; i < CH; ++i) { c[i][0] = i; c[i][1] = -i; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[threadIdx.x] = s;
}

template <int CH>
__global__ void dmma16816_kernel(double* out, int iters) {
  double a[8], b[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = 1.0 - threadIdx.x * 1e-4 + i;
  double c[CH][4];
#pragma unroll
  for (int i = 0; i < CH; ++i) { c[i][0] = i; c[i][1] = -i; c[i][2] = 0; c[i][3] = 1; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 12345.678) out[threadIdx.x] = s;
}

// DMMA and DFMA interleaved in one warp: do they share the FP64 pipe?
// NF DFMAs per thread ride along each group of 4 DMMAs (NF=0: DMMA only).
template <int NF>
__global__ void mixed_kernel(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[4][2];
  double f[NF > 0 ? NF : 1];
#pragma unroll
  for (int i = 0; i < 4; ++i) { c[i][0] = i; c[i][1] = -i; }
#pragma unroll
  for (int i = 0; i < (NF > 0 ? NF : 1); ++i) f[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
#pragma unroll
      for (int j = i; j < NF; j += 4) asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(f[j]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) s += c[i][0] + c[i][1];
#pragma unroll
  for (int i = 0; i < NF; ++i) s += f[i];
  if (s == 12345.678) out[threadIdx.x] = s;
}

template <int NF>
void run_mixed(int sms, double* out, int iters, cudaEvent_t e0, cudaEvent_t e1) {
  for (int threads : {256, 512}) {
    const int blocks = sms * 2;
    float ms;
    mixed_kernel<NF><<<blocks, threads>>>(out, 100);
    cudaEventRecord(e0);
    mixed_kernel<NF><<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    const double dmma_fl = 2.0 * 256 * 4 * (double)iters * blocks * (threads / 32);
    const double dfma_fl = 2.0 * NF * (double)iters * blocks * threads;
    printf("MIXED dfma/thread per 4 dmma=%d thr=%d : %.3f ms  dmma %.2f TF + dfma %.2f TF = %.2f TF\n", NF, threads,
           ms, dmma_fl / ms / 1e9, dfma_fl / ms / 1e9, (dmma_fl + dfma_fl) / ms / 1e9);
  }
}

__global__ void read_kernel(const double2* __restrict__ p, size_t n2, double* out) {
  double s0 = 0, s1 = 0;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n2; i += stride * 4) {
    double2 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      size_t j = i + u * stride;
      if (j < n2) {
        asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];" : "=d"(v[u].x), "=d"(v[u].y) : "l"(p + j));
      } else { v[u].x = v[u].y = 0; }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) { s0 += v[u].x * v[u].x; s1 += v[u].y * v[u].y; }
  }
  if (s0 + s1 == 12345.678) out[0] = s0;
}

int main() {
  int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  int clk; CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0));
  printf("SMs %d clock %d kHz\n", sms, clk);
  double* out; CK(cudaMalloc(&out, 1 << 20));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  const int iters = 20000;
  for (int bpsm : {1, 2, 4}) {
    for (int threads : {128, 256, 512}) {
      int blocks = sms * bpsm;
      dfma_kernel<8><<<blocks, threads>>>(out, 100, 1.0000001, 1e-9);
      cudaEventRecord(e0);
      dfma_kernel<8><<<blocks, threads>>>(out, iters, 1.0000001, 1e-9);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
      double fl = 2.0 * 8 * iters * (double)blocks * threads;
      printf("DFMA  ch=8  blocks=%d thr=%d : %.2f TFLOP/s\n", blocks, threads, fl / ms / 1e9);
    }
  }
  for (int bpsm : {1, 2, 4}) {
    for (int threads : {128, 256, 512}) {
      int blocks = sms * bpsm;
      dmma884_kernel<4><<<blocks, threads>>>(out, 100);
      cudaEventRecord(e0);
      dmma884_kernel<4><<<blocks, threads>>>(out, iters);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
      double fl = 2.0 * 8 * 8 * 4 * 4 * (double)iters * blocks * (threads / 32);
      printf("DMMA884 ch=4 blocks=%d thr=%d : %.2f TFLOP/s\n", blocks, threads, fl / ms / 1e9);
    }
  }
  for (int bpsm : {1, 2}) {
    for (int threads : {128, 256}) {
      int blocks = sms * bpsm;
      dmma16816_kernel<2><<<blocks, threads>>>(out, 100);
      cudaEventRecord(e0);
      dmma16816_kernel<2><<<blocks, threads>>>(out, iters / 4);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
      double fl = 2.0 * 16 * 8 * 16 * 2 * (double)(iters / 4) * blocks * (threads / 32);
      printf("DMMA16816 ch=2 blocks=%d thr=%d : %.2f TFLOP/s\n", blocks, threads, fl / ms / 1e9);
    }
  }
  run_mixed<0>(sms, out, iters, e0, e1);
  run_mixed<4>(sms, out, iters, e0, e1);
  run_mixed<8>(sms, out, iters, e0, e1);
  run_mixed<16>(sms, out, iters, e0, e1);
  run_mixed<32>(sms, out, iters, e0, e1);
  size_t bytes = (size_t)4 << 30;
  double2* buf; CK(cudaMalloc(&buf, bytes));
  CK(cudaMemset(buf, 0, bytes));
  for (int bpsm : {2, 4, 8}) {
    int blocks = sms * bpsm;
    read_kernel<<<blocks, 256>>>(buf, bytes / 16, out);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) read_kernel<<<blocks, 256>>>(buf, bytes / 16, out);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    printf("READ blocks=%d : %.1f GB/s\n", blocks, 5.0 * bytes / ms / 1e6);
  }
  CK(cudaGetLastError());
  return 0;
}
