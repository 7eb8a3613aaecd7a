// DMMA.8x8x4 dependent-chain latency and per-warp issue rate on one SM:
// one warp runs `chains` independent accumulator chains of `len` MMAs each.
#include <cstdio>
#include <cuda_runtime.h>

template <int CH>
__global__ void chain_kernel(double* out, long long* cycles, int len, double a, double b) {
    double acc[CH][2];
#pragma unroll
    for (int c = 0; c < CH; ++c) acc[c][0] = acc[c][1] = threadIdx.x * 1e-3 + c;
    __syncwarp();
    const long long t0 = clock64();
    for (int i = 0; i < len; ++i) {
#pragma unroll
        for (int c = 0; c < CH; ++c)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(acc[c][0]), "+d"(acc[c][1])
                         : "d"(a), "d"(b));
    }
    const long long t1 = clock64();
    double s = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) s += acc[c][0] + acc[c][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

template <int CH>
void run(int warps) {
    double* out;
    long long* cyc;
    cudaMalloc(&out, sizeof(double) * 32 * warps);
    cudaMalloc(&cyc, sizeof(long long));
    const int len = 4096;
    chain_kernel<CH><<<1, 32 * warps>>>(out, cyc, len, 1.0000001, 0.9999999);
    chain_kernel<CH><<<1, 32 * warps>>>(out, cyc, len, 1.0000001, 0.9999999);
    long long c;
    cudaMemcpy(&c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
    printf("warps/SM %2d chains/warp %2d: %6.1f cycles per MMA per chain, %5.2f cycles per MMA (SM)\n", warps, CH,
           double(c) / len, double(c) / (double(len) * CH * warps));
    cudaFree(out);
    cudaFree(cyc);
}

int main() {
    for (int w : {1, 4, 8, 16}) {
        run<1>(w);
        run<2>(w);
        run<4>(w);
        run<8>(w);
        run<16>(w);
    }
    return 0;
}
