// Dependent-chain latency microbenchmark (single warp), cycles per op.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false tools/microbench.cu -o /tmp/mb
#include <cstdio>
#include <cuda_runtime.h>

#define CHAIN 256

__global__ void k_dadd(double* out, long long* cyc, double a) {
  double x = a + threadIdx.x;
  long long t0 = clock64();
#pragma unroll
  for (int i = 0; i < CHAIN; ++i) x = __dadd_rn(x, a);
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_dmul(double* out, long long* cyc, double a) {
  double x = a + threadIdx.x;
  long long t0 = clock64();
#pragma unroll
  for (int i = 0; i < CHAIN; ++i) x = __dmul_rn(x, a);
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_f2f(double* out, long long* cyc, double a) {
  double x = a + threadIdx.x;
  long long t0 = clock64();
#pragma unroll
  for (int i = 0; i < CHAIN; ++i) x = (double)__double2float_rn(x);
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;  // pair: f64->f32->f64
}
__global__ void k_floor(double* out, long long* cyc, double a) {
  double x = a + threadIdx.x;
  long long t0 = clock64();
#pragma unroll
  for (int i = 0; i < CHAIN; ++i) x = floor(x) + 0.5;
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;  // floor + dadd
}
__global__ void k_shfl(double* out, long long* cyc, double a) {
  double x = a + threadIdx.x;
  long long t0 = clock64();
#pragma unroll
  for (int i = 0; i < CHAIN; ++i) x = __shfl_up_sync(0xffffffffu, x, 1);
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;  // 64-bit shfl (2 SHFL)
}
__global__ void k_ffadd(float* out, long long* cyc, float a) {
  float x = a + threadIdx.x;
  long long t0 = clock64();
#pragma unroll
  for (int i = 0; i < CHAIN; ++i) x = __fadd_rn(x, a);
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_lds(double* out, long long* cyc, double a) {
  __shared__ int s[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) s[i] = (i + 1) & 1023;
  __syncthreads();
  int p = threadIdx.x;
  long long t0 = clock64();
#pragma unroll
  for (int i = 0; i < CHAIN; ++i) p = s[p];
  long long t1 = clock64();
  out[threadIdx.x] = p;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
// throughput: many independent DADDs from all warps of a full SM
__global__ void k_dadd_tput(double* out, long long* cyc, double a) {
  double x0 = a + threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
  double x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  __syncthreads();
  long long t0 = clock64();
#pragma unroll
  for (int i = 0; i < CHAIN; ++i) {
    x0 = __dadd_rn(x0, a); x1 = __dadd_rn(x1, a); x2 = __dadd_rn(x2, a); x3 = __dadd_rn(x3, a);
    x4 = __dadd_rn(x4, a); x5 = __dadd_rn(x5, a); x6 = __dadd_rn(x6, a); x7 = __dadd_rn(x7, a);
  }
  __syncthreads();
  long long t1 = clock64();
  out[threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_f2f_tput(double* out, long long* cyc, double a) {
  double x0 = a + threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
  __syncthreads();
  long long t0 = clock64();
#pragma unroll
  for (int i = 0; i < CHAIN; ++i) {
    x0 = (double)__double2float_rn(x0); x1 = (double)__double2float_rn(x1);
    x2 = (double)__double2float_rn(x2); x3 = (double)__double2float_rn(x3);
  }
  __syncthreads();
  long long t1 = clock64();
  out[threadIdx.x] = x0 + x1 + x2 + x3;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 1 << 20);
  cudaMalloc(&cyc, 64);
  long long h;
  auto run = [&](const char* name, void (*k)(double*, long long*, double), int threads, double per) {
    k<<<1, threads>>>(out, cyc, 1.0000001);
    k<<<1, threads>>>(out, cyc, 1.0000001);
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("%-12s threads=%4d  %.2f cycles/op\n", name, threads, (double)h / (CHAIN * per));
  };
  run("dadd", k_dadd, 32, 1);
  run("dmul", k_dmul, 32, 1);
  run("f2f pair", k_f2f, 32, 1);
  run("floor+dadd", k_floor, 32, 1);
  run("shfl64", k_shfl, 32, 1);
  run("lds chain", k_lds, 32, 1);
  {
    float* fo = (float*)out;
    k_ffadd<<<1, 32>>>(fo, cyc, 1.0001f);
    k_ffadd<<<1, 32>>>(fo, cyc, 1.0001f);
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("%-12s threads=%4d  %.2f cycles/op\n", "fadd", 32, (double)h / CHAIN);
  }
  // throughput: cycles per warp-instruction per SM = cycles / (CHAIN*8*warps)
  for (int t : {256, 1024}) {
    k_dadd_tput<<<1, t>>>(out, cyc, 1.0000001);
    k_dadd_tput<<<1, t>>>(out, cyc, 1.0000001);
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("dadd tput   threads=%4d  %.3f SM-cycles per warp-DADD\n", t,
           (double)h / (CHAIN * 8.0 * (t / 32)));
    k_f2f_tput<<<1, t>>>(out, cyc, 1.0000001);
    k_f2f_tput<<<1, t>>>(out, cyc, 1.0000001);
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("f2f2 tput   threads=%4d  %.3f SM-cycles per warp-(F2F pair)\n", t,
           (double)h / (CHAIN * 4.0 * (t / 32)));
  }
  return 0;
}
