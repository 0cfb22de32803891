// Latency / throughput probe of the FP64 and conversion ops on the sweep's
// dependency chain (DADD, DMUL, FRND.FLOOR, F2F pair, SHFL).  Informs the
// sweep kernels' design; not part of the product.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -o /tmp/fp64_micro tools/fp64_micro.cu
#include <cstdio>

constexpr int kIters = 4096;

template <int OP>
__device__ __forceinline__ double step(double x, double y) {
  if (OP == 0) return __dadd_rn(x, y);
  if (OP == 1) return __dmul_rn(x, y);
  if (OP == 2) return floor(x) + 0.0 * y;  // FRND (+ folded)
  if (OP == 3) return (double)__double2float_rn(x);
  if (OP == 4) {
    double r;
    unsigned lo = __double2loint(x), hi = __double2hiint(x);
    lo = __shfl_xor_sync(0xffffffffu, lo, 1);
    hi = __shfl_xor_sync(0xffffffffu, hi, 1);
    r = __hiloint2double(hi, lo);
    return r;
  }
  if (OP == 5) return __int_as_float(__float_as_int((float)x) + 1) ;  // dummy
  return x;
}

template <int OP, int ILP>
__global__ void probe(double* out, long long* cyc, double y) {
  double x[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) x[i] = 1.0 + threadIdx.x * 1e-9 + i;
  __syncwarp();
  const long long t0 = clock64();
#pragma unroll 16
  for (int k = 0; k < kIters; ++k)
#pragma unroll
    for (int i = 0; i < ILP; ++i) x[i] = step<OP>(x[i], y);
  const long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int OP, int ILP>
void run(const char* name, int warps_per_block, int blocks) {
  double* out;
  long long* cyc;
  cudaMalloc(&out, sizeof(double) * blocks * warps_per_block * 32);
  cudaMalloc(&cyc, sizeof(long long) * blocks);
  probe<OP, ILP><<<blocks, warps_per_block * 32>>>(out, cyc, 1e-300);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  probe<OP, ILP><<<blocks, warps_per_block * 32>>>(out, cyc, 1e-300);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  long long c;
  cudaMemcpy(&c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
  const double ops = (double)kIters * ILP * blocks * warps_per_block;  // warp instrs
  printf("%-10s ilp=%d warps/blk=%2d blocks=%4d  cycles/iter/chain=%.2f  warp-ops/ns=%.1f  "
         "per-SM warp-ops/clk(@1.965GHz)=%.3f\n",
         name, ILP, warps_per_block, blocks, (double)c / kIters, ops / (ms * 1e6),
         ops / (ms * 1e-3) / 148 / 1.965e9);
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  // latency: one warp, one chain
  run<0, 1>("DADD", 1, 1);
  run<1, 1>("DMUL", 1, 1);
  run<2, 1>("FLOOR+", 1, 1);
  run<3, 1>("F2F pair", 1, 1);
  run<4, 1>("SHFLx2", 1, 1);
  // throughput: many warps, 4 chains each
  run<0, 4>("DADD", 16, 148 * 4);
  run<1, 4>("DMUL", 16, 148 * 4);
  run<3, 4>("F2F pair", 16, 148 * 4);
  run<4, 4>("SHFLx2", 16, 148 * 4);
  // latency hiding: warps per SMSP with 2 chains
  for (int w = 1; w <= 16; w *= 2) run<0, 2>("DADD", w * 4, 148);
  return 0;
}
