// hist.cu -- quantization-code histogram (ebzip/codec.py:107, np.bincount).
//
// One pass over the code array (1 byte per point for m <= 8), kept out of the
// wavefront sweep so the sweep's critical path stays short.  Each thread
// reads 16 consecutive codes with one 16-byte load and run-length-merges
// them (smooth fields produce long runs of the centre code), then adds the
// runs to a warp-private shared histogram (m <= 10) or a block histogram
// (m <= 13) or, beyond that, straight to global u64 counters.
#include "ebz_common.cuh"

namespace {

constexpr int kThreads = 256;

template <typename C>
__device__ __forceinline__ void load16(const C* codes, long long i0, long long n, int* out) {
  if (i0 + 16 <= n && (((uintptr_t)(codes + i0)) & 15) == 0) {
    if (sizeof(C) == 1) {
      const uint4 v = __ldcs(reinterpret_cast<const uint4*>(codes + i0));
      const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int j = 0; j < 16; ++j) out[j] = (w[j >> 2] >> (8 * (j & 3))) & 0xff;
    } else {
      const uint4 v0 = __ldcs(reinterpret_cast<const uint4*>(codes + i0));
      const uint4 v1 = __ldcs(reinterpret_cast<const uint4*>(codes + i0) + 1);
      const uint32_t w[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
#pragma unroll
      for (int j = 0; j < 16; ++j) out[j] = (w[j >> 1] >> (16 * (j & 1))) & 0xffff;
    }
  } else {
#pragma unroll
    for (int j = 0; j < 16; ++j) out[j] = (i0 + j < n) ? (int)codes[i0 + j] : -1;
  }
}

template <typename C>
__global__ void __launch_bounds__(kThreads)
code_hist_kernel(const C* __restrict__ codes, long long n, int m,
                 unsigned long long* __restrict__ hist) {
  extern __shared__ unsigned int sh[];
  const int nsym = 1 << m;
  const int mode = m <= 10 ? 0 : (m <= 13 ? 1 : 2);  // per-warp / per-block / global
  const int copies = mode == 0 ? kThreads / 32 : 1;
  unsigned int* h = sh + (mode == 0 ? (threadIdx.x >> 5) * nsym : 0);
  if (mode < 2) {
    for (int i = threadIdx.x; i < copies * nsym; i += kThreads) sh[i] = 0;
    __syncthreads();
  }
  const long long groups = (n + 15) / 16;
  for (long long g = (long long)blockIdx.x * kThreads + threadIdx.x; g < groups;
       g += (long long)gridDim.x * kThreads) {
    int c[16];
    load16<C>(codes, g * 16, n, c);
    // codes outside the alphabet (a skipped field's scratch) stay in range
#pragma unroll
    for (int j = 0; j < 16; ++j) c[j] &= (c[j] >> 31) | ((1 << m) - 1);
    int cur = c[0];
    unsigned int run = 1;
#pragma unroll
    for (int j = 1; j < 16; ++j) {
      if (c[j] == cur) {
        ++run;
      } else {
        if (cur >= 0) {
          if (mode < 2) atomicAdd(&h[cur], run);
          else atomicAdd(&hist[cur], (unsigned long long)run);
        }
        cur = c[j];
        run = 1;
      }
    }
    if (cur >= 0) {
      if (mode < 2) atomicAdd(&h[cur], run);
      else atomicAdd(&hist[cur], (unsigned long long)run);
    }
  }
  if (mode == 2) return;
  __syncthreads();
  for (int i = threadIdx.x; i < nsym; i += kThreads) {
    unsigned long long s = 0;
    for (int w = 0; w < copies; ++w) s += sh[w * nsym + i];
    if (s) atomicAdd(&hist[i], s);
  }
}

}  // namespace

cudaError_t launch_code_hist(const void* codes, int m, long long n, unsigned long long* hist,
                             int sms, cudaStream_t s) {
  const long long groups = (n + 15) / 16;
  long long blocks = (groups + kThreads - 1) / kThreads;
  const long long cap = (long long)sms * 4;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  const size_t smem = m <= 10 ? (size_t)(kThreads / 32) * 4 << m : (m <= 13 ? (size_t)4 << m : 0);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(code_hist_kernel<uint8_t>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         64 * 1024);
    cudaFuncSetAttribute(code_hist_kernel<uint16_t>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         64 * 1024);
    attr = true;
  }
  if (m > 8)
    code_hist_kernel<uint16_t><<<(unsigned)blocks, kThreads, smem, s>>>((const uint16_t*)codes, n,
                                                                        m, hist);
  else
    code_hist_kernel<uint8_t><<<(unsigned)blocks, kThreads, smem, s>>>((const uint8_t*)codes, n, m,
                                                                       hist);
  return cudaGetLastError();
}
