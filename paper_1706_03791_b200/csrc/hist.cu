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

struct HistTab {  // per-field pointers of a batched launch (blockIdx.y = field)
  const void* codes[kBatchMax];
  unsigned long long* hist[kBatchMax];
};

template <typename C>
__global__ void __launch_bounds__(kThreads)
code_hist_kernel(const __grid_constant__ HistTab tab, long long n, int m) {
  const C* __restrict__ codes = reinterpret_cast<const C*>(tab.codes[blockIdx.y]);
  unsigned long long* __restrict__ hist = tab.hist[blockIdx.y];
  extern __shared__ unsigned int sh[];
  const int nsym = 1 << m;
  // u8 codes index 256 bins (stray bytes of a skipped field land above 2^m and
  // are dropped at the merge), u16 codes are masked to the alphabet
  const int nbin = sizeof(C) == 1 ? 256 : nsym;
  const int mask = sizeof(C) == 1 ? 0xff : nsym - 1;
  const int mode = m <= 10 ? 0 : (m <= 13 ? 1 : 2);  // per-warp / per-block / global
  const int copies = mode == 0 ? kThreads / 32 : 1;
  unsigned int* h = sh + (mode == 0 ? (threadIdx.x >> 5) * nbin : 0);
  if (mode < 2) {
    for (int i = threadIdx.x; i < copies * nbin; i += kThreads) sh[i] = 0;
    __syncthreads();
  }
  auto add = [&](int sym, unsigned int run) {
    if (mode < 2) atomicAdd(&h[sym], run);
    else if (sym < nsym) atomicAdd(&hist[sym], (unsigned long long)run);
  };
  // run-length merge of 16 codes; lean path for full groups (every code valid)
  auto runs16 = [&](const int (&c)[16]) {
    int cur = c[0];
    unsigned int run = 1;
#pragma unroll
    for (int j = 1; j < 16; ++j) {
      if (c[j] == cur) {
        ++run;
      } else {
        add(cur, run);
        cur = c[j];
        run = 1;
      }
    }
    add(cur, run);
  };
  const long long groups = (n + 15) / 16;
  const long long full = n / 16;
  const long long stride = (long long)gridDim.x * kThreads;
  const bool aligned = (((uintptr_t)codes) & 15) == 0;
  auto load_full = [&](long long g, int (&c)[16]) {
    if (sizeof(C) == 1) {
      const uint4 v = __ldcs(reinterpret_cast<const uint4*>(codes + g * 16));
      const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int j = 0; j < 16; ++j) c[j] = (int)((w[j >> 2] >> (8 * (j & 3))) & 0xffu);
    } else {
      const uint4 v0 = __ldcs(reinterpret_cast<const uint4*>(codes + g * 16));
      const uint4 v1 = __ldcs(reinterpret_cast<const uint4*>(codes + g * 16) + 1);
      const uint32_t w[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
#pragma unroll
      for (int j = 0; j < 16; ++j) c[j] = (int)((w[j >> 1] >> (16 * (j & 1))) & 0xffffu) & mask;
    }
  };
  long long g = (long long)blockIdx.x * kThreads + threadIdx.x;
  if (aligned) {
    for (; g + stride < full; g += 2 * stride) {  // two groups in flight per thread
      int c0[16], c1[16];
      load_full(g, c0);
      load_full(g + stride, c1);
      runs16(c0);
      runs16(c1);
    }
  }
  for (; g < groups; g += stride) {  // remainder, unaligned or partial groups
    int c[16];
    load16<C>(codes, g * 16, n, c);
#pragma unroll
    for (int j = 0; j < 16; ++j)
      if (c[j] >= 0) add(c[j] & mask, 1u);
  }
  if (mode == 2) return;
  __syncthreads();
  for (int i = threadIdx.x; i < nsym; i += kThreads) {
    unsigned long long s = 0;
    for (int w = 0; w < copies; ++w) s += sh[w * nbin + i];
    if (s) atomicAdd(&hist[i], s);
  }
}

}  // namespace

cudaError_t launch_code_hist_batch(const void* const* codes, unsigned long long* const* hist,
                                   int nf, int m, long long n, int sms, cudaStream_t s) {
  if (nf < 1 || nf > kBatchMax) return cudaErrorInvalidValue;
  HistTab tab;
  for (int f = 0; f < nf; ++f) {
    tab.codes[f] = codes[f];
    tab.hist[f] = hist[f];
  }
  const long long groups = (n + 15) / 16;
  long long blocks = (groups + kThreads - 1) / kThreads;
  const long long cap = ((long long)sms * 8 + nf - 1) / nf;  // ~8 blocks / SM in all
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  const int nbin = m <= 8 ? 256 : 1 << m;
  const size_t smem = m <= 10 ? (size_t)(kThreads / 32) * 4 * nbin : (m <= 13 ? (size_t)4 << m : 0);
  static KernelAttr attr8, attr16;
  cudaError_t e = kernel_smem(attr8, code_hist_kernel<uint8_t>, 64 * 1024);
  if (e == cudaSuccess) e = kernel_smem(attr16, code_hist_kernel<uint16_t>, 64 * 1024);
  if (e != cudaSuccess) return e;
  const dim3 grid((unsigned)blocks, nf);
  if (m > 8)
    code_hist_kernel<uint16_t><<<grid, kThreads, smem, s>>>(tab, n, m);
  else
    code_hist_kernel<uint8_t><<<grid, kThreads, smem, s>>>(tab, n, m);
  return cudaGetLastError();
}

cudaError_t launch_code_hist(const void* codes, int m, long long n, unsigned long long* hist,
                             int sms, cudaStream_t s) {
  return launch_code_hist_batch(&codes, &hist, 1, m, n, sms, s);
}

// ---------------------------------------------------------------------------
// Batched interval trials (--auto-m, cli.py:146-154): every trial's sweep
// writes u16 codes; K (the code-0 count that decides the hitting rate,
// codec.py:121) is counted here, and the chosen trial's codes are narrowed to
// u8 when its m <= 8 so the back end reads the layout it always reads.
namespace {

struct ZeroTab {
  const uint16_t* codes[kBatchMax];
  unsigned long long* k[kBatchMax];
};

__global__ void __launch_bounds__(kThreads) zero_count_kernel(const __grid_constant__ ZeroTab tab,
                                                              long long n) {
  const uint16_t* __restrict__ codes = tab.codes[blockIdx.y];
  unsigned int c = 0;
  const long long n8 = n >> 3;
  for (long long i = blockIdx.x * (long long)kThreads + threadIdx.x; i < n8;
       i += (long long)gridDim.x * kThreads) {
    const uint4 v = __ldcs(reinterpret_cast<const uint4*>(codes) + i);
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int j = 0; j < 4; ++j)
      c += ((w[j] & 0xffffu) == 0) + ((w[j] >> 16) == 0);
  }
  if (blockIdx.x == 0)
    for (long long i = (n8 << 3) + threadIdx.x; i < n; i += kThreads) c += codes[i] == 0;
  c = __reduce_add_sync(EBZ_FULL, c);
  __shared__ unsigned int part[kThreads / 32];
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t = 0;
    for (int w = 0; w < kThreads / 32; ++w) t += part[w];
    if (t) atomicAdd(tab.k[blockIdx.y], t);
  }
}

__global__ void __launch_bounds__(kThreads) narrow_codes_kernel(const uint16_t* __restrict__ in,
                                                                uint8_t* __restrict__ out,
                                                                long long n) {
  for (long long i = blockIdx.x * (long long)kThreads + threadIdx.x; i < n;
       i += (long long)gridDim.x * kThreads)
    out[i] = (uint8_t)in[i];
}

}  // namespace

// k[f] += number of zero codes of field f (u16 codes, 16-byte aligned)
cudaError_t launch_zero_count_batch(const uint16_t* const* codes, unsigned long long* const* k,
                                    int nf, long long n, int sms, cudaStream_t s) {
  if (nf < 1 || nf > kBatchMax) return cudaErrorInvalidValue;
  ZeroTab tab;
  for (int f = 0; f < nf; ++f) {
    tab.codes[f] = codes[f];
    tab.k[f] = k[f];
  }
  long long blocks = ((n >> 3) + kThreads - 1) / kThreads;
  const long long cap = ((long long)sms * 8 + nf - 1) / nf;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  zero_count_kernel<<<dim3((unsigned)blocks, nf), kThreads, 0, s>>>(tab, n);
  return cudaGetLastError();
}

cudaError_t launch_narrow_codes(const uint16_t* in, uint8_t* out, long long n, int sms,
                                cudaStream_t s) {
  long long blocks = (n + kThreads - 1) / kThreads;
  if (blocks > (long long)sms * 8) blocks = (long long)sms * 8;
  if (blocks < 1) blocks = 1;
  narrow_codes_kernel<<<(unsigned)blocks, kThreads, 0, s>>>(in, out, n);
  return cudaGetLastError();
}
