// range.cu -- fused value-range / finiteness pass and effective bound.
//
// Replaces grid_range (ebzip/core.py:132-136), the DataGrid finiteness check
// (core.py:92-93) and ErrorBoundSpec.effective_bound (core.py:161-178).
// One HBM read of the grid (4N bytes for f32), one launch: per-thread
// min/max over ordered-integer keys with 16-byte vector loads, warp and block
// reduction, and the last block to finish resolves eb on the device so the
// sweep can start without a host round trip.
//
// The range is computed in the element precision, exactly as numpy does it:
// R = (double)(T)(max - min) (f32 subtraction for f32 grids).
#include "ebz_common.cuh"

namespace {

// order-preserving integer images of IEEE values (-0.0 < +0.0, NaN excluded)
__device__ __forceinline__ unsigned int okey(float v) {
  unsigned int b = __float_as_uint(v);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float okey_inv(unsigned int k) {
  unsigned int b = (k & 0x80000000u) ? (k & 0x7fffffffu) : ~k;
  return __uint_as_float(b);
}
__device__ __forceinline__ unsigned long long okey(double v) {
  unsigned long long b = (unsigned long long)__double_as_longlong(v);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double okey_inv(unsigned long long k) {
  unsigned long long b = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
  return __longlong_as_double((long long)b);
}

template <typename T> struct KeyOf;
template <> struct KeyOf<float> { typedef unsigned int K; typedef float4 V; enum { W = 4 }; };
template <> struct KeyOf<double> {
  typedef unsigned long long K;
  typedef double2 V;
  enum { W = 2 };
};

template <typename T>
__device__ __forceinline__ void acc(T v, typename KeyOf<T>::K& lo, typename KeyOf<T>::K& hi,
                                    int& bad) {
  if (!isfinite(v)) { bad = 1; return; }
  typename KeyOf<T>::K k = okey(v);
  lo = k < lo ? k : lo;
  hi = k > hi ? k : hi;
}

// per-field pointers of a batched launch (blockIdx.y = field)
struct RangeTab {
  const void* x[kBatchMax];
  Info* info[kBatchMax];
  unsigned int* scratch[kBatchMax];
  unsigned long long* hist[kBatchMax];  // zeroed here for the histogram pass (may be null)
};

// A fresh compress record: the range stage is the first stage of compress,
// so it initialises the whole record (and the field's histogram) instead of
// separate memsets.
__device__ __forceinline__ void write_record(Info* info, double eb, double vmin, double vmax,
                                             double range, int status) {
  Info z;
  memset(&z, 0, sizeof(Info));
  z.eb = eb;
  z.vmin = vmin;
  z.vmax = vmax;
  z.range = range;
  z.status = status;
  *info = z;
}
constexpr int kMaxBlocks = 1184;  // partial slots per field (148 SMs x 8)

template <typename T>
__global__ void __launch_bounds__(256)
range_kernel(const __grid_constant__ RangeTab tab, long long n, int has_abs, double abs_b,
             int has_rel, double rel_b, int nsym) {
  const int f = blockIdx.y;
  if (blockIdx.x == 0 && tab.hist[f])
    for (int i = threadIdx.x; i < nsym; i += blockDim.x) tab.hist[f][i] = 0ull;
  const T* __restrict__ x = reinterpret_cast<const T*>(tab.x[f]);
  Info* info = tab.info[f];
  unsigned long long* part = reinterpret_cast<unsigned long long*>(tab.scratch[f]);
  unsigned int* counter = reinterpret_cast<unsigned int*>(part + 3 * kMaxBlocks);
  typedef typename KeyOf<T>::K K;
  typedef typename KeyOf<T>::V V;
  const int W = KeyOf<T>::W;
  K lo = (K)~(K)0, hi = 0;
  int bad = 0;
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nthreads = (long long)gridDim.x * blockDim.x;
  // vector body (x from cudaMalloc / torch is >= 256B aligned; fall back if not)
  long long head = 0;
  if (((uintptr_t)x & 15) == 0) {
    const long long nv = n / W;
    const V* xv = reinterpret_cast<const V*>(x);
    for (long long i = tid; i < nv; i += nthreads) {
      V v = __ldcs(xv + i);
      const T* e = reinterpret_cast<const T*>(&v);
#pragma unroll
      for (int j = 0; j < W; ++j) acc<T>(e[j], lo, hi, bad);
    }
    head = nv * W;
  }
  for (long long i = head + tid; i < n; i += nthreads) acc<T>(x[i], lo, hi, bad);
  // warp + block reduction
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    K l2 = __shfl_xor_sync(EBZ_FULL, lo, o), h2 = __shfl_xor_sync(EBZ_FULL, hi, o);
    lo = l2 < lo ? l2 : lo;
    hi = h2 > hi ? h2 : hi;
  }
  bad = __any_sync(EBZ_FULL, bad);
  __shared__ K s_lo[8], s_hi[8];
  __shared__ int s_bad[8];
  __shared__ bool s_last;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) { s_lo[w] = lo; s_hi[w] = hi; s_bad[w] = bad; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 1; i < (int)(blockDim.x >> 5); ++i) {
      lo = s_lo[i] < lo ? s_lo[i] : lo;
      hi = s_hi[i] > hi ? s_hi[i] : hi;
      bad |= s_bad[i];
    }
    part[3 * blockIdx.x + 0] = (unsigned long long)lo;
    part[3 * blockIdx.x + 1] = (unsigned long long)hi;
    part[3 * blockIdx.x + 2] = (unsigned long long)bad;
    __threadfence();
    unsigned int done = atomicAdd(counter, 1u);
    s_last = (done == gridDim.x - 1);
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  // the last block reduces all block partials in parallel
  K glo = (K)~(K)0, ghi = 0;
  int gbad = 0;
  for (unsigned int b = threadIdx.x; b < gridDim.x; b += blockDim.x) {
    K l = (K)__ldcg(part + 3 * b), h = (K)__ldcg(part + 3 * b + 1);
    glo = l < glo ? l : glo;
    ghi = h > ghi ? h : ghi;
    gbad |= (int)__ldcg(part + 3 * b + 2);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    K l2 = __shfl_xor_sync(EBZ_FULL, glo, o), h2 = __shfl_xor_sync(EBZ_FULL, ghi, o);
    glo = l2 < glo ? l2 : glo;
    ghi = h2 > ghi ? h2 : ghi;
  }
  gbad = __any_sync(EBZ_FULL, gbad);
  __syncthreads();
  if (lane == 0) { s_lo[w] = glo; s_hi[w] = ghi; s_bad[w] = gbad; }
  __syncthreads();
  if (threadIdx.x != 0) return;
  for (int i = 1; i < (int)(blockDim.x >> 5); ++i) {
    glo = s_lo[i] < glo ? s_lo[i] : glo;
    ghi = s_hi[i] > ghi ? s_hi[i] : ghi;
    gbad |= s_bad[i];
  }
  *counter = 0;  // reusable without a memset
  const T vmin = okey_inv(glo), vmax = okey_inv(ghi);
  const T r = vmax - vmin;  // element-precision subtraction (numpy semantics)
  int st = gbad ? ST_NONFINITE_IN : 0;
  // min(candidates) in the reference's candidate order (absolute first)
  double eb = 0.0;
  bool have = false;
  if (has_abs) { eb = abs_b; have = true; }
  if (has_rel) {
    const double c = __dmul_rn(rel_b, (double)r);
    if (!have || c < eb) eb = c;
  }
  if (!(eb > 0.0)) st |= ST_EB_NONPOSITIVE;
  write_record(info, eb, (double)vmin, (double)vmax, (double)r, st);
}

// eb without a range pass (absolute-only bound; finiteness still checked)
template <typename T>
__global__ void finite_kernel(const T* __restrict__ x, long long n, Info* info) {
  int bad = 0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    bad |= !isfinite(x[i]);
  if (__any_sync(EBZ_FULL, bad) && (threadIdx.x & 31) == 0)
    atomicOr(&info->status, ST_NONFINITE_IN);
}

// absolute bound only: fresh records with eb (and zeroed histograms), one
// block per field
__global__ void set_abs_eb(const __grid_constant__ RangeTab tab, double eb, int nsym) {
  const int f = blockIdx.x;
  if (tab.hist[f])
    for (int i = threadIdx.x; i < nsym; i += blockDim.x) tab.hist[f][i] = 0ull;
  if (threadIdx.x == 0)
    write_record(tab.info[f], eb, 0.0, 0.0, 0.0, eb > 0.0 ? 0 : ST_EB_NONPOSITIVE);
}

}  // namespace

// scratch (per field): 3 * kMaxBlocks u64 partials followed by one u32
// counter (zeroed once; the last block re-arms it)
cudaError_t launch_range_batch(const void* const* values, Info* const* infos,
                               unsigned int* const* scratch, unsigned long long* const* hists,
                               int nsym, int nf, int width, long long n, int has_abs,
                               double abs_b, int has_rel, double rel_b, cudaStream_t s) {
  if (nf < 1 || nf > kBatchMax) return cudaErrorInvalidValue;
  RangeTab tab;
  for (int f = 0; f < nf; ++f) {
    tab.x[f] = values[f];
    tab.info[f] = infos[f];
    tab.scratch[f] = scratch[f];
    tab.hist[f] = hists ? hists[f] : nullptr;
  }
  if (!has_rel && has_abs >= 0) {
    // absolute bound: the reference does not compute the range at all; the
    // finiteness check only matters for device-resident inputs.
    set_abs_eb<<<nf, 256, 0, s>>>(tab, abs_b, nsym);
    return cudaGetLastError();
  }
  if (has_abs < 0) has_abs = 0;  // range requested without an absolute bound
  // ~2 waves of 8 blocks per SM over the whole batch, >= 1 block per field
  long long want = (n + 256LL * 16 - 1) / (256LL * 16);
  long long cap = (2LL * kMaxBlocks + nf - 1) / nf;
  if (cap > kMaxBlocks) cap = kMaxBlocks;
  const int blocks = (int)(want < 1 ? 1 : (want > cap ? cap : want));
  const dim3 grid(blocks, nf);
  if (width == 32)
    range_kernel<float><<<grid, 256, 0, s>>>(tab, n, has_abs, abs_b, has_rel, rel_b, nsym);
  else
    range_kernel<double><<<grid, 256, 0, s>>>(tab, n, has_abs, abs_b, has_rel, rel_b, nsym);
  return cudaGetLastError();
}

cudaError_t launch_range(const void* values, int width, long long n, int has_abs, double abs_b,
                         int has_rel, double rel_b, Info* info, unsigned int* scratch,
                         cudaStream_t s) {
  return launch_range_batch(&values, &info, &scratch, nullptr, 0, 1, width, n, has_abs, abs_b,
                            has_rel, rel_b, s);
}

cudaError_t launch_finite(const void* values, int width, long long n, Info* info, cudaStream_t s) {
  int blocks = (int)((n + 255) / 256);
  if (blocks > 1184) blocks = 1184;
  if (blocks < 1) blocks = 1;
  if (width == 32)
    finite_kernel<float><<<blocks, 256, 0, s>>>((const float*)values, n, info);
  else
    finite_kernel<double><<<blocks, 256, 0, s>>>((const double*)values, n, info);
  return cudaGetLastError();
}
