// analysis.cu -- callers of the hot path that the paper's methodology runs
// at scale:
//
//  * original_hits (ebzip/_kernels.py:108-121): points whose prediction from
//    the ORIGINAL neighbours lands within the bound.  No feedback, so every
//    point is independent: one thread per point, the reference's stencil bank
//    (same boundary rule, same term order, binary64 without contraction).
//  * fused distortion metrics (ebzip/metrics.py:93-137): max |a - b|, sums for
//    RMSE / means, centred dot products for Pearson, and the error
//    autocorrelation at lags 0..L.  Two passes (means first); block partial
//    sums reduced in a fixed order, so results are deterministic.
#include "ebz_common.cuh"

namespace {

constexpr int kHitThreads = 256;

template <typename T>
__global__ void __launch_bounds__(kHitThreads)
original_hits_kernel(const T* __restrict__ values, long long n, int ndim, long long d0,
                     long long d1, long long d2, int L, double bound,
                     const long long* __restrict__ deltas, const double* __restrict__ coeffs,
                     const long long* __restrict__ starts, const long long* __restrict__ counts,
                     unsigned long long* __restrict__ out) {
  unsigned long long hits = 0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    // coordinates, axis 0 fastest (core.py:71-76)
    long long c[4] = {0, 0, 0, 0};
    {
      long long r = i;
      c[0] = r % d0;
      r /= d0;
      if (ndim > 1) { c[1] = r % d1; r /= d1; }
      if (ndim > 2) { c[2] = r % d2; r /= d2; }
      if (ndim > 3) c[3] = r;
    }
    int mask = 0;
    long long deep = 0x7fffffffffffffffll;
    for (int ax = 0; ax < ndim; ++ax)
      if (c[ax] > 0) {
        mask |= 1 << ax;
        deep = c[ax] < deep ? c[ax] : deep;
      }
    double pred = 0.0;  // _predict_at (_kernels.py:18-36)
    if (mask) {
      const long long eff = (long long)L < deep ? (long long)L : deep;
      const long long slot = (long long)(mask - 1) * L + (eff - 1);
      const long long t0 = __ldg(starts + slot), t1 = t0 + __ldg(counts + slot);
      for (long long t = t0; t < t1; ++t)
        pred = __dadd_rn(pred, __dmul_rn(__ldg(coeffs + t), (double)values[i - __ldg(deltas + t)]));
    }
    hits += fabs(__dsub_rn((double)values[i], pred)) <= bound;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) hits += __shfl_xor_sync(EBZ_FULL, hits, o);
  if ((threadIdx.x & 31) == 0 && hits) atomicAdd(out, hits);
}

// ---------------------------------------------------------------- metrics
constexpr int kMetThreads = 256;
constexpr int kMetBlocks = 592;  // 148 SMs x 4; fixed so the reduction order is fixed
constexpr int kP1 = 5;           // max|e|, sum e^2, sum a, sum b, sum e

template <typename T>
__global__ void __launch_bounds__(kMetThreads)
metrics_pass1(const T* __restrict__ a, const T* __restrict__ b, long long n,
              double* __restrict__ part) {
  double mx = 0.0, se2 = 0.0, sa = 0.0, sb = 0.0, se = 0.0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const double av = (double)a[i], bv = (double)b[i];
    const double e = __dsub_rn(av, bv);
    mx = fmax(mx, fabs(e));
    se2 = __dadd_rn(se2, __dmul_rn(e, e));
    sa = __dadd_rn(sa, av);
    sb = __dadd_rn(sb, bv);
    se = __dadd_rn(se, e);
  }
  __shared__ double s[kP1][kMetThreads / 32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    mx = fmax(mx, __shfl_xor_sync(EBZ_FULL, mx, o));
    se2 = __dadd_rn(se2, __shfl_xor_sync(EBZ_FULL, se2, o));
    sa = __dadd_rn(sa, __shfl_xor_sync(EBZ_FULL, sa, o));
    sb = __dadd_rn(sb, __shfl_xor_sync(EBZ_FULL, sb, o));
    se = __dadd_rn(se, __shfl_xor_sync(EBZ_FULL, se, o));
  }
  if (lane == 0) {
    s[0][w] = mx; s[1][w] = se2; s[2][w] = sa; s[3][w] = sb; s[4][w] = se;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double r[kP1] = {0, 0, 0, 0, 0};
    for (int k = 0; k < kMetThreads / 32; ++k) {
      r[0] = fmax(r[0], s[0][k]);
      for (int q = 1; q < kP1; ++q) r[q] = __dadd_rn(r[q], s[q][k]);
    }
    for (int q = 0; q < kP1; ++q) part[(size_t)q * gridDim.x + blockIdx.x] = r[q];
  }
}

// pass 2: centred products.  Block-tiled: the tile's centred errors (plus the
// L following ones) sit in shared memory; thread t accumulates lags t + 1,
// t + 1 + kMetThreads, ... (up to kLagsPerThread * kMetThreads = EBZ_MAX_LAGS).
constexpr int kTile = 2048;
constexpr int kLagsPerThread = 4;
static_assert(kLagsPerThread * kMetThreads == EBZ_MAX_LAGS, "lag capacity");

template <typename T>
__global__ void __launch_bounds__(kMetThreads)
metrics_pass2(const T* __restrict__ a, const T* __restrict__ b, long long n, int lags,
              const double* __restrict__ means, double* __restrict__ part) {
  extern __shared__ double s_c[];  // kTile + lags centred errors
  const double ma = means[0], mb = means[1], me = means[2];
  double sab = 0.0, saa = 0.0, sbb = 0.0, scc = 0.0;
  double acc[kLagsPerThread] = {0.0, 0.0, 0.0, 0.0};
  const long long ntiles = (n + kTile - 1) / kTile;
  for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const long long i0 = tile * kTile;
    __syncthreads();
    for (int k = threadIdx.x; k < kTile + lags; k += blockDim.x) {
      const long long i = i0 + k;
      double cv = 0.0;
      if (i < n) {
        const double av = (double)a[i], bv = (double)b[i];
        cv = __dsub_rn(__dsub_rn(av, bv), me);
        if (k < kTile) {
          const double da = __dsub_rn(av, ma), db = __dsub_rn(bv, mb);
          sab = __dadd_rn(sab, __dmul_rn(da, db));
          saa = __dadd_rn(saa, __dmul_rn(da, da));
          sbb = __dadd_rn(sbb, __dmul_rn(db, db));
          scc = __dadd_rn(scc, __dmul_rn(cv, cv));
        }
      }
      s_c[k] = cv;
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kLagsPerThread; ++j) {
      const int lag = threadIdx.x + 1 + j * kMetThreads;
      if (lag > lags) break;
      // pairs (i, i + lag) with i in this tile and i + lag < n
      const long long lim = n - lag - i0;
      const int cnt = lim <= 0 ? 0 : (lim < kTile ? (int)lim : kTile);
      double r = acc[j];
      for (int k = 0; k < cnt; ++k) r = __dadd_rn(r, __dmul_rn(s_c[k], s_c[k + lag]));
      acc[j] = r;
    }
  }
  // block partials: 4 centred sums (reduced here) + one per lag
  __shared__ double s[4][kMetThreads / 32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    sab = __dadd_rn(sab, __shfl_xor_sync(EBZ_FULL, sab, o));
    saa = __dadd_rn(saa, __shfl_xor_sync(EBZ_FULL, saa, o));
    sbb = __dadd_rn(sbb, __shfl_xor_sync(EBZ_FULL, sbb, o));
    scc = __dadd_rn(scc, __shfl_xor_sync(EBZ_FULL, scc, o));
  }
  if (lane == 0) { s[0][w] = sab; s[1][w] = saa; s[2][w] = sbb; s[3][w] = scc; }
  __syncthreads();
  const size_t G = gridDim.x;
  if (threadIdx.x == 0) {
    double r[4] = {0, 0, 0, 0};
    for (int k = 0; k < kMetThreads / 32; ++k)
      for (int q = 0; q < 4; ++q) r[q] = __dadd_rn(r[q], s[q][k]);
    for (int q = 0; q < 4; ++q) part[(size_t)q * G + blockIdx.x] = r[q];
  }
#pragma unroll
  for (int j = 0; j < kLagsPerThread; ++j) {
    const int l = threadIdx.x + j * kMetThreads;  // lag l + 1
    if (l < lags) part[(size_t)(4 + l) * G + blockIdx.x] = acc[j];
  }
}

// fixed-order reduction of nq rows of G block partials (row 0 of pass 1 is a max)
__global__ void metrics_reduce(const double* __restrict__ part, int nq, int G, int max_row,
                               double* __restrict__ out) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nq) return;
  double r = 0.0;
  for (int k = 0; k < G; ++k)
    r = q == max_row ? fmax(r, part[(size_t)q * G + k]) : __dadd_rn(r, part[(size_t)q * G + k]);
  out[q] = r;
}

__global__ void metrics_means(const double* __restrict__ p1, long long n, double* __restrict__ m) {
  if (threadIdx.x == 0) {
    m[0] = __ddiv_rn(p1[2], (double)n);
    m[1] = __ddiv_rn(p1[3], (double)n);
    m[2] = __ddiv_rn(p1[4], (double)n);
  }
}

}  // namespace

cudaError_t launch_original_hits(const void* values, int width, int ndim, const long long* dims,
                                 int layers, double bound, const long long* deltas,
                                 const double* coeffs, const long long* starts,
                                 const long long* counts, unsigned long long* out, int sms,
                                 cudaStream_t s) {
  long long n = 1;
  for (int a = 0; a < ndim; ++a) n *= dims[a];
  long long blocks = (n + kHitThreads - 1) / kHitThreads;
  if (blocks > (long long)sms * 8) blocks = (long long)sms * 8;
  if (blocks < 1) blocks = 1;
  const long long d1 = ndim > 1 ? dims[1] : 1, d2 = ndim > 2 ? dims[2] : 1;
  if (width == 32)
    original_hits_kernel<float><<<(unsigned)blocks, kHitThreads, 0, s>>>(
        (const float*)values, n, ndim, dims[0], d1, d2, layers, bound, deltas, coeffs, starts,
        counts, out);
  else
    original_hits_kernel<double><<<(unsigned)blocks, kHitThreads, 0, s>>>(
        (const double*)values, n, ndim, dims[0], d1, d2, layers, bound, deltas, coeffs, starts,
        counts, out);
  return cudaGetLastError();
}

size_t metrics_scratch_bytes(int lags) {
  return (size_t)(kP1 + 4 + lags) * kMetBlocks * 8 + (size_t)(kP1 + 4 + lags + 8) * 8;
}

// out (device doubles): [max|e|, sum e^2, sum a, sum b, sum e, sum da*db,
// sum da^2, sum db^2, sum c^2, lag_1 .. lag_L]  (c = e - mean(e))
cudaError_t launch_metrics(const void* a, const void* b, int width, long long n, int lags,
                           double* scratch, double* out, cudaStream_t s) {
  double* part = scratch;
  double* means = scratch + (size_t)(kP1 + 4 + lags) * kMetBlocks;
  if (width == 32)
    metrics_pass1<float><<<kMetBlocks, kMetThreads, 0, s>>>((const float*)a, (const float*)b, n,
                                                            part);
  else
    metrics_pass1<double><<<kMetBlocks, kMetThreads, 0, s>>>((const double*)a,
                                                             (const double*)b, n, part);
  metrics_reduce<<<1, 32, 0, s>>>(part, kP1, kMetBlocks, 0, out);
  metrics_means<<<1, 32, 0, s>>>(out, n, means);
  const size_t smem = (size_t)(kTile + lags) * 8;
  if (width == 32)
    metrics_pass2<float><<<kMetBlocks, kMetThreads, smem, s>>>((const float*)a, (const float*)b,
                                                               n, lags, means, part);
  else
    metrics_pass2<double><<<kMetBlocks, kMetThreads, smem, s>>>(
        (const double*)a, (const double*)b, n, lags, means, part);
  metrics_reduce<<<(4 + lags + 127) / 128, 128, 0, s>>>(part, 4 + lags, kMetBlocks, -1,
                                                        out + kP1);
  return cudaGetLastError();
}
