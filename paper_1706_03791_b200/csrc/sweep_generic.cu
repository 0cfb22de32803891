// sweep_generic.cu -- row-pipelined wavefront for ANY shape (d = 1..4),
// any layer count n and both element widths.
//
// Restates compress_scan / decompress_scan (ebzip/_kernels.py:48-105) with
// the same stencil bank (codec.py:54-89) and identical arithmetic order, but
// runs the rows of the grid concurrently:
//
//  * a "row" is a line along axis 0 (the scan-fastest axis);
//  * a warp task owns 32 consecutive rows; lane t walks its row with a skew
//    of t steps (x = S - t at step S), so every in-warp dependency on an
//    earlier row has already been computed one or more steps before;
//  * dependencies on rows of earlier tasks are resolved with epoch-tagged
//    progress counters in global memory (release/acquire), checked once per
//    32-step chunk; tasks are handed out by an atomic ticket in row order, so
//    a task only ever waits on lower tickets (deadlock free).
//
// Neighbour values are read back from the recon buffer through L2
// (ld.global.cg).  This kernel is the correctness baseline for shapes the
// register-systolic kernels (sweep_fast.cu) do not cover: d = 1, d = 4,
// layers beyond the fast kernels' templates, and tiny axis-0 extents.
#include "ebz_common.cuh"

#include <climits>

namespace {

constexpr int kChunk = 32;
constexpr int kWarpsPerBlock = 8;
constexpr int kSmemHistMaxM = 12;

template <typename C>
__device__ __forceinline__ void hist_add(int code, bool valid, unsigned int* s_hist,
                                         unsigned long long* g_hist, bool smem) {
  const int key = valid ? code : -1;
  const unsigned int peers = __match_any_sync(EBZ_FULL, key);
  const int leader = __ffs(peers) - 1;
  if (valid && (int)(threadIdx.x & 31) == leader) {
    if (smem)
      atomicAdd(&s_hist[code], (unsigned int)__popc(peers));
    else
      atomicAdd(&g_hist[code], (unsigned long long)__popc(peers));
  }
}

template <typename T, typename C, bool COMPRESS>
__global__ void __launch_bounds__(32 * kWarpsPerBlock)
sweep_generic_kernel(SweepArgs a) {
  extern __shared__ unsigned int s_hist[];
  const bool smem_hist = COMPRESS && a.hist && a.m <= kSmemHistMaxM;
  const int nsym = 1 << a.m;
  if (smem_hist) {
    for (int i = threadIdx.x; i < nsym; i += blockDim.x) s_hist[i] = 0;
    __syncthreads();
  }
  const int lane = threadIdx.x & 31;
  const double eb = a.info->eb;
  const double two_eb = __dmul_rn(2.0, eb);
  const int nd = a.ndim;
  const int L = a.layers;
  const long long nx = a.dims[0];
  const long long ntasks = (a.nrows + 31) / 32;
  const long long steps_total = nx + 31;
  const unsigned long long tag = (unsigned long long)a.epoch << 32;
  const T* values = reinterpret_cast<const T*>(a.values);
  T* recon = reinterpret_cast<T*>(a.recon);
  C* codes = reinterpret_cast<C*>(a.codes);
  const T* unpred = reinterpret_cast<const T*>(a.unpred);
  const bool eb_bad = !(eb > 0.0);
  const unsigned long long n_unpred = COMPRESS ? 0ull : a.info->n_unpred;

  // distinct higher-axis offsets (ky, kz, kw) with ky..kw in [0, L]
  long long hi_count = 1;
  for (int ax = 1; ax < nd; ++ax) hi_count *= (L + 1);

  unsigned long long zeros_total = 0;

  for (;;) {
    long long task = 0;
    if (lane == 0) task = (long long)atomicAdd(a.ticket, 1u);
    task = __shfl_sync(EBZ_FULL, task, 0);
    if (task >= ntasks || eb_bad) break;

    const long long R0 = task * 32;
    const long long R = R0 + lane;
    const bool rv = R < a.nrows;
    long long rc[3] = {0, 0, 0};
    {
      long long r = rv ? R : 0;
      for (int ax = 1; ax < nd; ++ax) {
        rc[ax - 1] = r % a.dims[ax];
        r /= a.dims[ax];
      }
    }
    int rmask = 0;
    long long rdeep = LLONG_MAX;
    for (int ax = 1; ax < nd; ++ax)
      if (rc[ax - 1] > 0) {
        rmask |= 1 << ax;
        rdeep = rc[ax - 1] < rdeep ? rc[ax - 1] : rdeep;
      }
    const long long base = R * nx;
    unsigned long long zrank = 0;
    if (!COMPRESS && rv) zrank = a.rowbase[R] + a.rowblk[R >> 8];
    unsigned long long zeros = 0;

    for (long long S0 = 0; S0 < steps_total; S0 += kChunk) {
      const long long S1 = S0 + kChunk < steps_total ? S0 + kChunk : steps_total;
      // ---- wait for rows of earlier tasks (spread over lanes) ------------
      {
        const long long need_steps = (S1 - 1 + 32) < steps_total ? (S1 - 1 + 32) : steps_total;
        const unsigned long long need = tag | (unsigned long long)need_steps;
        for (long long c = 1 + lane; c < hi_count; c += 32) {
          long long rem = c, roff = 0, mul = 1;
          for (int ax = 1; ax < nd; ++ax) {
            roff += (rem % (L + 1)) * mul;
            rem /= (L + 1);
            mul *= a.dims[ax];
          }
          for (int side = 0; side < 2; ++side) {
            const long long rr = (side ? R0 + 31 : R0) - roff;
            if (rr < 0) continue;
            const long long dt = rr >> 5;
            if (dt >= task) continue;
            for (unsigned ns = 32; ld_acquire_u64(a.progress + (size_t)dt * kProgPad) < need;
                 ns = ns < 1024 ? 2 * ns : ns)
              __nanosleep(ns);
          }
        }
      }
      __syncwarp();
      for (long long S = S0; S < S1; ++S) {
        const long long x = S - lane;
        const bool act = rv && x >= 0 && x < nx;
        int code = 0;
        if (act) {
          const long long i = base + x;
          const int mask = rmask | (x > 0 ? 1 : 0);
          double pred = 0.0;
          if (mask) {
            long long deep = rdeep;
            if (x > 0 && x < deep) deep = x;
            const long long eff = (long long)L < deep ? (long long)L : deep;
            const long long slot = (long long)(mask - 1) * L + (eff - 1);
            const long long t0 = __ldg(a.starts + slot);
            const long long t1 = t0 + __ldg(a.counts + slot);
            for (long long t = t0; t < t1; ++t) {
              const double v = (double)__ldcg(recon + (i - __ldg(a.deltas + t)));
              pred = __dadd_rn(pred, __dmul_rn(__ldg(a.coeffs + t), v));
            }
          }
          if (COMPRESS) {
            T r;
            code = quantize_exact<T>(values[i], pred, eb, two_eb, a.center, r,
                                     a.trunc ? eb_exponent(eb) : kNoTrunc);
            codes[i] = (C)code;
            __stcg(recon + i, r);
            zeros += (code == 0);
          } else {
            code = (int)codes[i];
            T r;
            if (code == 0) {
              const unsigned long long rk = zrank + zeros;
              ++zeros;
              if (rk < n_unpred) {
                r = unpred[rk];
              } else {
                r = (T)0;
                atomicOr(&a.info_w->status, ST_UNDERRUN);
              }
            } else {
              r = Elem<T>::round(__dadd_rn(
                  pred, __dmul_rn((double)((long long)code - (long long)a.center), two_eb)));
            }
            if (!Elem<T>::finite(r)) atomicOr(&a.info_w->status, ST_NONFINITE_OUT);
            __stcg(recon + i, r);
          }
        }
        if (COMPRESS && a.hist) hist_add<C>(code, act, s_hist, a.hist, smem_hist);
        __syncwarp();
      }
      // ---- publish progress -------------------------------------------------
      __syncwarp();
      if (lane == 0) {
        __threadfence();
        st_release_u64(a.progress + (size_t)task * kProgPad, tag | (unsigned long long)S1);
      }
    }
    zeros_total += zeros;
  }
  // K (compress) / consumed count (decompress)
#pragma unroll
  for (int o = 16; o; o >>= 1) zeros_total += __shfl_xor_sync(EBZ_FULL, zeros_total, o);
  if (lane == 0 && zeros_total) {
    if (COMPRESS)
      atomicAdd(&a.info_w->n_unpred, zeros_total);
    else
      atomicAdd(&a.info_w->used, zeros_total);
  }
  if (smem_hist) {
    __syncthreads();
    for (int i = threadIdx.x; i < nsym; i += blockDim.x)
      if (s_hist[i]) atomicAdd(&a.hist[i], (unsigned long long)s_hist[i]);
  }
}

template <typename T, typename C, bool COMPRESS>
cudaError_t launch_generic_t(const SweepArgs& a, int sms, cudaStream_t s) {
  const long long ntasks = (a.nrows + 31) / 32;
  long long blocks = (ntasks + kWarpsPerBlock - 1) / kWarpsPerBlock;
  const long long cap = (long long)sms * 8;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  size_t smem = (COMPRESS && a.m <= kSmemHistMaxM) ? sizeof(unsigned int) << a.m : 0;
  sweep_generic_kernel<T, C, COMPRESS><<<(unsigned)blocks, 32 * kWarpsPerBlock, smem, s>>>(a);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_sweep_generic(const SweepArgs& a, int width, bool compress, int sms,
                                 cudaStream_t s) {
  const bool wide = a.wide != 0;
  if (width == 32) {
    if (compress)
      return wide ? launch_generic_t<float, uint16_t, true>(a, sms, s)
                  : launch_generic_t<float, uint8_t, true>(a, sms, s);
    return wide ? launch_generic_t<float, uint16_t, false>(a, sms, s)
                : launch_generic_t<float, uint8_t, false>(a, sms, s);
  }
  if (compress)
    return wide ? launch_generic_t<double, uint16_t, true>(a, sms, s)
                : launch_generic_t<double, uint8_t, true>(a, sms, s);
  return wide ? launch_generic_t<double, uint16_t, false>(a, sms, s)
              : launch_generic_t<double, uint8_t, false>(a, sms, s);
}
