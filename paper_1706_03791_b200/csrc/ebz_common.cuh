// ebz_common.cuh -- shared device helpers and internal interfaces of libebz200.
//
// Arithmetic contract: every floating-point op on the
// path is IEEE binary64 round-to-nearest with NO contraction.  All sums and
// products therefore go through __dadd_rn/__dsub_rn/__dmul_rn/__ddiv_rn
// (and the library is additionally built with -fmad=false).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include <mutex>

#include "../../include/ebz200.h"

#define EBZ_FULL 0xffffffffu

// ---------------------------------------------------------------- status bits
// Device-side status word (EbzInfo::status); the host maps the bits onto the
// reference's exceptions in the reference's order.
enum : int {
  ST_EB_NONPOSITIVE = 1 << 0,   // core.py:173-177
  ST_NONFINITE_IN = 1 << 1,     // core.py:92-93 (device-resident inputs)
  ST_DEPTH_GT_64 = 1 << 2,      // entropy.py:133-134
  ST_EMPTY_HIST = 1 << 3,
  ST_DEC_EXHAUSTED = 1 << 4,    // entropy.py:176-179
  ST_DEC_INVALID = 1 << 5,      // entropy.py:181-182
  ST_DEC_ANOMALY = 1 << 6,      // parallel decoder did not verify -> serial
  ST_UNPRED_MISMATCH = 1 << 7,  // codec.py:144-149
  ST_UNDERRUN = 1 << 8,         // _kernels.py:98-99 / codec.py:158-159
  ST_NONFINITE_OUT = 1 << 9,    // DataGrid check on the decompressed grid
  ST_CAPACITY = 1 << 10,        // output buffer too small (host regrows)
};

// Per-field device record.  Layout shared with the host (EbzInfo in ebz200.h).
typedef EbzInfo Info;

// ---------------------------------------------------------- memory ordering
__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned int ld_acquire_u32(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// ------------------------------------------------------------ numeric helpers
template <typename T> struct Elem;
template <> struct Elem<float> {
  __device__ __forceinline__ static float round(double v) { return __double2float_rn(v); }
  __device__ __forceinline__ static bool finite(float v) { return isfinite(v); }
};
template <> struct Elem<double> {
  __device__ __forceinline__ static double round(double v) { return v; }
  __device__ __forceinline__ static bool finite(double v) { return isfinite(v); }
};

// ---- truncated-mantissa coding of unpredictable values: the opt-in
// extension named by north_star (3) (the reference stores them verbatim,
// ebzip/codec.py:119; containers with it are format version 2).  A value
// keeps its sign, its exponent and the top k mantissa bits,
//     k = clamp(e(v) - e(eb), 0, M)      (e = unbiased binary exponent),
// zero and subnormal values stay whole, so |v - trunc(v)| < 2^e(eb) <= eb.
// The compressor predicts from trunc(v) at unpredictable points, exactly as
// the decompressor will.
constexpr int kNoTrunc = -0x7fffffff;
__host__ __device__ inline int eb_exponent(double eb) {  // floor(log2 eb), eb > 0 normal
  unsigned long long b;
  memcpy(&b, &eb, 8);
  const int E = (int)((b >> 52) & 0x7ff);
  return E ? E - 1023 : -1075;
}
template <typename T> struct TruncBits;
template <> struct TruncBits<float> {
  static constexpr int M = 23, EW = 8, BIAS = 127;
  typedef unsigned U;
  __device__ static U bits(float v) { return __float_as_uint(v); }
  __device__ static float from(U b) { return __uint_as_float(b); }
};
template <> struct TruncBits<double> {
  static constexpr int M = 52, EW = 11, BIAS = 1023;
  typedef unsigned long long U;
  __device__ static U bits(double v) { return (U)__double_as_longlong(v); }
  __device__ static double from(U b) { return __longlong_as_double((long long)b); }
};
// mantissa bits kept for a value with these bits
template <typename T>
__device__ __forceinline__ int trunc_keep(typename TruncBits<T>::U b, int e_eb) {
  typedef TruncBits<T> TB;
  const int E = (int)((b >> TB::M) & ((1u << TB::EW) - 1u));
  if (E == 0) return TB::M;
  const int k = E - TB::BIAS - e_eb;
  return k < 0 ? 0 : (k > TB::M ? TB::M : k);
}
template <typename T>
__device__ __forceinline__ T trunc_value(T v, int e_eb) {
  typedef TruncBits<T> TB;
  typedef typename TB::U U;
  const U b = TB::bits(v);
  const int k = trunc_keep<T>(b, e_eb);
  return TB::from(b & ~((U(1) << (TB::M - k)) - U(1)));
}

// Reference quantizer, exact (``_kernels.py:61-78``).  Returns the code
// (0 = unpredictable) and the stored reconstruction (tr_e != kNoTrunc: the
// truncated value at unpredictable points, the opt-in extension above).
template <typename T>
__device__ __forceinline__ int quantize_exact(T xv, double pred, double eb, double two_eb,
                                              int center, T& r_out, int tr_e = kNoTrunc) {
  const double x = (double)xv;
  const double s = __ddiv_rn(__dsub_rn(x, pred), two_eb);
  if (fabs(s) < (double)center + 1.0) {
    const double kd = s >= 0.0 ? floor(__dadd_rn(s, 0.5)) : ceil(__dsub_rn(s, 0.5));
    const long long k = (long long)kd;
    if (k >= -(long long)(center - 1) && k <= (long long)(center - 1)) {
      const T r = Elem<T>::round(__dadd_rn(pred, __dmul_rn((double)k, two_eb)));
      if (fabs(__dsub_rn(x, (double)r)) <= eb) {
        r_out = r;
        return center + (int)k;
      }
    }
  }
  r_out = tr_e == kNoTrunc ? xv : trunc_value<T>(xv, tr_e);
  return 0;
}

// Block-wide exclusive scan of one u64 per thread (NT threads); returns the
// exclusive prefix and the block total.  s_warp needs NT/32 entries.
template <int NT>
__device__ __forceinline__ unsigned long long block_exscan_u64(unsigned long long v,
                                                               unsigned long long* s_warp,
                                                               unsigned long long& total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  unsigned long long x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long t = __shfl_up_sync(EBZ_FULL, x, o);
    if (lane >= o) x += t;
  }
  if (lane == 31) s_warp[w] = x;
  __syncthreads();
  if (w == 0) {
    unsigned long long y = lane < NT / 32 ? s_warp[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long t = __shfl_up_sync(EBZ_FULL, y, o);
      if (lane >= o) y += t;
    }
    if (lane < NT / 32) s_warp[lane] = y;
  }
  __syncthreads();
  const unsigned long long pre = w ? s_warp[w - 1] : 0;
  total = s_warp[NT / 32 - 1];
  __syncthreads();
  return pre + x - v;
}

// ------------------------------------------------------ internal interfaces
struct SweepArgs {
  int ndim;
  long long dims[4];
  long long n;
  long long nrows;          // n / dims[0]
  int layers;
  int m;
  int center;
  const Info* info;         // eb lives in info->eb
  Info* info_w;             // status / counters
  const void* values;       // compress input (T)
  void* recon;              // T[n] (compress: scratch / faces, decompress: output)
  void* codes;              // u8 (m <= 8) or u16
  unsigned long long* hist; // compress: u64[2^m]
  const void* unpred;       // decompress
  unsigned long long n_unpred;
  const unsigned long long* rowbase;  // decompress: zero rank per row (within block)
  const unsigned long long* rowblk;   // ... + block prefix rowblk[row >> 8]
  // fast 2D/3D kernels: tagged patch-face buffers (see kTagBits)
  unsigned long long* yface;
  unsigned long long* zface;
  unsigned long long* progress;       // per task, epoch-tagged
  unsigned int* ticket;
  unsigned int epoch;
  // stencil bank (generic kernel)
  const long long* deltas;
  const double* coeffs;
  const long long* starts;
  const long long* counts;
  int wide;                 // u16 codes (m > 8, or forced: batched interval trials)
  int trunc;                // compress: truncated-mantissa unpredictable values (opt-in)
  unsigned jitter;          // test hook (EBZ_SCHED_JITTER): random per-chunk delays, ns
};
// Schedule perturbation (test hook): a warp sleeps up to `jitter` ns at one
// chunk in four, chosen by a hash of (ticket, chunk), so producers and
// consumers of the tagged faces meet in orders the normal schedule never
// produces; the outputs must not change (tests/test_gpu_stress.py).
__device__ __forceinline__ void sched_jitter(unsigned jitter, unsigned tk, int k) {
#ifdef EBZ_NO_JITTER_HOOK
  return;
#endif
  if (!jitter) return;
  unsigned h = tk * 0x9E3779B1u ^ (unsigned)k * 0x85EBCA77u;
  h ^= h >> 15;
  h *= 0x2C1B3C6Du;
  h ^= h >> 12;
  if ((h & 3u) == 0) __nanosleep(h % jitter);
}

// launchers (return cudaError_t).  *_batch launchers run one grid over up to
// kBatchMax fields of one geometry; per-field pointers travel as a
// __grid_constant__ kernel-parameter table.
constexpr int kBatchMax = 64;

// Patch-face words of the fast sweeps: the binary64 bit pattern of a
// reconstruction (always an exact float32 value, so its low 29 mantissa bits
// are zero) OR-ed with the launch's epoch in those 29 bits.  Consumers accept
// a word whose low bits equal their epoch and mask them off -- no float
// conversion on either side.  Epochs run in [1, kEpochMax] (0 = fresh memory).
constexpr unsigned kTagBits = 29;
constexpr unsigned kTagMask = (1u << kTagBits) - 1;
constexpr unsigned kEpochMax = kTagMask;
cudaError_t launch_range(const void* values, int width, long long n, int has_abs, double abs_b,
                         int has_rel, double rel_b, Info* info, unsigned int* scratch,
                         cudaStream_t s);
// also initialises each field's record (and zeroes its histogram when given)
cudaError_t launch_range_batch(const void* const* values, Info* const* infos,
                               unsigned int* const* scratch, unsigned long long* const* hists,
                               int nsym, int nf, int width, long long n, int has_abs,
                               double abs_b, int has_rel, double rel_b, cudaStream_t s);
cudaError_t launch_code_hist_batch(const void* const* codes, unsigned long long* const* hist,
                                   int nf, int m, long long n, int sms, cudaStream_t s);
cudaError_t launch_huffman_batch(const unsigned long long* const* hist, Info* const* info,
                                 uint8_t* const* lengths, unsigned long long* const* words,
                                 unsigned long long* const* scratch, int nf, int m,
                                 cudaStream_t s);
// encoder, per field: codes -> (count, scan + header, pack + verbatim gather)
struct EncodeJob {
  const void* codes;
  const uint8_t* lengths;
  const unsigned long long* words;
  unsigned long long* agg;     // 2 u64 per 4096-code chunk
  Info* info;
  uint8_t* bits;
  size_t bits_cap;
  uint8_t* head;               // container header + length table
  const void* values;          // code-0 values are gathered from here
  void* unpred;                // verbatim output (nullptr: skip the gather)
  int trunc;                   // gather trunc(value) (opt-in extension)
};
cudaError_t launch_encode_batch(const EncodeJob* jobs, int nf, int m, long long n, int width,
                                int ndim, const long long* dims, int layers, int sms,
                                cudaStream_t s);
size_t encode_pack_smem(int m, int width);
bool sweep_fast_supported(int ndim, int layers, long long dims0);
void fast_task_table(int npy, int npz, unsigned int* out, int wy, int wz);
bool sweep_r2_used(int ndim, int layers, bool compress);
void fast_patch_grid(int ndim, const long long* dims, int layers, bool compress, int* npy,
                     int* npz);
void fast_face_words(int ndim, const long long* dims, int layers, bool compress,
                     long long* ny_words, long long* nz_words);
// Per-field pointers of a batched fast sweep (all fields share one geometry).
// Passed by value as a __grid_constant__ kernel parameter (<= 4.6 KB).
struct FieldRef {
  const void* values;               // compress input
  void* recon;                      // decompress output
  void* codes;
  const void* unpred;               // decompress verbatim values
  const unsigned long long* rowbase;
  const unsigned long long* rowblk;
  unsigned long long* yface;
  unsigned long long* zface;
  Info* info;                       // eb, K, status, used
  unsigned long long* hist;         // compress: histogram the sweep fills, or null
};
struct FieldTable {
  FieldRef f[kBatchMax];
  int center[kBatchMax];            // compress: field's 2^(m-1) (interval trials), 0 = launch's
};
// One launch sweeps nf fields (geometry, m, ticket and epoch from `a`; the
// field pointers of `a` are ignored).  Tickets interleave the fields.
// 3D, n = 1, float32 compress / decompress with z-rows per lane (sweep3.cu): 32 x 4 patches
bool sweep3_used(int ndim, int layers, int width, const long long* dims, int nf, bool compress);
int sweep3_model_choice(const long long* dims, int nf);  // 0 two-row, 1 sweep3c, 2 sweep3b
void sweep3_patch_grid(const long long* dims, int* npy, int* npz);
void sweep3_face_words(const long long* dims, long long* ny_words, long long* nz_words);
cudaError_t launch_sweep3(const SweepArgs& a, const FieldTable& ft, int nf,
                          const unsigned int* d_tasks, int npy, int npz, bool compress, bool rec,
                          int sms, cudaStream_t s);
// 3D, n = 1, binary64: patch wavefront with 16-byte face words (sweep3b.cu)
bool sweep3b_used(int ndim, int layers, int width, const long long* dims, int nf, bool compress,
                  bool rec, bool trunc);
void sweep3b_face_words(const long long* dims, long long* ny_words, long long* nz_words);
cudaError_t launch_sweep3b(const SweepArgs& a, const FieldTable& ft, int nf,
                           const unsigned int* d_tasks, int npy, int npz, bool compress, int width,
                           int sms, cudaStream_t s);
// 2D, n = 1, 2, float32 / binary64: the low-latency block-speculative kernel (sweep2.cu)
bool sweep2_used(int ndim, int layers, int width, const long long* dims, bool rec, bool trunc);
cudaError_t launch_sweep2(const SweepArgs& a, const FieldTable& ft, int nf,
                          const unsigned int* d_tasks, int npy, bool compress, int width, int sms,
                          cudaStream_t s);
// rec (compress only): also store every point's reconstruction in FieldRef::recon.
cudaError_t launch_sweep_fast(const SweepArgs& a, const FieldTable& ft, int nf,
                              const unsigned int* d_tasks, int npy, int npz, bool compress,
                              bool rec, int sms, cudaStream_t s);
cudaError_t launch_huffman_build(const unsigned long long* hist, int m, Info* info,
                                 uint8_t* lengths, unsigned long long* words,
                                 unsigned long long* scratch, size_t scratch_bytes,
                                 cudaStream_t s);
cudaError_t launch_finite(const void* values, int width, long long n, Info* info, cudaStream_t s);
cudaError_t launch_sweep_generic(const SweepArgs& a, int width, bool compress, int sms,
                                 cudaStream_t s);
constexpr int kEncodeChunk = 4096;
// decoder, per field (record init, tables, sync, repair x2, verify, scan,
// write, serial fallback)
struct DecodeJob {
  const uint8_t* bits;
  long long nbytes;                      // budget, or capacity when dev_bitlen is set
  const uint8_t* lengths;
  void* codes;                           // output symbols
  Info* info;                            // decompress record (initialised here)
  unsigned long long* scratch;           // decode_scratch_bytes(nbytes, m)
  const unsigned long long* dev_bitlen;  // exact budget on the device, or nullptr
  const Info* src;                       // eb / K from this record, or ...
  double eb;                             // ... from the host
  unsigned long long k;
};
cudaError_t launch_decode_batch(const DecodeJob* jobs, int nf, int m, long long n, int sms,
                                cudaStream_t s);
cudaError_t launch_rowbase_batch(const void* const* codes, unsigned long long* const* rowbase,
                                 unsigned long long* const* rowblk, Info* const* info, int nf,
                                 int m, long long n, long long nx, cudaStream_t s);
cudaError_t launch_decode(const uint8_t* bits, long long nbytes, const uint8_t* lengths, int m,
                          long long n, void* codes, Info* info, unsigned long long* scratch,
                          size_t scratch_bytes, int sms, cudaStream_t s,
                          const unsigned long long* dev_bitlen);
size_t rowblk_words(long long nrows);
cudaError_t launch_rowbase(const void* codes, int m, long long n, long long nx,
                           unsigned long long* rowbase, unsigned long long* tmp,
                           unsigned long long n_unpred, Info* info, cudaStream_t s);
size_t decode_scratch_bytes(long long nbytes, int m);
size_t huffman_scratch_bytes(int m);
cudaError_t launch_code_hist(const void* codes, int m, long long n, unsigned long long* hist,
                             int sms, cudaStream_t s);
// batched interval trials: zero-code counts of u16 code arrays, u16 -> u8 narrowing
// truncated-mantissa block (trunc.cu, opt-in extension)
size_t tr_scratch_bytes(unsigned long long k);
cudaError_t launch_tr_pack(const void* values, int width, unsigned long long k, double eb,
                           uint8_t* bytes, unsigned long long* scratch, cudaStream_t s,
                           bool count_only);
cudaError_t launch_tr_unpack(const uint8_t* bytes, int width, unsigned long long k, double eb,
                             void* values, unsigned long long* scratch, cudaStream_t s);
cudaError_t launch_zero_count_batch(const uint16_t* const* codes, unsigned long long* const* k,
                                    int nf, long long n, int sms, cudaStream_t s);
cudaError_t launch_narrow_codes(const uint16_t* in, uint8_t* out, long long n, int sms,
                                cudaStream_t s);
// analysis (analysis.cu)
cudaError_t launch_original_hits(const void* values, int width, int ndim, const long long* dims,
                                 int layers, double bound, const long long* deltas,
                                 const double* coeffs, const long long* starts,
                                 const long long* counts, unsigned long long* out, int sms,
                                 cudaStream_t s);
size_t metrics_scratch_bytes(int lags);
cudaError_t launch_metrics(const void* a, const void* b, int width, long long n, int lags,
                           double* scratch, double* out, cudaStream_t s);
// Per-device launch attributes of one kernel.  cudaFuncSetAttribute (the
// dynamic shared-memory limit) applies to the calling thread's current
// device only, so the "already raised" record is kept per device, behind a
// mutex (one context per device may run on its own host thread, files.py).
constexpr int kMaxDevices = 64;
struct KernelAttr {
  std::mutex mu;
  size_t smem[kMaxDevices] = {};      // raised dynamic shared-memory limit
  size_t occ_smem[kMaxDevices] = {};  // occupancy cached for this smem size
  int occ[kMaxDevices] = {};
};
// Raise func's dynamic shared-memory limit to >= smem on the current device.
template <typename F>
inline cudaError_t kernel_smem(KernelAttr& k, F* func, size_t smem) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= kMaxDevices)
    return cudaFuncSetAttribute(reinterpret_cast<const void*>(func),
                                cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  std::lock_guard<std::mutex> g(k.mu);
  if (k.smem[dev] >= smem) return cudaSuccess;
  e = cudaFuncSetAttribute(reinterpret_cast<const void*>(func),
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e == cudaSuccess) k.smem[dev] = smem;
  return e;
}
// Resident blocks per SM of func at (threads, smem) on the current device (>= 1).
template <typename F>
inline int kernel_occupancy(KernelAttr& k, F* func, int threads, size_t smem) {
  int dev = 0;
  cudaGetDevice(&dev);
  const bool cache = dev >= 0 && dev < kMaxDevices;
  if (cache) {
    std::lock_guard<std::mutex> g(k.mu);
    if (k.occ_smem[dev] == smem && k.occ[dev] > 0) return k.occ[dev];
  }
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, func, threads, smem);
  if (per_sm < 1) per_sm = 1;
  if (cache) {
    std::lock_guard<std::mutex> g(k.mu);
    k.occ_smem[dev] = smem;
    k.occ[dev] = per_sm;
  }
  return per_sm;
}

// progress counters are spread 256 B apart (own L2 line / slice each)
constexpr int kProgPad = 32;
