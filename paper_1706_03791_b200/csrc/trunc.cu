// trunc.cu -- bit packing of truncated-mantissa unpredictable values: the
// opt-in extension named by north_star (3) ("truncated-mantissa binary-
// representation encoding"); the reference stores unpredictable values
// verbatim (ebzip/codec.py:119, core.py:19), so containers carrying this
// block are format version 2 and outside the parity claims.
//
// Value i (K values, scan order) keeps sign + biased exponent (HB = 9 bits
// for float32, 12 for float64) and the top k_i mantissa bits, where
// k_i = clamp(e(v_i) - e(eb), 0, M) is a function of the stored exponent and
// of the container's eb (ebz_common.cuh trunc_keep), so the reader recovers
// every length from the header fields alone:
//     bits [0, HB K)            header fields, HB bits each, MSB first
//     bits [HB K, HB K + sum k) mantissa fields, back to back
// padded with zero bits to a whole byte.
//
// Pack and unpack are three passes over chunks of 4096 values (count, one-CTA
// scan of the chunk totals, write); each chunk's header fields fill a
// word-aligned run (4096 x HB bits), its mantissa fields a run assembled in
// shared memory whose first and last words are OR-ed into the pre-zeroed
// output (they may be shared with the neighbouring chunks).
#include "ebz_common.cuh"

namespace {

constexpr int kTT = 256;                 // threads per chunk CTA
constexpr int kTPer = 16;                // values per thread
constexpr int kTChunk = kTT * kTPer;     // 4096

template <typename T> struct TrFmt {
  static constexpr int HB = TruncBits<T>::EW + 1;   // sign + exponent bits
  static constexpr int M = TruncBits<T>::M;
};

__device__ __forceinline__ unsigned bswap32(unsigned v) { return __byte_perm(v, 0, 0x0123); }

// big-endian 32-bit word w of a byte stream (4-byte aligned base, readable slack)
__device__ __forceinline__ unsigned long long be_word(const uint8_t* p, long long w) {
  return (unsigned long long)bswap32(reinterpret_cast<const unsigned*>(p)[w]);
}
// n <= 57 bits starting at bit position pos (MSB first)
__device__ __forceinline__ unsigned long long get_bits(const uint8_t* p, unsigned long long pos,
                                                       int n) {
  if (n == 0) return 0;
  const long long w = (long long)(pos >> 5);
  const int off = (int)(pos & 31);
  const unsigned long long hi = (be_word(p, w) << 32) | be_word(p, w + 1);
  const unsigned long long top = off ? (hi << off) | (be_word(p, w + 2) >> (32 - off)) : hi;
  return top >> (64 - n);
}
// OR an n-bit field (n <= 57) at bit position pos of a 32-bit-word window
// (word 0 = bit base); the words are MSB-first
__device__ __forceinline__ void or_bits(unsigned* win, unsigned long long pos,
                                        unsigned long long v, int n) {
  if (n == 0) return;
  const int w = (int)(pos >> 5), off = (int)(pos & 31);
  // the field occupies bits [off, off + n) of words w, w + 1, w + 2
  const int end = off + n;
  const unsigned long long x = v << (64 - n);  // MSB-aligned
  atomicOr(&win[w], (unsigned)(x >> (32 + off)));
  if (end > 32) atomicOr(&win[w + 1], (unsigned)(x >> off));
  if (end > 64) atomicOr(&win[w + 2], (unsigned)(x << (32 - off)));
}

struct TrJob {
  const void* values;      // pack: source values (K), unpack: destination
  uint8_t* bytes;          // pack: destination (zeroed), unpack: source
  unsigned long long k;    // number of values
  int e_eb;                // floor(log2 eb)
  unsigned long long* sums;  // per chunk: mantissa bits, then exclusive offsets
  unsigned long long* total; // [0] mantissa bits, [1] total bits
};

template <typename T>
__device__ __forceinline__ int keep_of(T v, int e_eb) {
  return trunc_keep<T>(TruncBits<T>::bits(v), e_eb);
}
// k from a stored header field (sign | biased exponent)
template <typename T>
__device__ __forceinline__ int keep_of_field(unsigned h, int e_eb) {
  typedef TruncBits<T> TB;
  const typename TB::U b = (typename TB::U)(h & ((1u << TB::EW) - 1u)) << TB::M;
  return trunc_keep<T>(b, e_eb);
}

// pass 1 (pack): mantissa bits per chunk
template <typename T>
__global__ void __launch_bounds__(kTT) tr_count_kernel(TrJob j) {
  const T* __restrict__ v = reinterpret_cast<const T*>(j.values);
  const unsigned long long i0 = (unsigned long long)blockIdx.x * kTChunk + threadIdx.x * kTPer;
  unsigned s = 0;
#pragma unroll
  for (int q = 0; q < kTPer; ++q)
    if (i0 + q < j.k) s += (unsigned)keep_of<T>(v[i0 + q], j.e_eb);
  __shared__ unsigned long long sw[kTT / 32];
  unsigned long long t;
  block_exscan_u64<kTT>(s, sw, t);
  if (threadIdx.x == 0) j.sums[blockIdx.x] = t;
}

// pass 1 (unpack): mantissa bits per chunk from the header fields
template <typename T>
__global__ void __launch_bounds__(kTT) tr_ucount_kernel(TrJob j) {
  constexpr int HB = TrFmt<T>::HB;
  const unsigned long long i0 = (unsigned long long)blockIdx.x * kTChunk + threadIdx.x * kTPer;
  unsigned s = 0;
#pragma unroll
  for (int q = 0; q < kTPer; ++q)
    if (i0 + q < j.k)
      s += (unsigned)keep_of_field<T>((unsigned)get_bits(j.bytes, (i0 + q) * HB, HB), j.e_eb);
  __shared__ unsigned long long sw[kTT / 32];
  unsigned long long t;
  block_exscan_u64<kTT>(s, sw, t);
  if (threadIdx.x == 0) j.sums[blockIdx.x] = t;
}

// pass 2: one CTA, exclusive scan of the chunk totals, grand totals
__global__ void __launch_bounds__(1024) tr_scan_kernel(TrJob j, long long nchunks, int hb) {
  __shared__ unsigned long long sw[32];
  unsigned long long run = 0;
  for (long long c0 = 0; c0 < nchunks; c0 += 1024) {
    const long long c = c0 + threadIdx.x;
    const unsigned long long v = c < nchunks ? j.sums[c] : 0ull;
    unsigned long long t;
    const unsigned long long ex = block_exscan_u64<1024>(v, sw, t);
    if (c < nchunks) j.sums[c] = run + ex;
    run += t;
  }
  if (threadIdx.x == 0) {
    j.total[0] = run;
    j.total[1] = (unsigned long long)hb * j.k + run;
  }
}

// pass 3 (pack): header fields and mantissa fields of one chunk
template <typename T>
__global__ void __launch_bounds__(kTT) tr_pack_kernel(TrJob j) {
  typedef TruncBits<T> TB;
  constexpr int HB = TrFmt<T>::HB, M = TB::M;
  constexpr int AW = kTChunk * HB / 32;               // header words per full chunk
  constexpr int BW = kTChunk * M / 32 + 3;            // mantissa window words
  __shared__ unsigned s_a[AW + 2];
  __shared__ unsigned s_b[BW];
  const T* __restrict__ v = reinterpret_cast<const T*>(j.values);
  unsigned* out = reinterpret_cast<unsigned*>(j.bytes);
  const unsigned long long c0 = (unsigned long long)blockIdx.x * kTChunk;
  const unsigned long long i0 = c0 + threadIdx.x * kTPer;
  for (int i = threadIdx.x; i < AW + 2; i += kTT) s_a[i] = 0u;
  for (int i = threadIdx.x; i < BW; i += kTT) s_b[i] = 0u;
  typename TB::U b[kTPer];
  int kk[kTPer];
  unsigned s = 0;
#pragma unroll
  for (int q = 0; q < kTPer; ++q) {
    b[q] = i0 + q < j.k ? TB::bits(v[i0 + q]) : (typename TB::U)0;
    kk[q] = i0 + q < j.k ? trunc_keep<T>(b[q], j.e_eb) : 0;
    s += (unsigned)kk[q];
  }
  __shared__ unsigned long long sw[kTT / 32];
  unsigned long long tot;
  const unsigned long long ex = block_exscan_u64<kTT>(s, sw, tot);  // also a barrier
  // mantissa run of the chunk: bits [B0, B0 + tot), B0 = HB K + chunk offset
  const unsigned long long B0 = (unsigned long long)HB * j.k + j.sums[blockIdx.x];
  const int bshift = (int)(B0 & 31);
  unsigned long long pos = ex + (unsigned long long)bshift;  // within the window
#pragma unroll
  for (int q = 0; q < kTPer; ++q) {
    if (i0 + q >= j.k) break;
    const unsigned h = (unsigned)(b[q] >> M);  // sign | biased exponent
    or_bits(s_a, (unsigned long long)(threadIdx.x * kTPer + q) * HB, h, HB);
    const unsigned long long mant = (unsigned long long)(b[q] & (((typename TB::U)1 << M) - 1));
    or_bits(s_b, pos, mant >> (M - kk[q]), kk[q]);
    pos += (unsigned long long)kk[q];
  }
  __syncthreads();
  // header run: word aligned (chunk start c0 HB is a multiple of 32); its
  // last word may be shared with the mantissa run (last chunk only)
  const unsigned long long nvals = j.k - c0 < (unsigned long long)kTChunk ? j.k - c0 : kTChunk;
  const long long aw0 = (long long)(c0 * HB / 32);
  const int an = (int)((nvals * HB + 31) / 32);
  const bool a_tail_shared = ((nvals * HB) & 31) != 0;
  for (int i = threadIdx.x; i < an; i += kTT) {
    const unsigned w = bswap32(s_a[i]);
    if (i == an - 1 && a_tail_shared) atomicOr(&out[aw0 + i], w);
    else out[aw0 + i] = w;
  }
  // mantissa run: first / last words may be shared with the neighbours
  if (tot) {
    const long long bw0 = (long long)(B0 >> 5);
    const int bn = (int)((bshift + tot + 31) / 32);
    const bool head = bshift != 0, tail = ((bshift + tot) & 31) != 0;
    for (int i = threadIdx.x; i < bn; i += kTT) {
      const unsigned w = bswap32(s_b[i]);
      if ((i == 0 && head) || (i == bn - 1 && tail)) atomicOr(&out[bw0 + i], w);
      else out[bw0 + i] = w;
    }
  }
}

// pass 3 (unpack): rebuild the values of one chunk
template <typename T>
__global__ void __launch_bounds__(kTT) tr_unpack_kernel(TrJob j) {
  typedef TruncBits<T> TB;
  typedef typename TB::U U;
  constexpr int HB = TrFmt<T>::HB, M = TB::M;
  T* __restrict__ v = reinterpret_cast<T*>(const_cast<void*>(j.values));
  const unsigned long long i0 = (unsigned long long)blockIdx.x * kTChunk + threadIdx.x * kTPer;
  unsigned h[kTPer];
  int kk[kTPer];
  unsigned s = 0;
#pragma unroll
  for (int q = 0; q < kTPer; ++q) {
    h[q] = i0 + q < j.k ? (unsigned)get_bits(j.bytes, (i0 + q) * HB, HB) : 0u;
    kk[q] = i0 + q < j.k ? keep_of_field<T>(h[q], j.e_eb) : 0;
    s += (unsigned)kk[q];
  }
  __shared__ unsigned long long sw[kTT / 32];
  unsigned long long tot;
  const unsigned long long ex = block_exscan_u64<kTT>(s, sw, tot);
  unsigned long long pos = (unsigned long long)HB * j.k + j.sums[blockIdx.x] + ex;
#pragma unroll
  for (int q = 0; q < kTPer; ++q) {
    if (i0 + q >= j.k) break;
    const U mant = (U)get_bits(j.bytes, pos, kk[q]) << (M - kk[q]);
    v[i0 + q] = TB::from(((U)h[q] << M) | mant);
    pos += (unsigned long long)kk[q];
  }
}

}  // namespace

size_t tr_scratch_bytes(unsigned long long k) {
  return (size_t)((k + kTChunk - 1) / kTChunk + 2) * 8 + 16;
}

// Pack K values (device) into the zeroed byte buffer; total bits -> tot[1]
// (tot[0] = mantissa bits).  scratch: tr_scratch_bytes(K).
cudaError_t launch_tr_pack(const void* values, int width, unsigned long long k, double eb,
                           uint8_t* bytes, unsigned long long* scratch, cudaStream_t s,
                           bool count_only) {
  const long long nchunks = (long long)((k + kTChunk - 1) / kTChunk);
  TrJob j;
  j.values = values;
  j.bytes = bytes;
  j.k = k;
  j.e_eb = eb_exponent(eb);
  j.total = scratch;
  j.sums = scratch + 2;
  if (nchunks == 0) return cudaMemsetAsync(scratch, 0, 16, s);
  if (width == 64) tr_count_kernel<double><<<(unsigned)nchunks, kTT, 0, s>>>(j);
  else tr_count_kernel<float><<<(unsigned)nchunks, kTT, 0, s>>>(j);
  tr_scan_kernel<<<1, 1024, 0, s>>>(j, nchunks, width == 64 ? TrFmt<double>::HB : TrFmt<float>::HB);
  if (count_only) return cudaGetLastError();
  if (width == 64) tr_pack_kernel<double><<<(unsigned)nchunks, kTT, 0, s>>>(j);
  else tr_pack_kernel<float><<<(unsigned)nchunks, kTT, 0, s>>>(j);
  return cudaGetLastError();
}

// Unpack K values from the byte buffer (with >= 12 readable slack bytes);
// total bits -> tot[1] (the caller checks it against the buffer size).
cudaError_t launch_tr_unpack(const uint8_t* bytes, int width, unsigned long long k, double eb,
                             void* values, unsigned long long* scratch, cudaStream_t s) {
  const long long nchunks = (long long)((k + kTChunk - 1) / kTChunk);
  TrJob j;
  j.values = values;
  j.bytes = const_cast<uint8_t*>(bytes);
  j.k = k;
  j.e_eb = eb_exponent(eb);
  j.total = scratch;
  j.sums = scratch + 2;
  if (nchunks == 0) return cudaMemsetAsync(scratch, 0, 16, s);
  if (width == 64) tr_ucount_kernel<double><<<(unsigned)nchunks, kTT, 0, s>>>(j);
  else tr_ucount_kernel<float><<<(unsigned)nchunks, kTT, 0, s>>>(j);
  tr_scan_kernel<<<1, 1024, 0, s>>>(j, nchunks, width == 64 ? TrFmt<double>::HB : TrFmt<float>::HB);
  if (width == 64) tr_unpack_kernel<double><<<(unsigned)nchunks, kTT, 0, s>>>(j);
  else tr_unpack_kernel<float><<<(unsigned)nchunks, kTT, 0, s>>>(j);
  return cudaGetLastError();
}
