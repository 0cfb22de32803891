// encode.cu -- canonical-Huffman encoder + unpredictable-value compaction.
//
// Replaces entropy.encode / pack_bits (ebzip/entropy.py:139-157,
// _kernels.py:124-148) and the boolean gather values[codes == 0]
// (codec.py:119).  Output bytes are identical: codewords MSB-first, back to
// back, last byte zero-padded; verbatim values in scan order.
//
// Three passes over the code array (1 byte per point for m <= 8):
//   count : per 4096-symbol chunk, sum of code lengths and number of zeros;
//   scan  : one CTA, exclusive scan of the (bits, zeros) pairs, totals into
//           EbzInfo, zero the first output word of every chunk (the only
//           words two CTAs may share), write the container header + table;
//   pack  : per chunk, CTA-local exclusive scan of per-thread bit counts;
//           each thread runs a bit writer over its 16 codes into a shared
//           word window (words it owns stored plainly, its two boundary
//           words OR-ed), the window leaves with coalesced stores (atomicOr
//           for the two words shared with neighbour chunks); chunks above 16
//           bits/code write to global memory directly.  The chunk's code-0
//           values are written to their scan-order slots.
#include "ebz_common.cuh"

namespace {

constexpr int kThreads = 256;
constexpr int kPer = 16;                       // codes per thread
constexpr int kChunk = kThreads * kPer;        // 4096 symbols per chunk
constexpr int kTableSmemMaxM = 12;
static_assert(kChunk == kEncodeChunk, "chunk size shared with the host");

struct EncTab {  // per-field pointers of a batched launch (blockIdx.y / .x = field)
  const void* codes[kBatchMax];
  const uint8_t* lengths[kBatchMax];
  const unsigned long long* words[kBatchMax];
  unsigned long long* agg[kBatchMax];
  Info* info[kBatchMax];
  uint8_t* bits[kBatchMax];
  size_t bits_cap[kBatchMax];
  uint8_t* head[kBatchMax];
  const void* values[kBatchMax];
  void* unpred[kBatchMax];
  int trunc[kBatchMax];  // gather trunc(value): the opt-in truncated-mantissa coding
};

template <typename C>
__device__ __forceinline__ void load16(const C* codes, long long i0, long long n, int* out) {
  if (i0 + kPer <= n && (((uintptr_t)(codes + i0)) & 15) == 0) {
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

// exact number of zero bytes / zero 16-bit halves of a 64-bit word
__device__ __forceinline__ unsigned zero_bytes64(unsigned long long v) {
  const unsigned long long t = (v & 0x7f7f7f7f7f7f7f7full) + 0x7f7f7f7f7f7f7f7full;
  return 8u - (unsigned)__popcll((t | v) & 0x8080808080808080ull);
}
__device__ __forceinline__ unsigned zero_halves64(unsigned long long v) {
  const unsigned long long t = (v & 0x7fff7fff7fff7fffull) + 0x7fff7fff7fff7fffull;
  return 4u - (unsigned)__popcll((t | v) & 0x8000800080008000ull);
}

// Fast code extraction of one full, 16-byte aligned group of 16 codes:
// codes (table index; u8 codes index a 256-entry zero-padded table, u16
// codes are masked to the alphabet) and the number of zero codes.
template <typename C>
__device__ __forceinline__ unsigned group16(const C* __restrict__ codes, long long i0, int mask,
                                            int (&c)[kPer]) {
  if (sizeof(C) == 1) {
    const uint4 v = __ldcs(reinterpret_cast<const uint4*>(codes + i0));
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int j = 0; j < 16; ++j) c[j] = (int)((w[j >> 2] >> (8 * (j & 3))) & 0xffu);
    return zero_bytes64(((unsigned long long)v.y << 32) | v.x) +
           zero_bytes64(((unsigned long long)v.w << 32) | v.z);
  } else {
    const uint4 v0 = __ldcs(reinterpret_cast<const uint4*>(codes + i0));
    const uint4 v1 = __ldcs(reinterpret_cast<const uint4*>(codes + i0) + 1);
    const uint32_t w[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
#pragma unroll
    for (int j = 0; j < 16; ++j) c[j] = (int)((w[j >> 1] >> (16 * (j & 1))) & 0xffffu) & mask;
    return zero_halves64(((unsigned long long)v0.y << 32) | v0.x) +
           zero_halves64(((unsigned long long)v0.w << 32) | v0.z) +
           zero_halves64(((unsigned long long)v1.y << 32) | v1.x) +
           zero_halves64(((unsigned long long)v1.w << 32) | v1.z);
  }
}

// group16 on already loaded words (v0; u16 codes also v1)
template <typename C>
__device__ __forceinline__ unsigned extract16(const uint4& v0, const uint4& v1, int mask,
                                              int (&c)[kPer]) {
  if (sizeof(C) == 1) {
    const uint32_t w[4] = {v0.x, v0.y, v0.z, v0.w};
#pragma unroll
    for (int j = 0; j < 16; ++j) c[j] = (int)((w[j >> 2] >> (8 * (j & 3))) & 0xffu);
    return zero_bytes64(((unsigned long long)v0.y << 32) | v0.x) +
           zero_bytes64(((unsigned long long)v0.w << 32) | v0.z);
  } else {
    const uint32_t w[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
#pragma unroll
    for (int j = 0; j < 16; ++j) c[j] = (int)((w[j >> 1] >> (16 * (j & 1))) & 0xffffu) & mask;
    return zero_halves64(((unsigned long long)v0.y << 32) | v0.x) +
           zero_halves64(((unsigned long long)v0.w << 32) | v0.z) +
           zero_halves64(((unsigned long long)v1.y << 32) | v1.x) +
           zero_halves64(((unsigned long long)v1.w << 32) | v1.z);
  }
}

// table entries held in shared memory: 2^m, padded to 256 for u8 codes so a
// stray byte code (a skipped field's scratch) reads a zero length
__device__ __forceinline__ int table_size(int m) { return m < 8 ? 256 : 1 << m; }

// Persistent: one warp per 4096-code chunk at a time (8 independent 16-code
// loads in flight per lane), the length table loaded once per block.
template <typename C>
__global__ void __launch_bounds__(kThreads)
encode_count_kernel(const __grid_constant__ EncTab tab, long long n, int m) {
  const C* __restrict__ codes = reinterpret_cast<const C*>(tab.codes[blockIdx.y]);
  const uint8_t* __restrict__ lengths = tab.lengths[blockIdx.y];
  unsigned long long* __restrict__ agg = tab.agg[blockIdx.y];
  __shared__ uint8_t s_len[1 << kTableSmemMaxM];
  const bool smem = m <= kTableSmemMaxM;
  const int nsym = 1 << m, mask = nsym - 1;
  if (smem)
    for (int i = threadIdx.x; i < table_size(m); i += kThreads)
      s_len[i] = i < nsym ? lengths[i] : 0;
  __syncthreads();
  const bool aligned = (((uintptr_t)codes) & 15) == 0;
  const int lane = threadIdx.x & 31;
  const long long nchunks = (n + kChunk - 1) / kChunk;
  const long long w0 = (long long)blockIdx.x * (kThreads / 32) + (threadIdx.x >> 5);
  const long long ws = (long long)gridDim.x * (kThreads / 32);
  for (long long chunk = w0; chunk < nchunks; chunk += ws) {
    unsigned bits = 0, zeros = 0;  // <= 4096 * 64 bits per chunk
    if (smem && aligned && (chunk + 1) * kChunk <= n) {
#pragma unroll 4
      for (int q = 0; q < kChunk / (32 * kPer); ++q) {
        int c[kPer];
        zeros += group16<C>(codes, chunk * kChunk + q * (32 * kPer) + lane * kPer, mask, c);
#pragma unroll
        for (int j = 0; j < kPer; ++j) bits += s_len[c[j]];
      }
    } else {
      for (int q = 0; q < kChunk / (32 * kPer); ++q) {
        int c[kPer];
        load16<C>(codes, chunk * kChunk + q * (32 * kPer) + lane * kPer, n, c);
#pragma unroll
        for (int j = 0; j < kPer; ++j) {
          c[j] &= (c[j] >> 31) | mask;  // stray codes stay in range; -1 = past n
          if (c[j] >= 0) {
            bits += smem ? s_len[c[j]] : __ldg(lengths + c[j]);
            zeros += c[j] == 0;
          }
        }
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      bits += __shfl_xor_sync(EBZ_FULL, bits, o);
      zeros += __shfl_xor_sync(EBZ_FULL, zeros, o);
    }
    if (lane == 0) {
      agg[2 * chunk] = bits;
      agg[2 * chunk + 1] = zeros;
    }
  }
}

// single CTA: exclusive scan of (bits, zeros) over nchunks + header
__global__ void __launch_bounds__(1024)
encode_scan_kernel(const __grid_constant__ EncTab tab, long long nchunks, int width, int ndim,
                   const unsigned long long dims0, const unsigned long long dims1,
                   const unsigned long long dims2, const unsigned long long dims3, int m,
                   int layers) {
  const int f = blockIdx.x;
  unsigned long long* __restrict__ agg = tab.agg[f];
  Info* info = tab.info[f];
  uint32_t* __restrict__ bits_words = reinterpret_cast<uint32_t*>(tab.bits[f]);
  const size_t bits_cap = tab.bits_cap[f];
  uint8_t* __restrict__ head = tab.head[f];
  const uint8_t* __restrict__ lengths = tab.lengths[f];
  __shared__ unsigned long long s_b[1024], s_z[1024];
  const long long per = (nchunks + 1023) / 1024;
  const long long lo = threadIdx.x * per;
  const long long hi = lo + per < nchunks ? lo + per : nchunks;
  unsigned long long b = 0, z = 0;
  for (long long i = lo; i < hi; ++i) {
    b += agg[2 * i];
    z += agg[2 * i + 1];
  }
  s_b[threadIdx.x] = b;
  s_z[threadIdx.x] = z;
  __syncthreads();
  // Hillis-Steele inclusive scan over 1024 partials
  for (int o = 1; o < 1024; o <<= 1) {
    unsigned long long tb = 0, tz = 0;
    if ((int)threadIdx.x >= o) {
      tb = s_b[threadIdx.x - o];
      tz = s_z[threadIdx.x - o];
    }
    __syncthreads();
    s_b[threadIdx.x] += tb;
    s_z[threadIdx.x] += tz;
    __syncthreads();
  }
  unsigned long long rb = threadIdx.x ? s_b[threadIdx.x - 1] : 0;
  unsigned long long rz = threadIdx.x ? s_z[threadIdx.x - 1] : 0;
  const unsigned long long total_bits = s_b[1023], total_z = s_z[1023];
  const bool fits = (total_bits + 7) / 8 + 8 <= bits_cap;
  for (long long i = lo; i < hi; ++i) {
    const unsigned long long cb = agg[2 * i], cz = agg[2 * i + 1];
    agg[2 * i] = rb;
    agg[2 * i + 1] = rz;
    if (fits) bits_words[rb >> 5] = 0u;  // shared boundary word of chunk i
    rb += cb;
    rz += cz;
  }
  if (fits && threadIdx.x == 0) bits_words[total_bits >> 5] = 0u;
  const int hsz = 36 + 8 * ndim;
  for (int i = threadIdx.x; i < (1 << m); i += 1024) head[hsz + i] = lengths[i];
  if (threadIdx.x == 0) {
    info->bit_length = total_bits;
    info->n_unpred = total_z;
    info->total_bytes = (unsigned long long)hsz + (1ull << m) + (total_bits + 7) / 8 +
                        total_z * (unsigned long long)(width / 8);
    if (!fits) atomicOr(&info->status, ST_CAPACITY);
    // header (ebzip/core.py:295-316), little-endian
    head[0] = 'E'; head[1] = 'B'; head[2] = 'Z'; head[3] = '1';
    head[4] = 1;
    head[5] = width == 64 ? 1 : 0;
    head[6] = (uint8_t)ndim;
    head[7] = (uint8_t)m;
    head[8] = (uint8_t)layers;
    head[9] = head[10] = head[11] = 0;
    const unsigned long long dd[4] = {dims0, dims1, dims2, dims3};
    int p = 12;
    for (int a = 0; a < ndim; ++a)
      for (int k = 0; k < 8; ++k) head[p++] = (uint8_t)(dd[a] >> (8 * k));
    const unsigned long long ebits = (unsigned long long)__double_as_longlong(info->eb);
    for (int k = 0; k < 8; ++k) head[p++] = (uint8_t)(ebits >> (8 * k));
    for (int k = 0; k < 8; ++k) head[p++] = (uint8_t)(total_z >> (8 * k));
    for (int k = 0; k < 8; ++k) head[p++] = (uint8_t)(total_bits >> (8 * k));
  }
}

__device__ __forceinline__ uint32_t bswap32(uint32_t v) { return __byte_perm(v, 0, 0x0123); }

// Shared output window per chunk: enough for 16 bits per code on average.
// Chunks above that (rare: long codes for rare symbols) write straight to
// global memory instead.
constexpr int kWinWords = kChunk * 16 / 32 + 2;

template <typename C, typename T>
__global__ void __launch_bounds__(kThreads)
encode_pack_kernel(const __grid_constant__ EncTab tab, long long n, int m) {
  const int f = blockIdx.y;
  const C* __restrict__ codes = reinterpret_cast<const C*>(tab.codes[f]);
  const uint8_t* __restrict__ lengths = tab.lengths[f];
  const unsigned long long* __restrict__ words = tab.words[f];
  const unsigned long long* __restrict__ agg = tab.agg[f];
  const Info* info = tab.info[f];
  uint32_t* __restrict__ out_words = reinterpret_cast<uint32_t*>(tab.bits[f]);
  const T* __restrict__ values = reinterpret_cast<const T*>(tab.values[f]);
  T* __restrict__ unpred_out = reinterpret_cast<T*>(tab.unpred[f]);
  if (info->status & ST_CAPACITY) return;
  // dynamic smem: [words 8 * T][lengths T][window][value staging], T =
  // table_size(m) entries (tables only for m <= 12)
  extern __shared__ __align__(16) unsigned char pk_smem[];
  const bool smem = m <= kTableSmemMaxM;
  const int nsym = 1 << m, mask = nsym - 1;
  const int tn = smem ? table_size(m) : 0;
  const int tsz = 9 * tn;
  unsigned long long* s_word = reinterpret_cast<unsigned long long*>(pk_smem);
  uint8_t* s_len = pk_smem + 8 * tn;
  uint32_t* s_win = reinterpret_cast<uint32_t*>(pk_smem + ((tsz + 15) & ~15));
  __shared__ unsigned int s_wsum[kThreads / 32];
  __shared__ unsigned int s_zsum[kThreads / 32];
  const long long chunk = blockIdx.x;
  const long long i0 = chunk * kChunk + (long long)threadIdx.x * kPer;
  // every global input of the chunk is requested before the table barrier,
  // so the code, aggregate and table latencies overlap (measured: the three
  // waited one after another, 16% of the stall samples)
  const bool fast_load = smem && (((uintptr_t)codes) & 15) == 0 && (chunk + 1) * kChunk <= n;
  uint4 raw0 = make_uint4(0, 0, 0, 0), raw1 = make_uint4(0, 0, 0, 0);
  if (fast_load) {
    raw0 = __ldcs(reinterpret_cast<const uint4*>(codes + i0));
    if (sizeof(C) == 2) raw1 = __ldcs(reinterpret_cast<const uint4*>(codes + i0) + 1);
  }
  const unsigned long long blk0 = agg[2 * chunk];
  const unsigned long long zoff = agg[2 * chunk + 1];
  int long_code = 0;
  for (int i = threadIdx.x; i < tn; i += kThreads) {
    const int l = i < nsym ? lengths[i] : 0;
    s_len[i] = (uint8_t)l;
    s_word[i] = i < nsym ? words[i] : 0ull;
    long_code |= l > 32;
  }
  // short codes (<= 32 bits, tables in smem): one-word accumulator writer
  const bool short_codes = smem && !__syncthreads_or(long_code);
  int c[kPer];
  unsigned bits = 0, zeros = 0;  // per thread <= 16 * 64 bits
  int L[kPer];
  if (fast_load) {
    // full aligned chunk: raw-word extraction, zero counts 8 at a time
    zeros = extract16<C>(raw0, raw1, mask, c);
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
      L[j] = s_len[c[j]];
      bits += L[j];
    }
  } else {
    load16<C>(codes, i0, n, c);
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
      c[j] &= (c[j] >> 31) | mask;  // stray codes stay in range; -1 = past n
      L[j] = c[j] >= 0 ? (smem ? s_len[c[j]] : __ldg(lengths + c[j])) : 0;
      bits += L[j];
      zeros += c[j] == 0;
    }
  }
  // CTA exclusive scan of (bits, zeros), 32-bit (a chunk holds < 2^19 bits)
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  unsigned ib = bits, iz = zeros;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned tb = __shfl_up_sync(EBZ_FULL, ib, o);
    const unsigned tz = __shfl_up_sync(EBZ_FULL, iz, o);
    if (lane >= o) {
      ib += tb;
      iz += tz;
    }
  }
  if (lane == 31) {
    s_wsum[wid] = ib;
    s_zsum[wid] = iz;
  }
  __syncthreads();
  unsigned wb = 0, blk_bits = 0;
  unsigned int wz = 0, blk_zeros = 0;
  for (int w = 0; w < kThreads / 32; ++w) {
    if (w < wid) {
      wb += s_wsum[w];
      wz += s_zsum[w];
    }
    blk_bits += s_wsum[w];
    blk_zeros += s_zsum[w];
  }
  const unsigned long long my_bits = blk0 + (wb + ib - bits);  // absolute
  const unsigned long long wbase = blk0 >> 5;                    // first output word
  const unsigned long long wlast = (blk0 + blk_bits + 31) >> 5;  // one past
  const int nwin = (int)(wlast - wbase);
  const bool head_shared = (blk0 & 31) != 0;
  const bool tail_shared = ((blk0 + blk_bits) & 31) != 0;
  const bool in_smem = nwin <= kWinWords;
  if (in_smem) {
    for (int i = threadIdx.x; i < nwin; i += kThreads) s_win[i] = 0u;
  } else {
    // global path: zero the words only this chunk touches (the shared
    // boundary words were zeroed by the scan)
    const long long lo = head_shared ? 1 : 0, hi = nwin - (tail_shared ? 1 : 0);
    for (long long i = lo + threadIdx.x; i < hi; i += kThreads) out_words[wbase + i] = 0u;
  }
  __syncthreads();
  // bit writer: whole words this thread owns are stored plainly; its first
  // word (if it starts mid-word) and its last partial word are OR-ed in
  unsigned long long wi = (my_bits >> 5) - wbase;
  int fill = (int)(my_bits & 31);
  bool lead = fill != 0;
  if (short_codes && in_smem) {
    // pending bits MSB-aligned in a 64-bit accumulator: fill < 32 before a
    // code and its length <= 32, so at most one word leaves per code
    unsigned long long acc = 0;
    auto append = [&](unsigned long long w, int len) {  // len <= 32, fill < 32
      if (len == 0) return;
      acc |= w << (64 - fill - len);
      fill += len;
      if (fill >= 32) {
        const uint32_t v = (uint32_t)(acc >> 32);
        if (lead) atomicOr(&s_win[wi], v);
        else s_win[wi] = v;
        lead = false;
        ++wi;
        acc <<= 32;
        fill -= 32;
      }
    };
    // groups of four codes whose total fits 32 bits are concatenated first
    // (one append instead of four)
#pragma unroll
    for (int j = 0; j < kPer; j += 4) {
      const int l4 = L[j] + L[j + 1] + L[j + 2] + L[j + 3];
      // zero-length entries (past the end: c = -1) contribute no bits
      const unsigned long long w0 = L[j] ? (uint32_t)s_word[c[j]] : 0u;
      const unsigned long long w1 = L[j + 1] ? (uint32_t)s_word[c[j + 1]] : 0u;
      const unsigned long long w2 = L[j + 2] ? (uint32_t)s_word[c[j + 2]] : 0u;
      const unsigned long long w3 = L[j + 3] ? (uint32_t)s_word[c[j + 3]] : 0u;
      if (l4 <= 32) {
        const unsigned long long w =
            (((((w0 << L[j + 1]) | w1) << L[j + 2]) | w2) << L[j + 3]) | w3;
        append(w, l4);
      } else {
        append(w0, L[j]);
        append(w1, L[j + 1]);
        append(w2, L[j + 2]);
        append(w3, L[j + 3]);
      }
    }
    if (fill > 0) atomicOr(&s_win[wi], (uint32_t)(acc >> 32));
    fill = 0;
  }
  uint32_t cur = 0;
  auto emit = [&](uint32_t v, bool shared) {
    if (in_smem) {
      if (shared) atomicOr(&s_win[wi], v);
      else s_win[wi] = v;
    } else {
      atomicOr(&out_words[wbase + wi], bswap32(v));
    }
  };
  if (!(short_codes && in_smem))
#pragma unroll
  for (int j = 0; j < kPer; ++j)
    if (c[j] >= 0) {
      int len = L[j];
      const unsigned long long w = smem ? s_word[c[j]] : __ldg(words + c[j]);
      while (len > 0) {
        const int take = len < 32 - fill ? len : 32 - fill;
        const uint32_t piece = (uint32_t)(w >> (len - take)) &
                               (take == 32 ? 0xffffffffu : ((1u << take) - 1u));
        cur |= piece << (32 - fill - take);
        fill += take;
        len -= take;
        if (fill == 32) {
          emit(cur, lead);
          lead = false;
          ++wi;
          cur = 0;
          fill = 0;
        }
      }
    }
  if (fill > 0) emit(cur, true);
  // verbatim values of code-0 points, scan order: compacted into shared
  // memory, then the chunk's contiguous slice leaves with coalesced stores
  if (unpred_out && zeros) {
    // (loaded here: issuing these loads before the scan raised the register
    // count past 4 blocks / SM, measured slower)
    T* s_val = reinterpret_cast<T*>(s_win + kWinWords);
    T v[kPer];
    const bool vec = i0 + kPer <= n && (((uintptr_t)values) & 15) == 0;
    if (vec && sizeof(T) == 4) {
#pragma unroll
      for (int q = 0; q < kPer / 4; ++q) {
        const float4 f = __ldcs(reinterpret_cast<const float4*>(values + i0) + q);
        v[4 * q] = (T)f.x; v[4 * q + 1] = (T)f.y; v[4 * q + 2] = (T)f.z; v[4 * q + 3] = (T)f.w;
      }
    } else if (vec) {
#pragma unroll
      for (int q = 0; q < kPer / 2; ++q) {
        const double2 f = __ldcs(reinterpret_cast<const double2*>(values + i0) + q);
        v[2 * q] = (T)f.x; v[2 * q + 1] = (T)f.y;
      }
    } else {
#pragma unroll
      for (int j = 0; j < kPer; ++j) v[j] = i0 + j < n ? values[i0 + j] : (T)0;
    }
    if (tab.trunc[f]) {  // uniform per field; off on the parity path
      const int tre = eb_exponent(info->eb);
#pragma unroll
      for (int j = 0; j < kPer; ++j) v[j] = trunc_value<T>(v[j], tre);
    }
    unsigned int z = wz + iz - zeros;  // block-local slot
#pragma unroll
    for (int j = 0; j < kPer; ++j)
      if (c[j] == 0) s_val[z++] = v[j];
  }
  __syncthreads();
  if (unpred_out && blk_zeros) {
    const T* s_val = reinterpret_cast<const T*>(s_win + kWinWords);
    T* dst = unpred_out + zoff;
    for (unsigned int i = threadIdx.x; i < blk_zeros; i += kThreads) dst[i] = s_val[i];
  }
  if (in_smem)
    for (int i = threadIdx.x; i < nwin; i += kThreads) {
      const uint32_t v = bswap32(s_win[i]);
      if ((i == 0 && head_shared) || (i == nwin - 1 && tail_shared))
        atomicOr(&out_words[wbase + i], v);  // shared with a neighbour chunk (pre-zeroed)
      else
        out_words[wbase + i] = v;
    }
}

}  // namespace

cudaError_t launch_encode_batch(const EncodeJob* jobs, int nf, int m, long long n, int width,
                                int ndim, const long long* dims, int layers, int sms,
                                cudaStream_t s) {
  if (nf < 1 || nf > kBatchMax) return cudaErrorInvalidValue;
  EncTab tab;
  for (int f = 0; f < nf; ++f) {
    tab.codes[f] = jobs[f].codes;
    tab.lengths[f] = jobs[f].lengths;
    tab.words[f] = jobs[f].words;
    tab.agg[f] = jobs[f].agg;
    tab.info[f] = jobs[f].info;
    tab.bits[f] = jobs[f].bits;
    tab.bits_cap[f] = jobs[f].bits_cap;
    tab.head[f] = jobs[f].head;
    tab.values[f] = jobs[f].values;
    tab.unpred[f] = jobs[f].unpred;
    tab.trunc[f] = jobs[f].trunc;
  }
  const long long nchunks = (n + kChunk - 1) / kChunk;
  {
    // persistent count: ~8 blocks (64 warps) per SM over the whole batch
    long long bpf = ((long long)sms * 8 + nf - 1) / nf;
    const long long need = (nchunks + kThreads / 32 - 1) / (kThreads / 32);
    if (bpf > need) bpf = need;
    if (bpf < 1) bpf = 1;
    const dim3 cgrid((unsigned)bpf, nf);
    if (m > 8)
      encode_count_kernel<uint16_t><<<cgrid, kThreads, 0, s>>>(tab, n, m);
    else
      encode_count_kernel<uint8_t><<<cgrid, kThreads, 0, s>>>(tab, n, m);
  }
  unsigned long long d[4] = {0, 0, 0, 0};
  for (int a = 0; a < ndim; ++a) d[a] = (unsigned long long)dims[a];
  encode_scan_kernel<<<nf, 1024, 0, s>>>(tab, nchunks, width, ndim, d[0], d[1], d[2], d[3], m,
                                         layers);
  const size_t win = encode_pack_smem(m, width);
  static KernelAttr attr[4];
  const int key = (m > 8 ? 2 : 0) + (width == 64 ? 1 : 0);
#define EBZ_PACK(C, T)                                                                        \
  do {                                                                                        \
    const cudaError_t e = kernel_smem(attr[key], encode_pack_kernel<C, T>,                    \
                                      encode_pack_smem(kTableSmemMaxM, 64));                  \
    if (e != cudaSuccess) return e;                                                           \
    encode_pack_kernel<C, T><<<dim3((unsigned)nchunks, nf), kThreads, win, s>>>(tab, n, m);   \
  } while (0)
  if (m > 8) {
    if (width == 64) EBZ_PACK(uint16_t, double); else EBZ_PACK(uint16_t, float);
  } else {
    if (width == 64) EBZ_PACK(uint8_t, double); else EBZ_PACK(uint8_t, float);
  }
#undef EBZ_PACK
  return cudaGetLastError();
}

size_t encode_pack_smem(int m, int width) {
  const size_t t = m <= kTableSmemMaxM ? (size_t)9 * (m < 8 ? 256 : (1u << m)) : 0;
  // + value staging for the verbatim compaction
  return ((t + 15) & ~(size_t)15) + (size_t)kWinWords * 4 + (size_t)kChunk * (width / 8);
}

