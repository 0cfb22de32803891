// decode.cu -- canonical-Huffman decode of exactly N symbols + zero ranks.
//
// Replaces entropy.decode / unpack_bits (ebzip/entropy.py:160-183,
// _kernels.py:151-183) with identical results and error classification:
// the bit budget is the WHOLE byte buffer (8 * nbytes, padding included),
// decoding stops after N symbols, "exhausted" when bits run out first,
// "invalid" when a prefix reaches max_len + 1 bits without matching.
//
// The container carries no chunk index, so the decoder finds codeword
// boundaries itself (self-synchronisation of prefix codes):
//   sync   : thread i warms up from bit i*B - W and decodes across its
//            subsequence [i*B, (i+1)*B), recording the first codeword
//            boundary at/after each end and the symbol count between;
//   verify : start_i == end_{i-1} for every i proves that all threads sit on
//            the true parse (induction from bit 0); counts are scanned;
//   write  : every thread re-decodes its span into its output slots;
//   serial : if verification fails or any thread met an invalid prefix, one
//            thread decodes bit-serially exactly like unpack_bits (rare:
//            malformed streams or pathological codes); otherwise a no-op.
// A 12-bit lookup table resolves codewords up to 12 bits in one probe;
// longer (or invalid) prefixes take the reference's depth-by-depth walk.
#include "ebz_common.cuh"

namespace {

constexpr int kLutBits = 12;
constexpr int kSubBits = 2048;   // B
constexpr int kWarmBits = 1024;  // W (measured sync distance <= 378 bits)

struct Tables {
  unsigned long long first[66];
  long long count[66];
  long long base[66];
  int max_len;
  int nused;
  unsigned int lut[1 << kLutBits];  // (symbol << 8) | len, 0 = no code <= 12 bits
  // ordered symbols follow (int32[nsym])
};

__device__ __forceinline__ int* ordered_of(Tables* t) { return reinterpret_cast<int*>(t + 1); }
__device__ __forceinline__ const int* ordered_of(const Tables* t) {
  return reinterpret_cast<const int*>(t + 1);
}

__global__ void __launch_bounds__(1024)
decode_tables_kernel(const uint8_t* __restrict__ lengths, int m, Tables* t, Info* info) {
  const int nsym = 1 << m;
  __shared__ int s_cnt[66];
  __shared__ int s_run[66];
  __shared__ int s_max;
  if (threadIdx.x < 66) s_cnt[threadIdx.x] = 0;
  if (threadIdx.x == 0) s_max = 0;
  __syncthreads();
  for (int s = threadIdx.x; s < nsym; s += blockDim.x) {
    const int l = lengths[s];
    if (l) {
      atomicAdd(&s_cnt[l], 1);
      atomicMax(&s_max, l);
    }
  }
  for (int i = threadIdx.x; i < (1 << kLutBits); i += blockDim.x) t->lut[i] = 0;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long w = 0;
    long long b = 0;
    t->first[0] = 0;
    t->count[0] = s_cnt[0];
    t->base[0] = 0;
    for (int l = 1; l <= 64; ++l) {
      b += s_cnt[l - 1];
      t->base[l] = b;
      t->count[l] = s_cnt[l];
      if (l <= s_max) {
        w <<= 1;
        t->first[l] = w;
        w += (unsigned long long)s_cnt[l];
      } else {
        t->first[l] = 0;
      }
    }
    t->max_len = s_max;
    t->nused = (int)(b + s_cnt[64]);
    info->max_len = s_max;
  }
  __syncthreads();
  // ordered symbols + LUT (one warp, symbol order within each length)
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    for (int i = lane; i < 66; i += 32) s_run[i] = 0;
    __syncwarp();
    int* ord = ordered_of(t);
    for (int s0 = 0; s0 < nsym; s0 += 32) {
      const int s = s0 + lane;
      const int l = s < nsym ? lengths[s] : 0;
      const unsigned int peers = __match_any_sync(EBZ_FULL, l);
      const int before = __popc(peers & ((1u << lane) - 1u));
      const int run = s_run[l];
      if (l) {
        const long long rank = run + before;
        ord[t->base[l] + rank] = s;
        if (l <= kLutBits) {
          const unsigned long long code = t->first[l] + (unsigned long long)rank;
          const unsigned int lo = (unsigned int)(code << (kLutBits - l));
          const unsigned int hi = lo + (1u << (kLutBits - l));
          for (unsigned int e = lo; e < hi; ++e) t->lut[e] = ((unsigned int)s << 8) | (unsigned)l;
        }
      }
      __syncwarp();
      if (l && before == 0) s_run[l] = run + __popc(peers);
      __syncwarp();
    }
  }
}

// 64 bits starting at bit position p of a big-endian bit stream (zero padded)
__device__ __forceinline__ unsigned long long peek64(const uint32_t* __restrict__ wds,
                                                     unsigned long long p) {
  const unsigned long long wi = p >> 5;
  const int sh = (int)(p & 31);
  const unsigned long long a = __byte_perm(__ldg(wds + wi), 0, 0x0123);
  const unsigned long long b = __byte_perm(__ldg(wds + wi + 1), 0, 0x0123);
  const unsigned long long c = __byte_perm(__ldg(wds + wi + 2), 0, 0x0123);
  const unsigned long long hi64 = (a << 32) | b;
  return sh ? (hi64 << sh) | (c << (sh)) >> 32 : hi64;
}

__device__ __forceinline__ int bit_at(const uint8_t* __restrict__ bytes, unsigned long long p) {
  return (bytes[p >> 3] >> (7 - (p & 7))) & 1;
}

// Decode one symbol at bit p.  Returns 1 and sets sym/len on success,
// -1 when the budget runs out first, -2 on an invalid prefix.
__device__ __forceinline__ int decode_one(const Tables* __restrict__ t,
                                          const uint32_t* __restrict__ wds,
                                          const uint8_t* __restrict__ bytes,
                                          unsigned long long nbits, unsigned long long p,
                                          int& sym, int& len) {
  const unsigned long long v = peek64(wds, p);
  const unsigned int e = t->lut[(unsigned int)(v >> (64 - kLutBits))];
  if (e) {
    len = (int)(e & 0xff);
    if (p + (unsigned long long)len > nbits) return -1;
    sym = (int)(e >> 8);
    return 1;
  }
  // reference walk: depth by depth (_kernels.py:165-180)
  unsigned long long word = 0;
  const int* ord = ordered_of(t);
  for (int depth = 1;; ++depth) {
    if (p + (unsigned long long)depth > nbits) return -1;
    word = (word << 1) | (unsigned long long)bit_at(bytes, p + depth - 1);
    if (depth > t->max_len) return -2;
    if (word >= t->first[depth]) {
      const unsigned long long off = word - t->first[depth];
      if (off < (unsigned long long)t->count[depth]) {
        sym = ord[t->base[depth] + (long long)off];
        len = depth;
        return 1;
      }
    }
  }
}

struct SubRec {
  unsigned long long start, end, count;
  int flag;  // 1 = invalid prefix met
  int pad;
};

// Bit budget: a host value, or (device-resident round trip) the bit length
// of a compress record on the device, rounded up to whole bytes -- the
// reference's budget is 8 * len(code_bits) (entropy.py:171-175).
struct Budget {
  unsigned long long nbits;
  const unsigned long long* dev_bitlen;
  __device__ __forceinline__ unsigned long long bits() const {
    return dev_bitlen ? ((*dev_bitlen + 7) / 8) * 8 : nbits;
  }
  __device__ __forceinline__ long long nsub() const {
    const unsigned long long b = bits();
    return b == 0 ? 1 : (long long)((b + kSubBits - 1) / kSubBits);
  }
};

__global__ void __launch_bounds__(256)
decode_sync_kernel(const Tables* __restrict__ t, const uint32_t* __restrict__ wds,
                   Budget bud, SubRec* __restrict__ rec) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const unsigned long long nbits = bud.bits();
  if (i >= bud.nsub()) return;
  const uint8_t* bytes = reinterpret_cast<const uint8_t*>(wds);
  const unsigned long long lo = (unsigned long long)i * kSubBits;
  const unsigned long long hi = lo + kSubBits;
  unsigned long long p = i == 0 ? 0 : (lo > kWarmBits ? lo - kWarmBits : 0);
  int flag = 0;
  int sym, len;
  // warm-up: first boundary >= lo
  while (p < lo) {
    const int r = decode_one(t, wds, bytes, nbits, p, sym, len);
    if (r != 1) {
      if (r == -2) flag = 1;
      break;
    }
    p += len;
  }
  const unsigned long long start = p;
  unsigned long long count = 0;
  bool stopped = p < lo;  // warm-up ended early (exhausted/invalid)
  while (!stopped && p < hi) {
    const int r = decode_one(t, wds, bytes, nbits, p, sym, len);
    if (r != 1) {
      if (r == -2) flag = 1;
      break;
    }
    p += len;
    ++count;
  }
  rec[i].start = start;
  rec[i].end = p;
  rec[i].count = count;
  rec[i].flag = flag;
}

// single CTA: verify the chain, exclusive-scan counts
__global__ void __launch_bounds__(1024)
decode_verify_kernel(SubRec* __restrict__ rec, Budget bud, long long want, Info* info) {
  const long long nsub = bud.nsub();
  __shared__ unsigned long long s_c[1024];
  __shared__ int s_bad;
  if (threadIdx.x == 0) s_bad = 0;
  __syncthreads();
  const long long per = (nsub + 1023) / 1024;
  const long long lo = threadIdx.x * per;
  const long long hi = lo + per < nsub ? lo + per : nsub;
  unsigned long long c = 0;
  int bad = 0;
  for (long long i = lo; i < hi; ++i) {
    c += rec[i].count;
    if (rec[i].flag) bad = 1;
    if (i > 0 && rec[i].start != rec[i - 1].end) bad = 1;
  }
  if (bad) atomicOr(&s_bad, 1);
  s_c[threadIdx.x] = c;
  __syncthreads();
  for (int o = 1; o < 1024; o <<= 1) {
    unsigned long long tv = (int)threadIdx.x >= o ? s_c[threadIdx.x - o] : 0;
    __syncthreads();
    s_c[threadIdx.x] += tv;
    __syncthreads();
  }
  unsigned long long run = threadIdx.x ? s_c[threadIdx.x - 1] : 0;
  for (long long i = lo; i < hi; ++i) {
    const unsigned long long ci = rec[i].count;
    rec[i].count = run;  // now the output offset
    run += ci;
  }
  if (threadIdx.x == 0) {
    const unsigned long long total = s_c[1023];
    if (s_bad) {
      atomicOr(&info->status, ST_DEC_ANOMALY);
    } else {
      info->decoded = (long long)(total < (unsigned long long)want ? total : want);
      if (total < (unsigned long long)want) atomicOr(&info->status, ST_DEC_EXHAUSTED);
    }
  }
}

template <typename C>
__global__ void __launch_bounds__(256)
decode_write_kernel(const Tables* __restrict__ t, const uint32_t* __restrict__ wds,
                    Budget bud, const SubRec* __restrict__ rec,
                    long long want, C* __restrict__ out, const Info* info) {
  if (info->status & (ST_DEC_ANOMALY | ST_DEC_EXHAUSTED)) return;
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const unsigned long long nbits = bud.bits();
  if (i >= bud.nsub()) return;
  const uint8_t* bytes = reinterpret_cast<const uint8_t*>(wds);
  unsigned long long p = rec[i].start;
  const unsigned long long end = rec[i].end;
  unsigned long long o = rec[i].count;  // offset after verify
  int sym, len;
  while (p < end && o < (unsigned long long)want) {
    decode_one(t, wds, bytes, nbits, p, sym, len);
    out[o++] = (C)sym;
    p += len;
  }
}

// exact bit-serial decoder (anomaly path), one thread
template <typename C>
__global__ void decode_serial_kernel(const Tables* __restrict__ t, const uint8_t* __restrict__ bytes,
                                     Budget bud, long long want, C* __restrict__ out,
                                     Info* info) {
  if (!(info->status & ST_DEC_ANOMALY)) return;
  const unsigned long long nbits = bud.bits();
  const int* ord = ordered_of(t);
  unsigned long long word = 0;
  int depth = 0;
  long long produced = 0;
  for (unsigned long long p = 0; p < nbits; ++p) {
    if (produced >= want) break;
    word = (word << 1) | (unsigned long long)bit_at(bytes, p);
    if (++depth > t->max_len) {
      info->decoded = -2;
      atomicOr(&info->status, ST_DEC_INVALID);
      return;
    }
    if (word >= t->first[depth]) {
      const unsigned long long off = word - t->first[depth];
      if (off < (unsigned long long)t->count[depth]) {
        out[produced++] = (C)ord[t->base[depth] + (long long)off];
        word = 0;
        depth = 0;
      }
    }
  }
  if (produced < want) {
    info->decoded = -1;
    atomicOr(&info->status, ST_DEC_EXHAUSTED);
    return;
  }
  info->decoded = produced;
}

// ------------------------------------------------------------ zero ranks
// Per-row count of code-0 symbols (a row = a line along axis 0), then an
// exclusive scan -> rowbase[r] = rank of the first verbatim value of row r.
template <typename C>
__global__ void __launch_bounds__(256)
row_zero_kernel(const C* __restrict__ codes, long long nrows, long long nx,
                unsigned long long* __restrict__ cnt) {
  const int lane = threadIdx.x & 31;
  if (nx <= 64) {
    const long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= nrows) return;
    unsigned long long z = 0;
    const C* row = codes + r * nx;
    for (long long x = 0; x < nx; ++x) z += row[x] == 0;
    cnt[r] = z;
    return;
  }
  const long long r = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (r >= nrows) return;
  const C* row = codes + r * nx;
  unsigned int z = 0;
  for (long long x = lane; x < nx; x += 32) z += __ldcs(row + x) == 0;
#pragma unroll
  for (int o = 16; o; o >>= 1) z += __shfl_xor_sync(EBZ_FULL, z, o);
  if (lane == 0) cnt[r] = z;
}

__global__ void __launch_bounds__(1024)
scan_rows_kernel(const unsigned long long* __restrict__ cnt, long long n,
                 unsigned long long* __restrict__ out, Info* info) {
  __shared__ unsigned long long s_c[1024];
  const long long per = (n + 1023) / 1024;
  const long long lo = threadIdx.x * per;
  const long long hi = lo + per < n ? lo + per : n;
  unsigned long long c = 0;
  for (long long i = lo; i < hi; ++i) c += cnt[i];
  s_c[threadIdx.x] = c;
  __syncthreads();
  for (int o = 1; o < 1024; o <<= 1) {
    unsigned long long tv = (int)threadIdx.x >= o ? s_c[threadIdx.x - o] : 0;
    __syncthreads();
    s_c[threadIdx.x] += tv;
    __syncthreads();
  }
  unsigned long long run = threadIdx.x ? s_c[threadIdx.x - 1] : 0;
  for (long long i = lo; i < hi; ++i) {
    const unsigned long long ci = cnt[i];
    out[i] = run;
    run += ci;
  }
  if (threadIdx.x == 0) {
    info->zeros_decoded = s_c[1023];
    if (s_c[1023] != info->n_unpred) atomicOr(&info->status, ST_UNPRED_MISMATCH);
  }
}

}  // namespace

size_t decode_scratch_bytes(long long nbytes, int m) {
  const long long nbits = nbytes * 8;
  const long long nsub = nbits / kSubBits + 1;
  size_t tables = sizeof(Tables) + sizeof(int) * ((size_t)1 << m);
  tables = (tables + 255) & ~(size_t)255;
  return tables + sizeof(SubRec) * (size_t)nsub + 256;
}

// nbytes: the byte budget, or (dev_bitlen != nullptr) an upper bound used
// only to size the grid; the exact budget is then read on the device.
cudaError_t launch_decode(const uint8_t* bits, long long nbytes, const uint8_t* lengths, int m,
                          long long n, void* codes, Info* info, unsigned long long* scratch,
                          size_t scratch_bytes, int sms, cudaStream_t s,
                          const unsigned long long* dev_bitlen) {
  (void)scratch_bytes;
  (void)sms;
  Tables* t = reinterpret_cast<Tables*>(scratch);
  size_t tables = sizeof(Tables) + sizeof(int) * ((size_t)1 << m);
  tables = (tables + 255) & ~(size_t)255;
  SubRec* rec = reinterpret_cast<SubRec*>(reinterpret_cast<char*>(scratch) + tables);
  Budget bud;
  bud.nbits = (unsigned long long)nbytes * 8ull;
  bud.dev_bitlen = dev_bitlen;
  decode_tables_kernel<<<1, 1024, 0, s>>>(lengths, m, t, info);
  if (n == 0) {
    return cudaGetLastError();
  }
  const unsigned long long nbits_max = (unsigned long long)nbytes * 8ull;
  const long long nsub_max =
      nbits_max == 0 ? 1 : (long long)((nbits_max + kSubBits - 1) / kSubBits);
  const unsigned grid = (unsigned)((nsub_max + 255) / 256);
  const uint32_t* wds = reinterpret_cast<const uint32_t*>(bits);
  decode_sync_kernel<<<grid, 256, 0, s>>>(t, wds, bud, rec);
  decode_verify_kernel<<<1, 1024, 0, s>>>(rec, bud, n, info);
  if (m > 8) {
    decode_write_kernel<uint16_t><<<grid, 256, 0, s>>>(t, wds, bud, rec, n, (uint16_t*)codes,
                                                       info);
    decode_serial_kernel<uint16_t><<<1, 1, 0, s>>>(t, bits, bud, n, (uint16_t*)codes, info);
  } else {
    decode_write_kernel<uint8_t><<<grid, 256, 0, s>>>(t, wds, bud, rec, n, (uint8_t*)codes, info);
    decode_serial_kernel<uint8_t><<<1, 1, 0, s>>>(t, bits, bud, n, (uint8_t*)codes, info);
  }
  return cudaGetLastError();
}

cudaError_t launch_rowbase(const void* codes, int m, long long n, long long nx,
                           unsigned long long* rowbase, unsigned long long* tmp,
                           unsigned long long n_unpred, Info* info, cudaStream_t s) {
  const long long nrows = n / nx;
  long long threads = nx <= 64 ? nrows : nrows * 32;
  const unsigned blocks = (unsigned)((threads + 255) / 256);
  if (m > 8)
    row_zero_kernel<uint16_t><<<blocks, 256, 0, s>>>((const uint16_t*)codes, nrows, nx, tmp);
  else
    row_zero_kernel<uint8_t><<<blocks, 256, 0, s>>>((const uint8_t*)codes, nrows, nx, tmp);
  (void)n_unpred;
  scan_rows_kernel<<<1, 1024, 0, s>>>(tmp, nrows, rowbase, info);
  return cudaGetLastError();
}
