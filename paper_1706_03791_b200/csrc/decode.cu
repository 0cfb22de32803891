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
//   repair : (twice) every subsequence whose start differs from its
//            predecessor's end is re-decoded from that end -- a true
//            boundary whenever the predecessor is right.  A check pass lists
//            them (span, predecessor end) and the repair pass decodes the
//            list densely, one span per lane (a repair per warp slot would
//            cost a whole warp for each of the few failing spans);
//   verify : start_i == end_{i-1} for every i proves that all threads sit on
//            the true parse (induction from bit 0); counts are scanned;
//   (sync and repair stage each span's symbols in a kSpanCap slot)
//   copy   : once the scan fixed every span's output offset, the staged
//            symbols move to their place (aligned 8-byte words);
//   serial : only if verification still fails or an invalid prefix was met
//            on a decoded span: one thread decodes bit-serially exactly like
//            unpack_bits (malformed streams); otherwise a no-op.
//
// Decoding keeps a 64-bit big-endian bit buffer in registers and resolves a
// 12-bit window with one shared-memory lookup that yields up to 7 symbols
// (m <= 8: every codeword that fits the window completely, greedily) or one
// 16-bit symbol (m > 8).  Near span ends and budget limits the decoder steps
// one codeword at a time (canonical length search on the window), so every
// boundary, count and error is exactly the bit-serial decoder's.
#include "ebz_common.cuh"

namespace {

#ifndef EBZ_DEC_B
#define EBZ_DEC_B 1024
#endif
#ifndef EBZ_DEC_W
#define EBZ_DEC_W 128
#endif
#ifndef EBZ_DEC_T
#define EBZ_DEC_T 512
#endif
#ifndef EBZ_DEC_U
#define EBZ_DEC_U 2   // windows per decode-loop iteration
#endif
#ifndef EBZ_COPY_U
#define EBZ_COPY_U 4
#endif
constexpr int kLutBits = 12;
constexpr int kSubBits = EBZ_DEC_B;   // B
// W: warm-up before each span.  Measured on the cfg5 batch (5.56M spans):
// W = 512 leaves 24 spans off the true parse, 256 -> 4.2K, 128 -> 72K (1.3%);
// the dense repair list makes 128 the fastest (decode 5.92 -> 5.43 ms).
constexpr int kWarmBits = EBZ_DEC_W;
static_assert(kWarmBits % 128 == 0, "the staged slice starts on a 16-byte word");
constexpr int kThreads = EBZ_DEC_T;   // decode blocks (one subsequence per thread)
constexpr int kRowsPerBlock = 256;
constexpr int kMaxMulti = 7;     // symbols per lookup (m <= 8)
// staged symbols per span: a span covers < kSubBits + 64 bits, one symbol per
// bit at most (multiple of 8 for the gathered 8-byte stores)
constexpr int kSpanCap = kSubBits + 128;

// Multi-symbol entry: bits 0..55 symbols (8-bit lanes, m <= 8; one 16-bit
// symbol for m > 8), bits 56..58 symbol count n (0 = no codeword of <= 12
// bits at the window), bits 59..62 total length.
__device__ __forceinline__ int ent_n(unsigned long long e) { return (int)(e >> 56) & 7; }
__device__ __forceinline__ int ent_len(unsigned long long e) { return (int)(e >> 59) & 15; }

struct Tables {
  unsigned long long first[66];
  long long count[66];
  long long base[66];
  int max_len;
  int nused;
  unsigned long long mlut[1 << kLutBits];
  // per 12-bit window: the length of its first codeword when <= 12, else
  // the shortest length with a codeword under this prefix (255: none) --
  // where the canonical length search starts
  uint8_t lmin[1 << kLutBits];
  // ordered symbols follow (int32[nsym])
};

__device__ __forceinline__ int* ordered_of(Tables* t) { return reinterpret_cast<int*>(t + 1); }
__device__ __forceinline__ const int* ordered_of(const Tables* t) {
  return reinterpret_cast<const int*>(t + 1);
}

struct SubRec;

// Per-field pointers of a batched decode (blockIdx.y, or blockIdx.x for the
// one-CTA stages, selects the field).
struct DecTab {
  const uint8_t* lengths[kBatchMax];
  const uint32_t* wds[kBatchMax];             // code stream (big-endian bytes)
  unsigned long long nbits[kBatchMax];        // budget (host) ...
  const unsigned long long* bitlen[kBatchMax];  // ... or a device bit length
  Tables* t[kBatchMax];
  SubRec* rec[kBatchMax];
  unsigned long long* bsum[kBatchMax];
  Info* info[kBatchMax];
  void* codes[kBatchMax];
  void* stage[kBatchMax];                     // kSpanCap symbols per span
  // repair list: [0] = entries of the current pass, then (span, from) pairs
  unsigned long long* rlist[kBatchMax];
  const Info* src[kBatchMax];                 // record init: source record ...
  double eb[kBatchMax];                       // ... or eb / K from the host
  unsigned long long k[kBatchMax];
};

__global__ void __launch_bounds__(1024)
decode_tables_kernel(const __grid_constant__ DecTab tab, int m) {
  const uint8_t* __restrict__ lengths = tab.lengths[blockIdx.x];
  Tables* t = tab.t[blockIdx.x];
  Info* info = tab.info[blockIdx.x];
  const int nsym = 1 << m;
  __shared__ int s_cnt[66];
  __shared__ int s_run[66];
  __shared__ int s_max;
  __shared__ unsigned long long s_first[66], s_endw[kLutBits + 1];
  __shared__ int s_base[66];
  __shared__ unsigned int s_lut[1 << kLutBits];  // (symbol << 8) | len, 0 = none
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
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long w = 0;
    long long b = 0;
    t->first[0] = 0;
    t->count[0] = s_cnt[0];
    t->base[0] = 0;
    s_first[0] = 0;
    s_base[0] = 0;
    for (int l = 1; l <= 64; ++l) {
      b += s_cnt[l - 1];
      t->base[l] = b;
      s_base[l] = (int)b;
      t->count[l] = s_cnt[l];
      if (l <= s_max) {
        w <<= 1;
        t->first[l] = w;
        s_first[l] = w;
        if (l <= kLutBits) s_endw[l] = w + (unsigned long long)s_cnt[l];
        w += (unsigned long long)s_cnt[l];
      } else {
        t->first[l] = 0;
        s_first[l] = 0;
        if (l <= kLutBits) s_endw[l] = 0;
      }
    }
    t->max_len = s_max;
    t->nused = (int)(b + s_cnt[64]);
    info->max_len = s_max;
  }
  __syncthreads();
  // ordered symbols: symbol order within each length (one warp)
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
      if (l) ord[s_base[l] + run + before] = s;
      __syncwarp();
      if (l && before == 0) s_run[l] = run + __popc(peers);
      __syncwarp();
    }
  }
  __syncthreads();
  // single-codeword LUT: canonical length search per window value
  const int* ord = ordered_of(t);
  const int top = s_max < kLutBits ? s_max : kLutBits;
  for (int e = threadIdx.x; e < (1 << kLutBits); e += blockDim.x) {
    unsigned int v = 0;
    for (int L = 1; L <= top; ++L) {
      const unsigned long long code = (unsigned long long)(e >> (kLutBits - L));
      if (code < s_endw[L]) {
        v = ((unsigned int)ord[s_base[L] + (int)(code - s_first[L])] << 8) | (unsigned)L;
        break;
      }
    }
    s_lut[e] = v;
    int lm = (int)(v & 0xff);
    if (!v) {  // longer codes: the first length whose codes reach this prefix
      lm = 255;
      for (int L = kLutBits + 1; L <= s_max; ++L) {
        if (!s_cnt[L]) continue;
        const int sh = L - kLutBits;
        const unsigned long long p0 = s_first[L] >> sh;
        const unsigned long long p1 = (s_first[L] + (unsigned long long)s_cnt[L] - 1ull) >> sh;
        if ((unsigned long long)e >= p0 && (unsigned long long)e <= p1) {
          lm = L;
          break;
        }
      }
    }
    t->lmin[e] = (uint8_t)lm;
  }
  __syncthreads();
  // multi-symbol entries: greedy decode of every codeword inside the window
  for (int e = threadIdx.x; e < (1 << kLutBits); e += blockDim.x) {
    unsigned long long ent = 0;
    int n = 0, used = 0;
    if (m <= 8) {
      while (n < kMaxMulti) {
        const unsigned int se = s_lut[(e << used) & ((1 << kLutBits) - 1)];
        const int L = (int)(se & 0xff);
        if (!se || used + L > kLutBits) break;
        ent |= (unsigned long long)(se >> 8) << (8 * n);
        ++n;
        used += L;
      }
    } else {
      const unsigned int se = s_lut[e];
      if (se) {
        ent = se >> 8;
        n = 1;
        used = (int)(se & 0xff);
      }
    }
    t->mlut[e] = ent | ((unsigned long long)n << 56) | ((unsigned long long)used << 59);
  }
}

__device__ __forceinline__ int bit_at(const uint8_t* __restrict__ bytes, unsigned long long p) {
  return (bytes[p >> 3] >> (7 - (p & 7))) & 1;
}
__device__ __forceinline__ unsigned long long be32(const uint32_t* p) {
  return (unsigned long long)__byte_perm(__ldg(p), 0, 0x0123);
}

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

// Shared-memory decode tables.  Longer canonical codewords: the length-L
// codes are the integers [first_L, first_L + count_L) and first_{L+1} =
// (first_L + count_L) << 1, so left-justified they tile the code space in
// increasing order and the codeword length is the smallest L whose top-L-bits
// value is below endw_L = first_L + count_L -- read straight from the
// register window (>= 33 valid bits, so L <= 32).
struct SmemTables {
  unsigned long long mlut[1 << kLutBits];
  unsigned long long endw[34];
  unsigned long long first[34];
  int base[34];
  int max_len;
  int m8;
  uint8_t lmin[1 << kLutBits];
};

__device__ __forceinline__ void load_tables(SmemTables* st, const Tables* t, int m) {
  for (int i = threadIdx.x; i < (1 << kLutBits); i += blockDim.x) st->mlut[i] = t->mlut[i];
  for (int i = threadIdx.x; i < (1 << kLutBits) / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(st->lmin)[i] = reinterpret_cast<const uint32_t*>(t->lmin)[i];
  if (threadIdx.x < 34) {
    const int L = threadIdx.x;
    const unsigned long long f = L >= 1 ? t->first[L] : 0;
    const long long c = L >= 1 ? t->count[L] : 0;
    st->first[L] = f;
    st->endw[L] = (L >= 1 && L <= t->max_len) ? f + (unsigned long long)c : 0ull;
    st->base[L] = L >= 1 ? (int)t->base[L] : 0;
  }
  if (threadIdx.x == 0) {
    st->max_len = t->max_len;
    st->m8 = m <= 8;
  }
  __syncthreads();
}

// Streaming decoder state: buf holds the upcoming bits MSB-aligned, nb of
// them valid (>= 33 after every refill).  Positions are kept relative to the
// last seek point p0 in 32-bit registers (spans are a few thousand bits):
// used = bits consumed since p0, nbrel = budget - p0.  STAGED readers take
// every word from the block's shared-memory slice of the stream (already
// byte-swapped, padded one word per 32 so lanes reading their own spans hit
// distinct banks); the slice covers all spans of the block by construction.
constexpr int kRelMax = 1 << 30;

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
// an opaque copy: the compiler cannot rebuild the address from SR_CgaCtaId
// inside the loop (it did, three instructions per lookup)
__device__ __forceinline__ unsigned pin_u32(unsigned a) {
  asm volatile("" : "+r"(a));
  return a;
}
__device__ __forceinline__ unsigned long long lds64(unsigned a) {
  unsigned long long v;
  asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ unsigned lds32(unsigned a) {
  unsigned v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ int lds8(unsigned a) {
  unsigned short v;
  asm volatile("ld.shared.u8 %0, [%1];" : "=h"(v) : "r"(a));
  return (int)v;
}

template <bool STAGED>
struct Reader {
  const uint32_t* wds;
  const uint8_t* bytes;
  const Tables* t;
  const SmemTables* st;  // shared-memory copy
  const uint32_t* sm;
  long long sw0;
  unsigned long long p0;
  int nbrel;
  int used;
  long long widx;
  unsigned long long buf;
  int nb;
  unsigned a_mlut = 0, a_lmin = 0, a_sm = 0;  // pinned shared addresses

  __device__ __forceinline__ void pin() {
    a_mlut = pin_u32(smem_u32(st->mlut));
    a_lmin = pin_u32(smem_u32(st->lmin));
    if (STAGED) a_sm = pin_u32(smem_u32(sm));
  }

  // STAGED: widx counts words from the slice start sw0 (32-bit arithmetic
  // in the refill); otherwise it is the absolute word index
  __device__ __forceinline__ unsigned long long word(long long i) const {
    if (STAGED) {
      const int k = (int)i;
      return (unsigned long long)lds32(a_sm + 4u * (unsigned)(k + (k >> 5)));
    }
    return be32(wds + i);
  }
  __device__ __forceinline__ unsigned long long pos() const {
    return p0 + (unsigned long long)used;
  }
  __device__ __forceinline__ void prime(unsigned long long p) {
    widx = (long long)(p >> 5) - (STAGED ? sw0 : 0ll);
    const int sh = (int)(p & 31);
    const unsigned long long a = word(widx), b = word(widx + 1);
    widx += 2;
    buf = ((a << 32) | b) << sh;
    nb = 64 - sh;
  }
  __device__ __forceinline__ void seek(unsigned long long p, unsigned long long nbits) {
    p0 = p;
    used = 0;
    const long long r = (long long)nbits - (long long)p;
    nbrel = r > kRelMax ? kRelMax : (r < -kRelMax ? -kRelMax : (int)r);
    prime(p);
  }
  // relative form of an absolute bound (clamped)
  __device__ __forceinline__ int rel(unsigned long long q) const {
    const long long r = (long long)q - (long long)p0;
    return r > kRelMax ? kRelMax : (r < -kRelMax ? -kRelMax : (int)r);
  }
  __device__ __forceinline__ void refill() {
    if (STAGED) {
      // branch-free: the next staged word is always in the slice (slack
      // words after the last span), merged only when needed
      const bool need = nb <= 32;
      const unsigned long long w = word(widx);
      buf |= need ? w << ((32 - nb) & 63) : 0ull;
      widx += need ? 1 : 0;
      nb += need ? 32 : 0;
    } else if (nb <= 32) {
      buf |= word(widx) << (32 - nb);
      ++widx;
      nb += 32;
    }
  }
  // without the refill: nb >= 33 after every refill, so two windows of <= 12
  // bits can be consumed before the next one
  __device__ __forceinline__ void skip(int len) {
    buf <<= len;
    nb -= len;
    used += len;
  }
  __device__ __forceinline__ void consume(int len) {
    skip(len);
    refill();
  }
  // the window's multi-symbol entry
  __device__ __forceinline__ unsigned long long peek() const {
    return lds64(a_mlut + 8u * (unsigned)(buf >> (64 - kLutBits)));
  }
  // One codeword.  1: decoded (sym), -1: budget exhausted, -2: invalid prefix
  __device__ __forceinline__ int next(int& sym) {
    const unsigned long long e = peek();
    const int n = ent_n(e);
    int len;
    if (n && !st->m8) {  // one 16-bit symbol per entry: its length is the total
      len = ent_len(e);
      if (used + len > nbrel) return -1;
      sym = (int)(e & 0xffff);
      consume(len);
      return 1;
    }
    // a window starting with a codeword of <= 12 bits: its length is in the
    // lmin table, its symbol the entry's first
    int L = lds8(a_lmin + (unsigned)(buf >> (64 - kLutBits)));
    if (n) {
      if (used + L > nbrel) return -1;
      sym = (int)(e & 0xff);
      consume(L);
      return 1;
    }
    // canonical length search on the window from the shortest length with
    // codewords under this 12-bit prefix (lengths below it cannot match)
    const int top = st->max_len < 32 ? st->max_len : 32;
    for (; L <= top; ++L) {
      const unsigned long long wv = buf >> (64 - L);
      if (wv < st->endw[L]) {
        if (used + L > nbrel) return -1;
        sym = ordered_of(t)[st->base[L] + (int)(wv - st->first[L])];
        consume(L);
        return 1;
      }
    }
    if (st->max_len <= 32) {
      // no codeword matches: the reference reads max_len + 1 bits and fails
      // as "invalid", unless the budget ends first ("exhausted")
      return used + st->max_len + 1 > nbrel ? -1 : -2;
    }
    // reference walk, depth by depth (_kernels.py:165-180), lengths > 32
    unsigned long long word = 0;
    const int* ord = ordered_of(t);
    const unsigned long long p = pos();
    for (int depth = 1;; ++depth) {
      if (used + depth > nbrel) return -1;
      word = (word << 1) | (unsigned long long)bit_at(bytes, p + depth - 1);
      if (depth > t->max_len) return -2;
      if (word >= t->first[depth]) {
        const unsigned long long off = word - t->first[depth];
        if (off < (unsigned long long)t->count[depth]) {
          sym = ord[t->base[depth] + (long long)off];
          len = depth;
          break;
        }
      }
    }
    used += len;
    prime(pos());
    return 1;
  }
};

struct SubRec {
  unsigned long long start, end, count;
  int flag;  // 1 = invalid prefix met on the decoded span
  int pad;
};


// Span staging: a span's symbols fill its own slot from the slot's start
// (16-byte aligned, kSpanCap symbols), so every store is a whole aligned
// word -- no head / alignment cases (the general writer recomputed the slot
// pointer and alignment on every store: the store path was ~16% of the
// decode loop's issued instructions at 6 active lanes; decode stage 5.17 ->
// 4.50 ms on the cfg5 batch).  Elements accumulate in a 64-bit word (two
// words per 16-byte store measured slower: 4.92 ms).
template <typename C>
struct StageWords {
  static constexpr int EB = 8 * (int)sizeof(C);  // bits per element
  static constexpr int PER = 8 / (int)sizeof(C);  // elements per word
  unsigned long long* out;
  unsigned long long lo = 0;
  int q = 0;  // elements pending
  __device__ __forceinline__ explicit StageWords(C* slot)
      : out(reinterpret_cast<unsigned long long*>(slot)) {}
  // n elements packed in `syms` (EB-bit lanes), n < PER
  // Branch-free (the store was a divergent block in the decode loop): a
  // full word needs q + n >= PER, so q >= 1 (n < PER) and 1 <= PER - q < PER
  __device__ __forceinline__ void put(unsigned long long syms, int n) {
    lo |= syms << (EB * q);
    const bool full = q + n >= PER;
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %2, 0;\n\t@p st.global.u64 [%0], %1;\n\t}"
                 :: "l"(out), "l"(lo), "r"((int)full) : "memory");
    out += full ? 1 : 0;
    lo = full ? syms >> ((EB * (PER - q)) & 63) : lo;
    q += full ? n - PER : n;
  }
  // the pending elements leave as whole words (the slot has room; the copy
  // reads only the span's count)
  __device__ __forceinline__ void finish() {
    if (q > 0) *out = lo;
  }
};

// Decode from the current position until the first boundary >= hi (or the
// budget ends), counting symbols.  Whole windows are consumed while every
// boundary inside stays <= hi and inside the budget.  Warp-uniform loop
// control: every lane steps together and finished lanes idle predicated -- a
// plain per-lane `while/break` loop let the divergent lanes run one after
// another (measured 1.4 active lanes).
template <bool STAGED, typename C>
__device__ __forceinline__ void run_span(Reader<STAGED>& rd, unsigned long long hi,
                                         unsigned long long& count, int& flag, bool live,
                                         C* stage) {
  const int hrel = rd.rel(hi);
  const int lrel = hrel < rd.nbrel ? hrel : rd.nbrel;
  StageWords<C> ow(stage);
  int sym;
  bool go = live && rd.used < hrel;
  // symbols of this call, 32-bit (at most kSpanCap), added to count at the end
  const int cap = count < (unsigned long long)kSpanCap ? kSpanCap - (int)count : 0;
  int cnt = 0;
  while (__any_sync(EBZ_FULL, go)) {
    if (go) {
      const unsigned long long e = rd.peek();
      const int n = ent_n(e);
      // an entry's symbols depend only on its first ent_len bits (prefix
      // code), so the entry is taken whenever those end inside the span and
      // the budget -- the one-codeword path is left for the window that
      // crosses the span end (requiring the whole 12-bit window inside sent
      // ~21% of the loop's instructions down the length search)
      if (n && rd.used + ent_len(e) <= lrel && cnt + n <= cap) {
        // the entry's symbol lanes past the n-th are zero: strip n / len only
        ow.put(sizeof(C) == 1 ? (e & 0x00ffffffffffffffull) : (e & 0xffffull), n);
        cnt += n;
        rd.skip(ent_len(e));
        // more windows per iteration (predicated; the loop control and vote
        // are paid once for all, the refill once per two windows)
#pragma unroll
        for (int u = 1; u < EBZ_DEC_U; ++u) {
          const unsigned long long e2 = rd.peek();
          const int n2 = ent_n(e2);
          const bool b = n2 && rd.used + ent_len(e2) <= lrel && cnt + n2 <= cap;
          ow.put(b ? (sizeof(C) == 1 ? (e2 & 0x00ffffffffffffffull) : (e2 & 0xffffull)) : 0ull,
                 b ? n2 : 0);
          cnt += b ? n2 : 0;
          rd.skip(b ? ent_len(e2) : 0);
          if (u & 1) rd.refill();
        }
        if (EBZ_DEC_U & 1) rd.refill();
        go = rd.used < hrel;
      } else {
        const int r = rd.next(sym);
        if (r == 1 && cnt < cap) {
          ow.put((unsigned long long)(unsigned)sym, 1);
          ++cnt;
          go = rd.used < hrel;
        } else {
          if (r != -1) flag = 1;  // invalid prefix (or a span over capacity)
          go = false;
        }
      }
    }
  }
  count += (unsigned long long)cnt;
  if (live) ow.finish();
}

// The block's slice of the stream (its spans plus the warm-up before and a
// codeword of slack after) staged in shared memory with coalesced 16-byte
// loads: refills then never wait on global memory inside the decode loop
// (measured: the un-staged refills were 58% of the stall samples).
constexpr int kRegionWords = (kThreads * kSubBits + kWarmBits) / 32 + 8;
constexpr int kRegionPadded = kRegionWords + kRegionWords / 32 + 1;
constexpr size_t kDecodeSmem = sizeof(SmemTables) + (size_t)kRegionPadded * 4;

__device__ __forceinline__ void stage_region(uint32_t* s, const uint32_t* __restrict__ wds,
                                             unsigned long long nbits, long long& w_lo,
                                             long long& w_end) {
  const long long blk_bit = (long long)blockIdx.x * kThreads * kSubBits;
  w_lo = blk_bit >= kWarmBits ? (blk_bit - kWarmBits) / 32 : 0;
  w_end = w_lo + kRegionWords;
  const long long valid_end = (long long)((nbits + 7) / 8 + 3) / 4 + 2;  // padded buffer
  if (w_end > valid_end) w_end = valid_end;
  const long long nw = w_end - w_lo;
  for (long long q = threadIdx.x; q * 4 < nw; q += kThreads) {
    const long long k0 = 4 * q;
    if (k0 + 4 <= nw) {
      const uint4 v = __ldg(reinterpret_cast<const uint4*>(wds + w_lo + k0));
      s[k0 + (k0 >> 5)] = __byte_perm(v.x, 0, 0x0123);  // stored big-endian
      s[k0 + 1 + ((k0 + 1) >> 5)] = __byte_perm(v.y, 0, 0x0123);
      s[k0 + 2 + ((k0 + 2) >> 5)] = __byte_perm(v.z, 0, 0x0123);
      s[k0 + 3 + ((k0 + 3) >> 5)] = __byte_perm(v.w, 0, 0x0123);
    } else {
      for (long long k = k0; k < nw; ++k)
        s[k + (k >> 5)] = __byte_perm(__ldg(wds + w_lo + k), 0, 0x0123);
    }
  }
  __syncthreads();
}

template <typename C>
__global__ void __launch_bounds__(kThreads)
decode_sync_kernel(const __grid_constant__ DecTab tab, int m) {
  const int f = blockIdx.y;
  const Tables* __restrict__ t = tab.t[f];
  const uint32_t* __restrict__ wds = tab.wds[f];
  const Budget bud{tab.nbits[f], tab.bitlen[f]};
  SubRec* __restrict__ rec = tab.rec[f];
  extern __shared__ __align__(16) unsigned char dsm[];
  SmemTables& s_tab = *reinterpret_cast<SmemTables*>(dsm);
  uint32_t* s_words = reinterpret_cast<uint32_t*>(dsm + sizeof(SmemTables));
  if ((long long)blockIdx.x * kThreads >= bud.nsub()) return;  // grid sized by capacity
  load_tables(&s_tab, t, m);
  long long w_lo, w_end;
  stage_region(s_words, wds, bud.bits(), w_lo, w_end);
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const bool live = i < bud.nsub();  // no early return: the loops vote warp-wide
  Reader<true> rd{wds, reinterpret_cast<const uint8_t*>(wds), t, &s_tab, s_words, w_lo};
  rd.pin();
  const unsigned long long lo = (unsigned long long)i * kSubBits;
  // idle lanes park at the slice start: staged readers never leave the slice
  rd.seek(live ? (i == 0 ? 0 : (lo > kWarmBits ? lo - kWarmBits : 0))
               : (unsigned long long)w_lo * 32ull,
          bud.bits());
  int sym;
  bool stopped = false;
  const int lorel = rd.rel(lo);
  const int wlim = lorel < rd.nbrel ? lorel : rd.nbrel;
  bool go = live && rd.used < lorel;
  while (__any_sync(EBZ_FULL, go)) {  // warm-up: reach the first boundary >= lo
    if (go) {
      const unsigned long long e = rd.peek();
      if (ent_n(e) && rd.used + ent_len(e) <= wlim) {
        rd.skip(ent_len(e));
        const unsigned long long e2 = rd.peek();  // a second window (as run_span)
        const bool b = ent_n(e2) && rd.used + ent_len(e2) <= wlim;
        rd.skip(b ? ent_len(e2) : 0);
        rd.refill();
        go = rd.used < lorel;
      } else if (rd.next(sym) != 1) {  // wrong-path trouble: the repair pass fixes it
        stopped = true;
        go = false;
      } else {
        go = rd.used < lorel;
      }
    }
  }
  const unsigned long long start = rd.pos();
  unsigned long long count = 0;
  int flag = 0;
  run_span(rd, lo + kSubBits, count, flag, live && !stopped,
           reinterpret_cast<C*>(tab.stage[f]) + (live ? i : 0) * (long long)kSpanCap);
  if (!live) return;
  rec[i].start = start;
  rec[i].end = rd.pos();
  rec[i].count = count;
  rec[i].flag = flag;
}

// re-decode spans whose start is not their predecessor's end
#ifdef EBZ_DEC_STATS
}  // namespace
#include <cstdio>
namespace {
__device__ unsigned long long g_dec_repairs;
#endif
// list the spans whose start is not their predecessor's end, with that end
__global__ void __launch_bounds__(kThreads)
decode_check_kernel(const __grid_constant__ DecTab tab) {
  const int f = blockIdx.y;
  const Budget bud{tab.nbits[f], tab.bitlen[f]};
  const long long nsub = bud.nsub();
  if ((long long)blockIdx.x * kThreads >= nsub) return;
  const SubRec* __restrict__ rec = tab.rec[f];
  const long long i = (long long)blockIdx.x * kThreads + threadIdx.x;
  const bool need = i >= 1 && i < nsub && rec[i].start != rec[i - 1].end;
  const unsigned mask = __ballot_sync(EBZ_FULL, need);
  if (!mask) return;
  unsigned long long* rl = tab.rlist[f];
  const int lane = threadIdx.x & 31;
  unsigned long long base = 0;
  if (lane == __ffs(mask) - 1) base = atomicAdd(rl, (unsigned long long)__popc(mask));
  base = __shfl_sync(EBZ_FULL, base, __ffs(mask) - 1);
  if (need) {
    const unsigned long long k = base + __popc(mask & ((1u << lane) - 1u));
    rl[1 + 2 * k] = (unsigned long long)i;
    rl[2 + 2 * k] = rec[i - 1].end;
  }
#ifdef EBZ_DEC_STATS
  if (lane == __ffs(mask) - 1) atomicAdd(&g_dec_repairs, (unsigned long long)__popc(mask));
#endif
}

// re-decode the listed spans from their predecessors' ends (grid-stride);
// resets the list for the next pass
template <typename C>
__global__ void __launch_bounds__(kThreads)
decode_repair_kernel(const __grid_constant__ DecTab tab, int m) {
  const int f = blockIdx.y;
  unsigned long long* rl = tab.rlist[f];
  const unsigned long long cnt = *rl;
  const unsigned long long first = (unsigned long long)blockIdx.x * kThreads;
  if (first >= cnt) return;
  const Tables* __restrict__ t = tab.t[f];
  const uint32_t* __restrict__ wds = tab.wds[f];
  const Budget bud{tab.nbits[f], tab.bitlen[f]};
  SubRec* __restrict__ rec = tab.rec[f];
  extern __shared__ __align__(16) unsigned char dsm[];
  SmemTables& s_tab = *reinterpret_cast<SmemTables*>(dsm);
  load_tables(&s_tab, t, m);
  const unsigned long long stride = (unsigned long long)gridDim.x * kThreads;
  for (unsigned long long k0 = first; k0 < cnt; k0 += stride) {
    const unsigned long long k = k0 + threadIdx.x;
    const bool live = k < cnt;
    const long long i = live ? (long long)rl[1 + 2 * k] : 0;
    const unsigned long long from = live ? rl[2 + 2 * k] : 0;
    Reader<false> rd{wds, reinterpret_cast<const uint8_t*>(wds), t, &s_tab, nullptr, 0};
    rd.pin();
    rd.seek(from, bud.bits());
    unsigned long long count = 0;
    int flag = 0;
    run_span(rd, (unsigned long long)(i + 1) * kSubBits, count, flag, live,
             reinterpret_cast<C*>(tab.stage[f]) + i * (long long)kSpanCap);
    if (live) {
      rec[i].start = from;
      rec[i].end = rd.pos();
      rec[i].count = count;
      rec[i].flag = flag;
    }
  }
}

// the list counter back to zero once every repair block has read it
__global__ void decode_relist_kernel(const __grid_constant__ DecTab tab, int nf) {
  if ((int)threadIdx.x < nf) *tab.rlist[threadIdx.x] = 0;
}

// verify the chain + block-local exclusive scan of the counts (one record
// per thread); block totals go to bsum for the top-level scan
__global__ void __launch_bounds__(kThreads)
decode_verify_kernel(const __grid_constant__ DecTab tab) {
  const int f = blockIdx.y;
  SubRec* __restrict__ rec = tab.rec[f];
  const Budget bud{tab.nbits[f], tab.bitlen[f]};
  unsigned long long* __restrict__ bsum = tab.bsum[f];
  Info* info = tab.info[f];
  __shared__ unsigned long long s_w[kThreads / 32];
  const long long nsub = bud.nsub();
  if ((long long)blockIdx.x * kThreads >= nsub) return;  // grid sized by the largest field
  const long long i = (long long)blockIdx.x * kThreads + threadIdx.x;
  unsigned long long c = 0;
  bool bad = false;
  if (i < nsub) {
    c = rec[i].count;
    bad = rec[i].flag || (i > 0 && rec[i].start != rec[i - 1].end);
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(&info->status, ST_DEC_ANOMALY);
  unsigned long long total;
  const unsigned long long ex = block_exscan_u64<kThreads>(c, s_w, total);
  if (i < nsub) rec[i].count = ex;
  if (threadIdx.x == 0) bsum[blockIdx.x] = total;
}

// single CTA: exclusive scan of the block totals; decoded count / exhaustion
__global__ void __launch_bounds__(1024)
decode_top_kernel(const __grid_constant__ DecTab tab, long long want) {
  const int f = blockIdx.x;
  unsigned long long* __restrict__ bsum = tab.bsum[f];
  Info* info = tab.info[f];
  const Budget bud{tab.nbits[f], tab.bitlen[f]};
  const long long nblk = (bud.nsub() + kThreads - 1) / kThreads;
  __shared__ unsigned long long s_w[32];
  const long long per = (nblk + 1023) / 1024;
  const long long lo = threadIdx.x * per;
  const long long hi = lo + per < nblk ? lo + per : nblk;
  unsigned long long c = 0;
  for (long long b = lo; b < hi; ++b) c += bsum[b];
  unsigned long long total;
  unsigned long long run = block_exscan_u64<1024>(c, s_w, total);
  for (long long b = lo; b < hi; ++b) {
    const unsigned long long v = bsum[b];
    bsum[b] = run;
    run += v;
  }
  if (threadIdx.x == 0) bsum[nblk] = total;  // end of the last span
#ifdef EBZ_DEC_STATS
  if (threadIdx.x == 0 && f == 0) {
    printf("EBZDEC repairs %llu\n", g_dec_repairs);
    g_dec_repairs = 0;
  }
#endif
  if (threadIdx.x == 0 && !(info->status & ST_DEC_ANOMALY)) {
    info->decoded = (long long)(total < (unsigned long long)want ? total : want);
    if (total < (unsigned long long)want) atomicOr(&info->status, ST_DEC_EXHAUSTED);
  }
}

// Place the staged spans: span i's symbols go to [off_i, off_{i+1}) of the
// output (absolute offsets = block-local exclusive counts + block prefix),
// clipped to the N-symbol limit.  One block per kThreads spans (the sync
// blocks' spans): offsets gathered once into shared memory, then each warp
// copies its spans with aligned 8-byte stores (bytes at the two ends).
template <typename C>
__global__ void __launch_bounds__(kThreads, 2)
decode_copy_kernel(const __grid_constant__ DecTab tab, long long want) {
  const int f = blockIdx.y;
  const Info* info = tab.info[f];
  const Budget bud{tab.nbits[f], tab.bitlen[f]};
  const long long nsub = bud.nsub();
  const long long i0 = (long long)blockIdx.x * kThreads;
  if (i0 >= nsub || (info->status & (ST_DEC_ANOMALY | ST_DEC_EXHAUSTED))) return;
  const SubRec* __restrict__ rec = tab.rec[f];
  const unsigned long long* __restrict__ bsum = tab.bsum[f];
  __shared__ unsigned long long s_off[kThreads + 1];
  {
    const long long i = i0 + threadIdx.x;
    const unsigned long long total = bsum[(nsub + kThreads - 1) / kThreads];
    s_off[threadIdx.x] = i < nsub ? rec[i].count + bsum[blockIdx.x] : total;
    if (threadIdx.x == 0)
      s_off[kThreads] = i0 + kThreads < nsub ? rec[i0 + kThreads].count + bsum[blockIdx.x + 1]
                                             : total;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const unsigned long long cap = (unsigned long long)want;
  // a warp copies U spans at a time, the loads of all U in flight before
  // the stores (one span at a time left each warp waiting on one load ->
  // store chain, ncu: long-scoreboard stalls, 1.9 TB/s).  Measured on the
  // cfg5 batch (decode stage): U = 1 5.43 ms, 2 5.29, 4 5.17, 6 5.39, 8 5.40
  constexpr int U = EBZ_COPY_U, NWARP = kThreads / 32;
  const int nk = (int)(nsub - i0 < kThreads ? nsub - i0 : kThreads);
  const C* __restrict__ stage = reinterpret_cast<const C*>(tab.stage[f]) + i0 * (long long)kSpanCap;
  C* __restrict__ codes = reinterpret_cast<C*>(tab.codes[f]);
  for (int k0 = threadIdx.x >> 5; k0 < nk; k0 += U * NWARP) {
    unsigned long long off[U];
    int nw[U], nbytes[U], head[U];
    int iters = 0;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int k = k0 + u * NWARP;
      off[u] = k < nk ? s_off[k] : 0;
      unsigned long long lim = k < nk ? s_off[k + 1] : 0;
      if (lim > cap) lim = cap;
      nbytes[u] = off[u] < lim ? (int)(lim - off[u]) * (int)sizeof(C) : 0;
      // bytes: the staged span starts 8-byte aligned, the destination
      // anywhere; aligned destination words come from two source words
      int h = (int)((8 - ((uintptr_t)(codes + off[u]) & 7)) & 7);
      if (h > nbytes[u]) h = nbytes[u];
      head[u] = h;
      nw[u] = (nbytes[u] - h) >> 3;
      const int it = (nw[u] + 31) >> 5;
      iters = it > iters ? it : iters;
    }
    for (int it = 0; it < iters; ++it) {
      const int w = lane + 32 * it;
      unsigned long long lo[U], hi[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const unsigned long long* s64 = reinterpret_cast<const unsigned long long*>(
            stage + (k0 + u * NWARP) * (long long)kSpanCap) + (head[u] >> 3);
        lo[u] = w < nw[u] ? s64[w] : 0ull;
        hi[u] = (w < nw[u] && (head[u] & 7)) ? s64[w + 1] : 0ull;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int sh = (head[u] & 7) * 8;
        unsigned long long* d64 =
            reinterpret_cast<unsigned long long*>(reinterpret_cast<uint8_t*>(codes + off[u]) + head[u]);
        if (w < nw[u]) d64[w] = sh ? (lo[u] >> sh) | (hi[u] << (64 - sh)) : lo[u];
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint8_t* sb =
          reinterpret_cast<const uint8_t*>(stage + (k0 + u * NWARP) * (long long)kSpanCap);
      uint8_t* db = reinterpret_cast<uint8_t*>(codes + off[u]);
      if (lane < head[u]) db[lane] = sb[lane];
      const int t0 = head[u] + 8 * nw[u];
      if (lane < nbytes[u] - t0) db[t0 + lane] = sb[t0 + lane];
    }
  }
}

// exact bit-serial decoder (anomaly path), one thread
template <typename C>
__global__ void decode_serial_kernel(const __grid_constant__ DecTab tab, long long want) {
  const int f = blockIdx.x;
  const Tables* __restrict__ t = tab.t[f];
  const uint8_t* __restrict__ bytes = reinterpret_cast<const uint8_t*>(tab.wds[f]);
  const Budget bud{tab.nbits[f], tab.bitlen[f]};
  C* __restrict__ out = reinterpret_cast<C*>(tab.codes[f]);
  Info* info = tab.info[f];
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

// fresh decompress records: eb and K from the source record or the host
__global__ void dec_init_kernel(const __grid_constant__ DecTab tab, int nf) {
  const int f = threadIdx.x;
  if (f >= nf) return;
  Info z;
  memset(&z, 0, sizeof(Info));
  z.eb = tab.src[f] ? tab.src[f]->eb : tab.eb[f];
  z.n_unpred = tab.src[f] ? tab.src[f]->n_unpred : tab.k[f];
  *tab.info[f] = z;
  *tab.rlist[f] = 0;
}

// ------------------------------------------------------------ zero ranks
// Per-row count of code-0 symbols (a row = a line along axis 0), then an
// exclusive scan -> rowbase[r] = rank of the first verbatim value of row r.
__device__ __forceinline__ int zero_bytes(unsigned long long v) {
  // number of zero bytes in v
  const unsigned long long t = (v & 0x7f7f7f7f7f7f7f7full) + 0x7f7f7f7f7f7f7f7full;
  return 8 - __popcll((t | v) & 0x8080808080808080ull);
}

// One block per kRowsPerBlock rows: per-row zero counts (warp per row,
// 8 codes per 64-bit load), then a block-local exclusive scan ->
// rowbase[r] (within-block prefix) and rowblk[block] (block total, scanned by
// rows_top_kernel).  Consumers use rowbase[r] + rowblk[r / kRowsPerBlock].
struct RowTab {  // per-field pointers of a batched zero-rank pass
  const void* codes[kBatchMax];
  unsigned long long* rowbase[kBatchMax];
  unsigned long long* rowblk[kBatchMax];
  Info* info[kBatchMax];
};

// Few long rows (a single 2D field: 1800 rows of 3600 codes are 8 blocks of
// row_zero_kernel, 75 us): one warp per row over the whole GPU first, the
// counts parked in rowbase; row_zero_kernel<.., true> then only scans them.
template <typename C>
__global__ void __launch_bounds__(256)
row_count_kernel(const __grid_constant__ RowTab tab, long long nrows, long long nx) {
  const C* __restrict__ codes = reinterpret_cast<const C*>(tab.codes[blockIdx.y]);
  unsigned long long* __restrict__ rowbase = tab.rowbase[blockIdx.y];
  const int lane = threadIdx.x & 31;
  const long long r = (long long)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (r >= nrows) return;
  const C* row = codes + r * nx;
  unsigned int z = 0;
  if (sizeof(C) == 1 && nx % 8 == 0) {  // 8 codes per 64-bit load
    const unsigned long long* rw = reinterpret_cast<const unsigned long long*>(row);
    for (long long q = lane; q < nx / 8; q += 32) z += zero_bytes(__ldcs(rw + q));
  } else {
    for (long long x = lane; x < nx; x += 32) z += __ldcs(row + x) == 0;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) z += __shfl_xor_sync(EBZ_FULL, z, o);
  if (lane == 0) rowbase[r] = z;
}

template <typename C, bool COUNTED = false>
__global__ void __launch_bounds__(256)
row_zero_kernel(const __grid_constant__ RowTab tab, long long nrows, long long nx) {
  const C* __restrict__ codes = reinterpret_cast<const C*>(tab.codes[blockIdx.y]);
  unsigned long long* __restrict__ rowbase = tab.rowbase[blockIdx.y];
  unsigned long long* __restrict__ rowblk = tab.rowblk[blockIdx.y];
  __shared__ unsigned int s_cnt[kRowsPerBlock];
  __shared__ unsigned long long s_w[8];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const long long r0 = (long long)blockIdx.x * kRowsPerBlock;
  if (COUNTED) {
    const long long r = r0 + threadIdx.x;
    s_cnt[threadIdx.x] = r < nrows ? (unsigned int)rowbase[r] : 0u;
  } else if (nx <= 64) {
    const long long r = r0 + threadIdx.x;
    unsigned int z = 0;
    if (r < nrows) {
      const C* row = codes + r * nx;
      for (long long x = 0; x < nx; ++x) z += row[x] == 0;
    }
    s_cnt[threadIdx.x] = z;
  } else if (sizeof(C) == 1 && nx % 256 == 0) {
    // rows of whole 256-code blocks (one 8-byte word per lane each): the
    // warp's rows are read four at a time with every load in flight before
    // the reductions (one row per iteration left the kernel waiting on each
    // load: 2.2 TB/s)
    const unsigned long long* base = reinterpret_cast<const unsigned long long*>(codes);
    const long long wpr = nx / 8;  // words per row
    for (int k0 = w; k0 < kRowsPerBlock; k0 += 32) {
      unsigned int z[4] = {0u, 0u, 0u, 0u};
      for (long long q = lane; q < wpr; q += 32) {
        unsigned long long v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const long long r = r0 + k0 + 8 * u;
          v[u] = r < nrows ? __ldcs(base + r * wpr + q) : ~0ull;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) z[u] += zero_bytes(v[u]);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        unsigned int t = z[u];
#pragma unroll
        for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(EBZ_FULL, t, o);
        if (lane == 0) s_cnt[k0 + 8 * u] = t;
      }
    }
  } else {
    for (int k = w; k < kRowsPerBlock; k += 8) {
      const long long r = r0 + k;
      unsigned int z = 0;
      if (r < nrows) {
        const C* row = codes + r * nx;
        if (sizeof(C) == 1 && nx % 8 == 0) {  // 8 codes per 64-bit load
          const unsigned long long* rw = reinterpret_cast<const unsigned long long*>(row);
          for (long long q = lane; q < nx / 8; q += 32) z += zero_bytes(__ldcs(rw + q));
        } else if (sizeof(C) == 1 && nx % 4 == 0) {  // 4 codes per load (cfg3: nx = 500)
          const unsigned int* rw = reinterpret_cast<const unsigned int*>(row);
          for (long long q = lane; q < nx / 4; q += 32)
            z += zero_bytes(0xffffffff00000000ull | __ldcs(rw + q));
        } else {
          for (long long x = lane; x < nx; x += 32) z += __ldcs(row + x) == 0;
        }
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) z += __shfl_xor_sync(EBZ_FULL, z, o);
      if (lane == 0) s_cnt[k] = z;
    }
  }
  __syncthreads();
  unsigned long long total;
  const unsigned long long ex = block_exscan_u64<256>(s_cnt[threadIdx.x], s_w, total);
  if (r0 + threadIdx.x < nrows) rowbase[r0 + threadIdx.x] = ex;
  if (threadIdx.x == 0) rowblk[blockIdx.x] = total;
}

__global__ void __launch_bounds__(1024)
rows_top_kernel(const __grid_constant__ RowTab tab, long long nblk) {
  unsigned long long* __restrict__ rowblk = tab.rowblk[blockIdx.x];
  Info* info = tab.info[blockIdx.x];
  __shared__ unsigned long long s_w[32];
  const long long per = (nblk + 1023) / 1024;
  const long long lo = threadIdx.x * per;
  const long long hi = lo + per < nblk ? lo + per : nblk;
  unsigned long long c = 0;
  for (long long b = lo; b < hi; ++b) c += rowblk[b];
  unsigned long long total;
  unsigned long long run = block_exscan_u64<1024>(c, s_w, total);
  for (long long b = lo; b < hi; ++b) {
    const unsigned long long v = rowblk[b];
    rowblk[b] = run;
    run += v;
  }
  if (threadIdx.x == 0) {
    info->zeros_decoded = total;
    if (total != info->n_unpred) atomicOr(&info->status, ST_UNPRED_MISMATCH);
  }
}

}  // namespace

size_t decode_scratch_bytes(long long nbytes, int m) {
  const long long nbits = nbytes * 8;
  const long long nsub = nbits / kSubBits + 1;
  size_t tables = sizeof(Tables) + sizeof(int) * ((size_t)1 << m);
  tables = (tables + 255) & ~(size_t)255;
  // tables | records | block sums | staged spans (kSpanCap symbols each)
  const size_t recs = ((sizeof(SubRec) * (size_t)(nsub + 1) + 8 * (size_t)(nsub / kThreads + 2)) +
                       255) & ~(size_t)255;
  const size_t stage = (((size_t)nsub * kSpanCap * (m > 8 ? 2 : 1)) + 255) & ~(size_t)255;
  return tables + recs + stage + 8 * (2 * (size_t)nsub + 2) + 512;
}

// Per field: nbytes is the byte budget, or (dev_bitlen != nullptr) an upper
// bound used only to size the grid; the exact budget is then read on the
// device.  One launch per stage for all nf fields.
cudaError_t launch_decode_batch(const DecodeJob* jobs, int nf, int m, long long n, int sms,
                                cudaStream_t s) {
  (void)sms;
  if (nf < 1 || nf > kBatchMax) return cudaErrorInvalidValue;
  static KernelAttr attr8, attr16;
  cudaError_t e = kernel_smem(attr8, decode_sync_kernel<uint8_t>, kDecodeSmem);
  if (e == cudaSuccess) e = kernel_smem(attr16, decode_sync_kernel<uint16_t>, kDecodeSmem);
  if (e != cudaSuccess) return e;
  DecTab tab;
  long long grid = 1;
  size_t tables = sizeof(Tables) + sizeof(int) * ((size_t)1 << m);
  tables = (tables + 255) & ~(size_t)255;
  for (int f = 0; f < nf; ++f) {
    const DecodeJob& j = jobs[f];
    const long long nsub_cap = (long long)(((unsigned long long)j.nbytes * 8ull) / kSubBits + 1);
    tab.lengths[f] = j.lengths;
    tab.wds[f] = reinterpret_cast<const uint32_t*>(j.bits);
    tab.nbits[f] = (unsigned long long)j.nbytes * 8ull;
    tab.bitlen[f] = j.dev_bitlen;
    tab.t[f] = reinterpret_cast<Tables*>(j.scratch);
    tab.rec[f] = reinterpret_cast<SubRec*>(reinterpret_cast<char*>(j.scratch) + tables);
    tab.bsum[f] = reinterpret_cast<unsigned long long*>(tab.rec[f] + nsub_cap + 1);
    const size_t recs = ((sizeof(SubRec) * (size_t)(nsub_cap + 1) +
                          8 * (size_t)(nsub_cap / kThreads + 2)) + 255) & ~(size_t)255;
    tab.stage[f] = reinterpret_cast<char*>(j.scratch) + tables + recs;
    const size_t stage =
        (((size_t)nsub_cap * kSpanCap * (m > 8 ? 2 : 1)) + 255) & ~(size_t)255;
    tab.rlist[f] = reinterpret_cast<unsigned long long*>(reinterpret_cast<char*>(tab.stage[f]) +
                                                         stage);
    tab.info[f] = j.info;
    tab.codes[f] = j.codes;
    tab.src[f] = j.src;
    tab.eb[f] = j.eb;
    tab.k[f] = j.k;
    const unsigned long long nbits_max = (unsigned long long)j.nbytes * 8ull;
    const long long nsub_max =
        nbits_max == 0 ? 1 : (long long)((nbits_max + kSubBits - 1) / kSubBits);
    const long long g = (nsub_max + kThreads - 1) / kThreads;
    if (g > grid) grid = g;
  }
  dec_init_kernel<<<1, kBatchMax, 0, s>>>(tab, nf);
  decode_tables_kernel<<<nf, 1024, 0, s>>>(tab, m);
  if (n == 0) return cudaGetLastError();
  const dim3 g2((unsigned)grid, nf);
  const dim3 gc = g2;  // copy: the sync blocks' spans
  // repair: the list is dense; blocks past its length exit, longer lists loop
  const dim3 gr((unsigned)((grid + 7) / 8), nf);
  const size_t tsm = sizeof(SmemTables);
#define EBZ_DEC(C)                                                                  \
  decode_sync_kernel<C><<<g2, kThreads, kDecodeSmem, s>>>(tab, m);                  \
  for (int pass = 0; pass < 2; ++pass) {                                            \
    decode_check_kernel<<<g2, kThreads, 0, s>>>(tab);                               \
    decode_repair_kernel<C><<<gr, kThreads, tsm, s>>>(tab, m);                      \
    decode_relist_kernel<<<1, kBatchMax, 0, s>>>(tab, nf);                          \
  }                                                                                 \
  decode_verify_kernel<<<g2, kThreads, 0, s>>>(tab);                                \
  decode_top_kernel<<<nf, 1024, 0, s>>>(tab, n);                                    \
  decode_copy_kernel<C><<<gc, kThreads, 0, s>>>(tab, n);                            \
  decode_serial_kernel<C><<<nf, 1, 0, s>>>(tab, n);
  if (m > 8) {
    EBZ_DEC(uint16_t)
  } else {
    EBZ_DEC(uint8_t)
  }
#undef EBZ_DEC
  return cudaGetLastError();
}

cudaError_t launch_decode(const uint8_t* bits, long long nbytes, const uint8_t* lengths, int m,
                          long long n, void* codes, Info* info, unsigned long long* scratch,
                          size_t scratch_bytes, int sms, cudaStream_t s,
                          const unsigned long long* dev_bitlen) {
  (void)scratch_bytes;
  // the caller initialised the record (eb / K) already: re-derive it from itself
  DecodeJob j;
  j.bits = bits;
  j.nbytes = nbytes;
  j.lengths = lengths;
  j.codes = codes;
  j.info = info;
  j.scratch = scratch;
  j.dev_bitlen = dev_bitlen;
  j.src = info;
  j.eb = 0.0;
  j.k = 0;
  return launch_decode_batch(&j, 1, m, n, sms, s);
}

size_t rowblk_words(long long nrows) { return (size_t)(nrows / kRowsPerBlock + 2); }

cudaError_t launch_rowbase_batch(const void* const* codes, unsigned long long* const* rowbase,
                                 unsigned long long* const* rowblk, Info* const* info, int nf,
                                 int m, long long n, long long nx, cudaStream_t s) {
  if (nf < 1 || nf > kBatchMax) return cudaErrorInvalidValue;
  RowTab tab;
  for (int f = 0; f < nf; ++f) {
    tab.codes[f] = codes[f];
    tab.rowbase[f] = rowbase[f];
    tab.rowblk[f] = rowblk[f];
    tab.info[f] = info[f];
  }
  const long long nrows = n / nx;
  const long long nblk = (nrows + kRowsPerBlock - 1) / kRowsPerBlock;
  const dim3 grid((unsigned)nblk, nf);
  if (nblk * nf < 128 && nx >= 1024) {  // few long rows: count them GPU-wide first
    const dim3 gcount((unsigned)((nrows + 7) / 8), nf);
    if (m > 8) {
      row_count_kernel<uint16_t><<<gcount, 256, 0, s>>>(tab, nrows, nx);
      row_zero_kernel<uint16_t, true><<<grid, 256, 0, s>>>(tab, nrows, nx);
    } else {
      row_count_kernel<uint8_t><<<gcount, 256, 0, s>>>(tab, nrows, nx);
      row_zero_kernel<uint8_t, true><<<grid, 256, 0, s>>>(tab, nrows, nx);
    }
  } else if (m > 8) {
    row_zero_kernel<uint16_t><<<grid, 256, 0, s>>>(tab, nrows, nx);
  } else {
    row_zero_kernel<uint8_t><<<grid, 256, 0, s>>>(tab, nrows, nx);
  }
  rows_top_kernel<<<nf, 1024, 0, s>>>(tab, nblk);
  return cudaGetLastError();
}

cudaError_t launch_rowbase(const void* codes, int m, long long n, long long nx,
                           unsigned long long* rowbase, unsigned long long* rowblk,
                           unsigned long long n_unpred, Info* info, cudaStream_t s) {
  (void)n_unpred;
  return launch_rowbase_batch(&codes, &rowbase, &rowblk, &info, 1, m, n, nx, s);
}
