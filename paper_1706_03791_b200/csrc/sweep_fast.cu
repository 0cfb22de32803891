// sweep_fast.cu -- register-systolic hyperplane wavefront for 2D / 3D grids
// (float32 elements, layers n in {1, 2}): the hot path of compress_scan and
// decompress_scan (ebzip/_kernels.py:48-105).
//
// Geometry.  A "row" is a line along axis 0 (x, scan-fastest).  A warp task
// owns a patch of 32 rows -- 32 (y) for 2D, 8 (y) x 4 (z) for 3D -- and walks
// x.  Lane (a, b) sits at row (y0 + a, z0 + b) and processes
//     x = S - (a + b)          at warp step S,
// i.e. the lanes form a 2-D systolic array skewed along the hyperplane
// x + y + z = const, so every in-patch dependency was produced one or more
// steps earlier by a neighbouring lane:
//   * values of row y-1 at column x arrive by __shfl_up(.., 1),
//   * values of plane z-1 at column x arrive by __shfl_up(.., 8),
//   * older columns (x-1 .. x-n) stay in registers (a (n+1)^d history cube;
//     the 16-step chunk is fully unrolled, so the history shift is register
//     renaming).
//
// Patch faces (rows y0-n..y0-1 and planes z0-n..z0-1) cross between warps
// through global memory as 64-bit tagged words (the binary64 value with the
// launch epoch in its 29 always-zero low mantissa bits, see kTagBits)
// written by the producer's face lanes at the step they are computed.  The
// consumer's boundary lanes load their face values DP steps ahead into a
// register FIFO and accept a word only when its tag equals this launch's
// epoch -- no progress counters, no fences, no chunk-level waits: a patch can
// trail its producer by just the producer's lane skew plus the prefetch
// distance.  A single aligned 64-bit store/load is atomic, so value and tag
// are always seen together.  Patches are handed out by an atomic ticket in
// hyperplane (Y + Z) order, so a task only ever waits on lower tickets.
//
// Memory traffic.  Inputs (values / codes) are staged per 16-column chunk
// into shared tiles with cp.async; outputs (codes / reconstructions) leave
// through shared tiles with row-coalesced stores.  Per point in compress:
// 4 B read, 1 B code written; decompress: 1 B read, 4 B written; face rows
// (11/32 of rows in 3D, 1/32 in 2D) additionally write 8 B.  The code
// histogram is a separate RLE pass (hist.cu), off the wavefront.
//
// Arithmetic is bit-identical to the reference: the stencil sum runs in the
// reference's term order (lexicographic offsets, axis 0 slowest) in binary64
// without contraction; missing neighbours are zeros, which reproduces the
// boundary-reduced stencils exactly (up to the sign of a zero prediction,
// which never changes a code or a stored value); points with a coordinate
// equal to 1 use the n = 1 stencil when n = 2 (eff = min(n, min coord)).
// The float32 rounding of reconstructions is round-to-nearest-even, the
// reference's float32 cast: the hardware conversion (F2F) in compress, the
// binary64 bit pattern for f32-normal results in decompress (hardware
// conversion otherwise) -- identical values either way.
#include <cstdlib>

#include "ebz_common.cuh"

namespace {

constexpr int CH = 16;        // steps per chunk (input/output staging)
constexpr int RS = 4;         // tile ring slots (chunks)
constexpr int RX = CH * RS;   // tile ring columns (power of two)
constexpr int WPB = 4;        // warps per block
// verbatim-value ring per row (decompress): a chunk consumes <= CH values,
// so keeping [cursor, cursor + 2 CH) loaded means every value arrives at
// least one chunk before it is used
constexpr int kURing = 2 * CH;
// 3D n = 1 (the batched decompress sweep): 40 slots -- refills in 16-byte
// aligned groups keep at most 2 CH + 3 values ahead of the cursor and 3
// behind it, so no live value is overwritten (measured: 2D single fields are
// slower with it, so they keep the 32-slot ring and scalar refills)
constexpr int kURingV = 2 * CH + 8;
static_assert(kURingV % 4 == 0 && kURingV >= 2 * CH + 6, "verbatim ring too small");

template <int D> struct Patch;
template <> struct Patch<2> { static constexpr int PY = 32, PZ = 1; };
template <> struct Patch<3> { static constexpr int PY = 8, PZ = 4; };

struct FastArgs {
  SweepArgs s;
  const unsigned int* tasks;  // task -> Y | Z << 16 (hyperplane order)
  int npy, npz;
  int nf;                     // fields in this launch (FieldTable entries)
};

// --- compile-time stencil ---------------------------------------------------
__host__ __device__ constexpr int cbin(int n, int k) {
  return k == 0 ? 1 : (n == 2 ? (k == 1 ? 2 : 1) : 1);
}
__host__ __device__ constexpr int coef(int n, int kx, int ky, int kz) {
  return -(((kx + ky + kz) & 1) ? -1 : 1) * cbin(n, kx) * cbin(n, ky) * cbin(n, kz);
}

template <int NN, int NB, int NA, int NC>
__device__ __forceinline__ double stencil_sum(const double (&H)[NB][NA][NC]) {
  // H[b][a][c] = value at (z-b, y-a, x-c); terms in (kx, ky, kz) lexicographic
  // order (x slowest): c outermost, then a, then b.
  double acc = 0.0;
  bool first = true;
#pragma unroll
  for (int c = 0; c <= NN; ++c)
#pragma unroll
    for (int a = 0; a <= NN; ++a)
#pragma unroll
      for (int b = 0; b <= (NB > 1 ? NN : 0); ++b) {
        if (a == 0 && b == 0 && c == 0) continue;
        const int k = coef(NN, c, a, b);
        const double v = H[b][a][c];
        if (first) {
          acc = k == 1 ? v : (k == -1 ? -v : __dmul_rn((double)k, v));
          first = false;
        } else if (k == 1) {
          acc = __dadd_rn(acc, v);
        } else if (k == -1) {
          acc = __dsub_rn(acc, v);
        } else {
          acc = __dadd_rn(acc, __dmul_rn((double)k, v));  // |k| = 2, 4, 8: exact
        }
      }
  return acc;
}

// --- cp.async helpers ----------------------------------------------------------
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem),
               "r"(src_bytes));
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem, int src_bytes) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(s), "l"(gmem),
               "r"(src_bytes));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::); }
__device__ __forceinline__ void cp_wait_1() { asm volatile("cp.async.wait_group 1;\n" ::); }
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, int src_bytes) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem),
               "r"(src_bytes));
}

// per-step shared-tile accesses through 32-bit shared-window addresses
// (generic pointers made the compiler rebuild the window base every step)
__device__ __forceinline__ unsigned smem_addr(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
// an address the compiler cannot rematerialise: it keeps the register
// instead of rebuilding the shared-window base (S2UR CgaCtaId, ULEA) at
// every access
__device__ __forceinline__ unsigned pinned(unsigned a) {
  asm volatile("" : "+r"(a));
  return a;
}
__device__ __forceinline__ float lds_f32(unsigned a) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ double lds_f64(unsigned a) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ int lds_code(unsigned a, bool wide) {
  unsigned v;
  if (wide) asm volatile("ld.shared.u16 %0, [%1];" : "=r"(v) : "r"(a));
  else asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(a));
  return (int)v;
}
__device__ __forceinline__ void sts_f32(unsigned a, float v) {
  asm volatile("st.shared.f32 [%0], %1;" ::"r"(a), "f"(v));
}
__device__ __forceinline__ void sts_code(unsigned a, int v, bool wide) {
  if (wide) asm volatile("st.shared.u16 [%0], %1;" ::"r"(a), "r"(v));
  else asm volatile("st.shared.u8 [%0], %1;" ::"r"(a), "r"(v));
}

// predicated face store (no branch around it: the step stays one basic block)
__device__ __forceinline__ void st_face_if(unsigned long long* p, unsigned long long w, bool pred) {
  asm volatile("{ .reg .pred q; setp.ne.u32 q, %2, 0; @q st.global.cg.u64 [%0], %1; }"
               ::"l"(p), "l"(w), "r"((unsigned)pred) : "memory");
}
// the same from the two halves of the tagged word (no 64-bit copy of the value)
__device__ __forceinline__ void st_face2_if(unsigned long long* p, unsigned lo, unsigned hi,
                                            bool pred) {
  asm volatile("{ .reg .pred q; setp.ne.u32 q, %3, 0; @q st.global.cg.v2.b32 [%0], {%1, %2}; }"
               ::"l"(p), "r"(lo), "r"(hi), "r"((unsigned)pred) : "memory");
}
// predicated shared load into v (v keeps its value when the predicate is off)
__device__ __forceinline__ void lds_f64_if(double& v, unsigned a, bool pred) {
  asm volatile("{ .reg .pred q; setp.ne.u32 q, %2, 0; @q ld.shared.f64 %0, [%1]; }"
               : "+d"(v) : "r"(a), "r"((unsigned)pred));
}
__device__ __forceinline__ unsigned long long ld_face(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.global.cg.u64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}

// tagged face words (ebz_common.cuh kTagBits)
__device__ __forceinline__ bool face_ok(unsigned long long w, unsigned ep) {
  return ((unsigned)w & kTagMask) == ep;
}
__device__ __forceinline__ double face_val(unsigned long long w) {
  return __longlong_as_double((long long)(w & ~(unsigned long long)kTagMask));
}
__device__ __forceinline__ unsigned long long face_word(double v, unsigned ep) {
  return (unsigned long long)__double_as_longlong(v) | ep;
}

template <int D, int N> struct Cfg {
  static constexpr int PY = Patch<D>::PY, PZ = Patch<D>::PZ;
  static constexpr int NB = D == 3 ? N + 1 : 1;     // z history depth
  static constexpr int SMAX = PY - 1 + PZ - 1;      // max lane skew
  static constexpr int NSY = N * NB;                // Y-face streams (la == 0 lanes)
  static constexpr int NSZ = NB - 1;                // Z-face streams (lb == 0 lanes)
  static constexpr int NS = NSY + NSZ;
  static constexpr int DP = N == 1 ? 4 : 2;         // face prefetch distance (steps)
  static constexpr int IN_STRIDE_F = D == 2 ? 64 : 68;   // floats per tile row
  static constexpr int IN_STRIDE_B = D == 2 ? 64 : 80;   // bytes per u8 tile row
  static constexpr int OUT_LAG = (SMAX + CH - 1) / CH;  // x-chunks still being written
  // output ring: OUT_LAG + 1 live chunks, rounded up to a power of two
  static constexpr int RSO = OUT_LAG + 1 <= 2 ? 2 : 4;
  static constexpr int RXO = CH * RSO;
  static constexpr int OUT_STRIDE_F = D == 2 ? 64 : RXO + 4;   // floats per out row
  static constexpr int OUT_STRIDE_B = D == 2 ? 64 : RXO + 16;  // codes per out row
};

template <int D, int N, typename C, bool COMPRESS>
struct Smem {
  typedef Cfg<D, N> K;
  static constexpr int IN_BYTES = COMPRESS ? 32 * K::IN_STRIDE_F * 4
                                           : 32 * K::IN_STRIDE_B * (int)sizeof(C);
  static constexpr int OUT_BYTES = COMPRESS ? 32 * K::OUT_STRIDE_B * (int)sizeof(C)
                                            : 32 * K::OUT_STRIDE_F * 4;
  static constexpr int IN_OFF = 0;
  static constexpr int OUT_OFF = ((IN_BYTES + 15) / 16) * 16;
  // decompress: per-row ring of upcoming verbatim values (kURing floats)
  static constexpr int RING_OFF = OUT_OFF + ((OUT_BYTES + 15) / 16) * 16;
  static constexpr int RING_BYTES =
      COMPRESS ? 0 : 32 * ((D == 3 && N == 1) ? kURingV : kURing) * 4;
  // 3D n = 1 decompress: staged patch-face words of two 8-step blocks
  // (Y 36 | corner 8 | Z 64 words each), see sweep_fast_kernel
  static constexpr int FST_OFF = RING_OFF + RING_BYTES;
  static constexpr int FST_WORDS = 36 + 8 + 64;
  static constexpr int FST_BYTES = (!COMPRESS && D == 3 && N == 1) ? 2 * FST_WORDS * 8 : 0;
  static constexpr int PER_WARP = FST_OFF + FST_BYTES;
};

// resident blocks per SM the register allocation must allow.  3D n = 1:
// 4 (128 registers; decompress measured 3% faster than at 96 registers /
// 5 blocks, where ptxas rematerialises shared addresses every step; a
// 102-register compress cap measured slower for the same reason).  The
// others keep the allocation the compiler picks on its own.
template <int D, int N, bool COMPRESS> struct MinBlocks {
  static constexpr int value =
      D == 3 ? (N == 1 ? 4 : 3)
             : (N == 1 ? (COMPRESS ? 7 : 8) : (COMPRESS ? 4 : 7));
};

// REC (compress only): also store every point's reconstruction into the
// field's recon array -- the full output of the reference's compress_scan
// (_kernels.py:71,77), for the C seam ebz_compress_scan; the pipelines run
// without it
template <int D, int N, typename C, bool COMPRESS, bool REC = false, bool TR = false>
__global__ void __launch_bounds__(32 * WPB, (MinBlocks<D, N, COMPRESS>::value))
sweep_fast_kernel(const __grid_constant__ FastArgs fa, const __grid_constant__ FieldTable ft) {
  typedef Cfg<D, N> K;
  typedef Smem<D, N, C, COMPRESS> SM;
  constexpr int PY = K::PY, PZ = K::PZ, NB = K::NB, NA = N + 1, NC = N + 1;
  // 3D, n = 1 decompress: the warp's 16 face streams (8 Y rows, 8 Z rows)
  // get one loader lane each, prefetched 8 steps ahead, and reach their
  // consumers by shuffles (measured: faster for decompress, not for
  // compress).  Otherwise every consumer lane loads its own NS streams.
  // 3D, n = 1 decompress (STG): the face words of each 8-step block are
  // staged in shared memory a block ahead -- Y and Z faces are contiguous
  // runs in the skew-major blocks (36 + 64 words), the corner word eight
  // single words -- tag-checked once per block and read by the consumer
  // lanes with one shared load each (measured: the former per-step loader
  // lanes + 8-step register FIFO + shuffle distribution cost ~34 issued
  // instructions and 6 shuffle wavefronts per point-step in an L1-bound kernel)
  constexpr bool STG = D == 3 && N == 1 && !COMPRESS;
  constexpr bool DIST = false;
  constexpr int NS = K::NS, DP = STG ? 8 : K::DP;
  constexpr int NSL = STG ? 1 : NS;  // stream slots per lane
  const SweepArgs& a = fa.s;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int la = lane % PY, lb = lane / PY;  // (a, b)
  const int sig = la + lb;
  unsigned char* wbase = smem_raw + warp * SM::PER_WARP;
  unsigned char* in_tile = wbase + SM::IN_OFF;
  unsigned char* out_tile = wbase + SM::OUT_OFF;
  const int nsym = 1 << a.m;
  // (code - center) exactly, without a conversion or a table: the binary64
  // with bit pattern 0x43300000:code is 2^52 + code, minus 2^52 + center
  // (a 256-entry shared table was measured: its random 8-byte lookups cost
  // bank-conflicted wavefronts in an L1-bound kernel)
  const double c52 = 0x1p52 + (double)a.center;

  const int nx = (int)a.dims[0], ny = (int)a.dims[1], nz = D == 3 ? (int)a.dims[2] : 1;
  const int npy = fa.npy, npz = fa.npz;
  const int nf = fa.nf;
  const int ntasks = npy * npz * nf;
  const int steps_total = nx + K::SMAX;
  const int nchunks = (steps_total + CH - 1) / CH;
  const unsigned epoch = a.epoch;
  const unsigned long long tag = epoch;  // tagged 0.0 (outside the domain)
  const bool al16_in = COMPRESS ? (nx % 4 == 0) : ((nx * (int)sizeof(C)) % 16 == 0);

  for (;;) {
    unsigned int tk = 0;
    if (lane == 0) tk = atomicAdd(a.ticket, 1u);
    tk = __shfl_sync(EBZ_FULL, tk, 0);
    if ((int)tk >= ntasks) break;
    sched_jitter(a.jitter, tk, 0);  // test hook: per task here (single fields are latency-bound)
    // ticket -> (task of the single-field order, field): every field advances
    // through the same hyperplane order, so a task waits only on lower tickets
    const int fi = (int)(tk % (unsigned)nf);
    const FieldRef& fr = ft.f[fi];
    // per-field interval count (batched --auto-m trials), else the launch's
    const int center = ft.center[fi] ? ft.center[fi] : a.center;
    const double lim = (double)(center - 1);  // |k| <= center - 1
    const double eb = fr.info->eb;
    if (!(eb > 0.0)) continue;  // whole field skipped; the host reports the bound
    const double two_eb = __dmul_rn(2.0, eb);
    const double inv = 1.0 / two_eb;
    const bool fast_ok = isfinite(inv) && inv > 0.0 && two_eb >= 0x1p-1000 &&
                         inv >= 0x1p-1000 && inv <= 0x1p1000;
    // fast-path margin, -1 (never met, NaN included) without a usable reciprocal
    const double guard = fast_ok ? 0.5 - 0x1p-30 : -1.0;
    const int tre = (COMPRESS && TR) ? eb_exponent(eb) : kNoTrunc;  // opt-in truncation
    const float* values = reinterpret_cast<const float*>(fr.values);
    float* recon = reinterpret_cast<float*>(fr.recon);
    C* codes = reinterpret_cast<C*>(fr.codes);
    const float* unpred = reinterpret_cast<const float*>(fr.unpred);
    const unsigned long long n_unpred = COMPRESS ? 0ull : fr.info->n_unpred;
    unsigned long long* yface = fr.yface;
    unsigned long long* zface = fr.zface;
    int bad = 0;
    unsigned hmax = 0;  // decompress: max |high word| of the stored values
    const unsigned int tv = fa.tasks[tk / (unsigned)nf];
    const int PYi = (int)(tv & 0xffff), PZi = (int)(tv >> 16);
    const int y0 = PYi * PY, z0 = PZi * PZ;
    const int y = y0 + la, z = z0 + lb;
    const bool rv = y < ny && z < nz;
    const long long rowi = (long long)z * ny + y;
    // face rows this lane writes (tagged); 32-bit word offsets (face buffers
    // hold < 2^31 words, checked by the host), -1 = none.
    // 3D n = 1 (SKEW): skew-major face blocks -- the Y face of patch (PY, PZ)
    // is a block of (nx + 4) x 4 words with face row zz = z - z0 at column x
    // in word 4 (x + zz) + zz, the Z face a block of (nx + 8) x 8 words with
    // zz = y - y0 in word 8 (x + zz) + zz.  A face's producer lanes all
    // compute x + zz = S - const at step S and a stream's consumers read
    // x + zz = S + const, so each warp-wide face access is one run of
    // consecutive words.  Otherwise: one row of nx words per face row.
    constexpr bool SKEW = D == 3 && N == 1;
    const int ybw = (nx + 4) * 4, zbw = (nx + 8) * 8;  // SKEW block words
    auto yblk = [&](int PY_, int PZ_) { return (PY_ * npz + PZ_) * ybw; };
    auto zblk = [&](int PY_, int PZ_) { return (PY_ * npz + PZ_) * zbw; };
    int wyo = -1, wzo = -1;
    if (SKEW) {
      if (rv && la == PY - 1) wyo = yblk(PYi, PZi) + 5 * lb;
      if (rv && lb == PZ - 1) wzo = zblk(PYi, PZi) + 9 * la;
    } else {
      if (rv && la >= PY - N) wyo = ((PYi * N + la - (PY - N)) + npy * N * z) * nx;
      if (D == 3 && rv && lb >= PZ - N) wzo = ((PZi * N + lb - (PZ - N)) * ny + y) * nx;
    }
    // word of column x of a SKEW Y stream of row zz (zz = -1: the last face
    // row of patch (PY - 1, PZ - 1)) / Z stream of row zz; the address is
    // base + (x << shift) with shift 2 (Y) or 3 (Z)
    auto yskew = [&](int zz) { return zz >= 0 ? yblk(PYi - 1, PZi) + 5 * zz : yblk(PYi - 1, PZi - 1) + 15; };
    // face streams this lane reads: la == 0 -> rows (y0 - aa, z - b);
    // lb == 0 -> rows (y, z0 - b).  Stream s reads base_s[ro[s] + x] for
    // (unsigned)x < rn[s]; rn = 0 outside the domain (zeros).
    int ro[NS > 0 ? NS : 1], rn[NS > 0 ? NS : 1], rsh[NS > 0 ? NS : 1];
#pragma unroll
    for (int b = 0; b < NB; ++b)
#pragma unroll
      for (int aa = 1; aa <= N; ++aa) {
        const int s = b * N + (aa - 1);
        const bool ok = rv && la == 0 && y0 - aa >= 0 && z - b >= 0;
        ro[s] = !ok ? 0 : (SKEW ? yskew(lb - b) : (((PYi - 1) * N + N - aa) + npy * N * (z - b)) * nx);
        rn[s] = ok ? nx : 0;
        rsh[s] = SKEW ? 2 : 0;
      }
#pragma unroll
    for (int b = 1; b < NB; ++b) {
      const bool ok = rv && lb == 0 && z0 - b >= 0;
      ro[K::NSY + b - 1] = !ok ? 0 : (SKEW ? zblk(PYi, PZi - 1) + 9 * la : (((PZi - 1) * N + N - b) * ny + y) * nx);
      rn[K::NSY + b - 1] = ok ? nx : 0;
      rsh[K::NSY + b - 1] = SKEW ? 3 : 0;
    }
    // loader lanes (DIST): lane L < 8 loads Y row (y0 - 1, z0 + L/2 - L%2) for
    // consumer lane (0, L/2); lane 8 + l loads Z row (y0 + l, z0 - 1) for
    // consumer lane (l, 0); the stream's x follows its consumer's skew
    const unsigned long long* l_base = yface;
    int l_sig = 0;
    if (DIST) {
      if (lane < 8) {
        const int cb = lane >> 1, b = lane & 1;
        l_sig = cb;
        l_base = yface;
        const bool ok = y0 < ny && z0 + cb < nz && y0 >= 1 && z0 + cb - b >= 0;
        ro[0] = !ok ? 0 : (SKEW ? yskew(cb - b) : ((PYi - 1) + npy * (z0 + cb - b)) * nx);
        rn[0] = ok ? nx : 0;
        rsh[0] = SKEW ? 2 : 0;
      } else if (lane < 16) {
        const int l = lane - 8;
        l_sig = l;
        l_base = zface;
        const bool ok = y0 + l < ny && z0 < nz && PZi >= 1;
        ro[0] = !ok ? 0 : (SKEW ? zblk(PYi, PZi - 1) + 9 * l : ((PZi - 1) * ny + y0 + l) * nx);
        rn[0] = ok ? nx : 0;
        rsh[0] = SKEW ? 3 : 0;
      } else {
        ro[0] = 0;
        rn[0] = 0;
        rsh[0] = 0;
      }
    }
    auto face_ptr = [&](int s) -> const unsigned long long* {
      if (DIST) return l_base + ro[0];
      return (s < K::NSY ? yface : zface) + ro[s];
    };
    const int fsig = DIST ? l_sig : sig;  // skew of the streams this lane loads
    // prefetch FIFO: fifo[s][j] holds the word for x = (step with st%DP==j)
    unsigned long long fifo[NSL > 0 ? NSL : 1][DP];
    if (!STG) {
#pragma unroll
      for (int s = 0; s < NSL; ++s)
#pragma unroll
        for (int j = 0; j < DP; ++j) {
          const int xx = j - fsig;
          fifo[s][j] = (unsigned)xx < (unsigned)rn[s] ? ld_face(face_ptr(s) + (xx << rsh[s])) : tag;
        }
    }
    // per-lane shared-memory rows
    const float* in_f = reinterpret_cast<const float*>(in_tile) + lane * K::IN_STRIDE_F;
    const C* in_c = reinterpret_cast<const C*>(in_tile) + lane * K::IN_STRIDE_B;
    C* out_c = reinterpret_cast<C*>(out_tile) + lane * K::OUT_STRIDE_B;
    float* out_f = reinterpret_cast<float*>(out_tile) + lane * K::OUT_STRIDE_F;
    const unsigned a_in_f = pinned(smem_addr(in_f)), a_in_c = pinned(smem_addr(in_c));
    // decompress code tile: the two 16-code slots of the rows of odd lb are
    // swapped (column ^ 16), which halves the bank conflicts of the skewed
    // per-step code reads (row stride 80 bytes: 4 -> 2.6 wavefronts)
    const int swz = (!COMPRESS && D == 3) ? (((lane / PY) & 1) * CH) : 0;
    const unsigned a_out_c = pinned(smem_addr(out_c)), a_out_f = pinned(smem_addr(out_f));
    constexpr bool WIDE = sizeof(C) == 2;
    // face rows this lane writes, as pointers (null = none)
    unsigned long long* const wyp = wyo >= 0 ? yface + wyo : nullptr;
    unsigned long long* const wzp = (D == 3 && wzo >= 0) ? zface + wzo : nullptr;
    const bool wy_ok = wyo >= 0, wz_ok = D == 3 && wzo >= 0;
    // face streams this lane reads, as pointers
    const unsigned long long* sp[NSL > 0 ? NSL : 1];
#pragma unroll
    for (int q = 0; q < NSL; ++q) sp[q] = face_ptr(q);

    // ---- STG: staged face blocks.  Block b covers steps [8b, 8b + 8) and
    // holds, in buffer b & 1: Y words [32b - 4, 32b + 32) of the Y face of
    // patch (PY - 1, PZ) (consumer (0, lb) reads word 4S + lb and, for lb > 0,
    // 4(S - 1) + lb - 1), the corner words 32b + 15 + 4i of patch
    // (PY - 1, PZ - 1) (consumer (0, 0): 4S + 15) and Z words [64b, 64b + 64)
    // of patch (PY, PZ - 1) (consumer (la, 0): 8S + la).  Words outside the
    // domain (x < 0, x >= nx, rows past the grid, no neighbour patch) are
    // zeros, never loaded or checked.
    unsigned long long* const fst =
        reinterpret_cast<unsigned long long*>(wbase + SM::FST_OFF);
    const bool hY = PYi > 0, hZ = PZi > 0, hC = PYi > 0 && PZi > 0;
    const unsigned long long* const gY = yface + (hY ? yblk(PYi - 1, PZi) : 0);
    const unsigned long long* const gC = yface + (hC ? yblk(PYi - 1, PZi - 1) : 0);
    const unsigned long long* const gZ = zface + (hZ ? zblk(PYi, PZi - 1) : 0);
    // this lane's staged words: Y pair (lanes 0-17), corner (lanes 18-25), Z pair (all)
    auto y_word_ok = [&](int w) {
      const int zz = w & 3, xx = (w >> 2) - zz;
      return hY && w >= 0 && w < ybw && (unsigned)xx < (unsigned)nx && z0 + zz < nz;
    };
    auto z_word_ok = [&](int w) {
      const int zz = w & 7, xx = (w >> 3) - zz;
      return hZ && w >= 0 && w < zbw && (unsigned)xx < (unsigned)nx && y0 + zz < ny;
    };
    // blocks whose every staged word lies inside the rows (b >= 1 and
    // 8b + 8 <= nx): each lane's five validity flags are task constants, one
    // packed register (the per-word index tests were ~100 issued
    // instructions per 8-step block)
    unsigned vmask = 0;
    if (STG) {
      const int zy = (2 * lane) & 3, zz8 = (2 * lane) & 7;
      vmask = (unsigned)(lane < 18 && hY && z0 + zy < nz) | (unsigned)(lane < 18 && hY && z0 + zy + 1 < nz) << 1 |
              (unsigned)(lane >= 18 && lane < 26 && hC) << 2 | (unsigned)(hZ && y0 + zz8 < ny) << 3 |
              (unsigned)(hZ && y0 + zz8 + 1 < ny) << 4;
    }
    auto stage_issue = [&](int b) {
      unsigned long long* buf = fst + (b & 1) * SM::FST_WORDS;
      if (lane < 18) {
        const int w = 32 * b - 4 + 2 * lane;
        if (hY && w >= 0 && w + 1 < ybw) cp_async16(buf + 2 * lane, gY + w, 16);
      } else if (lane < 26) {
        const int i = lane - 18, w = 32 * b + 15 + 4 * i;
        if (hC && w < ybw) cp_async8(buf + 36 + i, gC + w, 8);
      }
      const int wz = 64 * b + 2 * lane;
      if (hZ && wz + 1 < zbw) cp_async16(buf + 44 + 2 * lane, gZ + wz, 16);
    };
    // after the copies landed: check the tags of this lane's words (polling
    // the words a producer has not written yet), store them untagged
    auto stage_settle = [&](int b) {
      unsigned long long* buf = fst + (b & 1) * SM::FST_WORDS;
      const int wy = 32 * b - 4 + 2 * lane, wc = 32 * b + 15 + 4 * (lane - 18),
                wz = 64 * b + 2 * lane;
      bool yv0 = vmask & 1, yv1 = vmask & 2, cv = vmask & 4, zv0 = vmask & 8, zv1 = vmask & 16;
      if (!(b >= 1 && 8 * b + 8 <= nx)) {
        yv0 = lane < 18 && y_word_ok(wy);
        yv1 = lane < 18 && y_word_ok(wy + 1);
        cv = lane >= 18 && lane < 26 && hC && wc < ybw && (unsigned)(8 * b + lane - 18) < (unsigned)nx;
        zv0 = z_word_ok(wz);
        zv1 = z_word_ok(wz + 1);
      }
      unsigned long long w0 = tag, w1 = tag, w2 = tag, w3 = tag, w4 = tag;
      if (yv0) w0 = buf[2 * lane];
      if (yv1) w1 = buf[2 * lane + 1];
      if (cv) w2 = buf[36 + lane - 18];
      if (zv0) w3 = buf[44 + 2 * lane];
      if (zv1) w4 = buf[45 + 2 * lane];
      bool miss = !face_ok(w0, epoch) || !face_ok(w1, epoch) || !face_ok(w2, epoch) ||
                  !face_ok(w3, epoch) || !face_ok(w4, epoch);
      if (__any_sync(EBZ_FULL, miss)) {
        for (unsigned ns = 16;; ns = ns < 256 ? 2 * ns : ns) {
          if (miss) {
            if (!face_ok(w0, epoch)) w0 = ld_face(gY + wy);
            if (!face_ok(w1, epoch)) w1 = ld_face(gY + wy + 1);
            if (!face_ok(w2, epoch)) w2 = ld_face(gC + wc);
            if (!face_ok(w3, epoch)) w3 = ld_face(gZ + wz);
            if (!face_ok(w4, epoch)) w4 = ld_face(gZ + wz + 1);
            miss = !face_ok(w0, epoch) || !face_ok(w1, epoch) || !face_ok(w2, epoch) ||
                   !face_ok(w3, epoch) || !face_ok(w4, epoch);
          }
          if (!__any_sync(EBZ_FULL, miss)) break;
          __nanosleep(ns);
        }
      }
      double* db = reinterpret_cast<double*>(buf);
      if (lane < 18) {
        db[2 * lane] = face_val(w0);
        db[2 * lane + 1] = face_val(w1);
      } else if (lane < 26) {
        db[36 + lane - 18] = face_val(w2);
      }
      db[44 + 2 * lane] = face_val(w3);
      db[45 + 2 * lane] = face_val(w4);
      __syncwarp();
    };
    // consumer addresses within a staged buffer (words): Y (b = 0) 4 jj + lb + 4;
    // Y (b = 1) 4 jj + lb - 1, or the corner 36 + jj for lb = 0; Z 44 + 8 jj + la
    const unsigned a_fst = pinned(smem_addr(fst));

    // history cube: H[b][a][c] = r(z-b, y-a, x-c)
    double H[NB][NA][NC];
#pragma unroll
    for (int b = 0; b < NB; ++b)
#pragma unroll
      for (int aa = 0; aa < NA; ++aa)
#pragma unroll
        for (int c = 0; c < NC; ++c) H[b][aa][c] = 0.0;

    // decompress: verbatim values of this row in scan order, staged through
    // the ring; uload = first value not yet requested
    // Value u lives in ring slot u % RING; rc / rl track the slots of ucur
    // and uload.  3D n = 1 with a 16-byte aligned verbatim array: refills are
    // aligned 4-value groups (one sector request per 4 values instead of 1).
    constexpr int RING = (D == 3 && N == 1) ? kURingV : kURing;
    unsigned long long ucur = 0, ustart = 0, uload = 0;
    float* ring = reinterpret_cast<float*>(wbase + SM::RING_OFF) + lane * RING;
    const unsigned a_ring = pinned(smem_addr(ring));
    const bool uvec = RING == kURingV && (reinterpret_cast<uintptr_t>(unpred) & 15) == 0;
    unsigned rc = 0, rl = 0;
    if (!COMPRESS && rv) {
      ucur = ustart = fr.rowbase[rowi] + fr.rowblk[rowi >> 8];
      uload = uvec ? (ucur & ~3ull) : ucur;
      rc = (unsigned)(ucur % RING);
      rl = (unsigned)(uload % RING);
    }
    auto ring_fill = [&]() {  // request up to cursor + 2 CH (cp.async, no wait)
      if (COMPRESS || !rv) return;
      unsigned long long want = ucur + 2 * CH;
      if (want > n_unpred) want = n_unpred;
      if (uvec) {
        for (; uload < want; uload += 4) {
          const unsigned long long rem = n_unpred - uload;
          cp_async16(ring + rl, unpred + uload, rem >= 4 ? 16 : (int)rem * 4);
          rl = rl + 4 == RING ? 0 : rl + 4;
        }
      } else if (RING == kURing) {
        for (; uload < want; ++uload) cp_async4(ring + (uload & (kURing - 1)), unpred + uload, 4);
      } else {
        for (; uload < want; ++uload) {
          cp_async4(ring + rl, unpred + uload, 4);
          rl = rl + 1 == RING ? 0 : rl + 1;
        }
      }
    };

    // decompress lookahead (off the recurrence, one step ahead): the next
    // step's dequantised value (code - center) * 2eb and code == 0 flag, and
    // the next verbatim value of the row (as float bits and binary64)
    double qn = 0.0, und = 0.0;
    bool zn = false;
    float un = 0.f;
    auto dequant = [&](int xx) {
      const int code = sizeof(C) == 1
          ? lds_code(a_in_c + (unsigned)((xx & (RX - 1)) ^ swz), false)
          : lds_code(a_in_c + 2u * (unsigned)((xx & (RX - 1)) ^ swz), true);
      qn = __dmul_rn(__dsub_rn(__hiloint2double(0x43300000, code), c52), two_eb);
      zn = code == 0;
    };
    auto next_verbatim = [&]() {
      un = lds_f32(a_ring + 4u * (RING == kURing ? (unsigned)ucur & (kURing - 1) : rc));
      und = (double)un;
    };

    // ---- staging helpers ---------------------------------------------------
    auto load_in = [&](int j) {
      const int x0 = j * CH;
      if (x0 >= nx) return;
      const int slot = j & (RS - 1);
      if (COMPRESS) {
        float* tile = reinterpret_cast<float*>(in_tile);
        if (al16_in) {
#pragma unroll
          for (int i = 0; i < (32 * CH / 4) / 32; ++i) {
            const int p = lane + 32 * i;
            const int r = p / (CH / 4), c4 = p % (CH / 4);
            const int yy = y0 + r % PY, zz = z0 + r / PY;
            const int xx = x0 + 4 * c4;
            float* dst = tile + r * K::IN_STRIDE_F + slot * CH + 4 * c4;
            const int rem = nx - xx;
            const int bytes = (yy < ny && zz < nz && rem > 0) ? (rem >= 4 ? 16 : rem * 4) : 0;
            const float* src = values + (bytes ? ((long long)zz * ny + yy) * nx + xx : 0);
            cp_async16(dst, src, bytes);
          }
        } else {
#pragma unroll 4
          for (int i = 0; i < CH; ++i) {
            const int p = lane + 32 * i;
            const int r = p / CH, c = p % CH;
            const int yy = y0 + r % PY, zz = z0 + r / PY, xx = x0 + c;
            float* dst = tile + r * K::IN_STRIDE_F + slot * CH + c;
            const int bytes = (yy < ny && zz < nz && xx < nx) ? 4 : 0;
            const float* src = values + (bytes ? ((long long)zz * ny + yy) * nx + xx : 0);
            cp_async4(dst, src, bytes);
          }
        }
        cp_commit();
      } else {
        C* tile = reinterpret_cast<C*>(in_tile);
        constexpr int CB = CH * (int)sizeof(C);  // bytes of a row's chunk
        if (al16_in || (nx * (int)sizeof(C)) % 4 == 0) {
          // each lane stages its own row's 16 codes.  Rows on 16-byte
          // boundaries: 16-byte async copies; on 4-byte boundaries (cfg3's
          // nx = 500; 16-bit codes of even nx): 4-byte async copies,
          // zero-filled past the row's end.  (The element-wise path below
          // waits for its loads at every chunk: cfg3 0.73 -> 0.49 ms.)
          const int r = lane;
          const int yy = y0 + r % PY, zz = z0 + r / PY;
          const int rem = nx - x0;
          const int nb = (yy < ny && zz < nz && rem > 0) ? (rem >= CH ? CB : rem * (int)sizeof(C)) : 0;
          unsigned char* dst = reinterpret_cast<unsigned char*>(tile + r * K::IN_STRIDE_B + ((slot * CH) ^ swz));
          const unsigned char* src = reinterpret_cast<const unsigned char*>(
              codes + (nb ? ((long long)zz * ny + yy) * nx + x0 : 0));
          if (al16_in && nb == CB) {
#pragma unroll
            for (int v = 0; v < CB / 16; ++v) cp_async16(dst + 16 * v, src + 16 * v, 16);
          } else {
#pragma unroll
            for (int q = 0; q < CB / 4; ++q) {
              const int b4 = nb - 4 * q >= 4 ? 4 : 0;
              cp_async4(dst + 4 * q, b4 ? src + 4 * q : reinterpret_cast<const unsigned char*>(codes), b4);
            }
          }
          cp_commit();
        } else {
#pragma unroll 4
          for (int i = 0; i < CH; ++i) {
            const int p = lane + 32 * i;
            const int r = p / CH, c = p % CH;
            const int yy = y0 + r % PY, zz = z0 + r / PY, xx = x0 + c;
            C v = 0;
            if (yy < ny && zz < nz && xx < nx) v = codes[((long long)zz * ny + yy) * nx + xx];
            const int sw = (D == 3) ? (((r / PY) & 1) * CH) : 0;  // row r's swizzle
            tile[r * K::IN_STRIDE_B + ((slot * CH + c) ^ sw)] = v;
          }
        }
      }
    };
    // each lane drains its own row segment with 16-byte vector stores
    const bool al16_out = COMPRESS ? (nx % (16 / (int)sizeof(C)) == 0) : (nx % 4 == 0);
    // STG (PY = 8, CH = 16): in a full-chunk drain lane pairs write the
    // sectors of rows (y0 + lane / 4, z0 + i), i < 4, at columns c_l and
    // c_l + 4 of the pair's half -- per task one row pointer and one shared
    // address (the generic index math below was ~140 issued instructions
    // per chunk, rebuilt from the task registers at every drain)
    static_assert(!STG || (PY == 8 && PZ == 4 && CH == 16), "STG drain geometry");
    const int d_c = ((lane >> 1) & 1) * 8 + (lane & 1) * 4;
    float* const d_row = STG ? recon + (((long long)z0 * ny + y0 + (lane >> 2)) * nx + d_c) : nullptr;
    const bool d_yok = y0 + (lane >> 2) < ny;
    const long long d_plane = (long long)ny * nx;
    const unsigned a_drain =
        STG ? pinned(smem_addr(reinterpret_cast<const float*>(out_tile) + (lane >> 2) * K::OUT_STRIDE_F + d_c))
            : 0u;
    auto flush_out = [&](int j) {
      const int x0 = j * CH;
      if (STG && al16_out && x0 + CH <= nx) {
        const unsigned sa = a_drain + 4u * (unsigned)((j & (K::RSO - 1)) * CH);
        float* const g = d_row + x0;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          float4 v;
          asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                       : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                       : "r"(sa + 4u * (unsigned)(8 * i * K::OUT_STRIDE_F)));
          if (d_yok && z0 + i < nz) *reinterpret_cast<float4*>(g + i * d_plane) = v;
        }
        return;
      }
      if (!COMPRESS && al16_out && x0 + CH <= nx) {
        // full chunk (warp-uniform): lane pairs write whole 32-byte sectors,
        // 16 sectors per instruction (a lane writing its own row's 64 bytes
        // as 4 x 16 B would touch every sector twice)
        const int slot = j & (K::RSO - 1);
#pragma unroll
        for (int i = 0; i < CH / 4; ++i) {
          const int q = i * 16 + (lane >> 1);  // sector: row tr, half sc of the chunk
          const int tr = q / (CH / 8), sc = q % (CH / 8), h = lane & 1;
          const int yy = y0 + tr % PY, zz = z0 + tr / PY;
          const int c = sc * 8 + h * 4;
          const float4 v = *reinterpret_cast<const float4*>(
              reinterpret_cast<const float*>(out_tile) + tr * K::OUT_STRIDE_F + slot * CH + c);
          if (yy < ny && zz < nz)
            *reinterpret_cast<float4*>(recon + ((long long)zz * ny + yy) * nx + x0 + c) = v;
        }
        return;
      }
      if (x0 >= nx || !rv) return;
      const int slot = j & (K::RSO - 1);
      const int cnt = nx - x0 < CH ? nx - x0 : CH;
      const long long gi = rowi * nx + x0;
      if (COMPRESS) {
        const C* src = reinterpret_cast<const C*>(out_tile) + lane * K::OUT_STRIDE_B + slot * CH;
        if (al16_out && cnt == CH) {
#pragma unroll
          for (int v = 0; v < CH * (int)sizeof(C) / 16; ++v)
            reinterpret_cast<uint4*>(codes + gi)[v] = reinterpret_cast<const uint4*>(src)[v];
        } else if ((nx * (int)sizeof(C)) % 4 == 0 && cnt == CH) {  // 4-byte boundaries: word stores
#pragma unroll
          for (int q = 0; q < CH * (int)sizeof(C) / 4; ++q)
            reinterpret_cast<unsigned*>(codes + gi)[q] = reinterpret_cast<const unsigned*>(src)[q];
        } else {
          for (int c = 0; c < cnt; ++c) codes[gi + c] = src[c];
        }
      } else {
        const float* src = reinterpret_cast<const float*>(out_tile) + lane * K::OUT_STRIDE_F +
                           slot * CH;
        if (al16_out && cnt == CH) {
#pragma unroll
          for (int v = 0; v < CH / 4; ++v)
            reinterpret_cast<float4*>(recon + gi)[v] = reinterpret_cast<const float4*>(src)[v];
        } else {
          for (int c = 0; c < cnt; ++c) recon[gi + c] = src[c];
        }
      }
    };

    if (!COMPRESS)  // ring columns read at x < 0 must hold valid codes
      for (int c = RX - K::SMAX; c < RX; ++c)
        reinterpret_cast<C*>(in_tile)[lane * K::IN_STRIDE_B + (c ^ swz)] = (C)0;
    ring_fill();
    load_in(0);
    if (STG) stage_issue(0);
    cp_commit();
    cp_wait_all();
    __syncwarp();
    if (STG) stage_settle(0);

#ifdef EBZ_DEBUG_CLOCKS
    long long dbg_t[4] = {0, 0, 0, 0};
    long long dbg_c0 = clock64();
#endif
    for (int k = 0; k < nchunks; ++k) {
      const int S0 = k * CH;
#ifdef EBZ_DEBUG_CLOCKS
      long long t_a = clock64();
#endif
      if (STG) {  // faces of this chunk's second block (waited at its start)
        stage_issue(2 * k + 1);
        cp_commit();
      }
      ring_fill();
      load_in(k + 1);
      if (!COMPRESS) cp_commit();
#ifdef EBZ_DEBUG_CLOCKS
      long long t_b = clock64();
      dbg_t[0] += t_b - t_a;
#endif
      // unrolled by the FIFO depth only: a fully unrolled 16-step chunk
      // overflows the instruction cache (measured: 20% no_inst stalls)
      if (!COMPRESS) {  // this chunk's columns and verbatim values are resident
        dequant(S0 - sig);
        next_verbatim();
      }
#pragma unroll 1
      for (int st0 = 0; st0 < CH; st0 += DP) {
      if (STG && st0 == DP) {
        // second block: its faces landed (the newer group is the next
        // chunk's codes); stage the next chunk's first block
        cp_wait_1();
        __syncwarp();
        stage_settle(2 * k + 1);
        stage_issue(2 * k + 2);
        cp_commit();
      }
      const unsigned a_fb = a_fst + 8u * (unsigned)(((S0 + st0) / DP) & 1) * SM::FST_WORDS;
      // face-store bases of this block of DP steps (immediate offsets below)
      const long long xb = S0 + st0 - sig;
      unsigned long long* const wyb = wyp + xb * (SKEW ? 4 : 1);
      unsigned long long* const wzb = wzp + xb * (SKEW ? 8 : 1);
#pragma unroll
      for (int jj = 0; jj < DP; ++jj) {
        const int st = st0 + jj;
        const int x = S0 + st - sig;
        const int col = x & (RX - 1);            // input ring column
        const int colo = x & (K::RXO - 1);       // output ring column
        const bool act = rv && (unsigned)x < (unsigned)nx;
        // ---- face words for column x (prefetched DP steps ago)
        double fv[NS > 0 ? NS : 1];
        if (STG) {
          // (consumer lanes load their staged face values after the shuffles)
        } else if (NS > 0) {
          const int xs = DIST ? S0 + st - fsig : x;  // column of this lane's streams
          bool miss = false;
#pragma unroll
          for (int s = 0; s < NSL; ++s) miss |= !face_ok(fifo[s][jj], epoch);
          if (__any_sync(EBZ_FULL, miss)) {
            // producer not there yet: spin on the words still missing
            for (unsigned ns = 16;; ns = ns < 256 ? 2 * ns : ns) {
              bool m2 = false;
#pragma unroll
              for (int s = 0; s < NSL; ++s)
                if (!face_ok(fifo[s][jj], epoch)) {
                  fifo[s][jj] = ld_face(sp[s] + (xs << rsh[s]));
                  m2 |= !face_ok(fifo[s][jj], epoch);
                }
              if (!__any_sync(EBZ_FULL, m2)) break;
              __nanosleep(ns);
            }
          }
          double lv[NSL > 0 ? NSL : 1];
#pragma unroll
          for (int s = 0; s < NSL; ++s) {
            lv[s] = face_val(fifo[s][jj]);
            const int xp = xs + DP;
            fifo[s][jj] = (unsigned)xp < (unsigned)rn[s] ? ld_face(sp[s] + (xp << rsh[s])) : tag;
          }
          if (DIST) {  // consumers: (0, b) <- lanes 2b, 2b + 1; (a, 0) <- lane 8 + a
            fv[0] = __shfl_sync(EBZ_FULL, lv[0], 2 * lb);
            fv[1] = __shfl_sync(EBZ_FULL, lv[0], 2 * lb + 1);
            fv[2] = __shfl_sync(EBZ_FULL, lv[0], 8 + la);
          } else {
#pragma unroll
            for (int s = 0; s < NSL; ++s) fv[s] = lv[s];
          }
        }
        // ---- receive column x from neighbour lanes (previous step's column 0)
        double nw[NB][NA];
#pragma unroll
        for (int b = 0; b < NB; ++b)
#pragma unroll
          for (int aa = 0; aa < NA; ++aa) {
            if (aa == 0 && b == 0) continue;
            if (aa >= 1) nw[b][aa] = __shfl_up_sync(EBZ_FULL, H[b][aa - 1][0], 1);
            else nw[b][aa] = __shfl_up_sync(EBZ_FULL, H[b - 1][0][0], PY);
          }
        if (STG) {  // face values straight into the neighbour slots
          lds_f64_if(nw[0][1], a_fb + 8u * (unsigned)(4 * jj + lb + 4), la == 0);
          lds_f64_if(nw[1][1], a_fb + 8u * (unsigned)(lb ? 4 * jj + lb - 1 : 36 + jj), la == 0);
          lds_f64_if(nw[1][0], a_fb + 8u * (unsigned)(44 + 8 * jj + la), lb == 0);
        } else {
        if (la == 0) {
#pragma unroll
          for (int b = 0; b < NB; ++b)
#pragma unroll
            for (int aa = 1; aa < NA; ++aa) nw[b][aa] = fv[b * N + aa - 1];
        }
        if (D == 3 && lb == 0) {
#pragma unroll
          for (int b = 1; b < NB; ++b) nw[b][0] = fv[K::NSY + b - 1];
        }
        }
        // shift history, install the new column
#pragma unroll
        for (int b = 0; b < NB; ++b)
#pragma unroll
          for (int aa = 0; aa < NA; ++aa) {
#pragma unroll
            for (int c = NC - 1; c >= 1; --c) H[b][aa][c] = H[b][aa][c - 1];
            if (!(aa == 0 && b == 0)) H[b][aa][0] = nw[b][aa];
          }
        // ---- predict
        double pred;
        if (N == 2) {
          const bool eff1 = x == 1 || y == 1 || (D == 3 && z == 1);
          double h1[NB == 1 ? 1 : 2][2][2];
#pragma unroll
          for (int b = 0; b < (NB == 1 ? 1 : 2); ++b)
#pragma unroll
            for (int aa = 0; aa < 2; ++aa)
#pragma unroll
              for (int c = 0; c < 2; ++c) h1[b][aa][c] = H[b][aa][c];
          pred = eff1 ? stencil_sum<1, (NB == 1 ? 1 : 2), 2, 2>(h1)
                      : stencil_sum<N, NB, NA, NC>(H);
        } else {
          pred = stencil_sum<N, NB, NA, NC>(H);
        }
        double r64;
        if (COMPRESS) {
          const float xv = lds_f32(a_in_f + 4 * col);
          const double x64 = (double)xv;
          // reciprocal quantizer, bit-identical to quantize_exact: k = rint(q)
          // through the 1.5 * 2^52 magic constant, exact whenever q is at
          // least 2^-30 from a half-integer (the guard; see quantize_fast2 for
          // why the reference's |s| < center + 1 test needs none)
          constexpr double M = 0x1.8p52;
          const double q = __dmul_rn(__dsub_rn(x64, pred), inv);
          const double t = __dadd_rn(q, M);
          const double kd = __dsub_rn(t, M);  // never -0.0
          const double rr = __dadd_rn(pred, __dmul_rn(kd, two_eb));
          // T(pred + k * 2eb): hardware round-to-nearest-even to float32
          const float rf = __double2float_rn(rr);
          const double rq = (double)rf;
          const bool safe = fabs(__dsub_rn(q, kd)) < guard;
          const bool good = fabs(kd) <= lim && fabs(__dsub_rn(x64, rq)) <= eb;
          // branch-free selects (bit masks) keep the common path free of
          // reconvergence points
          const long long gm = -(long long)good;
          const double xs = TR ? (double)trunc_value<float>(xv, tre) : x64;
          r64 = __longlong_as_double((__double_as_longlong(rq) & gm) |
                                     (__double_as_longlong(xs) & ~gm));
          int code = (center + __double2loint(t)) & (int)gm;
          const bool slow = !safe && act;
          if (__any_sync(EBZ_FULL, slow)) {  // rare: exact IEEE division path
            if (slow) {
              float rf;
              code = quantize_exact<float>(xv, pred, eb, two_eb, center, rf, tre);
              r64 = (double)rf;
            }
          }
          // unguarded: columns outside [0, nx) land in ring slots that are
          // either rewritten before their drain or never drained
          sts_code(a_out_c + (unsigned)sizeof(C) * colo, code, WIDE);
          if (REC && act) recon[rowi * nx + x] = (float)r64;
        } else {
          const double qv = qn;
          const bool zc = zn;
          if (st + 1 < CH) dequant(x + 1);  // next step, same chunk (resident)
          const double rr = __dadd_rn(pred, qv);
          // T(pred + q) by the hardware conversion pair (measured: the
          // binary64 bit-pattern rounding cost ~12 more instructions per
          // point, 5.78 vs 5.49 ms on the cfg5 batch)
          r64 = (double)__double2float_rn(rr);
          if (act && zc) {
            // (a value read past this chunk's resident ones is re-read at the
            // next chunk start, after the ring's cp.async wait)
            // (a cursor past the block is an underrun: detected from the
            // final cursor, the value is then never used)
            r64 = und;
            ++ucur;
            if (RING != kURing) rc = rc + 1 == RING ? 0 : rc + 1;
            next_verbatim();
          }
          // non-finite output: exponent field all ones (checked per task)
          hmax = max(hmax, act ? ((unsigned)__double2hiint(r64) & 0x7fffffffu) : 0u);
          // r64 is a float32 value: the conversion is exact (off the recurrence)
          sts_f32(a_out_f + 4 * colo, __double2float_rn(r64));  // unguarded, as in compress
        }
        {
          const unsigned lo = (unsigned)__double2loint(r64) | epoch;
          const unsigned hi = (unsigned)__double2hiint(r64);
          st_face2_if(wyb + jj * (SKEW ? 4 : 1), lo, hi, act && wy_ok);
          if (D == 3) st_face2_if(wzb + jj * (SKEW ? 8 : 1), lo, hi, act && wz_ok);
        }
        H[0][0][0] = act ? r64 : 0.0;
      }
      }
      // ---- end of chunk: drain outputs, land the next input chunk
#ifdef EBZ_DEBUG_CLOCKS
      long long t_c = clock64();
      dbg_t[1] += t_c - t_b;
#endif
      __syncwarp();
      if (k - K::OUT_LAG >= 0) flush_out(k - K::OUT_LAG);
#ifdef EBZ_DEBUG_CLOCKS
      long long t_d = clock64();
      dbg_t[2] += t_d - t_c;
#endif
      cp_wait_all();
      __syncwarp();
      if (STG && k + 1 < nchunks) stage_settle(2 * k + 2);
#ifdef EBZ_DEBUG_CLOCKS
      dbg_t[3] += clock64() - t_d;
#endif
    }
#ifdef EBZ_DEBUG_CLOCKS
    if (tk == 0 && lane == 0)
      printf("EBZDBG D=%d N=%d C=%d nchunks=%d total=%lld load_in=%lld steps=%lld "
             "flush=%lld wait=%lld per_step=%.1f\n",
             D, N, (int)COMPRESS, nchunks, clock64() - dbg_c0, dbg_t[0], dbg_t[1], dbg_t[2],
             dbg_t[3], (double)dbg_t[1] / (nchunks * CH));
#endif
    for (int j = nchunks - K::OUT_LAG; j < nchunks; ++j)
      if (j >= 0) flush_out(j);
    __syncwarp();
    if (!COMPRESS) {  // per task: consecutive tasks may belong to different fields
      unsigned long long used = ucur - ustart;
      if (ucur > n_unpred) bad |= ST_UNDERRUN;
#pragma unroll
      for (int o = 16; o; o >>= 1) used += __shfl_xor_sync(EBZ_FULL, used, o);
      if (hmax >= 0x7ff00000u) bad |= ST_NONFINITE_OUT;
      bad = __reduce_or_sync(EBZ_FULL, bad);
      if (lane == 0) {
        if (used) atomicAdd(&fr.info->used, used);
        if (bad) atomicOr(&fr.info->status, bad);
      }
    }
  }
}

template <int D, int N, typename C, bool COMPRESS, bool REC = false, bool TR = false>
cudaError_t launch_fast_t(const FastArgs& fa, const FieldTable& ft, int sms, cudaStream_t s) {
  typedef Smem<D, N, C, COMPRESS> SM;
  const int m = fa.s.m;
  const size_t tail = 0;
  const size_t smem = (size_t)WPB * SM::PER_WARP + tail;
  static KernelAttr attr;
  cudaError_t e = kernel_smem(attr, sweep_fast_kernel<D, N, C, COMPRESS, REC, TR>, smem);
  if (e != cudaSuccess) return e;
  const int per_sm_cached =
      kernel_occupancy(attr, sweep_fast_kernel<D, N, C, COMPRESS, REC, TR>, 32 * WPB, smem);
  const long long ntasks = (long long)fa.npy * fa.npz * fa.nf;
  // Launch only as many warps as the wavefronts keep busy (a single field
  // leaves SMs to concurrent work on other streams; a batch fills the GPU).
  long long active = (long long)fa.npy + fa.npz + 64;
  if (D == 3) {
    const long long diag = fa.npy < fa.npz ? fa.npy : fa.npz;
    // a task runs ~nx steps and its successors start ~14 steps behind it, so
    // about diag * nx / 14 tasks are runnable at once (measured on cfg3:
    // the former diag * (nx / 64 + 8) starved the wavefront, 1.18 -> 0.96 ms;
    // launching every task's warp is slower again -- idle warps spin)
    active = diag * ((fa.s.dims[0] + 14) / 14 + 1) + 64;
  }
  active *= fa.nf;
  {  // EBZ_ACTIVE_SCALE: A/B experiments on the launch size
    static const char* sc = getenv("EBZ_ACTIVE_SCALE");
    if (sc) active = (long long)(active * atof(sc));
  }
  if (active > ntasks) active = ntasks;
  long long blocks = (active + WPB - 1) / WPB;
  if (blocks > (long long)sms * per_sm_cached) blocks = (long long)sms * per_sm_cached;
  if (blocks < 1) blocks = 1;
  sweep_fast_kernel<D, N, C, COMPRESS, REC, TR><<<(unsigned)blocks, 32 * WPB, smem, s>>>(fa, ft);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// 3D, n = 1, two rows per lane.  A warp owns an 8 (y) x 8 (z) patch; lane
// (a, b), b < 4, carries rows (y0 + a, z0 + b) and (y0 + a, z0 + b + 4) and
// processes x_r = S - (a + b + 4r) at step S, i.e. its second row trails the
// first by four steps.  Every row dependency keeps the one-step systolic form
// of the one-row kernel: y - 1 from lane a - 1 (same row slot), z - 1 from
// lane b - 1 (same slot) or, for b = 0's second row, from lane (a, 3)'s first
// row -- one rotate-by-8 shuffle whose source sends the right slot.  Two
// independent recurrences per lane (ILP) and half the per-point loop, face
// and staging overhead.  Chunks are 8 steps (the 64-row tiles stay small).
constexpr int CH2 = 8;                 // steps per chunk
constexpr int RS2 = 4;                 // input ring slots
constexpr int RX2 = CH2 * RS2;         // input ring columns
constexpr int SMAX2 = 7 + 3 + 4;       // max row skew
constexpr int OUT_LAG2 = (SMAX2 + CH2 - 1) / CH2;
constexpr int RSO2 = 4;                // output ring slots (>= OUT_LAG2 + 1)
constexpr int RXO2 = CH2 * RSO2;
constexpr int INF2 = RX2 + 4;          // floats per input row (f32 tile)
// code tile row: 72 B for u8 codes (2.3-way instead of 4-way bank conflicts
// on the per-step byte stores)
constexpr int OUTB2 = RXO2 + 40;
constexpr int NS2 = 5;                 // face streams: Y(r, b) x 4, Z(row 0)
constexpr int DP2 = 4;                 // face prefetch distance (steps)
// Padded, skew-major face blocks (see the kernel): word index x + zz runs
// over [-7, nx + SMAX2 + CH2 + DP2 + 6] -- producers store every step from
// x + zz = -7, consumers prefetch up to DP2 steps ahead and the corner stream
// reads x + 7 -- so with the pads every access is inside its block and pad
// columns carry tagged zeros (the right pad past a producer's last step is
// filled when its task ends).
constexpr int kFPadL2 = 16;
constexpr int kFPadR2 = 32;
constexpr int kFPad2 = kFPadL2 + kFPadR2;
static_assert(kFPadL2 >= 7 && kFPadR2 >= SMAX2 + CH2 + DP2 + 6, "face pads too small");
static_assert(OUT_LAG2 + 1 <= RSO2, "output ring too small");

// per-warp shared memory: 64-row f32 input ring, 64-row code output ring,
// and (u8 codes) the warp's code histogram of its current task
template <typename C>
struct Smem2 {
  static constexpr int IN_BYTES = 64 * INF2 * 4;
  static constexpr int OUT_BYTES = 64 * OUTB2 * (int)sizeof(C);
  static constexpr int OUT_OFF = ((IN_BYTES + 15) / 16) * 16;
  static constexpr int HIST_OFF = OUT_OFF + ((OUT_BYTES + 15) / 16) * 16;
  // 256 bins + a dummy bin for inactive points (16-byte multiple)
  static constexpr int HIST_BYTES = sizeof(C) == 1 ? 260 * 4 : 0;
  static constexpr int PER_WARP = HIST_OFF + HIST_BYTES;
};

// 3D n = 1 stencil of both rows, term by term in the reference's order
// (stencil_sum), the rows' independent chains in lockstep
__device__ __forceinline__ void stencil2(const double (&H)[2][2][2][2], double (&p)[2]) {
#pragma unroll
  for (int r = 0; r < 2; ++r) p[r] = __dadd_rn(H[r][1][0][0], H[r][0][1][0]);
#pragma unroll
  for (int r = 0; r < 2; ++r) p[r] = __dsub_rn(p[r], H[r][1][1][0]);
#pragma unroll
  for (int r = 0; r < 2; ++r) p[r] = __dadd_rn(p[r], H[r][0][0][1]);
#pragma unroll
  for (int r = 0; r < 2; ++r) p[r] = __dsub_rn(p[r], H[r][1][0][1]);
#pragma unroll
  for (int r = 0; r < 2; ++r) p[r] = __dsub_rn(p[r], H[r][0][1][1]);
#pragma unroll
  for (int r = 0; r < 2; ++r) p[r] = __dadd_rn(p[r], H[r][1][1][1]);
}

// fast-path quantizer of both rows in lockstep, without the fallback;
// slow[r] = needs the exact division.  k = rint(q) through the 1.5 * 2^52
// magic constant (two DADDs instead of DADD + FRND): it equals the
// reference's round-half-away-from-zero floor(|s| + 0.5) * sign(s) whenever
// the guard below holds (q at least 2^-30 from a half-integer), its low
// word is the signed code offset, and it is never -0.0.  The stored value's
// zero sign may differ from the reference's only when pred = -0 and k = 0;
// a zero's sign never changes a code or a verbatim decision, and compress
// emits only those.
__device__ __forceinline__ void quantize_fast2(const float (&xv)[2], const double (&pred)[2],
                                               double eb, double two_eb, double inv,
                                               double guard, double lim, int center,
                                               double (&r64)[2],
                                               int (&code)[2], bool (&slow)[2],
                                               int tre = kNoTrunc) {
  constexpr double M = 0x1.8p52;
  double x64[2], q[2], t[2], kr[2], rr[2], rq[2];
  float rf[2];
#pragma unroll
  for (int r = 0; r < 2; ++r) x64[r] = (double)xv[r];
#pragma unroll
  for (int r = 0; r < 2; ++r) q[r] = __dmul_rn(__dsub_rn(x64[r], pred[r]), inv);
#pragma unroll
  for (int r = 0; r < 2; ++r) t[r] = __dadd_rn(q[r], M);
#pragma unroll
  for (int r = 0; r < 2; ++r) kr[r] = __dsub_rn(t[r], M);
#pragma unroll
  for (int r = 0; r < 2; ++r) rr[r] = __dadd_rn(pred[r], __dmul_rn(kr[r], two_eb));
  // T(rr): the hardware F2F pair (measured faster here than the bit-pattern
  // rounding, whose extra integer ops cost more than the latency they save)
#pragma unroll
  for (int r = 0; r < 2; ++r) rf[r] = __double2float_rn(rr[r]);
#pragma unroll
  for (int r = 0; r < 2; ++r) rq[r] = (double)rf[r];
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    // guard: q at least 2^-30 from a half-integer.  q - kr is exact (kr = 0
    // for |q| < 1/2, Sterbenz otherwise).  The reference's |s| < center + 1
    // test needs no guard of its own: when it fails, |k| >= center + 1 >
    // center - 1 and both paths emit code 0; and for |q| >= 2^16 (where q's
    // error could exceed the margin) |kr| > center - 1 likewise.
    slow[r] = !(fabs(__dsub_rn(q[r], kr[r])) < guard);
    const bool good = fabs(kr[r]) <= lim && fabs(__dsub_rn(x64[r], rq[r])) <= eb;
    const long long gm = -(long long)good;
    const double xs = tre == kNoTrunc ? x64[r] : (double)trunc_value<float>(xv[r], tre);
    r64[r] = __longlong_as_double((__double_as_longlong(rq[r]) & gm) |
                                  (__double_as_longlong(xs) & ~gm));
    code[r] = (center + (int)__double2loint(t[r])) & (int)gm;
  }
}

// compress only (decompress measured slower with two rows per lane)
// REC: also store every point's reconstruction (see sweep_fast_kernel)
template <typename C, bool REC = false, bool TR = false>
#ifndef EBZ_R2_MINB
#define EBZ_R2_MINB 3
#endif
__global__ void __launch_bounds__(32 * WPB, EBZ_R2_MINB)
sweep_r2_kernel(const __grid_constant__ FastArgs fa, const __grid_constant__ FieldTable ft) {
  typedef Smem2<C> SM;
  const SweepArgs& a = fa.s;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int la = lane & 7, lb = lane >> 3;
  const int sig = la + lb;  // row 0; row 1 is sig + 4
  unsigned char* wbase = smem_raw + warp * SM::PER_WARP;
  unsigned char* in_tile = wbase;
  unsigned char* out_tile = wbase + SM::OUT_OFF;
  // u8 codes: the code histogram (codec.py:107) is counted here, as the codes
  // are produced, instead of in a second pass over the code array
  constexpr bool FH = sizeof(C) == 1;
  unsigned int* whist = reinterpret_cast<unsigned int*>(wbase + SM::HIST_OFF);

  const int nx = (int)a.dims[0], ny = (int)a.dims[1], nz = (int)a.dims[2];
  const int npy = fa.npy, npz = fa.npz;
  const int nf = fa.nf;
  const int ntasks = npy * npz * nf;
  const int nchunks = (nx + SMAX2 + CH2 - 1) / CH2;
  const unsigned epoch = a.epoch;
  const unsigned long long tag = epoch;  // tagged 0.0 (outside the domain)
  const bool al_in = nx % 4 == 0;
  // drains write CH2 = 8 codes: 8- (u8) or 16-byte (u16) stores
  const bool al_out = nx % 8 == 0;
  const bool al4_out = (nx * (int)sizeof(C)) % 4 == 0;
  // rotate-by-8 source lane: (a, b - 1 mod 4)
  const int zsrc = (lane + 24) & 31;

  for (;;) {
    unsigned int tk = 0;
    if (lane == 0) tk = atomicAdd(a.ticket, 1u);
    tk = __shfl_sync(EBZ_FULL, tk, 0);
    if ((int)tk >= ntasks) break;
    sched_jitter(a.jitter, tk, 0);  // test hook: per task here (single fields are latency-bound)
    const int fi = (int)(tk % (unsigned)nf);
    const FieldRef& fr = ft.f[fi];
    const int center = ft.center[fi] ? ft.center[fi] : a.center;  // per-field m (auto-m trials)
    const double lim = (double)(center - 1);
    const double eb = fr.info->eb;
    if (!(eb > 0.0)) continue;
    const double two_eb = __dmul_rn(2.0, eb);
    const double inv = 1.0 / two_eb;
    const bool fast_ok = isfinite(inv) && inv > 0.0 && two_eb >= 0x1p-1000 &&
                         inv >= 0x1p-1000 && inv <= 0x1p1000;
    const double guard = fast_ok ? 0.5 - 0x1p-30 : -1.0;
    const int tre = TR ? eb_exponent(eb) : kNoTrunc;  // opt-in truncation
    const float* values = reinterpret_cast<const float*>(fr.values);
    float* const recon = reinterpret_cast<float*>(fr.recon);
    C* codes = reinterpret_cast<C*>(fr.codes);
    unsigned long long* yface = fr.yface;
    unsigned long long* zface = fr.zface;
    unsigned long long* const ghist = FH ? fr.hist : nullptr;
    if (ghist) {
#pragma unroll
      for (int b = 0; b < 8; ++b) whist[lane + 32 * b] = 0u;
      __syncwarp();
    }
    const unsigned int tv = fa.tasks[tk / (unsigned)nf];
    const int PYi = (int)(tv & 0xffff), PZi = (int)(tv >> 16);
    const int y0 = PYi * 8, z0 = PZi * 8;
    const int y = y0 + la;
    int zr[2];
    bool rv[2];
    long long rowi[2];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      zr[r] = z0 + lb + 4 * r;
      rv[r] = y < ny && zr[r] < nz;
      rowi[r] = (long long)zr[r] * ny + y;
    }
    // Skew-major patch faces.  The face words of patch (PY, PZ) form a block
    // of fsx x 8 words; face row zz (Y face: z - z0, Z face: y - y0) at
    // column x sits at word (kFPadL2 + x + zz) * 8 + zz of the block.  The
    // eight producer lanes of a face all compute x + zz = S - 7 at step S,
    // and the consumer lanes of a stream read x + zz = S + const, so every
    // warp-wide face store or load is one run of consecutive words (one or
    // two sectors) instead of one sector per lane.
    const long long fsx = nx + kFPad2;
    auto fblk = [&](int PY, int PZ) { return ((long long)PY * npz + PZ) * fsx * 8; };
    // faces written: Y by la == 7 (both rows, zz = lb + 4r), Z by lb == 3's
    // row 1 (zz = la); pointers at step 0
    bool wyh[2];
    unsigned long long* wy[2];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      wyh[r] = rv[r] && la == 7;
      wy[r] = yface + (wyh[r] ? fblk(PYi, PZi) + (kFPadL2 - 7) * 8 + lb + 4 * r : 0);
    }
    const bool wzh = rv[1] && lb == 3;
    unsigned long long* const wz = zface + (wzh ? fblk(PYi, PZi) + (kFPadL2 - 7) * 8 + la : 0);
    // face streams: s = 2r + b -> Y row (y0 - 1, z_r - b); s = 4 -> Z row (y, z0 - 1);
    // fh = the lane has the stream (otherwise tagged zeros); pointers at step 0
    bool fh[NS2];
    const unsigned long long* fp[NS2];
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
      for (int b = 0; b < 2; ++b) {
        const bool ok = rv[r] && la == 0 && y0 >= 1 && zr[r] - b >= 0;
        const int zz = lb + 4 * r - b;
        // zz = -1: row z0 - 1, the last face row of patch (PY - 1, PZ - 1)
        const long long off = zz >= 0 ? fblk(PYi - 1, PZi) + (kFPadL2 - b) * 8 + zz
                                      : fblk(PYi - 1, PZi - 1) + (kFPadL2 + 7) * 8 + 7;
        fh[2 * r + b] = ok;
        fp[2 * r + b] = yface + (ok ? off : 0);
      }
    fh[4] = rv[0] && lb == 0 && PZi >= 1;
    fp[4] = zface + (fh[4] ? fblk(PYi, PZi - 1) + kFPadL2 * 8 + la : 0);
    unsigned long long fifo[NS2][DP2];
#pragma unroll
    for (int s = 0; s < NS2; ++s)
#pragma unroll
      for (int j = 0; j < DP2; ++j) fifo[s][j] = fh[s] ? ld_face(fp[s] + j * 8) : tag;
    // tile rows of this lane: lane (row 0) and lane + 32 (row 1)
    const float* in_f[2] = {reinterpret_cast<const float*>(in_tile) + lane * INF2,
                            reinterpret_cast<const float*>(in_tile) + (lane + 32) * INF2};
    C* out_c[2] = {reinterpret_cast<C*>(out_tile) + lane * OUTB2,
                   reinterpret_cast<C*>(out_tile) + (lane + 32) * OUTB2};
    // history cubes: H[r][b][a][c] = r(z_r - b, y - a, x_r - c)
    double H[2][2][2][2];
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
      for (int b = 0; b < 2; ++b)
#pragma unroll
        for (int aa = 0; aa < 2; ++aa)
#pragma unroll
          for (int c = 0; c < 2; ++c) H[r][b][aa][c] = 0.0;
    // tile row t (0..63) <-> (y0 + (t & 7), z0 + ((t >> 3) & 3) + 4 * (t >> 5))
    auto tile_row = [&](int t, int& yy, int& zz) {
      yy = y0 + (t & 7);
      zz = z0 + ((t >> 3) & 3) + 4 * (t >> 5);
    };
    auto load_in = [&](int j) {
      const int x0 = j * CH2;
      if (x0 >= nx) return;
      const int slot = j & (RS2 - 1);
      float* tile = reinterpret_cast<float*>(in_tile);
      if (al_in) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {  // 64 rows x 2 float4
          const int p = lane + 32 * i;
          const int t = p >> 1, c4 = p & 1;
          int yy, zz;
          tile_row(t, yy, zz);
          const int xx = x0 + 4 * c4;
          const int rem = nx - xx;
          const int bytes = (yy < ny && zz < nz && rem > 0) ? (rem >= 4 ? 16 : rem * 4) : 0;
          const float* src = values + (bytes ? ((long long)zz * ny + yy) * nx + xx : 0);
          cp_async16(tile + t * INF2 + slot * CH2 + 4 * c4, src, bytes);
        }
      } else {
#pragma unroll 4
        for (int i = 0; i < 16; ++i) {  // 64 rows x 8 floats
          const int p = lane + 32 * i;
          const int t = p >> 3, c = p & 7;
          int yy, zz;
          tile_row(t, yy, zz);
          const int xx = x0 + c;
          const int bytes = (yy < ny && zz < nz && xx < nx) ? 4 : 0;
          const float* src = values + (bytes ? ((long long)zz * ny + yy) * nx + xx : 0);
          cp_async4(tile + t * INF2 + slot * CH2 + c, src, bytes);
        }
      }
      cp_commit();
    };
    auto flush_out = [&](int j) {
      const int x0 = j * CH2;
      if (x0 >= nx) return;
      const int slot = j & (RSO2 - 1);
      const int cnt = nx - x0 < CH2 ? nx - x0 : CH2;
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        if (!rv[r]) continue;
        const long long gi = rowi[r] * nx + x0;
        const C* src = out_c[r] + slot * CH2;
        if (al_out && cnt == CH2) {
          if (sizeof(C) == 1)
            *reinterpret_cast<uint2*>(codes + gi) = *reinterpret_cast<const uint2*>(src);
          else
            *reinterpret_cast<uint4*>(codes + gi) = *reinterpret_cast<const uint4*>(src);
        } else if (al4_out && cnt == CH2) {  // rows on 4-byte boundaries: word stores
#pragma unroll
          for (int q = 0; q < CH2 * (int)sizeof(C) / 4; ++q)
            reinterpret_cast<unsigned*>(codes + gi)[q] = reinterpret_cast<const unsigned*>(src)[q];
        } else {
          for (int c = 0; c < cnt; ++c) codes[gi + c] = src[c];
        }
      }
    };

    // ring columns read at x < 0 (the last two slots, x in [-SMAX2, 0)) hold +0.0
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
      for (int c = RX2 - 16; c < RX2; c += 4)
        *reinterpret_cast<float4*>(const_cast<float*>(in_f[r]) + c) = make_float4(0.f, 0.f, 0.f, 0.f);
    static_assert(SMAX2 <= 16 && RX2 - 16 >= 2 * CH2, "x < 0 columns must be the last two slots");
    load_in(0);
    cp_commit();
    cp_wait_all();
    __syncwarp();

    for (int k = 0; k < nchunks; ++k) {
      const int S0 = k * CH2;
      load_in(k + 1);
#pragma unroll 1
      for (int st0 = 0; st0 < CH2; st0 += DP2) {
      // this group's face addresses: base + jj (immediate offsets per step)
      const int G = S0 + st0;
      const unsigned long long* gp[NS2];
#pragma unroll
      for (int s = 0; s < NS2; ++s) gp[s] = fp[s] + (G + DP2) * 8;
      unsigned long long* gy[2];
#pragma unroll
      for (int r = 0; r < 2; ++r) gy[r] = wy[r] + G * 8;
      unsigned long long* const gz = wz + G * 8;
#pragma unroll
      for (int jj = 0; jj < DP2; ++jj) {
        const int S = G + jj;
        int xr[2], col[2], colo[2];
        bool act[2];
#pragma unroll
        for (int r = 0; r < 2; ++r) {
          xr[r] = S - sig - 4 * r;
          col[r] = xr[r] & (RX2 - 1);
          colo[r] = xr[r] & (RXO2 - 1);
          act[r] = rv[r] && (unsigned)xr[r] < (unsigned)nx;
        }
        // ---- face words (prefetched DP2 steps ago)
        double fv[NS2];
        {
          unsigned d = 0;  // tag mismatch bits of all streams (XOR/OR folds into LOP3s)
#pragma unroll
          for (int s = 0; s < NS2; ++s) d |= (unsigned)fifo[s][jj] ^ epoch;
          if (__any_sync(EBZ_FULL, (d & kTagMask) != 0)) {
            for (unsigned ns = 16;; ns = ns < 256 ? 2 * ns : ns) {
              bool m2 = false;
#pragma unroll
              for (int s = 0; s < NS2; ++s)
                if (!face_ok(fifo[s][jj], epoch)) {
                  fifo[s][jj] = ld_face(gp[s] + (jj - DP2) * 8);
                  m2 |= !face_ok(fifo[s][jj], epoch);
                }
              if (!__any_sync(EBZ_FULL, m2)) break;
              __nanosleep(ns);
            }
          }
#pragma unroll
          for (int s = 0; s < NS2; ++s) {
            fv[s] = face_val(fifo[s][jj]);
            // (the explicit tag keeps each FIFO slot in one register across
            // the group loop; a conditional-only load made ptxas copy the
            // slot at the back-edge, waiting on the load just issued)
            fifo[s][jj] = fh[s] ? ld_face(gp[s] + jj * 8) : tag;
          }
        }
        // ---- neighbours of column x_r (neighbour lanes' previous column 0)
        double n01[2], n11[2], n10[2];
#pragma unroll
        for (int r = 0; r < 2; ++r) {
          n01[r] = __shfl_up_sync(EBZ_FULL, H[r][0][0][0], 1);  // (z, y-1)
          n11[r] = __shfl_up_sync(EBZ_FULL, H[r][1][0][0], 1);  // (z-1, y-1)
        }
        // (z-1, y): lane b-1's same row; for b = 0, row 1's is lane (a, 3)'s row 0
        const double z0v = __shfl_sync(EBZ_FULL, H[0][0][0][0], zsrc);
        const double z1v = __shfl_sync(EBZ_FULL, H[1][0][0][0], zsrc);
        n10[0] = z0v;
        n10[1] = lb == 0 ? z0v : z1v;
        if (la == 0) {
          n01[0] = fv[0];
          n11[0] = fv[1];
          n01[1] = fv[2];
          n11[1] = fv[3];
        }
        if (lb == 0) n10[0] = fv[4];
#pragma unroll
        for (int r = 0; r < 2; ++r) {
#pragma unroll
          for (int b = 0; b < 2; ++b)
#pragma unroll
            for (int aa = 0; aa < 2; ++aa) H[r][b][aa][1] = H[r][b][aa][0];
          H[r][0][1][0] = n01[r];
          H[r][1][1][0] = n11[r];
          H[r][1][0][0] = n10[r];
        }
        // ---- predict + quantize both rows: fast paths first (independent
        // chains), one vote for the exact-division fallback
        double rq64[2], pr[2];
        float xv[2];
        int code[2];
        bool slow[2];
#pragma unroll
        for (int r = 0; r < 2; ++r) xv[r] = in_f[r][col[r]];
        stencil2(H, pr);
        quantize_fast2(xv, pr, eb, two_eb, inv, guard, lim, center, rq64, code,
                       slow, tre);
#pragma unroll
        for (int r = 0; r < 2; ++r) slow[r] = slow[r] && act[r];
#ifndef EBZ_EXP_NOSLOW
        if (__any_sync(EBZ_FULL, slow[0] || slow[1])) {
#else
        if (false) {
#endif
#pragma unroll
          for (int r = 0; r < 2; ++r)
            if (slow[r]) {
              float rf2;
              code[r] = quantize_exact<float>(xv[r], pr[r], eb, two_eb, center, rf2, tre);
              rq64[r] = (double)rf2;
            }
        }
#pragma unroll
        for (int r = 0; r < 2; ++r) {
          out_c[r][colo[r]] = (C)code[r];  // unguarded
          // one shared atomic per point, result unused (measured cheaper
          // than run-merging the drained codes, and than per-lane copies)
          // (unconditional, inactive points into the dummy bin: a guarded
          // atomic is a branch region per point)
          if (FH) atomicAdd(&whist[(ghist && act[r]) ? code[r] : 256], 1u);
          // no activity mask: columns x < 0 compute exact +0.0 from the zeroed
          // ring columns; values at x >= nx or on rows outside the grid only
          // reach inactive points and pad words no active point reads
          H[r][0][0][0] = rq64[r];
          if (REC && act[r]) recon[rowi[r] * nx + xr[r]] = (float)rq64[r];
          // every step, inside the padded row
          const unsigned long long w = face_word(rq64[r], epoch);
          if (wyh[r]) __stcg(gy[r] + jj * 8, w);
          if (r == 1 && wzh) __stcg(gz + jj * 8, w);
        }
      }
      }
      __syncwarp();
      if (k - OUT_LAG2 >= 0) flush_out(k - OUT_LAG2);
      cp_wait_all();
      __syncwarp();
    }
    for (int j = nchunks - OUT_LAG2; j < nchunks; ++j)
      if (j >= 0) flush_out(j);
    if (ghist) {  // the task's counts into the field's histogram
      __syncwarp();
#pragma unroll
      for (int b = 0; b < 8; ++b) {
        const unsigned v = whist[lane + 32 * b];
        if (v) atomicAdd(&ghist[lane + 32 * b], (unsigned long long)v);
      }
    }
    // right pads past the last step: tagged zeros (x + zz up to nx + kFPadR2 - 1)
    for (int S = nchunks * CH2; S < nx + kFPadR2 + 7; ++S) {
      if (wyh[0]) __stcg(wy[0] + S * 8, tag);
      if (wyh[1]) __stcg(wy[1] + S * 8, tag);
      if (wzh) __stcg(wz + S * 8, tag);
    }
    __syncwarp();
  }
}

template <typename C, bool REC = false, bool TR = false>
cudaError_t launch_r2_t(const FastArgs& fa, const FieldTable& ft, int sms, cudaStream_t s) {
  const size_t smem = (size_t)WPB * Smem2<C>::PER_WARP;
  static KernelAttr attr;
  cudaError_t e = kernel_smem(attr, sweep_r2_kernel<C, REC, TR>, smem);
  if (e != cudaSuccess) return e;
  const int per_sm_cached = kernel_occupancy(attr, sweep_r2_kernel<C, REC, TR>, 32 * WPB, smem);
  const long long ntasks = (long long)fa.npy * fa.npz * fa.nf;
  const long long diag = fa.npy < fa.npz ? fa.npy : fa.npz;
  long long active = (diag * ((fa.s.dims[0] + 14) / 14 + 1) + 64) * fa.nf;  // see launch_fast_t
  {  // EBZ_ACTIVE_SCALE: A/B experiments on the launch size
    static const char* sc = getenv("EBZ_ACTIVE_SCALE");
    if (sc) active = (long long)(active * atof(sc));
  }
  if (active > ntasks) active = ntasks;
  long long blocks = (active + WPB - 1) / WPB;
  if (blocks > (long long)sms * per_sm_cached) blocks = (long long)sms * per_sm_cached;
  if (blocks < 1) blocks = 1;
  sweep_r2_kernel<C, REC, TR><<<(unsigned)blocks, 32 * WPB, smem, s>>>(fa, ft);
  return cudaGetLastError();
}

}  // namespace

bool sweep_fast_supported(int ndim, int layers, long long dims0) {
  return (ndim == 2 || ndim == 3) && (layers == 1 || layers == 2) && dims0 < (1ll << 30);
}

// host: task table for a patch grid, ordered by wy * Y + wz * Z (ties by Y):
// a task's producers (Y - 1, Z), (Y, Z - 1), (Y - 1, Z - 1) always come
// first (deadlock-free ticket order for any positive weights), and weights
// proportional to the consumer's lag behind each producer hand out tickets
// in the order the tasks become runnable
void fast_task_table(int npy, int npz, unsigned int* out, int wy, int wz) {
  int t = 0;
  const int dmax = wy * (npy - 1) + wz * (npz - 1);
  for (int d = 0; d <= dmax; ++d)
    for (int Y = 0; Y < npy; ++Y) {
      const int r = d - wy * Y;
      if (r < 0 || r % wz) continue;
      const int Z = r / wz;
      if (Z >= npz) continue;
      out[t++] = (unsigned)Y | ((unsigned)Z << 16);
    }
}

// 3D, n = 1 compress runs the two-rows-per-lane kernel (8 x 8 patches;
// measured faster for compress, slower for decompress); EBZ_NO_R2 disables
// it for A/B comparisons
bool sweep_r2_used(int ndim, int layers, bool compress) {
  static const bool off = getenv("EBZ_NO_R2") != nullptr;
  return ndim == 3 && layers == 1 && compress && !off;
}

void fast_patch_grid(int ndim, const long long* dims, int layers, bool compress, int* npy,
                     int* npz) {
  if (ndim == 2) {
    *npy = (int)((dims[1] + 31) / 32);
    *npz = 1;
  } else {
    const int pz = sweep_r2_used(ndim, layers, compress) ? 8 : 4;
    *npy = (int)((dims[1] + 7) / 8);
    *npz = (int)((dims[2] + pz - 1) / pz);
  }
}

// tagged face buffer sizes (u64 words) for a grid
void fast_face_words(int ndim, const long long* dims, int layers, bool compress,
                     long long* ny_words, long long* nz_words) {
  int npy, npz;
  fast_patch_grid(ndim, dims, layers, compress, &npy, &npz);
  const long long ny = dims[1], nz = ndim == 3 ? dims[2] : 1;
  if (sweep_r2_used(ndim, layers, compress)) {  // skew-major blocks of 8 padded rows
    *ny_words = *nz_words = (long long)npy * npz * 8 * (dims[0] + kFPad2);
    return;
  }
  if (ndim == 3 && layers == 1) {  // skew-major blocks (nx + 4) x 4 and (nx + 8) x 8
    *ny_words = (long long)npy * npz * (dims[0] + 4) * 4;
    *nz_words = (long long)npy * npz * (dims[0] + 8) * 8;
    return;
  }
  const long long nx = dims[0];
  *ny_words = (long long)npy * layers * nz * nx;
  *nz_words = ndim == 3 ? (long long)npz * layers * ny * nx : 0;
}

cudaError_t launch_sweep_fast(const SweepArgs& a, const FieldTable& ft, int nf,
                              const unsigned int* d_tasks, int npy, int npz, bool compress,
                              bool rec, int sms, cudaStream_t s) {
  if (nf < 1 || nf > kBatchMax) return cudaErrorInvalidValue;
  FastArgs fa;
  fa.s = a;
  fa.tasks = d_tasks;
  fa.npy = npy;
  fa.npz = npz;
  fa.nf = nf;
  const bool wide = a.wide != 0;
  if (sweep_r2_used(a.ndim, a.layers, compress)) {
    if (a.trunc) {  // opt-in truncated-mantissa coding
      if (rec) return cudaErrorInvalidValue;
      return wide ? launch_r2_t<uint16_t, false, true>(fa, ft, sms, s)
                  : launch_r2_t<uint8_t, false, true>(fa, ft, sms, s);
    }
    if (rec)
      return wide ? launch_r2_t<uint16_t, true>(fa, ft, sms, s)
                  : launch_r2_t<uint8_t, true>(fa, ft, sms, s);
    return wide ? launch_r2_t<uint16_t>(fa, ft, sms, s) : launch_r2_t<uint8_t>(fa, ft, sms, s);
  }
#define EBZ_FAST(D, N)                                                                   \
  if (compress && a.trunc)                                                               \
    return rec ? cudaErrorInvalidValue                                                   \
               : (wide ? launch_fast_t<D, N, uint16_t, true, false, true>(fa, ft, sms, s) \
                       : launch_fast_t<D, N, uint8_t, true, false, true>(fa, ft, sms, s)); \
  if (compress && rec)                                                                   \
    return wide ? launch_fast_t<D, N, uint16_t, true, true>(fa, ft, sms, s)              \
                : launch_fast_t<D, N, uint8_t, true, true>(fa, ft, sms, s);              \
  if (compress)                                                                          \
    return wide ? launch_fast_t<D, N, uint16_t, true>(fa, ft, sms, s)                    \
                : launch_fast_t<D, N, uint8_t, true>(fa, ft, sms, s);                    \
  return wide ? launch_fast_t<D, N, uint16_t, false>(fa, ft, sms, s)                     \
              : launch_fast_t<D, N, uint8_t, false>(fa, ft, sms, s);
  if (a.ndim == 2 && a.layers == 1) { EBZ_FAST(2, 1) }
  if (a.ndim == 2 && a.layers == 2) { EBZ_FAST(2, 2) }
  if (a.ndim == 3 && a.layers == 1) { EBZ_FAST(3, 1) }
  if (a.ndim == 3 && a.layers == 2) { EBZ_FAST(3, 2) }
#undef EBZ_FAST
  return cudaErrorInvalidValue;
}
