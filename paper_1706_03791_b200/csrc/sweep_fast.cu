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
//   * older columns (x-1 .. x-n) stay in registers (a (n+1)^d history cube).
// Only the patch faces (rows y0-n..y0-1 and planes z0-n..z0-1) come from
// memory: producer patches store their face rows to the recon buffer as they
// go and publish epoch-tagged progress counters (release/acquire); consumers
// poll them per 16-step chunk and stage the face columns in a per-warp shared
// ring (double), prefetching the next chunk when its producers are ahead.
// Patches are handed out by an atomic ticket in hyperplane (Y + Z) order, so a
// task only waits on lower tickets -- deadlock free.
//
// Memory traffic.  Inputs (values / codes) are staged per 16-column chunk
// into shared tiles with cp.async (16-byte pieces when rows are aligned);
// outputs (codes / reconstructions) leave through shared tiles with
// row-coalesced stores.  Per point in compress: 4 B read, 1 B code written
// (+ 4 B for face rows only); decompress: 1 B code read, 4 B written.
//
// Arithmetic is bit-identical to the reference: the stencil sum runs in the
// reference's term order (lexicographic offsets, axis 0 slowest) in binary64
// without contraction; missing neighbours are zeros, which reproduces the
// boundary-reduced stencils exactly (up to the sign of a zero prediction,
// which never changes a code or a stored value); points with a coordinate
// equal to 1 use the n = 1 stencil when n = 2 (eff = min(n, min coord)).
#include "ebz_common.cuh"

namespace {

constexpr int CH = 16;        // steps per chunk
constexpr int RS = 4;         // ring slots (chunks)
constexpr int RX = CH * RS;   // ring columns
constexpr int WPB = 4;        // warps per block

template <int D> struct Patch;
template <> struct Patch<2> { static constexpr int PY = 32, PZ = 1; };
template <> struct Patch<3> { static constexpr int PY = 8, PZ = 4; };

struct FastArgs {
  SweepArgs s;
  const unsigned int* tasks;  // ticket -> Y | Z << 16
  int npy, npz;
  double inv_two_eb_unused;
};

// --- compile-time stencil ---------------------------------------------------
__host__ __device__ constexpr int cbin(int n, int k) {
  return k == 0 ? 1 : (n == 2 ? (k == 1 ? 2 : 1) : (n == 3 ? (k == 1 || k == 2 ? 3 : 1) : 1));
}
__host__ __device__ constexpr int coef(int n, int kx, int ky, int kz) {
  // -prod (-1)^k C(n, k)
  return -(((kx + ky + kz) & 1) ? -1 : 1) * cbin(n, kx) * cbin(n, ky) * cbin(n, kz);
}

template <int NN, int NB, int NA, int NC>
struct StencilSum {
  // H[b][a][c] = value at (z-b, y-a, x-c); terms in (kx, ky, kz) lexicographic
  // order (x slowest), i.e. c outermost, then a, then b.
  __device__ __forceinline__ static double eval(const double (&H)[NB][NA][NC]) {
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
          double t;
          if (k == 1) t = v;
          else if (k == -1) t = -v;
          else t = __dmul_rn((double)k, v);  // |k| = 2, 4, 8: exact
          if (first) { acc = t; first = false; }   // 0.0 + t == t (up to -0)
          else acc = __dadd_rn(acc, t);
        }
    return acc;
  }
};

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

template <int D, int N> struct Cfg {
  static constexpr int PY = Patch<D>::PY, PZ = Patch<D>::PZ;
  static constexpr int NB = D == 3 ? N + 1 : 1;     // z history depth
  static constexpr int SMAX = PY - 1 + PZ - 1;      // max lane skew
  static constexpr int NFY = D == 3 ? N * (PZ + N) : N;  // Y-face rows
  static constexpr int NFZ = D == 3 ? N * PY : 0;        // Z-face rows
  static constexpr int NFR = NFY + NFZ;
  static constexpr int IN_STRIDE_F = D == 2 ? 64 : 68;   // floats per tile row
  static constexpr int IN_STRIDE_B = D == 2 ? 64 : 80;   // bytes per u8 tile row
  static constexpr int FACE_PER_LANE = (NFR * CH + 31) / 32;
};

template <int D, int N, typename C, bool COMPRESS>
struct Smem {
  typedef Cfg<D, N> K;
  // inputs: compress -> float values; decompress -> codes (C)
  static constexpr int IN_BYTES = COMPRESS ? 32 * K::IN_STRIDE_F * 4
                                           : 32 * K::IN_STRIDE_B * (int)sizeof(C);
  // outputs: compress -> codes (C); decompress -> float recon
  static constexpr int OUT_BYTES = COMPRESS ? 32 * K::IN_STRIDE_B * (int)sizeof(C)
                                            : 32 * K::IN_STRIDE_F * 4;
  static constexpr int FACE_BYTES = K::NFR * RX * 8;
  static constexpr int PER_WARP = ((IN_BYTES + 15) / 16 + (OUT_BYTES + 15) / 16 +
                                   (FACE_BYTES + 15) / 16) * 16;
};

template <int D, int N, typename C, bool COMPRESS>
__global__ void __launch_bounds__(32 * WPB)
sweep_fast_kernel(FastArgs fa) {
  typedef Cfg<D, N> K;
  typedef Smem<D, N, C, COMPRESS> SM;
  constexpr int PY = K::PY, PZ = K::PZ, NB = K::NB, NA = N + 1, NC = N + 1;
  const SweepArgs& a = fa.s;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int la = lane % PY, lb = lane / PY;  // (a, b)
  const int sig = la + lb;
  unsigned char* wbase = smem_raw + warp * SM::PER_WARP;
  unsigned char* in_tile = wbase;
  unsigned char* out_tile = wbase + ((SM::IN_BYTES + 15) / 16) * 16;
  double* face = reinterpret_cast<double*>(out_tile + ((SM::OUT_BYTES + 15) / 16) * 16);
  // block-shared tail: histogram (compress, m <= 12) or dequant table (decompress)
  unsigned char* tail = smem_raw + WPB * SM::PER_WARP;
  unsigned int* s_hist = reinterpret_cast<unsigned int*>(tail);
  double* s_qtab = reinterpret_cast<double*>(tail);

  const int nsym = 1 << a.m;
  const bool smem_hist = COMPRESS && a.m <= 12;
  const double eb = a.info->eb;
  const double two_eb = __dmul_rn(2.0, eb);
  const double inv = 1.0 / two_eb;
  const bool fast_ok = isfinite(inv) && inv > 0.0 && two_eb >= 0x1p-1000 && inv >= 0x1p-1000 &&
                       inv <= 0x1p1000;
  const bool qtab = !COMPRESS && a.m <= 12;
  if (smem_hist)
    for (int i = threadIdx.x; i < nsym; i += blockDim.x) s_hist[i] = 0;
  if (qtab)
    for (int i = threadIdx.x; i < nsym; i += blockDim.x)
      s_qtab[i] = __dmul_rn((double)(i - a.center), two_eb);
  __syncthreads();
  if (!(eb > 0.0)) return;

  const long long nx = a.dims[0], ny = a.dims[1], nz = D == 3 ? a.dims[2] : 1;
  const long long ntasks = (long long)fa.npy * fa.npz;
  const long long steps_total = nx + K::SMAX;
  const unsigned long long tag = (unsigned long long)a.epoch << 32;
  const float* values = reinterpret_cast<const float*>(a.values);
  float* recon = reinterpret_cast<float*>(a.recon);
  C* codes = reinterpret_cast<C*>(a.codes);
  const float* unpred = reinterpret_cast<const float*>(a.unpred);
  const unsigned long long n_unpred = COMPRESS ? 0ull : a.info->n_unpred;
  const bool al16_in = COMPRESS ? (nx % 4 == 0) : (nx % 16 == 0 && sizeof(C) == 1);

  unsigned long long zeros_total = 0;
  int hist_code = -1;
  unsigned int hist_run = 0;

  for (;;) {
    unsigned int tk = 0;
    if (lane == 0) tk = atomicAdd(a.ticket, 1u);
    tk = __shfl_sync(EBZ_FULL, tk, 0);
    if ((long long)tk >= ntasks) break;
    const unsigned int tv = fa.tasks[tk];
    const int PYi = (int)(tv & 0xffff), PZi = (int)(tv >> 16);
    const long long y0 = (long long)PYi * PY, z0 = (long long)PZi * PZ;
    const long long y = y0 + la, z = z0 + lb;
    const bool rv = y < ny && z < nz;
    const long long rowi = z * ny + y;
    const long long base = rowi * nx;
    const int self = PZi * fa.npy + PYi;
    // producers (patch ids) or -1
    const int prodY = PYi > 0 ? self - 1 : -1;
    const int prodZ = (D == 3 && PZi > 0) ? self - fa.npy : -1;
    const int prodYZ = (D == 3 && PYi > 0 && PZi > 0) ? self - fa.npy - 1 : -1;
    // face lanes store their outputs for consumer patches
    const bool face_lane = rv && (la >= PY - N || (D == 3 && lb >= PZ - N));

    // history cube: H[b][a][c] = r(z-b, y-a, x-c)
    double H[NB][NA][NC];
#pragma unroll
    for (int b = 0; b < NB; ++b)
#pragma unroll
      for (int aa = 0; aa < NA; ++aa)
#pragma unroll
        for (int c = 0; c < NC; ++c) H[b][aa][c] = 0.0;

    // decompress: verbatim-value cursor for this row
    unsigned long long ucur = 0;
    float u0 = 0.f, u1 = 0.f;
    if (!COMPRESS && rv) {
      ucur = a.rowbase[rowi];
      if (ucur < n_unpred) u0 = __ldg(unpred + ucur);
      if (ucur + 1 < n_unpred) u1 = __ldg(unpred + ucur + 1);
    }
    unsigned long long zeros = 0;

    // --- staging helpers (lambdas capture the task geometry) ----------------
    // input x-chunk j -> in_tile ring slot (j % RS)
    auto load_in = [&](long long j) {
      const long long x0 = j * CH;
      if (x0 >= nx) return;
      const int slot = (int)(j % RS);
      if (COMPRESS) {
        float* tile = reinterpret_cast<float*>(in_tile);
        if (al16_in) {
#pragma unroll
          for (int i = 0; i < (32 * CH / 4) / 32; ++i) {
            const int p = lane + 32 * i;
            const int r = p / (CH / 4), c4 = p % (CH / 4);
            const int ra = r % PY, rb = r / PY;
            const long long yy = y0 + ra, zz = z0 + rb;
            const long long xx = x0 + 4 * c4;
            float* dst = tile + r * K::IN_STRIDE_F + slot * CH + 4 * c4;
            long long rem = nx - xx;
            const int bytes = (yy < ny && zz < nz && rem > 0) ? (rem >= 4 ? 16 : (int)rem * 4) : 0;
            const float* src = values + (bytes ? (zz * ny + yy) * nx + xx : 0);
            cp_async16(dst, src, bytes);
          }
        } else {
#pragma unroll 4
          for (int i = 0; i < CH; ++i) {
            const int p = lane + 32 * i;
            const int r = p / CH, c = p % CH;
            const int ra = r % PY, rb = r / PY;
            const long long yy = y0 + ra, zz = z0 + rb, xx = x0 + c;
            float* dst = tile + r * K::IN_STRIDE_F + slot * CH + c;
            const int bytes = (yy < ny && zz < nz && xx < nx) ? 4 : 0;
            const float* src = values + (bytes ? (zz * ny + yy) * nx + xx : 0);
            cp_async4(dst, src, bytes);
          }
        }
        cp_commit();
      } else {
        C* tile = reinterpret_cast<C*>(in_tile);
        if (al16_in) {
          // 16 one-byte codes per row piece
          const int r = lane;
          const int ra = r % PY, rb = r / PY;
          const long long yy = y0 + ra, zz = z0 + rb;
          long long rem = nx - x0;
          const int bytes = (yy < ny && zz < nz && rem > 0) ? (rem >= 16 ? 16 : (int)rem) : 0;
          C* dst = tile + r * K::IN_STRIDE_B + slot * CH;
          const C* src = codes + (bytes ? (zz * ny + yy) * nx + x0 : 0);
          if (bytes == 16) {
            cp_async16(dst, src, 16);
          } else {
            for (int c = 0; c < CH; ++c) dst[c] = c < bytes ? src[c] : (C)0;
          }
          cp_commit();
        } else {
#pragma unroll 4
          for (int i = 0; i < CH; ++i) {
            const int p = lane + 32 * i;
            const int r = p / CH, c = p % CH;
            const int ra = r % PY, rb = r / PY;
            const long long yy = y0 + ra, zz = z0 + rb, xx = x0 + c;
            C v = 0;
            if (yy < ny && zz < nz && xx < nx) v = codes[(zz * ny + yy) * nx + xx];
            tile[r * K::IN_STRIDE_B + slot * CH + c] = v;
          }
        }
      }
    };
    // face x-chunk j: registers first (prefetch), then shared ring
    double freg[K::FACE_PER_LANE];
    auto face_fetch = [&](long long j) {
      const long long x0 = j * CH;
#pragma unroll
      for (int i = 0; i < K::FACE_PER_LANE; ++i) {
        const int p = lane + 32 * i;
        double v = 0.0;
        if (p < K::NFR * CH) {
          const int fr = p / CH, c = p % CH;
          long long yy, zz;
          if (fr < K::NFY) {
            const int ap = fr / (D == 3 ? PZ + N : 1) + 1;
            const int zo = D == 3 ? fr % (PZ + N) : N;
            yy = y0 - ap;
            zz = z0 + zo - N;
          } else {
            const int q = fr - K::NFY;
            const int bp = q / PY + 1;
            yy = y0 + q % PY;
            zz = z0 - bp;
          }
          const long long xx = x0 + c;
          if (yy >= 0 && zz >= 0 && yy < ny && zz < nz && xx < nx)
            v = (double)__ldcg(recon + (zz * ny + yy) * nx + xx);
        }
        freg[i] = v;
      }
    };
    auto face_store = [&](long long j) {
      const int slot = (int)(j % RS);
#pragma unroll
      for (int i = 0; i < K::FACE_PER_LANE; ++i) {
        const int p = lane + 32 * i;
        if (p < K::NFR * CH) {
          const int fr = p / CH, c = p % CH;
          face[fr * RX + slot * CH + c] = freg[i];
        }
      }
    };
    auto deps_need = [&](long long j) -> unsigned long long {
      long long need = (j + 1) * CH + K::SMAX;
      if (need > steps_total) need = steps_total;
      return tag | (unsigned long long)need;
    };
    auto deps_ready = [&](long long j) -> bool {  // non-blocking, warp-uniform
      const unsigned long long need = deps_need(j);
      bool ok = true;
      if (lane == 0 && prodY >= 0) ok = ld_acquire_u64(a.progress + prodY) >= need;
      if (lane == 1 && prodZ >= 0) ok = ld_acquire_u64(a.progress + prodZ) >= need;
      if (lane == 2 && prodYZ >= 0) ok = ld_acquire_u64(a.progress + prodYZ) >= need;
      return __all_sync(EBZ_FULL, ok);
    };
    auto deps_wait = [&](long long j) {
      const unsigned long long need = deps_need(j);
      int p = -1;
      if (lane == 0) p = prodY;
      if (lane == 1) p = prodZ;
      if (lane == 2) p = prodYZ;
      if (p >= 0)
        while (ld_acquire_u64(a.progress + p) < need) __nanosleep(40);
      __syncwarp();
    };
    // output x-chunk j: shared tile -> global, row-coalesced
    auto flush_out = [&](long long j) {
      const long long x0 = j * CH;
      if (x0 >= nx) return;
      const int slot = (int)(j % RS);
#pragma unroll 4
      for (int i = 0; i < CH; ++i) {
        const int p = lane + 32 * i;
        const int r = p / CH, c = p % CH;
        const int ra = r % PY, rb = r / PY;
        const long long yy = y0 + ra, zz = z0 + rb, xx = x0 + c;
        if (yy < ny && zz < nz && xx < nx) {
          const long long gi = (zz * ny + yy) * nx + xx;
          if (COMPRESS) {
            codes[gi] = reinterpret_cast<C*>(out_tile)[r * K::IN_STRIDE_B + slot * CH + c];
          } else {
            recon[gi] = reinterpret_cast<float*>(out_tile)[r * K::IN_STRIDE_F + slot * CH + c];
          }
        }
      }
    };

    // prologue: inputs for x-chunks 0 (and 1 prefetched later), faces chunk 0
    load_in(0);
    deps_wait(0);
    face_fetch(0);
    face_store(0);
    bool face_next = false;
    cp_wait_all();
    __syncwarp();

    const long long nchunks = (steps_total + CH - 1) / CH;
    constexpr int OUT_LAG = (K::SMAX + CH - 1) / CH;  // x-chunks still being written
    for (long long k = 0; k < nchunks; ++k) {
      const long long S0 = k * CH;
      // faces for x-chunk k must be in the ring
      if (k > 0 && !face_next) {
        deps_wait(k);
        face_fetch(k);
        face_store(k);
        __syncwarp();
      }
      // prefetch next chunk's inputs (async) and, if producers are ahead, faces
      load_in(k + 1);
      face_next = deps_ready(k + 1);
      if (face_next) face_fetch(k + 1);

#pragma unroll 1
      for (int st = 0; st < CH; ++st) {
        const long long S = S0 + st;
        const long long x = S - sig;
        const bool act = rv && x >= 0 && x < nx;
        // ---- receive column x from neighbour lanes (previous step's column 0)
        double nw[NB][NA];
#pragma unroll
        for (int b = 0; b < NB; ++b)
#pragma unroll
          for (int aa = 0; aa < NA; ++aa) {
            if (aa == 0 && b == 0) continue;
            double v;
            if (aa >= 1) v = __shfl_up_sync(EBZ_FULL, H[b][aa - 1][0], 1);
            else v = __shfl_up_sync(EBZ_FULL, H[b - 1][0][0], PY);
            nw[b][aa] = v;
          }
        // boundary lanes take face values from the ring
        const int fcol = (int)(((x % RX) + RX) % RX);
        const bool xin = x >= 0;
#pragma unroll
        for (int b = 0; b < NB; ++b)
#pragma unroll
          for (int aa = 0; aa < NA; ++aa) {
            if (aa == 0 && b == 0) continue;
            if (aa >= 1 && la == 0) {
              const int fr = (aa - 1) * (D == 3 ? PZ + N : 1) + (D == 3 ? lb - b + N : 0);
              nw[b][aa] = xin ? face[fr * RX + fcol] : 0.0;
            } else if (aa == 0 && lb == 0) {
              const int fr = K::NFY + (b - 1) * PY + la;
              nw[b][aa] = xin ? face[fr * RX + fcol] : 0.0;
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
          if (eff1) {
            double h1[NB == 1 ? 1 : 2][2][2];
#pragma unroll
            for (int b = 0; b < (NB == 1 ? 1 : 2); ++b)
#pragma unroll
              for (int aa = 0; aa < 2; ++aa)
#pragma unroll
                for (int c = 0; c < 2; ++c) h1[b][aa][c] = H[b][aa][c];
            pred = StencilSum<1, (NB == 1 ? 1 : 2), 2, 2>::eval(h1);
          } else {
            pred = StencilSum<N, NB, NA, NC>::eval(H);
          }
        } else {
          pred = StencilSum<N, NB, NA, NC>::eval(H);
        }
        const int col = (int)(((x % RX) + RX) % RX);
        float r = 0.f;
        if (COMPRESS) {
          const float xv = act ? reinterpret_cast<const float*>(in_tile)[lane * K::IN_STRIDE_F + col]
                               : 0.f;
          int code = 0;
          if (act) {
            code = quantize_fast<float>(xv, pred, eb, two_eb, inv, fast_ok, a.center, r);
            reinterpret_cast<C*>(out_tile)[lane * K::IN_STRIDE_B + col] = (C)code;
            zeros += code == 0;
            // run-length histogram
            if (code == hist_code) {
              ++hist_run;
            } else {
              if (hist_run) {
                if (smem_hist) atomicAdd(&s_hist[hist_code], hist_run);
                else atomicAdd(&a.hist[hist_code], (unsigned long long)hist_run);
              }
              hist_code = code;
              hist_run = 1;
            }
          }
        } else {
          if (act) {
            const int code = (int)reinterpret_cast<const C*>(in_tile)[lane * K::IN_STRIDE_B + col];
            if (code == 0) {
              if (ucur < n_unpred) {
                r = u0;
              } else {
                atomicOr(&a.info_w->status, ST_UNDERRUN);
              }
              ++ucur;
              ++zeros;
              u0 = u1;
              if (ucur + 1 < n_unpred) u1 = __ldg(unpred + ucur + 1);
            } else {
              const double q = qtab ? s_qtab[code]
                                    : __dmul_rn((double)(code - a.center), two_eb);
              r = __double2float_rn(__dadd_rn(pred, q));
            }
            if (!isfinite(r)) atomicOr(&a.info_w->status, ST_NONFINITE_OUT);
            reinterpret_cast<float*>(out_tile)[lane * K::IN_STRIDE_F + col] = r;
          }
        }
        if (act && face_lane) __stcg(recon + base + x, r);
        H[0][0][0] = act ? (double)r : 0.0;
      }
      // ---- end of chunk: publish progress, drain outputs, stage next faces
      __syncwarp();
      if (lane == 0) {
        __threadfence();
        const long long done = S0 + CH < steps_total ? S0 + CH : steps_total;
        st_release_u64(a.progress + self, tag | (unsigned long long)done);
      }
      if (k - OUT_LAG >= 0) flush_out(k - OUT_LAG);
      if (face_next) face_store(k + 1);
      cp_wait_all();
      __syncwarp();
    }
    // flush remaining output chunks
    for (long long j = nchunks - OUT_LAG; j < nchunks; ++j)
      if (j >= 0) flush_out(j);
    __syncwarp();
    zeros_total += zeros;
  }
  // histogram tail + counters
  if (COMPRESS && hist_run) {
    if (smem_hist) atomicAdd(&s_hist[hist_code], hist_run);
    else atomicAdd(&a.hist[hist_code], (unsigned long long)hist_run);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) zeros_total += __shfl_xor_sync(EBZ_FULL, zeros_total, o);
  if (lane == 0 && zeros_total) {
    if (COMPRESS) atomicAdd(&a.info_w->n_unpred, zeros_total);
    else atomicAdd(&a.info_w->used, zeros_total);
  }
  if (smem_hist) {
    __syncthreads();
    for (int i = threadIdx.x; i < nsym; i += blockDim.x)
      if (s_hist[i]) atomicAdd(&a.hist[i], (unsigned long long)s_hist[i]);
  }
}

template <int D, int N, typename C, bool COMPRESS>
cudaError_t launch_fast_t(const FastArgs& fa, int sms, cudaStream_t s) {
  typedef Smem<D, N, C, COMPRESS> SM;
  const int m = fa.s.m;
  size_t tail = COMPRESS ? (m <= 12 ? ((size_t)4 << m) : 0) : (m <= 12 ? ((size_t)8 << m) : 0);
  const size_t smem = (size_t)WPB * SM::PER_WARP + tail;
  static size_t attr = 0;
  if (attr < smem) {
    cudaError_t e = cudaFuncSetAttribute(sweep_fast_kernel<D, N, C, COMPRESS>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    attr = smem;
  }
  const long long ntasks = (long long)fa.npy * fa.npz;
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sweep_fast_kernel<D, N, C, COMPRESS>,
                                                32 * WPB, smem);
  if (per_sm < 1) per_sm = 1;
  long long blocks = (ntasks + WPB - 1) / WPB;
  if (blocks > (long long)sms * per_sm) blocks = (long long)sms * per_sm;
  if (blocks < 1) blocks = 1;
  sweep_fast_kernel<D, N, C, COMPRESS><<<(unsigned)blocks, 32 * WPB, smem, s>>>(fa);
  return cudaGetLastError();
}

}  // namespace

bool sweep_fast_supported(int ndim, int layers, long long dims0) {
  (void)dims0;
  return (ndim == 2 || ndim == 3) && (layers == 1 || layers == 2);
}

// host: hyperplane-ordered task table for a patch grid
void fast_task_table(int npy, int npz, unsigned int* out) {
  int t = 0;
  for (int d = 0; d <= npy + npz - 2; ++d)
    for (int Y = 0; Y < npy; ++Y) {
      const int Z = d - Y;
      if (Z < 0 || Z >= npz) continue;
      out[t++] = (unsigned)Y | ((unsigned)Z << 16);
    }
}

void fast_patch_grid(int ndim, const long long* dims, int* npy, int* npz) {
  if (ndim == 2) {
    *npy = (int)((dims[1] + 31) / 32);
    *npz = 1;
  } else {
    *npy = (int)((dims[1] + 7) / 8);
    *npz = (int)((dims[2] + 3) / 4);
  }
}

cudaError_t launch_sweep_fast(const SweepArgs& a, const unsigned int* d_tasks, int npy, int npz,
                              bool compress, int sms, cudaStream_t s) {
  FastArgs fa;
  fa.s = a;
  fa.tasks = d_tasks;
  fa.npy = npy;
  fa.npz = npz;
  fa.inv_two_eb_unused = 0.0;
  const bool wide = a.m > 8;
#define EBZ_FAST(D, N)                                                                   \
  if (compress)                                                                          \
    return wide ? launch_fast_t<D, N, uint16_t, true>(fa, sms, s)                        \
                : launch_fast_t<D, N, uint8_t, true>(fa, sms, s);                        \
  return wide ? launch_fast_t<D, N, uint16_t, false>(fa, sms, s)                         \
              : launch_fast_t<D, N, uint8_t, false>(fa, sms, s);
  if (a.ndim == 2 && a.layers == 1) { EBZ_FAST(2, 1) }
  if (a.ndim == 2 && a.layers == 2) { EBZ_FAST(2, 2) }
  if (a.ndim == 3 && a.layers == 1) { EBZ_FAST(3, 1) }
  if (a.ndim == 3 && a.layers == 2) { EBZ_FAST(3, 2) }
#undef EBZ_FAST
  return cudaErrorInvalidValue;
}
