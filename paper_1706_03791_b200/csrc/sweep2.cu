// sweep2.cu -- low-latency hyperplane wavefront for 2D grids, layers n = 1, 2
// (float32 or binary64 elements): compress_scan / decompress_scan of ebzip/_kernels.py:48-105
// for 2D fields, where the sweep is one dependent chain of nx + ny
// point-steps and a lone warp's step latency is all that counts.
//
// Geometry as in sweep_fast.cu: a warp task owns 32 rows (lines along x);
// lane a processes column x = S - a at warp step S; row y - 1 arrives by one
// shuffle (n = 2: row y - 2 is relayed, lane a receives what lane a - 1
// received a step earlier); the patch above hands its last n rows over as
// epoch-tagged 64-bit face words in global memory (same face layout: rows
// n PY .. n PY + n - 1 of the Y-face buffer belong to patch PY).  What differs
// is the step itself.  The one-row kernel's step is three basic blocks
// (slow-path vote, face-tag vote, spin loop) of ~120 instructions; measured on
// B200 a lone warp needs ~520 cycles for it, against a dependent chain (2
// SHFL, 9 FP64 ops, the F2F pair, a compare, a select) of ~200.  Here a block
// of 8 steps (4 for n = 2) is ONE basic block:
//   * compress runs the reciprocal quantizer speculatively for the whole
//     block and OR-s the (2^-30-rare) "needs the exact division" flags; ONE
//     vote per block covers them and the tag check of the next block's face
//     words; on a hit the block is replayed from the saved history with the
//     exact quantizer.  Face words of the block are stored after the vote, so
//     no consumer ever sees a speculative value;
//   * lane 0's face words are requested a block ahead (predicated loads into
//     registers preset to the tagged zero);
//   * interior blocks (every lane inside its row, past the n = 1 boundary
//     columns) carry no range selects and no boundary rule;
//   * per step and lane: one shared load (value / code), one shared store
//     (code / reconstruction); everything else is the recurrence.
// Decompress has no slow path; its verbatim values are fetched a block ahead
// from the row's cursor (the codes of the next block are already resident)
// and prefetched into L2 a few blocks further.
//
// Arithmetic is the same as sweep_fast.cu (binary64, reference term order --
// n = 1: (up + left) - upleft; n = 2: the eight terms x offset outermost --
// no contraction; points with a coordinate equal to 1 use the n = 1 stencil;
// RNE float32 cast by the F2F pair, none for binary64 elements), so the bytes
// are identical to the one-row / generic kernel's and to the reference's.
// binary64 elements use 16-byte face words {value, epoch} (struct Face) and
// 4-step blocks; everything else is shared.
#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include "ebz_common.cuh"

namespace {

constexpr int RX = 64;         // tile ring columns
#ifndef EBZ_S2_AHEAD
#define EBZ_S2_AHEAD 32
#endif
constexpr int kUnpredAhead = EBZ_S2_AHEAD;  // verbatim values prefetched ahead of a row's cursor
// warps per block (measured on cfg2: compress 0.84 ms at 1, 2 or 4; decompress
// 0.75 / 0.73 / 0.77 ms)
#ifndef EBZ_S2_WPB
#define EBZ_S2_WPB 2
#endif
constexpr int WPB = EBZ_S2_WPB;

// steps per block: 8 for n = 1; 4 for n = 2 (two face streams and a
// nine-value history: the register budget of an 8-step block is not there)
// (binary64 elements: 4 as well -- twice the registers per value and face word)
template <int N, typename T> struct Blk {
  static constexpr int BS = (N == 1 && sizeof(T) == 4) ? 8 : 4;
  static constexpr int NCH = RX / BS;                 // ring slots (chunks of BS columns)
  static constexpr int PD = BS == 8 ? 3 : 6;          // input prefetch distance (blocks)
  static constexpr int WLAST = (BS + 30) / BS;        // chunk c is last written in block c + WLAST
};

struct S2Args {
  SweepArgs s;
  const unsigned int* tasks;   // task -> patch row (hyperplane order = row order)
  int npy;
  int nf;
};

template <typename C, typename T> struct Sm2 {
  // element tile (row stride 64 elements: the skewed per-step accesses are
  // conflict-free for float32) and code tile (row stride 80 codes)
  static constexpr int CODE_STRIDE = RX + 16;
  static constexpr int F_BYTES = 32 * RX * (int)sizeof(T);
  static constexpr int C_BYTES = 32 * CODE_STRIDE * (int)sizeof(C);
  static constexpr int F_OFF = 0;
  static constexpr int C_OFF = F_BYTES;
  static constexpr int PER_WARP = F_BYTES + C_BYTES;
};

__device__ __forceinline__ void cpa16(unsigned s, const void* g, int bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(g), "r"(bytes));
}
__device__ __forceinline__ void cpa4(unsigned s, const void* g, int bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(s), "l"(g), "r"(bytes));
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int K> __device__ __forceinline__ void cpa_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(K));
}
__device__ __forceinline__ unsigned saddr(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ unsigned pin(unsigned a) {
  asm volatile("" : "+r"(a));
  return a;
}
__device__ __forceinline__ float lds32(unsigned a) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts32(unsigned a, float v) {
  asm volatile("st.shared.f32 [%0], %1;" ::"r"(a), "f"(v));
}
// element accesses by type (float32 / binary64)
__device__ __forceinline__ void lds_t(unsigned a, float& v) { v = lds32(a); }
__device__ __forceinline__ void lds_t(unsigned a, double& v) {
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
}
__device__ __forceinline__ void sts_t(unsigned a, float, double r) { sts32(a, __double2float_rn(r)); }
__device__ __forceinline__ void sts_t(unsigned a, double, double r) {
  asm volatile("st.shared.f64 [%0], %1;" ::"r"(a), "d"(r));
}
__device__ __forceinline__ void cpa8(unsigned s, const void* g, int bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(g), "r"(bytes));
}
__device__ __forceinline__ void ldg_nc_if(float& v, const float* p, unsigned ok) {
  asm volatile("{ .reg .pred q; setp.ne.u32 q, %2, 0; @q ld.global.nc.f32 %0, [%1]; }"
               : "+f"(v) : "l"(p), "r"(ok));
}
__device__ __forceinline__ void ldg_nc_if(double& v, const double* p, unsigned ok) {
  asm volatile("{ .reg .pred q; setp.ne.u32 q, %2, 0; @q ld.global.nc.f64 %0, [%1]; }"
               : "+d"(v) : "l"(p), "r"(ok));
}
template <typename C> __device__ __forceinline__ int lds_c(unsigned a) {
  unsigned v;
  if (sizeof(C) == 2) asm volatile("ld.shared.u16 %0, [%1];" : "=r"(v) : "r"(a));
  else asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(a));
  return (int)v;
}
template <typename C> __device__ __forceinline__ void sts_c(unsigned a, int v) {
  if (sizeof(C) == 2) asm volatile("st.shared.u16 [%0], %1;" ::"r"(a), "r"(v));
  else asm volatile("st.shared.u8 [%0], %1;" ::"r"(a), "r"(v));
}
__device__ __forceinline__ void st_face_if(unsigned long long* p, unsigned lo, unsigned hi,
                                           bool pred) {
  asm volatile("{ .reg .pred q; setp.ne.u32 q, %3, 0; @q st.global.cg.v2.b32 [%0], {%1, %2}; }"
               ::"l"(p), "r"(lo), "r"(hi), "r"((unsigned)pred) : "memory");
}
__device__ __forceinline__ unsigned long long ld_face(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.global.cg.u64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ double untag(unsigned long long w) {
  return __longlong_as_double((long long)(w & ~(unsigned long long)kTagMask));
}

// Face words.  float32: the binary64 of the reconstruction with the launch
// epoch in its 29 always-zero low mantissa bits (one aligned 8-byte access
// carries value and tag).  binary64 has no spare bits: the word is 16 bytes
// {value, epoch}, read and written with ONE aligned 16-byte access (a single
// transaction on the memory path, the same reliance as 16-byte status words
// in decoupled look-back scans).
template <typename T> struct Face;
template <> struct Face<float> {
  typedef unsigned long long W;
  __device__ static W zero(unsigned ep) { return ep; }
  __device__ static unsigned diff(const W& w, unsigned ep) { return ((unsigned)w ^ ep) & kTagMask; }
  __device__ static double val(const W& w) { return untag(w); }
  __device__ static void ld_if(W& w, const W* p, unsigned ok) {
    asm volatile("{ .reg .pred q; setp.ne.u32 q, %2, 0; @q ld.global.cg.u64 %0, [%1]; }"
                 : "+l"(w) : "l"(p), "r"(ok));
  }
  __device__ static W ld(const W* p) { return ld_face(p); }
  __device__ static void st_if(W* p, double r, unsigned ep, bool pred) {
    st_face_if(p, (unsigned)__double2loint(r) | ep, (unsigned)__double2hiint(r), pred);
  }
};
template <> struct Face<double> {
  typedef ulonglong2 W;
  __device__ static W zero(unsigned ep) { return make_ulonglong2(0ull, (unsigned long long)ep); }
  __device__ static unsigned diff(const W& w, unsigned ep) {
    return (unsigned)(w.y != (unsigned long long)ep);
  }
  __device__ static double val(const W& w) { return __longlong_as_double((long long)w.x); }
  __device__ static void ld_if(W& w, const W* p, unsigned ok) {
    asm volatile("{ .reg .pred q; setp.ne.u32 q, %3, 0; @q ld.global.cg.v2.u64 {%0, %1}, [%2]; }"
                 : "+l"(w.x), "+l"(w.y) : "l"(p), "r"(ok));
  }
  __device__ static W ld(const W* p) {
    W w;
    asm volatile("ld.global.cg.v2.u64 {%0, %1}, [%2];" : "=l"(w.x), "=l"(w.y) : "l"(p));
    return w;
  }
  __device__ static void st_if(W* p, double r, unsigned ep, bool pred) {
    asm volatile("{ .reg .pred q; setp.ne.u32 q, %3, 0; @q st.global.cg.v2.u64 [%0], {%1, %2}; }"
                 ::"l"(p), "l"((unsigned long long)__double_as_longlong(r)),
                   "l"((unsigned long long)ep), "r"((unsigned)pred) : "memory");
  }
};

// Face words of one block for lane 0: columns [x0, x0 + BS) of the N face
// rows above the patch (stream s = row y0 - 1 - s); outside [0, nx) (or
// without a producer patch) the tagged zero.
template <int N, typename T> struct FaceIn {
  static constexpr int BS = Blk<N, T>::BS;
  typedef typename Face<T>::W W;
  const W* row[N];  // null: no producer patch / not lane 0
  int nx;
  unsigned ep;
  // predicated loads into registers preset to the tagged zero (a select
  // after the load would wait for the data on the spot)
  __device__ __forceinline__ void load(int x0, W (&w)[N][BS]) const {
#pragma unroll
    for (int s = 0; s < N; ++s)
#pragma unroll
      for (int j = 0; j < BS; ++j) {
        w[s][j] = Face<T>::zero(ep);
        const unsigned ok = row[s] != nullptr && (unsigned)(x0 + j) < (unsigned)nx;
        Face<T>::ld_if(w[s][j], row[s] + x0 + j, ok);
      }
  }
  __device__ __forceinline__ bool missing(const W (&w)[N][BS]) const {
    unsigned d = 0;
#pragma unroll
    for (int s = 0; s < N; ++s)
#pragma unroll
      for (int j = 0; j < BS; ++j) d |= Face<T>::diff(w[s][j], ep);
    return d != 0;
  }
  // spin until every word carries this launch's tag (warp-uniform call)
  __device__ __forceinline__ void settle(int x0, W (&w)[N][BS]) const {
    bool miss = missing(w);
    if (!__any_sync(EBZ_FULL, miss)) return;
    for (unsigned ns = 16;; ns = ns < 256 ? 2 * ns : ns) {
      if (miss) {
        miss = false;
#pragma unroll
        for (int s = 0; s < N; ++s)
#pragma unroll
          for (int j = 0; j < BS; ++j)
            if (Face<T>::diff(w[s][j], ep)) {
              w[s][j] = Face<T>::ld(row[s] + x0 + j);
              miss |= Face<T>::diff(w[s][j], ep) != 0;
            }
      }
      if (!__any_sync(EBZ_FULL, miss)) break;
      __nanosleep(ns);
    }
  }
};

// The recurrence state of a lane: its own row's last N values and the N rows
// above at columns x .. x - N.  step() takes the values arriving for column x
// (row y - 1 from lane - 1's newest value, row y - 2 relayed from what lane - 1
// received a step earlier; lane 0: the face words) and returns the prediction.
template <int N> struct Hist {
  double L[N];         // r(y, x - 1 - i)
  double U[N][N + 1];  // r(y - 1 - s, x - c)
  __device__ __forceinline__ void clear() {
#pragma unroll
    for (int i = 0; i < N; ++i) L[i] = 0.0;
#pragma unroll
    for (int s = 0; s < N; ++s)
#pragma unroll
      for (int c = 0; c <= N; ++c) U[s][c] = 0.0;
  }
  // shift in column x of the rows above; EFF1: this point has a coordinate
  // equal to 1 and uses the n = 1 stencil (eff = min(n, min coordinate))
  __device__ __forceinline__ double predict(const double (&fv)[N], int lane, bool eff1) {
    double in[N];
    in[0] = __shfl_up_sync(EBZ_FULL, L[0], 1);
    if (N == 2) in[1] = __shfl_up_sync(EBZ_FULL, U[0][0], 1);
#pragma unroll
    for (int s = 0; s < N; ++s) {
      if (lane == 0) in[s] = fv[s];
#pragma unroll
      for (int c = N; c >= 1; --c) U[s][c] = U[s][c - 1];
      U[s][0] = in[s];
    }
    // reference term order: x offset outermost, then y; binary64, no contraction
    const double p1 = __dsub_rn(__dadd_rn(U[0][0], L[0]), U[0][1]);
    if (N == 1) return p1;
    double acc = __dmul_rn(2.0, U[0][0]);
    acc = __dsub_rn(acc, U[N - 1][0]);
    acc = __dadd_rn(acc, __dmul_rn(2.0, L[0]));
    acc = __dadd_rn(acc, __dmul_rn(-4.0, U[0][1]));
    acc = __dadd_rn(acc, __dmul_rn(2.0, U[N - 1][1]));
    acc = __dsub_rn(acc, L[N - 1]);
    acc = __dadd_rn(acc, __dmul_rn(2.0, U[0][N]));
    acc = __dsub_rn(acc, U[N - 1][N]);
    return eff1 ? p1 : acc;
  }
  __device__ __forceinline__ void push(double r) {
#pragma unroll
    for (int i = N - 1; i >= 1; --i) L[i] = L[i - 1];
    L[0] = r;
  }
};

// ---------------------------------------------------------------------------
// compress.  Per block b (steps [BS b, BS b + BS), lane's columns xb .. xb +
// BS - 1, xb = BS b - lane), in program order:
//   request the next block's face words (lane 0) and the input columns of
//   block b + PD (cp.async); flush the code chunk completed two blocks ago;
//   the chain, with the validated codes of block b - 1 (tile stores) and the
//   value loads of block b + 1 in its latency shadows;
//   ONE vote: a lane needs the exact division (replay the block) or a face
//   word of the next block is not there yet (spin on it);
//   the block's face words leave.
template <int N, typename C, typename T>
__global__ void __launch_bounds__(32 * WPB, (sizeof(T) == 8 ? 4 : 12 / WPB))
sweep2c_kernel(const __grid_constant__ S2Args fa, const __grid_constant__ FieldTable ft) {
  typedef Sm2<C, T> SM;
  typedef Blk<N, T> B;
  typedef typename Face<T>::W W;
  constexpr int BS = B::BS;
  constexpr int EP = 16 / (int)sizeof(T);  // elements per 16-byte copy
  const SweepArgs& a = fa.s;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char* wbase = smem_raw + warp * SM::PER_WARP;
  T* in_tile = reinterpret_cast<T*>(wbase + SM::F_OFF);
  C* out_tile = reinterpret_cast<C*>(wbase + SM::C_OFF);
  const unsigned a_in = pin(saddr(in_tile + lane * RX));
  const unsigned a_out = pin(saddr(out_tile + lane * SM::CODE_STRIDE));
  const int nx = (int)a.dims[0], ny = (int)a.dims[1];
  const int npy = fa.npy, nf = fa.nf, ntasks = npy * nf;
  // codes are stored one block after they are computed; chunk c is flushed
  // at block c + WLAST + 2
  const int nblk = (nx + BS - 1) / BS + B::WLAST + 2;
  const unsigned epoch = a.epoch;
  const bool al_in = nx % EP == 0;
  const bool al_out = nx % 8 == 0;
  const bool al4_out = (nx * (int)sizeof(C)) % 4 == 0;
  constexpr double M = 0x1.8p52;

  for (;;) {
    unsigned int tk = 0;
    if (lane == 0) tk = atomicAdd(a.ticket, 1u);
    tk = __shfl_sync(EBZ_FULL, tk, 0);
    if ((int)tk >= ntasks) break;
    sched_jitter(a.jitter, tk, 0);
    const int fi = (int)(tk % (unsigned)nf);
    const FieldRef& fr = ft.f[fi];
    const int center = ft.center[fi] ? ft.center[fi] : a.center;
    const double lim = (double)(center - 1);
    const double eb = fr.info->eb;
    if (!(eb > 0.0)) continue;
    const double two_eb = __dmul_rn(2.0, eb);
    const double inv = 1.0 / two_eb;
    const bool fast_ok = isfinite(inv) && inv > 0.0 && two_eb >= 0x1p-1000 &&
                         inv >= 0x1p-1000 && inv <= 0x1p1000;
    const double guard = fast_ok ? 0.5 - 0x1p-30 : -1.0;
    const T* values = reinterpret_cast<const T*>(fr.values);
    C* codes = reinterpret_cast<C*>(fr.codes);
    const int PYi = (int)(fa.tasks[tk / (unsigned)nf] & 0xffff);
    const int y0 = PYi * 32, y = y0 + lane;
    const bool rv = y < ny;
    // interior blocks need every lane inside its row, past its n = 1 columns
    // (x >= N), and no row with y = 1 (n = 2: patch 0 stays on the edge path)
    const bool plain_rows = y0 + 32 <= ny && (N == 1 || PYi > 0);
    C* const row_out = codes + (long long)(rv ? y : 0) * nx;
    W* const faces = reinterpret_cast<W*>(fr.yface);
    FaceIn<N, T> fin;
#pragma unroll
    for (int s = 0; s < N; ++s)
      fin.row[s] = (lane == 0 && PYi > 0)
                       ? faces + (long long)((PYi - 1) * N + N - 1 - s) * nx : nullptr;
    fin.nx = nx;
    fin.ep = epoch;
    // face rows this patch hands on: its last N rows (lanes 32 - N .. 31)
    W* const fout = faces + (long long)(PYi * N + (lane >= 32 - N ? lane - (32 - N) : 0)) * nx;
    const bool f_ok = lane >= 32 - N && rv && PYi + 1 < npy;

    // input columns [BS j, BS j + BS) of the patch's 32 rows (zeros outside the grid)
    auto load_in = [&](int j) {
      const int x0 = j * BS;
      const int slot = (j & (B::NCH - 1)) * BS;
      if (al_in) {
        constexpr int G = BS / EP;  // 16-byte groups per row and block
#pragma unroll
        for (int i = 0; i < G; ++i) {
          const int p = lane + 32 * i, r = p / G, g = p % G;
          const int xx = x0 + EP * g, rem = nx - xx;
          const int bytes =
              (y0 + r < ny && rem > 0) ? (rem >= EP ? 16 : rem * (int)sizeof(T)) : 0;
          const T* src = values + (bytes ? (long long)(y0 + r) * nx + xx : 0);
          cpa16(saddr(in_tile + r * RX + slot + EP * g), src, bytes);
        }
      } else {
#pragma unroll
        for (int i = 0; i < BS; ++i) {
          const int p = lane + 32 * i, r = p / BS, c = p % BS;
          const int bytes = (y0 + r < ny && x0 + c < nx) ? (int)sizeof(T) : 0;
          const T* src = values + (bytes ? (long long)(y0 + r) * nx + x0 + c : 0);
          if (sizeof(T) == 4) cpa4(saddr(in_tile + r * RX + slot + c), src, bytes);
          else cpa8(saddr(in_tile + r * RX + slot + c), src, bytes);
        }
      }
      cpa_commit();
    };
    // each lane writes its own row's BS codes of chunk j
    auto flush_out = [&](int j) {
      const int x0 = j * BS;
      if (j < 0 || x0 >= nx || !rv) return;
      const C* src = out_tile + lane * SM::CODE_STRIDE + (j & (B::NCH - 1)) * BS;
      if (al_out) {
        constexpr int NB = BS * (int)sizeof(C);
        if (NB == 4) *reinterpret_cast<unsigned*>(row_out + x0) = *reinterpret_cast<const unsigned*>(src);
        else if (NB == 8) *reinterpret_cast<uint2*>(row_out + x0) = *reinterpret_cast<const uint2*>(src);
        else *reinterpret_cast<uint4*>(row_out + x0) = *reinterpret_cast<const uint4*>(src);
      } else if (al4_out && x0 + BS <= nx) {  // rows on 4-byte boundaries: word stores
#pragma unroll
        for (int q = 0; q < BS * (int)sizeof(C) / 4; ++q)
          reinterpret_cast<unsigned*>(row_out + x0)[q] = reinterpret_cast<const unsigned*>(src)[q];
      } else {
        const int cnt = nx - x0 < BS ? nx - x0 : BS;
        for (int c = 0; c < cnt; ++c) row_out[x0 + c] = src[c];
      }
    };

    W fw[N][BS], fnext[N][BS];
    fin.load(0, fw);
#pragma unroll
    for (int j = 0; j < B::PD; ++j) load_in(j);
    cpa_wait<B::PD - 1>();
    __syncwarp();
    fin.settle(0, fw);
    T xv[BS], xn[BS];
#pragma unroll
    for (int j = 0; j < BS; ++j)
      lds_t(a_in + (unsigned)sizeof(T) * (unsigned)((j - lane) & (RX - 1)), xv[j]);

    Hist<N> H;
    H.clear();
    int cp[BS];  // previous block's codes (validated)
#pragma unroll
    for (int j = 0; j < BS; ++j) cp[j] = 0;
#ifdef EBZ_DEBUG_CLOCKS
    long long dbg_t0 = clock64();
#endif
#pragma unroll 1
    for (int b = 0; b < nblk; ++b) {
      const int S0 = b * BS;
      const int xb = S0 - lane;  // this lane's column at the block's first step
      sched_jitter(a.jitter, tk, b + 1);  // test hook (a uniform branch at the loop head)
      // next block's face words (lane 0), checked at this block's end
      // (issued before the cp.async wait below: measured, a wait right after
      // plain loads waits for them too)
      fin.load(S0 + BS, fnext);
      load_in(b + B::PD);
      flush_out(b - (B::WLAST + 2));
      cpa_wait<B::PD - 1>();  // block b + 1's input columns have landed
      __syncwarp();
      const bool edge = !(S0 >= 31 + N && S0 + BS <= nx && plain_rows);
      const Hist<N> Hs = H;  // block-start state (replay)
      double rj[BS];
      int code[BS];
      bool slow = false;
      auto pass = [&](auto edge_c, auto exact_c) {
        constexpr bool EDGE = decltype(edge_c)::value, EXACT = decltype(exact_c)::value;
#pragma unroll
        for (int j = 0; j < BS; ++j) {
          double fv[N];
#pragma unroll
          for (int s = 0; s < N; ++s) fv[s] = Face<T>::val(fw[s][j]);
          const bool eff1 = N == 2 && EDGE && (xb + j == 1 || y == 1);
          const double pred = H.predict(fv, lane, eff1);
          const double x64 = (double)xv[j];
          const double q = __dmul_rn(__dsub_rn(x64, pred), inv);
          const double t = __dadd_rn(q, M);
          const double kd = __dsub_rn(t, M);
          // |k| > center - 1 fails the bound test below through a negative
          // bound (set before the rounding: one compare after it)
          const double ebk = fabs(kd) <= lim ? eb : -1.0;
          const double rr = __dadd_rn(pred, __dmul_rn(kd, two_eb));
          const double rq = (double)Elem<T>::round(rr);  // float32: the RNE cast (F2F pair)
          const bool safe = fabs(__dsub_rn(q, kd)) < guard;
          // branch-free (a short-circuit && compiles to a divergent branch per step)
          const bool good = fabs(__dsub_rn(x64, rq)) <= ebk;
          const long long gm = -(long long)good;
          double r = __longlong_as_double((__double_as_longlong(rq) & gm) |
                                          (__double_as_longlong(x64) & ~gm));
          int c = (center + __double2loint(t)) & (int)gm;
          const bool act = !EDGE || (rv && (unsigned)(xb + j) < (unsigned)nx);
          if (EXACT) {
            if (!safe && act) {  // the reference's division, bit for bit
              T rf;
              c = quantize_exact<T>(xv[j], pred, eb, two_eb, center, rf);
              r = (double)rf;
            }
            __syncwarp();
          } else {
            slow |= !safe && act;
            // in the chain's shadow: block b - 1's codes, block b + 1's values
            sts_c<C>(a_out + (unsigned)sizeof(C) * (unsigned)((xb - BS + j) & (RX - 1)), cp[j]);
            lds_t(a_in + (unsigned)sizeof(T) * (unsigned)((xb + BS + j) & (RX - 1)), xn[j]);
          }
          if (EDGE) r = act ? r : 0.0;
          rj[j] = r;
          code[j] = c;
          H.push(r);
        }
      };
      typedef std::true_type Yes;
      typedef std::false_type No;
      if (edge) pass(Yes(), No());
      else pass(No(), No());
      const bool miss = fin.missing(fnext);
      if (__any_sync(EBZ_FULL, slow | miss)) {
        if (__any_sync(EBZ_FULL, slow)) {  // replay the block with the exact quantizer
          H = Hs;
          pass(Yes(), Yes());
        }
        fin.settle(S0 + BS, fnext);
      }
      // the block is final: its face words leave now, its codes go to the
      // tile during the next block
#pragma unroll
      for (int j = 0; j < BS; ++j)
        Face<T>::st_if(fout + (xb + j), rj[j], epoch, f_ok && (unsigned)(xb + j) < (unsigned)nx);
#pragma unroll
      for (int j = 0; j < BS; ++j) {
#pragma unroll
        for (int s = 0; s < N; ++s) fw[s][j] = fnext[s][j];
        xv[j] = xn[j];
        cp[j] = code[j];
      }
    }
    cpa_wait<0>();
#ifdef EBZ_DEBUG_CLOCKS
    if (lane == 0 && (PYi == 0 || PYi == npy - 1 || PYi == npy / 2))
      printf("EBZDBG2 C N=%d PY=%d nblk=%d total=%lld per_step=%.1f\n", N, PYi, nblk,
             clock64() - dbg_t0, (double)(clock64() - dbg_t0) / (nblk * BS));
#endif
    __syncwarp();
  }
}

// ---------------------------------------------------------------------------
// decompress: no slow path, so no speculation; 16-column chunks (measured:
// the per-block staging of the compress kernel is slower here, 0.96 vs 0.91
// ms on cfg2 -- the step is bound by its fetch / store overhead, not by the
// recurrence).  The verbatim values of a block are fetched a block ahead
// from the row's cursor (the codes of the next block are already resident).
template <int N, typename C, typename T>
__global__ void __launch_bounds__(32 * WPB, (sizeof(T) == 8 ? 4 : 16 / WPB))
sweep2d_kernel(const __grid_constant__ S2Args fa, const __grid_constant__ FieldTable ft) {
  typedef Sm2<C, T> SM;
  typedef typename Face<T>::W W;
  constexpr int BS = Blk<N, T>::BS;
  constexpr int CH = 16;      // columns per staged chunk
  constexpr int OUT_LAG = 2;  // chunks still being written (skew 31)
  const SweepArgs& a = fa.s;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char* wbase = smem_raw + warp * SM::PER_WARP;
  T* out_tile = reinterpret_cast<T*>(wbase + SM::F_OFF);
  C* in_tile = reinterpret_cast<C*>(wbase + SM::C_OFF);
  const unsigned a_out = pin(saddr(out_tile + lane * RX));
  const unsigned a_in = pin(saddr(in_tile + lane * SM::CODE_STRIDE));
  const int nx = (int)a.dims[0], ny = (int)a.dims[1];
  const int npy = fa.npy, nf = fa.nf, ntasks = npy * nf;
  const int nchunks = (nx + 31 + CH - 1) / CH;
  const unsigned epoch = a.epoch;
  const bool al_in = nx % (16 / (int)sizeof(C)) == 0;
  const bool al4_in = (nx * (int)sizeof(C)) % 4 == 0;
  const bool al_out = nx % (16 / (int)sizeof(T)) == 0;
  const double c52 = 0x1p52 + (double)a.center;

  for (;;) {
    unsigned int tk = 0;
    if (lane == 0) tk = atomicAdd(a.ticket, 1u);
    tk = __shfl_sync(EBZ_FULL, tk, 0);
    if ((int)tk >= ntasks) break;
    sched_jitter(a.jitter, tk, 0);
    const int fi = (int)(tk % (unsigned)nf);
    const FieldRef& fr = ft.f[fi];
    const double eb = fr.info->eb;
    if (!(eb > 0.0)) continue;
    const double two_eb = __dmul_rn(2.0, eb);
    T* recon = reinterpret_cast<T*>(fr.recon);
    const C* codes = reinterpret_cast<const C*>(fr.codes);
    const T* unpred = reinterpret_cast<const T*>(fr.unpred);
    const unsigned long long n_unpred = fr.info->n_unpred;
    const int PYi = (int)(fa.tasks[tk / (unsigned)nf] & 0xffff);
    const int y0 = PYi * 32, y = y0 + lane;
    const bool rv = y < ny;
    const C* const row_in = codes + (long long)(rv ? y : 0) * nx;
    T* const row_out = recon + (long long)(rv ? y : 0) * nx;
    W* const faces = reinterpret_cast<W*>(fr.yface);
    FaceIn<N, T> fin;
#pragma unroll
    for (int s = 0; s < N; ++s)
      fin.row[s] = (lane == 0 && PYi > 0)
                       ? faces + (long long)((PYi - 1) * N + N - 1 - s) * nx : nullptr;
    fin.nx = nx;
    fin.ep = epoch;
    W* const fout = faces + (long long)(PYi * N + (lane >= 32 - N ? lane - (32 - N) : 0)) * nx;
    const bool f_ok = lane >= 32 - N && rv && PYi + 1 < npy;
    unsigned long long ucur = 0, ustart = 0;
    if (rv) ucur = ustart = fr.rowbase[y] + fr.rowblk[y >> 8];
    unsigned hmax = 0;

    // each lane stages its own row's 16 codes of chunk j (zeros past the row)
    auto load_in = [&](int j) {
      const int x0 = j * CH;
      if (x0 >= nx) return;
      C* dst = in_tile + lane * SM::CODE_STRIDE + (j & 3) * CH;
      const int rem = rv ? nx - x0 : 0;
      if (al_in && rem >= CH) {
#pragma unroll
        for (int v = 0; v < CH * (int)sizeof(C) / 16; ++v)
          cpa16(saddr(dst) + 16u * v, reinterpret_cast<const uint4*>(row_in + x0) + v, 16);
      } else if (al4_in) {
        // rows on 4-byte boundaries: 4-byte async copies, zero-filled past the
        // row's end (element-wise loads are waited for on the spot)
        const int nb = (rem > CH ? CH : (rem > 0 ? rem : 0)) * (int)sizeof(C);  // multiple of 4
#pragma unroll
        for (int q = 0; q < CH * (int)sizeof(C) / 4; ++q) {
          const int b4 = nb - 4 * q >= 4 ? 4 : 0;
          cpa4(saddr(dst) + 4u * q,
               b4 ? reinterpret_cast<const unsigned char*>(row_in + x0) + 4 * q
                  : reinterpret_cast<const unsigned char*>(codes), b4);
        }
      } else {
        for (int c = 0; c < CH; ++c) dst[c] = c < rem ? row_in[x0 + c] : (C)0;
      }
    };
    auto flush_out = [&](int j) {
      const int x0 = j * CH;
      if (x0 >= nx || !rv) return;
      const int cnt = nx - x0 < CH ? nx - x0 : CH;
      const T* src = out_tile + lane * RX + (j & 3) * CH;
      if (al_out && cnt == CH) {
#pragma unroll
        for (int v = 0; v < CH * (int)sizeof(T) / 16; ++v)
          reinterpret_cast<uint4*>(row_out + x0)[v] = reinterpret_cast<const uint4*>(src)[v];
      } else {
        for (int c = 0; c < cnt; ++c) row_out[x0 + c] = src[c];
      }
    };
    // the row's values a few blocks ahead into L2 (only where the cursor
    // moved): a sector's first touch is a DRAM access of about one block's
    // time, and a block's value loads are waited for at its end.  Measured on
    // cfg2: rel 1e-5 (63% / 84% verbatim) 1.05 -> 0.92 ms (n = 1), 1.60 ->
    // 1.36 ms (n = 2).  Predicated, not branched: the block stays one basic
    // block.  Issued from the fetch for n = 2 and at the block end for n = 1
    // (measured: the other placement costs each 4-6% at high hit rates).
    unsigned long long upf = 0;
    auto prefetch_values = [&]() {
      asm volatile("{ .reg .pred q; setp.ne.u32 q, %1, 0; @q prefetch.global.L2 [%0]; }"
                   ::"l"(unpred + ucur + kUnpredAhead),
                     "r"((unsigned)(ucur != upf && ucur + kUnpredAhead < n_unpred)));
      upf = ucur;
    };
    // codes and verbatim values of the block starting at step S0 (this
    // lane's columns S0 - lane .. + BS - 1): the values are requested from
    // the row's cursor, which moves past them
    auto fetch = [&](int S0, int (&cd)[BS], T (&vv)[BS]) {
      const int xb = S0 - lane;
#pragma unroll
      for (int j = 0; j < BS; ++j) {
        const bool act = rv && (unsigned)(xb + j) < (unsigned)nx;
        // (columns outside the row read ring slots of other columns, never an
        // out-of-bounds address; they are masked here)
        const int c = lds_c<C>(a_in + (unsigned)sizeof(C) * (unsigned)((xb + j) & (RX - 1)));
        cd[j] = act ? c : -1;
        vv[j] = (T)0;
        const unsigned take = act && c == 0;
        const unsigned ok = take && ucur < n_unpred;
        ldg_nc_if(vv[j], unpred + ucur, ok);
        ucur += take;
      }
      if (N == 2) prefetch_values();
    };

    load_in(0);
    cpa_commit();
    W fw[N][BS], fnext[N][BS];
    fin.load(0, fw);
    cpa_wait<0>();
    __syncwarp();
    int cd[BS], cdn[BS];
    T vv[BS], vvn[BS];
    fetch(0, cd, vv);
    fin.settle(0, fw);

    Hist<N> H;
    H.clear();
    for (int k = 0; k < nchunks; ++k) {
      load_in(k + 1);
      cpa_commit();
#pragma unroll 1
      for (int h = 0; h < CH / BS; ++h) {
        const int S0 = k * CH + h * BS;
        const int xb = S0 - lane;
        sched_jitter(a.jitter, tk, S0 / BS + 1);  // test hook
        fin.load(S0 + BS, fnext);
        if (h + 1 == CH / BS) {  // the next block's codes are in the chunk being staged
          cpa_wait<0>();
          __syncwarp();
        }
        fetch(S0 + BS, cdn, vvn);
        double rj[BS];
#pragma unroll
        for (int j = 0; j < BS; ++j) {
          const bool act = cd[j] >= 0;
          const double qv = __dmul_rn(__dsub_rn(__hiloint2double(0x43300000, cd[j]), c52), two_eb);
          const double und = (double)vv[j];
          double fv[N];
#pragma unroll
          for (int s = 0; s < N; ++s) fv[s] = Face<T>::val(fw[s][j]);
          const bool eff1 = N == 2 && (xb + j == 1 || y == 1);
          const double pred = H.predict(fv, lane, eff1);
          double r = (double)Elem<T>::round(__dadd_rn(pred, qv));
          r = cd[j] == 0 ? und : r;
          r = act ? r : 0.0;
          hmax = max(hmax, (unsigned)__double2hiint(r) & 0x7fffffffu);
          sts_t(a_out + (unsigned)sizeof(T) * (unsigned)((xb + j) & (RX - 1)), T(), r);
          rj[j] = r;
          H.push(r);
        }
#pragma unroll
        for (int j = 0; j < BS; ++j)
          Face<T>::st_if(fout + (xb + j), rj[j], epoch, f_ok && (unsigned)(xb + j) < (unsigned)nx);
        fin.settle(S0 + BS, fnext);
        if (N == 1) prefetch_values();
#pragma unroll
        for (int j = 0; j < BS; ++j) {
#pragma unroll
          for (int s = 0; s < N; ++s) fw[s][j] = fnext[s][j];
          cd[j] = cdn[j];
          vv[j] = vvn[j];
        }
      }
      __syncwarp();
      if (k - OUT_LAG >= 0) flush_out(k - OUT_LAG);
      __syncwarp();
    }
    for (int j = nchunks - OUT_LAG; j < nchunks; ++j)
      if (j >= 0) flush_out(j);
    __syncwarp();
    {
      // (the prefetch of the block past the last one moved no cursor: its
      // columns are outside the row)
      unsigned long long used = ucur - ustart;
      int bad = 0;
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

template <int N, typename C, typename T, bool COMPRESS>
cudaError_t launch2_t(const S2Args& fa, const FieldTable& ft, int sms, cudaStream_t s) {
  const size_t smem = (size_t)WPB * Sm2<C, T>::PER_WARP;
  static KernelAttr attr;
  auto* kern = COMPRESS ? sweep2c_kernel<N, C, T> : sweep2d_kernel<N, C, T>;
  cudaError_t e = kernel_smem(attr, kern, smem);
  if (e != cudaSuccess) return e;
  const int per_sm = kernel_occupancy(attr, kern, 32 * WPB, smem);
  const long long ntasks = (long long)fa.npy * fa.nf;
  long long blocks = (ntasks + WPB - 1) / WPB;
  if (blocks > (long long)sms * per_sm) blocks = (long long)sms * per_sm;
  if (blocks < 1) blocks = 1;
  kern<<<(unsigned)blocks, 32 * WPB, smem, s>>>(fa, ft);
  return cudaGetLastError();
}

template <int N, typename T>
cudaError_t launch2_n(const S2Args& fa, const FieldTable& ft, bool compress, int sms,
                      cudaStream_t s) {
  const bool wide = fa.s.wide != 0;
  if (compress)
    return wide ? launch2_t<N, uint16_t, T, true>(fa, ft, sms, s)
                : launch2_t<N, uint8_t, T, true>(fa, ft, sms, s);
  return wide ? launch2_t<N, uint16_t, T, false>(fa, ft, sms, s)
              : launch2_t<N, uint8_t, T, false>(fa, ft, sms, s);
}

}  // namespace

// 2D, n = 1 or 2, float32 or binary64, without the full-reconstruction
// output (REC) or the truncated coding (TR) of the one-row kernel;
// EBZ_NO_SWEEP2 keeps the one-row (float32) / generic (binary64) kernel
// (A/B, tests)
bool sweep2_used(int ndim, int layers, int width, const long long* dims, bool rec, bool trunc) {
  if (getenv("EBZ_NO_SWEEP2")) return false;
  return ndim == 2 && (layers == 1 || layers == 2) && (width == 32 || width == 64) && !rec &&
         !trunc && dims[0] < (1ll << 30);
}

cudaError_t launch_sweep2(const SweepArgs& a, const FieldTable& ft, int nf,
                          const unsigned int* d_tasks, int npy, bool compress, int width, int sms,
                          cudaStream_t s) {
  if (nf < 1 || nf > kBatchMax) return cudaErrorInvalidValue;
  S2Args fa;
  fa.s = a;
  fa.tasks = d_tasks;
  fa.npy = npy;
  fa.nf = nf;
  if (width == 64)
    return a.layers == 2 ? launch2_n<2, double>(fa, ft, compress, sms, s)
                         : launch2_n<1, double>(fa, ft, compress, sms, s);
  return a.layers == 2 ? launch2_n<2, float>(fa, ft, compress, sms, s)
                       : launch2_n<1, float>(fa, ft, compress, sms, s);
}
