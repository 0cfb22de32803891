// sweep3.cu -- 3D, n = 1, float32 predict/quantize sweep with z-rows per
// lane: the compress_scan hot loop (ebzip/_kernels.py:48-80) for the 3D
// configs (cfg3, cfg4, cfg5).
//
// Geometry.  A warp task owns a patch of 32 (y) x R3 = 4 (z) rows.  Lane a
// holds the rows (y0 + a, z0 + j), j = 0..3, and processes row j at
//     x = S - a - j            at warp step S,
// so every dependency of a point was produced one step earlier (or two, or
// three) either by the lane itself or by lane a - 1:
//   * (x, y, z - 1), (x - 1, y, z - 1), (x - 1, y, z): the lane's own rows j - 1
//     and j, kept in registers (row j - 1 computed x one step before row j);
//   * (x, y - 1, z): lane a - 1's row j of the previous step -- ONE shuffle per
//     row and step; (x - 1, y - 1, z), (x, y - 1, z - 1), (x - 1, y - 1, z - 1)
//     are the values received one and two steps earlier (rows j and j - 1).
// Compared with lanes on a 2-D (y, z) grid, every point needs one neighbour
// exchange instead of three.  Row j = -1 is a "virtual" row carrying the Z
// face of the patch below (z0 - 1), loaded one step ahead; the Y face (row
// y0 - 1) enters at lane 0 through the same shuffle: the exchange is a
// rotate by one lane and lane 31 -- whose own values nobody in the warp
// needs -- sends the face words lane 0 wants.
//
// Faces cross between warps as 64-bit tagged words (the binary64 value with
// the launch epoch in its 29 always-zero low mantissa bits, ebz_common.cuh),
// in hyperplane-major blocks so every warp-wide access is one contiguous run:
//   Y face of patch (PY, PZ): word [h * 4 + j] = value of (x = h - j, y0 + 31,
//     z0 + j), written by lane 31 at step h + 31;
//   Z face: word [h * 32 + a] = value of (x = h - a, y0 + a, z0 + 3), written
//     by row 3 of every lane at step h + 3.
// A consumer stages the next chunk's face words while computing the current
// one and checks their tags once per chunk (spinning only if a producer is
// behind); tasks are ticketed in hyperplane (PY + PZ) order, so a task waits
// only on lower tickets.
//
// Staging.  Inputs go through a per-row ring in shared memory (16 values +
// a 4-value front guard), rotated per row by 4 * ((a + j) / 4) so that a
// chunk of 4 steps reads 4 consecutive slots at a per-row base and every
// aligned 16-byte group of a row lands at the same slot for all rows (one
// cp.async per row and chunk, uniform destination, no per-step address
// arithmetic).  Rows are laid out so the 32 lanes' reads hit 32 banks.
// Codes leave through a per-row ring of 32 (same rotation), drained every
// four chunks as one 16-code block per row.
//
// Arithmetic: as sweep_fast.cu (reference term order, binary64 without
// contraction, reciprocal quantizer with the exact-division fallback); the
// stencil here is written out in the reference's order
//   (0,0,1) + (0,1,0) - (0,1,1) + (1,0,0) - (1,0,1) - (1,1,0) + (1,1,1)
// with (kx, ky, kz) offsets, x slowest (predictor.py:41-56).
#include <cmath>
#include <cstdlib>
#include <cstring>
#include "ebz_common.cuh"

namespace {

constexpr int R3 = 4;                 // z rows per lane
constexpr int CH3 = 4;                // steps per chunk
constexpr int SK3 = 31 + R3 - 1;      // largest lane/row skew
constexpr int WI3 = 16;               // input ring (values) per row
constexpr int GD3 = 4;                // front guard (mirror of the ring's last group)
constexpr int IRW = WI3 + GD3;        // floats per input row
constexpr int WO3 = 32;               // output ring (codes) per row
constexpr int WPB3 = 4;               // warps per block
constexpr int YPAD3 = 48;             // face hyperplanes past nx (pads hold tagged zeros)

__host__ __device__ constexpr int face3_h(long long nx) { return (int)nx + YPAD3; }

template <typename C>
struct Sm3 {
  static constexpr int IN_BYTES = 32 * R3 * IRW * 4;                        // 10240
  static constexpr int ORW = (WO3 + GD3) * (int)sizeof(C);                  // bytes per out row
  static constexpr int OUT_OFF = IN_BYTES;
  static constexpr int OUT_BYTES = 32 * R3 * ORW;
  static constexpr int YST_OFF = ((OUT_OFF + OUT_BYTES + 15) / 16) * 16;
  static constexpr int YST_BYTES = 2 * (4 * CH3 + CH3) * 8;                 // 2 chunks x 20 words
  static constexpr int ZST_OFF = YST_OFF + YST_BYTES;
  static constexpr int ZST_BYTES = 2 * CH3 * 32 * 8;                        // 2 chunks x 128 words
  static constexpr int HIST_OFF = ZST_OFF + ZST_BYTES;
  // 256 bins + one dummy bin (lanes outside their row count there: an
  // unconditional atomic keeps the step free of branch regions)
  static constexpr int HIST_BYTES = sizeof(C) == 1 ? 257 * 4 : 0;
  static constexpr int PER_WARP = ((HIST_OFF + HIST_BYTES + 15) / 16) * 16;
};

struct F3Args {
  SweepArgs s;
  const unsigned int* tasks;
  int npy, npz, nf;
};

__device__ __forceinline__ void cpa16(unsigned smem, const void* g, int bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem), "l"(g), "r"(bytes));
}
__device__ __forceinline__ void cpa8(unsigned smem, const void* g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem), "l"(g));
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cpa_wait0() { asm volatile("cp.async.wait_group 0;\n" ::); }
__device__ __forceinline__ unsigned sm_addr(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ float ld_sf(unsigned a) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ unsigned long long ld_cg64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.global.cg.u64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}
// predicated global stores (one instruction, no branch around them)
__device__ __forceinline__ void st_if(unsigned long long* p, unsigned long long w, bool pred) {
  asm volatile("{ .reg .pred q; setp.ne.u32 q, %2, 0; @q st.global.cg.u64 [%0], %1; }"
               ::"l"(p), "l"(w), "r"((unsigned)pred) : "memory");
}
__device__ __forceinline__ void st2_if(unsigned long long* p, unsigned long long w0,
                                       unsigned long long w1, bool pred) {
  asm volatile("{ .reg .pred q; setp.ne.u32 q, %3, 0; @q st.global.cg.v2.u64 [%0], {%1, %2}; }"
               ::"l"(p), "l"(w0), "l"(w1), "r"((unsigned)pred) : "memory");
}
__device__ __forceinline__ bool tag_ok(unsigned long long w, unsigned ep) {
  return ((unsigned)w & kTagMask) == ep;
}
__device__ __forceinline__ double untag(unsigned long long w) {
  return __longlong_as_double((long long)(w & ~(unsigned long long)kTagMask));
}
__device__ __forceinline__ unsigned long long tagged(double v, unsigned ep) {
  return (unsigned long long)__double_as_longlong(v) | ep;
}

// row slot of lane a's row j: 32 lanes of one j read 32 distinct banks
// (row stride 20 words; lanes a = 4p + e sit at n = 8e + p)
__device__ __forceinline__ int row_slot(int a, int j) { return j * 32 + (a & 3) * 8 + (a >> 2); }

#ifndef EBZ_S3_MINB
#define EBZ_S3_MINB 3  // 168 registers, 12 warps per SM (2: 255 registers, 6.75 ms vs 5.37 ms on cfg5)
#endif
// PF: per-field interval counts (FieldRef::center, the batched --auto-m
// trials); the pipelines keep the launch's centre as a kernel constant
// TR: unpredictable points reconstruct to trunc(x) (the opt-in truncated-
// mantissa coding, ebz_common.cuh); the pipelines instantiate TR = false
// JIT: the schedule-perturbation test hook (EBZ_SCHED_JITTER), compiled into
// its own instantiation so the pipeline kernel carries no per-chunk test
template <typename C, bool REC, bool PF, bool TR = false, bool JIT = false>
__global__ void __launch_bounds__(32 * WPB3, EBZ_S3_MINB)
sweep3c_kernel(const __grid_constant__ F3Args fa, const __grid_constant__ FieldTable ft) {
  typedef Sm3<C> SM;
  const SweepArgs& A = fa.s;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5, a = threadIdx.x & 31;
  unsigned char* wbase = smem_raw + warp * SM::PER_WARP;
  constexpr bool FH = sizeof(C) == 1;
  unsigned int* whist = reinterpret_cast<unsigned int*>(wbase + SM::HIST_OFF);
  double* yst = reinterpret_cast<double*>(wbase + SM::YST_OFF);
  unsigned long long* zst = reinterpret_cast<unsigned long long*>(wbase + SM::ZST_OFF);
  const unsigned a_in = sm_addr(wbase);
  const unsigned a_zst = sm_addr(zst);
  const unsigned a_out = sm_addr(wbase + SM::OUT_OFF);
  const unsigned a_yst = sm_addr(yst);
  // the histogram base stays in its register (rebuilt from SR_CgaCtaId at
  // every code otherwise: 5.17 -> 5.07 ms on cfg5)
  unsigned a_hist = sm_addr(whist);
  asm volatile("" : "+r"(a_hist));

  const double lim0 = (double)(A.center - 1);
  const int nx = (int)A.dims[0], ny = (int)A.dims[1], nz = (int)A.dims[2];
  const int npy = fa.npy, npz = fa.npz, nf = fa.nf;
  const int ntasks = npy * npz * nf;
  const int nsteps = nx + SK3;
  const int nchunks = (nsteps + CH3 - 1) / CH3;
  const unsigned ep = A.epoch;
  const unsigned long long tag0 = ep;  // tagged +0.0
  const int HY = face3_h(nx);
  const long long plane = (long long)nx * ny;
  const int src = (a + 31) & 31;       // rotate: lane a receives from lane a - 1

  for (;;) {
    unsigned int tk = 0;
    if (a == 0) tk = atomicAdd(A.ticket, 1u);
    tk = __shfl_sync(EBZ_FULL, tk, 0);
    if ((int)tk >= ntasks) break;
    const int fi = (int)(tk % (unsigned)nf);
    const FieldRef& fr = ft.f[fi];
    // per-field interval count (batched --auto-m trials), else the launch's
    const int center = PF ? ft.center[fi] : 0;
    const double lim = PF ? (double)(center - 1) : lim0;
    const double eb = fr.info->eb;
    if (!(eb > 0.0)) continue;
    const double two_eb = __dmul_rn(2.0, eb);
    const double inv = 1.0 / two_eb;
    const bool fast_ok = isfinite(inv) && inv > 0.0 && two_eb >= 0x1p-1000 &&
                         inv >= 0x1p-1000 && inv <= 0x1p1000;
    // fast-path margin; a field without a usable reciprocal takes the exact
    // path at every point (|q - kd| < -1 never holds, NaN included)
    const double guard = fast_ok ? 0.5 - 0x1p-21 : -1.0;
    const int tre = TR ? eb_exponent(eb) : kNoTrunc;
    const float* values = reinterpret_cast<const float*>(fr.values);
    C* codes = reinterpret_cast<C*>(fr.codes);
    float* const recon = reinterpret_cast<float*>(fr.recon);
    unsigned long long* const ghist = FH ? fr.hist : nullptr;
    if (ghist) {
#pragma unroll
      for (int b = 0; b < 8; ++b) whist[a + 32 * b] = 0u;
      __syncwarp();
    }
    const unsigned int tv = fa.tasks[tk / (unsigned)nf];
    const int PY = (int)(tv & 0xffff), PZ = (int)(tv >> 16);
    const int y0 = PY * 32, z0 = PZ * R3;
    const int y = y0 + a;
    bool rv[R3];
    int s_[R3], q_[R3], r_[R3];
#pragma unroll
    for (int j = 0; j < R3; ++j) {
      rv[j] = y < ny && z0 + j < nz;
      s_[j] = a + j;
      q_[j] = s_[j] >> 2;
      r_[j] = s_[j] & 3;
    }
    // ---- faces: own blocks (written) and the neighbours' (read)
    unsigned long long* const yfw = fr.yface + (long long)(PY * npz + PZ) * HY * 4;
    unsigned long long* const zfw = fr.zface + (long long)(PY * npz + PZ) * HY * 32;
    const bool hasY = PY > 0, hasZ = PZ > 0, hasC = PY > 0 && PZ > 0;
    const unsigned long long* const yfr =
        fr.yface + (long long)((hasY ? PY - 1 : 0) * npz + PZ) * HY * 4;
    const unsigned long long* const cfr =
        fr.yface + (long long)((hasC ? PY - 1 : 0) * npz + (hasC ? PZ - 1 : 0)) * HY * 4;
    const unsigned long long* const zfb =
        fr.zface + (long long)(PY * npz + (hasZ ? PZ - 1 : 0)) * HY * 32;
    const unsigned long long* const zfr = zfb + a;  // this lane's column

    // ---- per-row ring addresses (bytes in the shared window), less the row's
    // rotation residue r: a chunk's step t reads slot P0 + t - r at base + 4 t
    unsigned in_b[R3], out_b[R3];
#pragma unroll
    for (int j = 0; j < R3; ++j) {
      in_b[j] = a_in + (unsigned)(row_slot(a, j) * IRW * 4) - 4u * (unsigned)r_[j];
      out_b[j] = a_out + (unsigned)(row_slot(a, j) * SM::ORW) - (unsigned)(sizeof(C) * r_[j]);
    }
    const long long row0 = ((long long)z0 * ny + y) * nx;  // element index of (0, y, z0)
    const int ngroups = nx >> 2;

    // input loader: the aligned group of row j that chunk k + 1 needs last,
    // x0 = 4 (k + 1 - q_j), lands at slot GD3 + (4 (k + 1) mod 16) of every
    // row (and in the guard when that slot is the ring's last group)
    auto load_group = [&](int k) {
      const unsigned col = (unsigned)(GD3 + ((4 * (k + 1)) & (WI3 - 1))) * 4u;
      const bool mirror = ((4 * (k + 1)) & (WI3 - 1)) == WI3 - 4;
#pragma unroll
      for (int j = 0; j < R3; ++j) {
        const int g = k + 1 - q_[j];
        const bool in = rv[j] && (unsigned)g < (unsigned)ngroups;
        const float* gp = values + (in ? row0 + j * plane + 4 * g : 0);
        const unsigned dst = in_b[j] + 4u * (unsigned)r_[j];
        cpa16(dst + col, gp, in ? 16 : 0);
        if (mirror) cpa16(dst, gp, in ? 16 : 0);
      }
    };
    // face words of chunk k into staging buffer k & 1: Y -- lanes 0-7 the four
    // words of hyperplanes 4k..4k+3 (16 B each), lanes 8-11 the corner words
    // (row 3 of patch (PY - 1, PZ - 1)) of hyperplanes 4k + 4..4k + 7; Z --
    // hyperplanes 4k + 1..4k + 4 (1 KB), two 16-byte pieces per lane
    auto load_faces = [&](int k) {
      const unsigned yb = a_yst + (unsigned)((k & 1) * 20 * 8);
      if (hasY && a < 8) cpa16(yb + a * 16, yfr + (long long)16 * k + 2 * a, 16);
      if (hasC && a >= 8 && a < 12)
        cpa8(yb + 128 + (a - 8) * 8, cfr + (long long)(4 * k + 4 + (a - 8)) * 4 + 3);
      if (hasZ) {
        const unsigned zb = a_zst + (unsigned)((k & 1) * CH3 * 32 * 8);
        const unsigned long long* g = zfb + (long long)(4 * k + 1) * 32 + 2 * a;
        cpa16(zb + a * 16, g, 16);
        cpa16(zb + 512 + a * 16, g + 64, 16);
      }
    };
    // after the copies of chunk k landed: check every staged word's tag
    // (spinning on the ones a producer has not written yet), clear the Y tags
    auto settle = [&](int k) {
      double* yb = yst + (k & 1) * 20;
      unsigned long long* zb = zst + (k & 1) * CH3 * 32;
      const bool ymine = hasY && (a < 8 || (a < 12 && hasC));
      const int w0 = a < 8 ? 2 * a : 16 + (a - 8);
      unsigned long long yw0 = tag0, yw1 = tag0;
      if (ymine) {
        yw0 = (unsigned long long)__double_as_longlong(yb[w0]);
        if (a < 8) yw1 = (unsigned long long)__double_as_longlong(yb[w0 + 1]);
      }
      unsigned long long zw[CH3];
#pragma unroll
      for (int t = 0; t < CH3; ++t) zw[t] = hasZ ? zb[t * 32 + a] : tag0;
      unsigned d = ((unsigned)yw0 ^ ep) | ((unsigned)yw1 ^ ep);
#pragma unroll
      for (int t = 0; t < CH3; ++t) d |= (unsigned)zw[t] ^ ep;
      bool miss = (d & kTagMask) != 0;
      if (__any_sync(EBZ_FULL, miss)) {
        // a producer is behind: poll the missing words directly
        for (unsigned ns = 32;; ns = ns < 512 ? 2 * ns : ns) {
          if (miss) {
            if (!tag_ok(yw0, ep))
              yw0 = a < 8 ? ld_cg64(yfr + (long long)16 * k + 2 * a)
                          : ld_cg64(cfr + (long long)(4 * k + 4 + (a - 8)) * 4 + 3);
            if (!tag_ok(yw1, ep)) yw1 = ld_cg64(yfr + (long long)16 * k + 2 * a + 1);
#pragma unroll
            for (int t = 0; t < CH3; ++t)
              if (!tag_ok(zw[t], ep)) {
                zw[t] = ld_cg64(zfr + (long long)(4 * k + 1 + t) * 32);
                zb[t * 32 + a] = zw[t];
              }
            miss = !tag_ok(yw0, ep) || !tag_ok(yw1, ep);
#pragma unroll
            for (int t = 0; t < CH3; ++t) miss |= !tag_ok(zw[t], ep);
          }
          if (!__any_sync(EBZ_FULL, miss)) break;
          __nanosleep(ns);
        }
      }
      if (ymine) {
        yb[w0] = untag(yw0);
        if (a < 8) yb[w0 + 1] = untag(yw1);
      }
      __syncwarp();
    };

    // ---- state: rows -1 (virtual, Z face) .. 3.  R = latest value, P = the
    // one before, B / B1 / B2 = values received from lane a - 1 this step,
    // one and two steps ago (lane 0: the Y face / corner sent by lane 31)
    double Rv[R3 + 1], Pv[R3 + 1], Bv[R3 + 1], B1[R3 + 1], B2[R3 + 1];
#pragma unroll
    for (int j = 0; j <= R3; ++j) Rv[j] = Pv[j] = Bv[j] = B1[j] = B2[j] = 0.0;

    // ---- prologue: staging words no producer fills hold zeros for the whole
    // task (Y words: +0.0 itself -- settle() untags only the words it loads,
    // and a tagged zero read as a double is a tiny denormal that would leak
    // into the prediction; Z words: tagged, settle() checks them); the
    // groups and faces of chunk 0
    for (int i = a; i < 40; i += 32)
      if (!hasY || (!hasC && (i % 20) >= 16))
        reinterpret_cast<unsigned long long*>(yst)[i] = 0ull;
    if (!hasZ)
      for (int i = a; i < 2 * CH3 * 32; i += 32) zst[i] = tag0;
    __syncwarp();
    load_group(-2);
    load_group(-1);
    load_faces(0);
    cpa_commit();
    // virtual row before step 0: Z word of hyperplane 0; lane 0's B of the
    // virtual row "received at step -1": the corner word of hyperplane 3
    {
      unsigned long long w = hasZ ? ld_cg64(zfr) : tag0;
      unsigned long long c = (hasC && a == 0) ? ld_cg64(cfr + 3 * 4 + 3) : tag0;
      bool miss = !tag_ok(w, ep) || !tag_ok(c, ep);
      for (unsigned ns = 32; __any_sync(EBZ_FULL, miss); ns = ns < 512 ? 2 * ns : ns) {
        __nanosleep(ns);
        if (!tag_ok(w, ep)) w = ld_cg64(zfr);
        if (!tag_ok(c, ep)) c = ld_cg64(cfr + 3 * 4 + 3);
        miss = !tag_ok(w, ep) || !tag_ok(c, ep);
      }
      Rv[0] = untag(w);
      Bv[0] = untag(c);
    }
    cpa_wait0();
    __syncwarp();
    settle(0);

    for (int k = 0; k < nchunks; ++k) {
      if (JIT) sched_jitter(A.jitter, tk, k);
      const int S0 = k * CH3;
      // next chunk's inputs and faces (in flight during this chunk)
      if (k + 1 < nchunks) {
        load_group(k);
        load_faces(k + 1);
      }
      cpa_commit();
      const unsigned P0 = (unsigned)(GD3 + (S0 & (WI3 - 1))) * 4u;
      const unsigned Q0 = (unsigned)(GD3 + (S0 & (WO3 - 1))) * (unsigned)sizeof(C);
      const double* yb = yst + (k & 1) * 20;
      const unsigned long long* zb = zst + (k & 1) * CH3 * 32;
      unsigned ia[R3], oa[R3];
      int xl[R3];
#pragma unroll
      for (int j = 0; j < R3; ++j) {
        ia[j] = in_b[j] + P0;
        oa[j] = out_b[j] + Q0;
        xl[j] = rv[j] ? S0 - s_[j] : (int)0x80000000;  // x at t = 0 (invalid rows: never active)
      }
      // exchange for step t: Bn_j <- lane a - 1's value of row j after step
      // t - 1 (lane 0: the Y face / corner words lane 31 sends).  Issued one
      // step ahead, right after the values it sends are known, so that the
      // four rows of the next step can start together.
      double Bn[R3 + 1];
      auto exchange = [&](int t) {
        const double2 y01 = *reinterpret_cast<const double2*>(yb + 4 * t);
        const double2 y23 = *reinterpret_cast<const double2*>(yb + 4 * t + 2);
        const double yf[R3 + 1] = {yb[16 + t], y01.x, y01.y, y23.x, y23.y};
#pragma unroll
        for (int j = 0; j <= R3; ++j) Bn[j] = __shfl_sync(EBZ_FULL, a == 31 ? yf[j] : Rv[j], src);
      };
      exchange(0);
#pragma unroll
      for (int t = 0; t < CH3; ++t) {
        const int S = S0 + t;
        const double zn = untag(zb[t * 32 + a]);  // virtual row, next value
#pragma unroll
        for (int j = 0; j <= R3; ++j) {
          B2[j] = B1[j];
          B1[j] = Bv[j];
          Bv[j] = Bn[j];
        }
        // ---- predict + quantize rows 0..3: four independent chains, written
        // operation by operation across the rows so they interleave
        double rq[R3], pr[R3];
        int code[R3];
        bool slow[R3];
        float xv[R3];
#pragma unroll
        for (int j = 0; j < R3; ++j) xv[j] = ld_sf(ia[j] + 4u * t);
        // (z-1) + (y-1) - (y-1,z-1) + (x-1) - (x-1,z-1) - (x-1,y-1) + (x-1,y-1,z-1)
#pragma unroll
        for (int j = 0; j < R3; ++j) pr[j] = __dadd_rn(Rv[j], Bv[j + 1]);
#pragma unroll
        for (int j = 0; j < R3; ++j) pr[j] = __dsub_rn(pr[j], B1[j]);
#pragma unroll
        for (int j = 0; j < R3; ++j) pr[j] = __dadd_rn(pr[j], Rv[j + 1]);
#pragma unroll
        for (int j = 0; j < R3; ++j) pr[j] = __dsub_rn(pr[j], Pv[j]);
#pragma unroll
        for (int j = 0; j < R3; ++j) pr[j] = __dsub_rn(pr[j], B1[j + 1]);
#pragma unroll
        for (int j = 0; j < R3; ++j) pr[j] = __dadd_rn(pr[j], B2[j]);
        {
          constexpr double M = 0x1.8p52;
          double x64[R3], q[R3], tq[R3], kd[R3], rd[R3];
#pragma unroll
          for (int j = 0; j < R3; ++j) x64[j] = (double)xv[j];
#pragma unroll
          for (int j = 0; j < R3; ++j) q[j] = __dmul_rn(__dsub_rn(x64[j], pr[j]), inv);
#pragma unroll
          for (int j = 0; j < R3; ++j) tq[j] = __dadd_rn(q[j], M);
#pragma unroll
          for (int j = 0; j < R3; ++j) kd[j] = __dsub_rn(tq[j], M);
#pragma unroll
          for (int j = 0; j < R3; ++j) rd[j] = __dadd_rn(pr[j], __dmul_rn(kd[j], two_eb));
#pragma unroll
          for (int j = 0; j < R3; ++j) rd[j] = (double)__double2float_rn(rd[j]);
#pragma unroll
          for (int j = 0; j < R3; ++j) {
            slow[j] = !(fabs(__dsub_rn(q[j], kd[j])) < guard);
            const bool good = fabs(kd[j]) <= lim && fabs(__dsub_rn(x64[j], rd[j])) <= eb;
            const long long gm = -(long long)good;
            const double xs = TR ? (double)trunc_value<float>(xv[j], tre) : x64[j];
            rq[j] = __longlong_as_double((__double_as_longlong(rd[j]) & gm) |
                                         (__double_as_longlong(xs) & ~gm));
            code[j] = ((PF ? center : A.center) + (int)__double2loint(tq[j])) & (int)gm;
          }
        }
        if (__any_sync(EBZ_FULL, slow[0] | slow[1] | slow[2] | slow[3])) {
#pragma unroll
          for (int j = 0; j < R3; ++j)
            if (slow[j]) {
              float rf;
              code[j] = quantize_exact<float>(xv[j], pr[j], eb, two_eb, PF ? center : A.center, rf,
                                              tre);
              rq[j] = (double)rf;
            }
        }
        // ---- outputs of the step: code (ring), histogram, faces
#pragma unroll
        for (int j = 0; j < R3; ++j) {
          const int x = xl[j] + t;
          const unsigned act = (unsigned)x < (unsigned)nx;
          const unsigned o = oa[j] + (unsigned)(t * sizeof(C));
          // unguarded: a column outside [0, nx) lands in a ring slot that is
          // rewritten by its in-row position before that block drains, or
          // that no drain reads (the ring invariant holds for every column)
          if (sizeof(C) == 1)
            asm volatile("st.shared.u8 [%0], %1;" ::"r"(o), "r"(code[j]));
          else
            asm volatile("st.shared.u16 [%0], %1;" ::"r"(o), "r"(code[j]));
          if (FH) {
            // (a predicated red.shared compiles to a branch region around a
            // warp-aggregated atomic: four reconvergence points per step)
            const unsigned h = a_hist + 4u * ((act && ghist != nullptr) ? (unsigned)code[j] : 256u);
            asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(h) : "memory");
          }
          if (REC && act) recon[row0 + j * plane + x] = (float)rq[j];
        }
        // Y face (lane 31, hyperplane S - 31) and Z face (row 3, hyperplane S - 3)
        {  // predicated stores: 5.36 -> 5.17 ms on cfg5 against a branch around them
          const bool ys = a == 31 && S >= 31;
          unsigned long long* const yp = yfw + (long long)(S - 31) * 4;  // 32-byte aligned
          st2_if(yp, tagged(rq[0], ep), tagged(rq[1], ep), ys);
          st2_if(yp + 2, tagged(rq[2], ep), tagged(rq[3], ep), ys);
          st_if(zfw + (long long)(S - 3) * 32 + a, tagged(rq[R3 - 1], ep), S >= 3);
        }
        // ---- shift the rows: P <- R, R <- new (virtual row: the next Z word)
        Pv[0] = Rv[0];
        Rv[0] = zn;
#pragma unroll
        for (int j = 0; j < R3; ++j) {
          Pv[j + 1] = Rv[j + 1];
          Rv[j + 1] = rq[j];
        }
        if (t + 1 < CH3) exchange(t + 1);
      }
      // ---- every four chunks: drain one 16-code block per row
      if ((k & 3) == 3) {
        const int m = k >> 2;
#pragma unroll
        for (int j = 0; j < R3; ++j) {
          const int d = m - ((s_[j] + 15) >> 4);
          const int xb = 16 * d;
          if (!rv[j] || xb < 0 || xb >= nx) continue;
          const unsigned rb = out_b[j] + (unsigned)(sizeof(C) * r_[j]);  // physical slot 0
          // logical slots (16 d + 4 q) mod 32 .. +15 (physical + GD3); the
          // group at logical 28..31 has its elements e >= 4 - r in the guard
          unsigned w[4 * sizeof(C)];
#pragma unroll
          for (int g = 0; g < 4; ++g) {
            const int gi = (4 * d + q_[j] + g) & 7;
            const unsigned ad = rb + (unsigned)((GD3 + 4 * gi) * sizeof(C));
            if (sizeof(C) == 1) {
              unsigned v;
              asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(ad));
              if (gi == 7) {
                unsigned gv;
                asm volatile("ld.shared.u32 %0, [%1];" : "=r"(gv) : "r"(rb));
                // bytes e < 4 - r from v, the rest from the guard word
                const unsigned sel = 0x3210u + (0x4444u & (0xFFFFu << (4 * (4 - r_[j]))));
                v = __byte_perm(v, gv, sel);
              }
              w[g] = v;
            } else {
              unsigned v0, v1;
              asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v0), "=r"(v1) : "r"(ad));
              if (gi == 7) {
                unsigned g0, g1;
                asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(g0), "=r"(g1) : "r"(rb));
                const int keep = 4 - r_[j];  // elements 0..keep-1 from v, the rest from g
                if (keep <= 2) v1 = g1;
                if (keep == 1) v0 = __byte_perm(v0, g0, 0x7610);
                if (keep == 3) v1 = __byte_perm(v1, g1, 0x7610);
              }
              w[2 * g] = v0;
              w[2 * g + 1] = v1;
            }
          }
          unsigned char* dst = reinterpret_cast<unsigned char*>(codes + row0 + j * plane + xb);
          const int cnt = nx - xb < 16 ? nx - xb : 16;  // multiple of 4 (nx % 4 == 0)
          if (cnt == 16 && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
#pragma unroll
            for (int i = 0; i < (int)sizeof(C); ++i)
              *reinterpret_cast<uint4*>(dst + 16 * i) =
                  make_uint4(w[4 * i], w[4 * i + 1], w[4 * i + 2], w[4 * i + 3]);
          } else {
            const int nw = cnt * (int)sizeof(C) / 4;
#pragma unroll
            for (int i = 0; i < 4 * (int)sizeof(C); ++i)
              if (i < nw) reinterpret_cast<unsigned*>(dst)[i] = w[i];
          }
        }
      }
      if (k + 1 < nchunks) {
        cpa_wait0();
        __syncwarp();
        settle(k + 1);
      }
    }
    // ---- final drain: every block not drained yet (x up to nx - 1)
    {
      const int mlast = nchunks / 4;  // first drain index not performed
      __syncwarp();
#pragma unroll
      for (int j = 0; j < R3; ++j) {
        if (!rv[j]) continue;
        const unsigned rb = out_b[j] + (unsigned)(sizeof(C) * r_[j]);
        for (int d = mlast - ((s_[j] + 15) >> 4); 16 * d < nx; ++d) {
          if (d < 0) continue;
          const int xb = 16 * d;
          C* dst = codes + row0 + j * plane + xb;
          const int cnt = nx - xb < 16 ? nx - xb : 16;
          for (int e = 0; e < cnt; ++e) {
            const int x = xb + e;
            // slot of x: logical (x + 4q) mod 32, in the guard when it was a
            // wrapped write (logical >= 28 and in the last r of the group)
            const int L = (x + 4 * q_[j]) & (WO3 - 1);
            const bool g = L >= WO3 - 4 && (L - (WO3 - 4)) >= 4 - r_[j];
            const unsigned addr = rb + (unsigned)((g ? L - (WO3 - 4) : GD3 + L) * sizeof(C));
            unsigned u;
            if (sizeof(C) == 1) asm volatile("ld.shared.u8 %0, [%1];" : "=r"(u) : "r"(addr));
            else asm volatile("ld.shared.u16 %0, [%1];" : "=r"(u) : "r"(addr));
            dst[e] = (C)u;
          }
        }
      }
    }
    if (ghist) {
      __syncwarp();
#pragma unroll
      for (int b = 0; b < 8; ++b) {
        const unsigned v = whist[a + 32 * b];
        if (v) atomicAdd(&ghist[a + 32 * b], (unsigned long long)v);
      }
    }
    // pads past the last written hyperplane hold tagged zeros
    for (int h = nsteps - 31 + a; h < HY; h += 32) {
      if (h >= 0) {
#pragma unroll
        for (int j = 0; j < R3; ++j) __stcg(yfw + (long long)h * 4 + j, tag0);
      }
    }
    for (int h = nsteps - 3; h < HY; ++h) __stcg(zfw + (long long)h * 32 + a, tag0);
    __syncwarp();
  }
}

// ---------------------------------------------------------------------------
// Decompress: the mirror sweep (decompress_scan, _kernels.py:83-105) on the
// same geometry, faces and ticket order as sweep3c_kernel (the face staging
// and checks below are the compress kernel's).  Per row:
//   * codes through a ring of 16 codes + a 4-code guard -- the compress input
//     ring with code-sized elements, one 4- (u8) or 8-byte (u16) cp.async per
//     row and chunk;
//   * the row's verbatim values (contiguous in the block: scan order) through
//     a ring of 16, refilled each chunk in aligned 4-value groups up to
//     cursor + 8 (a chunk consumes at most 4; indices past the block are
//     zero-filled, an underrun is detected from the final cursors);
//   * the reconstruction through a ring of 8 floats + a 4-float guard, drained
//     every chunk as one aligned 16-byte group.
// A point outside the row (x < 0 or x >= nx) reads the code `center` (the
// loader stores it in place of groups outside the row), so it consumes no
// verbatim value and its value is its prediction: +0.0 before the row
// starts (every term is a +0.0), the zero neighbour of the boundary rule.
constexpr int ORD = 8;    // recon ring per row (two groups)
constexpr int VRL = 16;   // verbatim ring per row (four aligned groups)
constexpr int WPB3D = 6;  // warps per block (2 blocks = 12 warps per SM in 228 KB)

template <typename C>
struct Sm3d {
  static constexpr int IRB = (WI3 + GD3) * (int)sizeof(C);  // bytes per code row
  static constexpr int IN_BYTES = 32 * R3 * IRB;
  static constexpr int OUT_OFF = ((IN_BYTES + 15) / 16) * 16;
  static constexpr int ORB = (ORD + GD3) * 4;                // 48 bytes per recon row
  static constexpr int OUT_BYTES = 32 * R3 * ORB;
  static constexpr int VR_OFF = OUT_OFF + OUT_BYTES;
  static constexpr int VR_BYTES = 32 * R3 * VRL * 4;
  static constexpr int YST_OFF = ((VR_OFF + VR_BYTES + 15) / 16) * 16;
  static constexpr int YST_BYTES = 2 * (4 * CH3 + CH3) * 8;
  static constexpr int ZST_OFF = YST_OFF + YST_BYTES;
  static constexpr int ZST_BYTES = 2 * CH3 * 32 * 8;
  static constexpr int PER_WARP = ((ZST_OFF + ZST_BYTES + 15) / 16) * 16;
};

__device__ __forceinline__ void cpa4z(unsigned smem, const void* g, int bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(smem), "l"(g), "r"(bytes));
}
__device__ __forceinline__ void cpa8z(unsigned smem, const void* g, int bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(smem), "l"(g), "r"(bytes));
}

#ifndef EBZ_S3D_MINB
#define EBZ_S3D_MINB 2
#endif
template <typename C>
__global__ void __launch_bounds__(32 * WPB3D, EBZ_S3D_MINB)
sweep3d_kernel(const __grid_constant__ F3Args fa, const __grid_constant__ FieldTable ft) {
  typedef Sm3d<C> SM;
  const SweepArgs& A = fa.s;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5, a = threadIdx.x & 31;
  unsigned char* wbase = smem_raw + warp * SM::PER_WARP;
  double* yst = reinterpret_cast<double*>(wbase + SM::YST_OFF);
  unsigned long long* zst = reinterpret_cast<unsigned long long*>(wbase + SM::ZST_OFF);
  const unsigned a_in = sm_addr(wbase);
  const unsigned a_out = sm_addr(wbase + SM::OUT_OFF);
  const unsigned a_vr = sm_addr(wbase + SM::VR_OFF);
  const unsigned a_zst = sm_addr(zst);
  const unsigned a_yst = sm_addr(yst);

  const int center = A.center;
  const double c52 = 0x1p52 + (double)center;  // (code - center) = (2^52 + code) - c52, exact
  const int nx = (int)A.dims[0], ny = (int)A.dims[1], nz = (int)A.dims[2];
  const int npy = fa.npy, npz = fa.npz, nf = fa.nf;
  const int ntasks = npy * npz * nf;
  const int nsteps = nx + SK3;
  const int nchunks = (nsteps + CH3 - 1) / CH3;
  const unsigned ep = A.epoch;
  const unsigned long long tag0 = ep;  // tagged +0.0
  const int HY = face3_h(nx);
  const long long plane = (long long)nx * ny;
  const int src = (a + 31) & 31;

  for (;;) {
    unsigned int tk = 0;
    if (a == 0) tk = atomicAdd(A.ticket, 1u);
    tk = __shfl_sync(EBZ_FULL, tk, 0);
    if ((int)tk >= ntasks) break;
    const int fi = (int)(tk % (unsigned)nf);
    const FieldRef& fr = ft.f[fi];
    const double eb = fr.info->eb;
    if (!(eb > 0.0)) continue;
    const double two_eb = __dmul_rn(2.0, eb);
    const C* const codes = reinterpret_cast<const C*>(fr.codes);
    float* const recon = reinterpret_cast<float*>(fr.recon);
    const float* const unpred = reinterpret_cast<const float*>(fr.unpred);
    const unsigned long long n_unpred = fr.info->n_unpred;
    const unsigned int tv = fa.tasks[tk / (unsigned)nf];
    const int PY = (int)(tv & 0xffff), PZ = (int)(tv >> 16);
    const int y0 = PY * 32, z0 = PZ * R3;
    const int y = y0 + a;
    bool rv[R3];
    int s_[R3], q_[R3], r_[R3];
#pragma unroll
    for (int j = 0; j < R3; ++j) {
      rv[j] = y < ny && z0 + j < nz;
      s_[j] = a + j;
      q_[j] = s_[j] >> 2;
      r_[j] = s_[j] & 3;
    }
    unsigned long long* const yfw = fr.yface + (long long)(PY * npz + PZ) * HY * 4;
    unsigned long long* const zfw = fr.zface + (long long)(PY * npz + PZ) * HY * 32;
    const bool hasY = PY > 0, hasZ = PZ > 0, hasC = PY > 0 && PZ > 0;
    const unsigned long long* const yfr =
        fr.yface + (long long)((hasY ? PY - 1 : 0) * npz + PZ) * HY * 4;
    const unsigned long long* const cfr =
        fr.yface + (long long)((hasC ? PY - 1 : 0) * npz + (hasC ? PZ - 1 : 0)) * HY * 4;
    const unsigned long long* const zfb =
        fr.zface + (long long)(PY * npz + (hasZ ? PZ - 1 : 0)) * HY * 32;
    const unsigned long long* const zfr = zfb + a;

    // ring addresses less the row's rotation residue r (as in the compress kernel)
    unsigned in_b[R3], out_b[R3], vr_b[R3];
#pragma unroll
    for (int j = 0; j < R3; ++j) {
      in_b[j] = a_in + (unsigned)(row_slot(a, j) * SM::IRB) - (unsigned)(sizeof(C) * r_[j]);
      out_b[j] = a_out + (unsigned)(row_slot(a, j) * SM::ORB) - 4u * (unsigned)r_[j];
      vr_b[j] = a_vr + (unsigned)(row_slot(a, j) * VRL * 4);
    }
    const long long row0 = ((long long)z0 * ny + y) * nx;
    const int ngroups = nx >> 2;
    // verbatim cursors: rank of the row's first code-0 point (zero-rank
    // pass); cursors are kept relative to ub = that rank rounded down to a
    // group (ring slot = relative position & 15)
    const bool uvec = (reinterpret_cast<uintptr_t>(unpred) & 15) == 0;
    const float* ubp[R3];  // unpred + the row's group-aligned base rank
    unsigned uc[R3], ul[R3], us[R3], un_rem[R3];  // un_rem: values left in the block past ubp
#pragma unroll
    for (int j = 0; j < R3; ++j) {
      const long long ri = (long long)(z0 + j) * ny + y;
      const unsigned long long u0 = rv[j] ? fr.rowbase[ri] + fr.rowblk[ri >> 8] : 0ull;
      const unsigned long long b0 = u0 & ~3ull;
      ubp[j] = unpred + b0;
      const unsigned long long rem = b0 < n_unpred ? n_unpred - b0 : 0ull;
      un_rem[j] = rem > 0x7fffffffull ? 0x7fffffffu : (unsigned)rem;
      uc[j] = us[j] = (unsigned)(u0 & 3);
      ul[j] = 0;
    }
    const unsigned cfill = sizeof(C) == 1 ? (unsigned)center * 0x01010101u
                                          : (unsigned)center * 0x00010001u;

    auto load_group = [&](int k) {
      const unsigned col = (unsigned)(GD3 + ((4 * (k + 1)) & (WI3 - 1))) * (unsigned)sizeof(C);
      const bool mirror = ((4 * (k + 1)) & (WI3 - 1)) == WI3 - 4;
#pragma unroll
      for (int j = 0; j < R3; ++j) {
        const int g = k + 1 - q_[j];
        const bool in = rv[j] && (unsigned)g < (unsigned)ngroups;
        const C* gp = codes + (in ? row0 + j * plane + 4 * g : 0);
        const unsigned dst = in_b[j] + (unsigned)(sizeof(C) * r_[j]);
        if (in) {
          if (sizeof(C) == 1) {
            cpa4z(dst + col, gp, 4);
            if (mirror) cpa4z(dst, gp, 4);
          } else {
            cpa8z(dst + col, gp, 8);
            if (mirror) cpa8z(dst, gp, 8);
          }
        } else {  // outside the row: codes `center`
          if (sizeof(C) == 1) {
            asm volatile("st.shared.u32 [%0], %1;" ::"r"(dst + col), "r"(cfill));
            if (mirror) asm volatile("st.shared.u32 [%0], %1;" ::"r"(dst), "r"(cfill));
          } else {
            asm volatile("st.shared.v2.u32 [%0], {%1, %1};" ::"r"(dst + col), "r"(cfill));
            if (mirror) asm volatile("st.shared.v2.u32 [%0], {%1, %1};" ::"r"(dst), "r"(cfill));
          }
        }
      }
    };
    // one verbatim group (4 values, aligned) of row j while the ring holds
    // fewer than cursor + 8 (values past the block are zero-filled).  The
    // prologue calls it three times; afterwards once per chunk keeps
    // ul >= uc + 8 (a chunk consumes at most 4)
    auto refill_one = [&](int j) {
      if (rv[j] && ul[j] < uc[j] + 8) {
        const int nv = ul[j] >= un_rem[j] ? 0 : (un_rem[j] - ul[j] >= 4 ? 4 : (int)(un_rem[j] - ul[j]));
        const float* g = nv ? ubp[j] + ul[j] : unpred;
        const unsigned d = vr_b[j] + 4u * (ul[j] & (VRL - 1));
        if (uvec) {
          cpa16(d, g, 4 * nv);
        } else {
#pragma unroll
          for (int e = 0; e < 4; ++e) cpa4z(d + 4 * e, e < nv ? g + e : unpred, e < nv ? 4 : 0);
        }
        ul[j] += 4;
      }
    };
    auto refill = [&]() {
#pragma unroll
      for (int j = 0; j < R3; ++j) refill_one(j);
    };
    auto load_faces = [&](int k) {
      const unsigned yb = a_yst + (unsigned)((k & 1) * 20 * 8);
      if (hasY && a < 8) cpa16(yb + a * 16, yfr + (long long)16 * k + 2 * a, 16);
      if (hasC && a >= 8 && a < 12)
        cpa8(yb + 128 + (a - 8) * 8, cfr + (long long)(4 * k + 4 + (a - 8)) * 4 + 3);
      if (hasZ) {
        const unsigned zb = a_zst + (unsigned)((k & 1) * CH3 * 32 * 8);
        const unsigned long long* g = zfb + (long long)(4 * k + 1) * 32 + 2 * a;
        cpa16(zb + a * 16, g, 16);
        cpa16(zb + 512 + a * 16, g + 64, 16);
      }
    };
    auto settle = [&](int k) {
      double* yb = yst + (k & 1) * 20;
      unsigned long long* zb = zst + (k & 1) * CH3 * 32;
      const bool ymine = hasY && (a < 8 || (a < 12 && hasC));
      const int w0 = a < 8 ? 2 * a : 16 + (a - 8);
      unsigned long long yw0 = tag0, yw1 = tag0;
      if (ymine) {
        yw0 = (unsigned long long)__double_as_longlong(yb[w0]);
        if (a < 8) yw1 = (unsigned long long)__double_as_longlong(yb[w0 + 1]);
      }
      unsigned long long zw[CH3];
#pragma unroll
      for (int t = 0; t < CH3; ++t) zw[t] = hasZ ? zb[t * 32 + a] : tag0;
      unsigned d = ((unsigned)yw0 ^ ep) | ((unsigned)yw1 ^ ep);
#pragma unroll
      for (int t = 0; t < CH3; ++t) d |= (unsigned)zw[t] ^ ep;
      bool miss = (d & kTagMask) != 0;
      if (__any_sync(EBZ_FULL, miss)) {
        for (unsigned ns = 32;; ns = ns < 512 ? 2 * ns : ns) {
          if (miss) {
            if (!tag_ok(yw0, ep))
              yw0 = a < 8 ? ld_cg64(yfr + (long long)16 * k + 2 * a)
                          : ld_cg64(cfr + (long long)(4 * k + 4 + (a - 8)) * 4 + 3);
            if (!tag_ok(yw1, ep)) yw1 = ld_cg64(yfr + (long long)16 * k + 2 * a + 1);
#pragma unroll
            for (int t = 0; t < CH3; ++t)
              if (!tag_ok(zw[t], ep)) {
                zw[t] = ld_cg64(zfr + (long long)(4 * k + 1 + t) * 32);
                zb[t * 32 + a] = zw[t];
              }
            miss = !tag_ok(yw0, ep) || !tag_ok(yw1, ep);
#pragma unroll
            for (int t = 0; t < CH3; ++t) miss |= !tag_ok(zw[t], ep);
          }
          if (!__any_sync(EBZ_FULL, miss)) break;
          __nanosleep(ns);
        }
      }
      if (ymine) {
        yb[w0] = untag(yw0);
        if (a < 8) yb[w0 + 1] = untag(yw1);
      }
      __syncwarp();
    };
    // drain recon group d of every row (complete, still in the ring): logical
    // group (d + q) & 1 == gi for all rows; group 1's elements e >= 4 - r were
    // written past the ring's end, into the guard
    unsigned fmax = 0;  // max |bits| of the stored values (non-finite check)
    auto drain = [&](int dk, int gi) {
#pragma unroll
      for (int j = 0; j < R3; ++j) {
        const int d = dk - q_[j];
        if (!rv[j] || d < 0 || d >= ngroups) continue;
        const unsigned rb = out_b[j] + 4u * (unsigned)r_[j];  // physical slot 0
        uint4 v;
        asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                     : "r"(rb + (unsigned)((GD3 + 4 * gi) * 4)));
        if (gi) {
          uint4 g;
          asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                       : "=r"(g.x), "=r"(g.y), "=r"(g.z), "=r"(g.w)
                       : "r"(rb));
          const int keep = 4 - r_[j];
          if (keep <= 3) v.w = g.w;
          if (keep <= 2) v.z = g.z;
          if (keep <= 1) v.y = g.y;
        }
        fmax = max(fmax, max(max(v.x & 0x7fffffffu, v.y & 0x7fffffffu),
                             max(v.z & 0x7fffffffu, v.w & 0x7fffffffu)));
        *reinterpret_cast<uint4*>(recon + row0 + j * plane + 4 * d) = v;
      }
    };

    double Rv[R3 + 1], Pv[R3 + 1], Bv[R3 + 1], B1[R3 + 1], B2[R3 + 1];
#pragma unroll
    for (int j = 0; j <= R3; ++j) Rv[j] = Pv[j] = Bv[j] = B1[j] = B2[j] = 0.0;

    for (int i = a; i < 40; i += 32)
      if (!hasY || (!hasC && (i % 20) >= 16))
        reinterpret_cast<unsigned long long*>(yst)[i] = 0ull;
    if (!hasZ)
      for (int i = a; i < 2 * CH3 * 32; i += 32) zst[i] = tag0;
    __syncwarp();
    load_group(-2);
    load_group(-1);
    load_faces(0);
    cpa_commit();
    {
      unsigned long long w = hasZ ? ld_cg64(zfr) : tag0;
      unsigned long long c = (hasC && a == 0) ? ld_cg64(cfr + 3 * 4 + 3) : tag0;
      bool miss = !tag_ok(w, ep) || !tag_ok(c, ep);
      for (unsigned ns = 32; __any_sync(EBZ_FULL, miss); ns = ns < 512 ? 2 * ns : ns) {
        __nanosleep(ns);
        if (!tag_ok(w, ep)) w = ld_cg64(zfr);
        if (!tag_ok(c, ep)) c = ld_cg64(cfr + 3 * 4 + 3);
        miss = !tag_ok(w, ep) || !tag_ok(c, ep);
      }
      Rv[0] = untag(w);
      Bv[0] = untag(c);
    }
    refill();
    refill();
    refill();
    cpa_commit();
    cpa_wait0();
    __syncwarp();
    settle(0);

    for (int k = 0; k < nchunks; ++k) {
      sched_jitter(A.jitter, tk, k);
      const int S0 = k * CH3;
      if (k + 1 < nchunks) {
        load_group(k);
        load_faces(k + 1);
      }
      // this chunk's verbatim values [cursor, cursor + 4) landed with the
      // previous chunk's copies; request up to cursor + 8 for the next one
      float un[R3];
#pragma unroll
      for (int j = 0; j < R3; ++j) un[j] = ld_sf(vr_b[j] + 4u * (uc[j] & (VRL - 1)));
      refill();
      cpa_commit();
      const unsigned P0 = (unsigned)(GD3 + (S0 & (WI3 - 1))) * (unsigned)sizeof(C);
      const unsigned Q0 = (unsigned)(GD3 + (S0 & (ORD - 1))) * 4u;
      const double* yb = yst + (k & 1) * 20;
      const unsigned long long* zb = zst + (k & 1) * CH3 * 32;
      unsigned ia[R3], oa[R3];
      int xl[R3];
#pragma unroll
      for (int j = 0; j < R3; ++j) {
        ia[j] = in_b[j] + P0;
        oa[j] = out_b[j] + Q0;
        xl[j] = rv[j] ? S0 - s_[j] : (int)0x80000000;
      }
      double Bn[R3 + 1];
      auto exchange = [&](int t) {
        const double2 y01 = *reinterpret_cast<const double2*>(yb + 4 * t);
        const double2 y23 = *reinterpret_cast<const double2*>(yb + 4 * t + 2);
        const double yf[R3 + 1] = {yb[16 + t], y01.x, y01.y, y23.x, y23.y};
#pragma unroll
        for (int j = 0; j <= R3; ++j) Bn[j] = __shfl_sync(EBZ_FULL, a == 31 ? yf[j] : Rv[j], src);
      };
      exchange(0);
#pragma unroll
      for (int t = 0; t < CH3; ++t) {
        const int S = S0 + t;
        const double zn = untag(zb[t * 32 + a]);
#pragma unroll
        for (int j = 0; j <= R3; ++j) {
          B2[j] = B1[j];
          B1[j] = Bv[j];
          Bv[j] = Bn[j];
        }
        // codes (off the recurrence): (code - center) * 2eb
        int code[R3];
        double qv[R3];
#pragma unroll
        for (int j = 0; j < R3; ++j) {
          unsigned c;
          if (sizeof(C) == 1)
            asm volatile("ld.shared.u8 %0, [%1];" : "=r"(c) : "r"(ia[j] + (unsigned)t));
          else
            asm volatile("ld.shared.u16 %0, [%1];" : "=r"(c) : "r"(ia[j] + 2u * (unsigned)t));
          code[j] = (int)c;
          qv[j] = __dmul_rn(__dsub_rn(__hiloint2double(0x43300000, code[j]), c52), two_eb);
        }
        double pr[R3];
#pragma unroll
        for (int j = 0; j < R3; ++j) pr[j] = __dadd_rn(Rv[j], Bv[j + 1]);
#pragma unroll
        for (int j = 0; j < R3; ++j) pr[j] = __dsub_rn(pr[j], B1[j]);
#pragma unroll
        for (int j = 0; j < R3; ++j) pr[j] = __dadd_rn(pr[j], Rv[j + 1]);
#pragma unroll
        for (int j = 0; j < R3; ++j) pr[j] = __dsub_rn(pr[j], Pv[j]);
#pragma unroll
        for (int j = 0; j < R3; ++j) pr[j] = __dsub_rn(pr[j], B1[j + 1]);
#pragma unroll
        for (int j = 0; j < R3; ++j) pr[j] = __dadd_rn(pr[j], B2[j]);
        // recon = T(pred + (code - center) 2eb), or the next verbatim value
        double rq[R3];
#pragma unroll
        for (int j = 0; j < R3; ++j) {
          const float rf = __double2float_rn(__dadd_rn(pr[j], qv[j]));
          const bool zc = code[j] == 0;
          const float vf = zc ? un[j] : rf;
          rq[j] = (double)vf;
          asm volatile("st.shared.f32 [%0], %1;" ::"r"(oa[j] + 4u * (unsigned)t), "f"(vf));
          if (zc) {
            ++uc[j];
            un[j] = ld_sf(vr_b[j] + 4u * (uc[j] & (VRL - 1)));
          }
        }
        {
          const bool ys = a == 31 && S >= 31;
          unsigned long long* const yp = yfw + (long long)(S - 31) * 4;
          st2_if(yp, tagged(rq[0], ep), tagged(rq[1], ep), ys);
          st2_if(yp + 2, tagged(rq[2], ep), tagged(rq[3], ep), ys);
          st_if(zfw + (long long)(S - 3) * 32 + a, tagged(rq[R3 - 1], ep), S >= 3);
        }
        Pv[0] = Rv[0];
        Rv[0] = zn;
#pragma unroll
        for (int j = 0; j < R3; ++j) {
          Pv[j + 1] = Rv[j + 1];
          Rv[j + 1] = rq[j];
        }
        if (t + 1 < CH3) exchange(t + 1);
      }
      __syncwarp();
      drain(k - 1, (k - 1) & 1);
      if (k + 1 < nchunks) {
        cpa_wait0();
        __syncwarp();
        settle(k + 1);
      }
    }
    drain(nchunks - 1, (nchunks - 1) & 1);
    cpa_wait0();  // no copy may land after the next task reuses the rings
    // per task (consecutive tasks may belong to different fields)
    {
      unsigned long long used = 0;
      bool under = false;
#pragma unroll
      for (int j = 0; j < R3; ++j) {
        used += uc[j] - us[j];
        under |= uc[j] > un_rem[j];
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) used += __shfl_xor_sync(EBZ_FULL, used, o);
      int bad = (under ? ST_UNDERRUN : 0) | (fmax >= 0x7f800000u ? ST_NONFINITE_OUT : 0);
      bad = __reduce_or_sync(EBZ_FULL, bad);
      if (a == 0) {
        if (used) atomicAdd(&fr.info->used, used);
        if (bad) atomicOr(&fr.info->status, bad);
      }
    }
    for (int h = nsteps - 31 + a; h < HY; h += 32) {
      if (h >= 0) {
#pragma unroll
        for (int j = 0; j < R3; ++j) __stcg(yfw + (long long)h * 4 + j, tag0);
      }
    }
    for (int h = nsteps - 3; h < HY; ++h) __stcg(zfw + (long long)h * 32 + a, tag0);
    __syncwarp();
  }
}

template <typename C>
cudaError_t launch3d_t(const F3Args& fa, const FieldTable& ft, int sms, cudaStream_t s) {
  typedef Sm3d<C> SM;
  const size_t smem = (size_t)WPB3D * SM::PER_WARP;
  static KernelAttr attr;
  cudaError_t e = kernel_smem(attr, sweep3d_kernel<C>, smem);
  if (e != cudaSuccess) return e;
  const int per_sm = kernel_occupancy(attr, sweep3d_kernel<C>, 32 * WPB3D, smem);
  const long long ntasks = (long long)fa.npy * fa.npz * fa.nf;
  long long blocks = (ntasks + WPB3D - 1) / WPB3D;
  if (blocks > (long long)sms * per_sm) blocks = (long long)sms * per_sm;
  if (blocks < 1) blocks = 1;
  sweep3d_kernel<C><<<(unsigned)blocks, 32 * WPB3D, smem, s>>>(fa, ft);
  return cudaGetLastError();
}

template <typename C, bool REC, bool PF = false, bool TR = false, bool JIT = false>
cudaError_t launch3_t(const F3Args& fa, const FieldTable& ft, int sms, cudaStream_t s) {
  typedef Sm3<C> SM;
  const size_t smem = (size_t)WPB3 * SM::PER_WARP;
  static KernelAttr attr;
  cudaError_t e = kernel_smem(attr, sweep3c_kernel<C, REC, PF, TR, JIT>, smem);
  if (e != cudaSuccess) return e;
  const int per_sm = kernel_occupancy(attr, sweep3c_kernel<C, REC, PF, TR, JIT>, 32 * WPB3, smem);
  const long long ntasks = (long long)fa.npy * fa.npz * fa.nf;
  long long blocks = (ntasks + WPB3 - 1) / WPB3;
  if (blocks > (long long)sms * per_sm) blocks = (long long)sms * per_sm;
  if (blocks < 1) blocks = 1;
  sweep3c_kernel<C, REC, PF, TR, JIT><<<(unsigned)blocks, 32 * WPB3, smem, s>>>(fa, ft);
  return cudaGetLastError();
}

}  // namespace

// 3D, n = 1, float32, nx a multiple of 4 (aligned row groups).  Compress by
// default (EBZ_NO_SWEEP3 turns it off); the decompress kernel only with
// EBZ_SWEEP3D=1 -- bit-exact, but measured slower than sweep_fast.cu's
// decompress kernel on cfg5 (7.5-7.9 ms vs 6.25 ms: per-chunk ring and
// verbatim bookkeeping and the verbatim cursor updates cost more issue slots
// than the shared neighbour exchange saves)
// Kernel choice for 3D, n = 1, float32 compress.  Three kernels write the same
// bytes: sweep3c (32 x 4 patches, four z-rows per lane) has the highest
// throughput (cfg5 batch: 4.6 vs 5.6 ms), the two-row kernel (8 x 8 patches,
// sweep_fast.cu) a shorter wavefront ramp, the block-speculative one-row
// kernel with 16-byte face words (8 x 4 patches, sweep3b.cu) the shortest
// ramp and the lowest throughput (a lone 256^3 field: 0.75 / 0.59 / 0.49 ms;
// 16 of them: 1.41 / 1.61 / 2.41 ms).  The launch takes the one a fitted time
// model predicts fastest:
//   t = hypot(ramp, work),  u = [nx % 16 != 0],
//   ramp = (c0 nx + c1 npy + c2 npz) (1 + v u)   (ms, critical path),
//   work = w * Mpoints * (1 + r u)               (ms, throughput),
// constants fitted to 52 (shape, field count) measurements per kernel on B200
// (tools/kernel_choice_probe.py, profiles/r02_kernel_choice.md: model error
// 3-5% mean; the choice costs 0.2% over the best kernel on average, 3.5% at
// worst, and 11% less than the best of the first two kernels).
// Returns 0 two-row, 1 sweep3c, 2 sweep3b.
int sweep3_model_choice(const long long* dims, int nf) {
  const long long nx = dims[0];
  const double ny = (double)dims[1], nz = (double)dims[2];
  const double mpts = (double)(nf > 0 ? nf : 1) * (double)nx * ny * nz * 1e-6;
  const double unal = nx % 16 ? 1.0 : 0.0;
  const double ramp3 = (0.000540 * (double)nx + 0.026845 * ceil(ny / 32.0) +
                        0.007053 * ceil(nz / R3)) * (1.0 + 0.050 * unal);
  const double work3 = 0.004318 * mpts * (1.0 + 0.120 * unal);
  const double ramp2 = 0.000413 * (double)nx + 0.007720 * ceil(ny / 8.0) + 0.006496 * ceil(nz / 8.0);
  const double work2 = 0.005356 * mpts * (1.0 + 0.084 * unal);
  const double rampb = 0.000229 * (double)nx + 0.004665 * ceil(ny / 8.0) + 0.003263 * ceil(nz / 4.0);
  const double workb = 0.007760 * mpts * (1.0 + 0.063 * unal);
  const double t3 = nx % 4 == 0 ? hypot(ramp3, work3) : 1e30;  // sweep3c needs nx % 4 == 0
  const double t2 = hypot(ramp2, work2), tb = hypot(rampb, workb);
  if (tb < t2 && tb < t3) return 2;
  return t3 < t2 ? 1 : 0;
}

// EBZ_SWEEP3 = always | never | auto overrides (read at every call, so tests
// can cover both kernels in one process); EBZ_NO_SWEEP3 = never.
bool sweep3_used(int ndim, int layers, int width, const long long* dims, int nf, bool compress) {
  const long long nx = dims[0];
  const bool able = ndim == 3 && layers == 1 && width == 32 && nx % 4 == 0 && nx < (1ll << 28);
  if (!able) return false;
  if (!compress) return getenv("EBZ_SWEEP3D") != nullptr;
  const char* mode = getenv("EBZ_SWEEP3");
  if (getenv("EBZ_NO_SWEEP3") || (mode && !strcmp(mode, "never"))) return false;
  if (mode && !strcmp(mode, "always")) return true;
  return sweep3_model_choice(dims, nf) == 1;
}

void sweep3_patch_grid(const long long* dims, int* npy, int* npz) {
  *npy = (int)((dims[1] + 31) / 32);
  *npz = (int)((dims[2] + R3 - 1) / R3);
}

void sweep3_face_words(const long long* dims, long long* ny_words, long long* nz_words) {
  int npy, npz;
  sweep3_patch_grid(dims, &npy, &npz);
  const long long hy = face3_h(dims[0]);
  *ny_words = (long long)npy * npz * hy * 4;
  *nz_words = (long long)npy * npz * hy * 32;
}

cudaError_t launch_sweep3(const SweepArgs& a, const FieldTable& ft, int nf,
                          const unsigned int* d_tasks, int npy, int npz, bool compress, bool rec,
                          int sms, cudaStream_t s) {
  if (nf < 1 || nf > kBatchMax) return cudaErrorInvalidValue;
  F3Args fa;
  fa.s = a;
  fa.tasks = d_tasks;
  fa.npy = npy;
  fa.npz = npz;
  fa.nf = nf;
  const bool wide = a.wide != 0;
  if (!compress) return wide ? launch3d_t<uint16_t>(fa, ft, sms, s) : launch3d_t<uint8_t>(fa, ft, sms, s);
  // per-field centres (interval trials: u16 codes, no recon)
  if (ft.center[0]) {
    if (!wide || rec) return cudaErrorInvalidValue;
    return launch3_t<uint16_t, false, true>(fa, ft, sms, s);
  }
  if (a.trunc) {  // opt-in truncated-mantissa coding (no recon output there)
    if (rec) return cudaErrorInvalidValue;
    return wide ? launch3_t<uint16_t, false, false, true>(fa, ft, sms, s)
                : launch3_t<uint8_t, false, false, true>(fa, ft, sms, s);
  }
  if (rec) return wide ? launch3_t<uint16_t, true>(fa, ft, sms, s) : launch3_t<uint8_t, true>(fa, ft, sms, s);
  if (a.jitter)  // test hook instantiation
    return wide ? launch3_t<uint16_t, false, false, false, true>(fa, ft, sms, s)
                : launch3_t<uint8_t, false, false, false, true>(fa, ft, sms, s);
  return wide ? launch3_t<uint16_t, false>(fa, ft, sms, s) : launch3_t<uint8_t, false>(fa, ft, sms, s);
}
