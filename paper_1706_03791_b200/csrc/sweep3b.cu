// sweep3b.cu -- patch wavefront with 16-byte face words for 3D grids, layer
// n = 1: compress_scan / decompress_scan of ebzip/_kernels.py:48-105 for
// binary64 fields, which the float32 kernels cannot take (the generic kernel
// hands a field's 32-row tasks out in flat row order, one chain per field:
// 128^3 float64 took 74 ms), and -- compress -- for lone float32 fields,
// where it has the shortest ramp of the three compress kernels.
//
// Geometry of the one-row kernel (sweep_fast.cu): a warp owns 8 (y) x 4 (z)
// rows, lane (a, b) processes x = S - (a + b) at step S; rows y - 1 / z - 1
// arrive by shuffles (1 / 8 lanes up), the diagonal row (y - 1, z - 1) is
// relayed (what lane - 1 received from its z - 1 neighbour a step earlier);
// patches are handed out by an atomic ticket in hyperplane (Y + Z) order.
// The step is sweep2.cu's: blocks of 4 steps as one basic block, compress
// speculating on the reciprocal quantizer with ONE vote per block (replay
// with the reference's division on a hit), face words stored after it.
//
// Patch faces: binary64 has no spare mantissa bits for the epoch tag of the
// float32 kernels, so a face word is 16 bytes {value, epoch}, read and
// written with one aligned 16-byte access (sweep2.cu, struct Face).  Layout
// as the one-row kernel's skew-major blocks: the Y face of patch (PY, PZ) is
// (nx + 4) x 4 words with row zz at column x in word 4 (x + zz) + zz, the Z
// face (nx + 8) x 8 words with row zz in word 8 (x + zz) + zz.  The words a
// block of 4 steps consumes (20 Y, 4 corner, 32 Z) are staged in shared
// memory a block ahead (one 16-byte async copy each), tag-checked once per
// block and handed to the boundary lanes as plain doubles.
//
// Arithmetic: the reference's term order ((((((z-1 + y-1) - yz) + x-1) - xz)
// - xy) + xyz), binary64, no contraction, no rounding of the stored value
// (the element type is binary64) -- the bytes of the generic kernel and of
// the reference.
#include <cstdlib>
#include <cstring>
#include <type_traits>

#include "ebz_common.cuh"

namespace {

typedef ulonglong2 W;           // face word {value bits, epoch}
constexpr int BS = 4;           // steps per block
constexpr int RX = 64;          // tile ring columns
constexpr int NCH = RX / BS;    // input ring slots (compress)
constexpr int PD = 6;           // input prefetch distance (blocks, compress)
constexpr int PY = 8, PZ = 4;   // patch rows
constexpr int SMAX = PY - 1 + PZ - 1;        // max lane skew
constexpr int WLAST = (BS + SMAX - 1) / BS;  // code chunk c is last written in block c + WLAST
constexpr int WPB = 2;          // warps per block
constexpr int FY = 4 * BS + 4, FC = BS, FZ = 8 * BS;  // staged words per block
constexpr int FW = FY + FC + FZ;
constexpr int CH = 16;          // columns per staged code chunk (decompress)
constexpr int OUT_LAG = 1;      // (decompress) chunks still being written: skew 10 < 16

struct S3bArgs {
  SweepArgs s;
  const unsigned int* tasks;    // task -> PY | PZ << 16 (hyperplane order)
  int npy, npz;
  int nf;
};

template <typename C, typename T> struct Sm3b {
  static constexpr int CODE_STRIDE = RX + 16;
  static constexpr int F_BYTES = 32 * RX * (int)sizeof(T);
  static constexpr int C_BYTES = 32 * CODE_STRIDE * (int)sizeof(C);
  static constexpr int F_OFF = 0;
  static constexpr int C_OFF = F_BYTES;
  static constexpr int FST_OFF = C_OFF + C_BYTES;            // raw face words, 2 blocks
  static constexpr int FVAL_OFF = FST_OFF + 2 * FW * 16;     // their values, 2 blocks
  // u8 codes: the warp's code histogram of its current task (256 bins + a
  // dummy bin for points outside their row), flushed per task
  static constexpr int HIST_OFF = FVAL_OFF + 2 * FW * 8;
  static constexpr int HIST_BYTES = sizeof(C) == 1 ? 260 * 4 : 0;
  static constexpr int PER_WARP = HIST_OFF + HIST_BYTES;
};

__device__ __forceinline__ void cpa16(unsigned s, const void* g, int bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(g), "r"(bytes));
}
__device__ __forceinline__ void cpa8(unsigned s, const void* g, int bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(g), "r"(bytes));
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
// element accesses by type (float32 / binary64)
__device__ __forceinline__ void lds_t(unsigned a, float& v) {
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
}
__device__ __forceinline__ void lds_t(unsigned a, double& v) {
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
}
__device__ __forceinline__ void sts_t(unsigned a, float, double r) {
  asm volatile("st.shared.f32 [%0], %1;" ::"r"(a), "f"(__double2float_rn(r)));
}
__device__ __forceinline__ void sts_t(unsigned a, double, double r) {
  asm volatile("st.shared.f64 [%0], %1;" ::"r"(a), "d"(r));
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
// predicated shared load into v (v keeps its value when the predicate is off)
__device__ __forceinline__ void lds_f64_if(double& v, unsigned a, bool pred) {
  asm volatile("{ .reg .pred q; setp.ne.u32 q, %2, 0; @q ld.shared.f64 %0, [%1]; }"
               : "+d"(v) : "r"(a), "r"((unsigned)pred));
}
__device__ __forceinline__ W ld_face(const W* p) {
  W w;
  asm volatile("ld.global.cg.v2.u64 {%0, %1}, [%2];" : "=l"(w.x), "=l"(w.y) : "l"(p));
  return w;
}
__device__ __forceinline__ void st_face_if(W* p, double r, unsigned ep, bool pred) {
  asm volatile("{ .reg .pred q; setp.ne.u32 q, %3, 0; @q st.global.cg.v2.u64 [%0], {%1, %2}; }"
               ::"l"(p), "l"((unsigned long long)__double_as_longlong(r)),
                 "l"((unsigned long long)ep), "r"((unsigned)pred) : "memory");
}

// Everything a task's face traffic needs: the neighbours' blocks, this lane's
// staged words, their validity.
struct Faces {
  const W* gY;  // Y face of patch (PY - 1, PZ)
  const W* gC;  // Y face of patch (PY - 1, PZ - 1) (corner row zz = 3)
  const W* gZ;  // Z face of patch (PY, PZ - 1)
  bool hY, hC, hZ;
  int nx, ny, nz, y0, z0, ybw, zbw;
  unsigned ep;
  W* fst;        // shared: raw words [2][FW]
  double* fval;  // shared: values [2][FW]
  int lane;
  // blocks whose every staged word lies inside the rows (b >= 2 and
  // 4b + 8 <= nx): this lane's two validity flags are task constants
  // (bit 0: its Y / corner word, bit 1: its Z word)
  unsigned vmask;
  __device__ __forceinline__ void init_mask() {
    const bool y = lane < FY ? (hY && z0 + (lane & 3) < nz) : (lane < FY + FC && hC);
    const bool z = hZ && y0 + (lane & 7) < ny;
    vmask = (unsigned)y | (unsigned)z << 1;
  }
  __device__ __forceinline__ bool interior(int b) const { return b >= 2 && 4 * b + 8 <= nx; }
  __device__ __forceinline__ bool v0(int b) const {
    return interior(b) ? (vmask & 1u) != 0 : (y_ok(wy(b)) || c_ok(b));
  }
  __device__ __forceinline__ bool v1(int b) const {
    return interior(b) ? (vmask & 2u) != 0 : z_ok(wz(b));
  }

  // this lane's words of block b: (Y or corner) and Z
  __device__ __forceinline__ int wy(int b) const { return 4 * BS * b - 4 + lane; }
  __device__ __forceinline__ int wc(int b) const { return 4 * BS * b + 15 + 4 * (lane - FY); }
  __device__ __forceinline__ int wz(int b) const { return 8 * BS * b + lane; }
  __device__ __forceinline__ bool y_ok(int w) const {
    const int zz = w & 3, xx = (w >> 2) - zz;
    return lane < FY && hY && w >= 0 && w < ybw && (unsigned)xx < (unsigned)nx && z0 + zz < nz;
  }
  __device__ __forceinline__ bool c_ok(int b) const {
    return lane >= FY && lane < FY + FC && hC && wc(b) < ybw &&
           (unsigned)(BS * b + lane - FY) < (unsigned)nx;
  }
  __device__ __forceinline__ bool z_ok(int w) const {
    const int zz = w & 7, xx = (w >> 3) - zz;
    return hZ && w >= 0 && w < zbw && (unsigned)xx < (unsigned)nx && y0 + zz < ny;
  }
  __device__ __forceinline__ void issue(int b) const {
    W* buf = fst + (b & 1) * FW;
    // (Y words by lanes < FY, corner words by lanes FY .. FY + FC - 1: slot = lane)
    if (v0(b)) cpa16(saddr(buf + lane), lane < FY ? gY + wy(b) : gC + wc(b), 16);
    if (v1(b)) cpa16(saddr(buf + FY + FC + lane), gZ + wz(b), 16);
    cpa_commit();
  }
  // after the block's copies landed: this lane's two words (tagged zero where
  // the word lies outside the domain)
  __device__ __forceinline__ void read(int b, W (&w)[2]) const {
    const W* buf = fst + (b & 1) * FW;
    const W zero = make_ulonglong2(0ull, (unsigned long long)ep);
    w[0] = v0(b) ? buf[lane] : zero;
    w[1] = v1(b) ? buf[FY + FC + lane] : zero;
  }
  __device__ __forceinline__ bool missing(const W (&w)[2]) const {
    return w[0].y != (unsigned long long)ep || w[1].y != (unsigned long long)ep;
  }
  // spin on the late words (warp-uniform call)
  __device__ __forceinline__ void settle(int b, W (&w)[2]) const {
    bool miss = missing(w);
    if (!__any_sync(EBZ_FULL, miss)) return;
    for (unsigned ns = 16;; ns = ns < 256 ? 2 * ns : ns) {
      if (miss) {
        if (w[0].y != (unsigned long long)ep)
          w[0] = lane < FY ? ld_face(gY + wy(b)) : ld_face(gC + wc(b));
        if (w[1].y != (unsigned long long)ep) w[1] = ld_face(gZ + wz(b));
        miss = missing(w);
      }
      if (!__any_sync(EBZ_FULL, miss)) break;
      __nanosleep(ns);
    }
  }
  // the values for the consumers of block b
  __device__ __forceinline__ void store(int b, const W (&w)[2]) const {
    double* v = fval + (b & 1) * FW;
    if (lane < FY + FC) v[lane] = __longlong_as_double((long long)w[0].x);
    v[FY + FC + lane] = __longlong_as_double((long long)w[1].x);
    __syncwarp();
  }
};

// history: own row at x - 1; rows (y-1, z), (y, z-1), (y-1, z-1) at x and x - 1
struct Hist3 {
  double L, Uy0, Uy1, Uz0, Uz1, Uc0, Uc1;
  // shift in column x of the three neighbour rows (patch-boundary lanes take
  // the staged face values) and predict
  __device__ __forceinline__ double predict(unsigned a_fv, int j, int la, int lb) {
    double iny = __shfl_up_sync(EBZ_FULL, L, 1);
    double inz = __shfl_up_sync(EBZ_FULL, L, PY);
    double inc = __shfl_up_sync(EBZ_FULL, Uz0, 1);
    lds_f64_if(iny, a_fv + 8u * (unsigned)(4 * j + lb + 4), la == 0);
    lds_f64_if(inc, a_fv + 8u * (unsigned)(lb ? 4 * j + lb - 1 : FY + j), la == 0);
    lds_f64_if(inz, a_fv + 8u * (unsigned)(FY + FC + 8 * j + la), lb == 0);
    Uy1 = Uy0;
    Uz1 = Uz0;
    Uc1 = Uc0;
    Uy0 = iny;
    Uz0 = inz;
    Uc0 = inc;
    // reference term order (x offset outermost, then y, then z)
    double p = __dadd_rn(Uz0, Uy0);
    p = __dsub_rn(p, Uc0);
    p = __dadd_rn(p, L);
    p = __dsub_rn(p, Uz1);
    p = __dsub_rn(p, Uy1);
    p = __dadd_rn(p, Uc1);
    return p;
  }
};

// task geometry shared by both directions
struct Task {
  int PYi, PZi, y0, z0, y, z;
  bool rv, full_rows;
};

template <typename C, typename T, bool COMPRESS>
__global__ void __launch_bounds__(32 * WPB, 4)
sweep3b_kernel(const __grid_constant__ S3bArgs fa, const __grid_constant__ FieldTable ft) {
  typedef Sm3b<C, T> SM;
  constexpr int EP = 16 / (int)sizeof(T);  // elements per 16-byte copy
  const SweepArgs& a = fa.s;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int la = lane % PY, lb = lane / PY, sig = la + lb;
  unsigned char* wbase = smem_raw + warp * SM::PER_WARP;
  T* f_tile = reinterpret_cast<T*>(wbase + SM::F_OFF);   // compress: input; decompress: output
  C* c_tile = reinterpret_cast<C*>(wbase + SM::C_OFF);   // compress: codes out; decompress: codes in
  const unsigned a_f = pin(saddr(f_tile + lane * RX));
  const unsigned a_c = pin(saddr(c_tile + lane * SM::CODE_STRIDE));
  const unsigned a_fval = pin(saddr(wbase + SM::FVAL_OFF));
  unsigned int* const whist = reinterpret_cast<unsigned int*>(wbase + SM::HIST_OFF);
  const unsigned a_hist = pin(saddr(whist));
  const int nx = (int)a.dims[0], ny = (int)a.dims[1], nz = (int)a.dims[2];
  const int npy = fa.npy, npz = fa.npz, nf = fa.nf;
  const int ntasks = npy * npz * nf;
  const unsigned epoch = a.epoch;
  const int ybw = (nx + 4) * 4, zbw = (nx + 8) * 8;  // face block words
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
    const unsigned int tv = fa.tasks[tk / (unsigned)nf];
    Task t;
    t.PYi = (int)(tv & 0xffff);
    t.PZi = (int)(tv >> 16);
    t.y0 = t.PYi * PY;
    t.z0 = t.PZi * PZ;
    t.y = t.y0 + la;
    t.z = t.z0 + lb;
    t.rv = t.y < ny && t.z < nz;
    t.full_rows = t.y0 + PY <= ny && t.z0 + PZ <= nz;
    const bool rv = t.rv;
    const long long rowi = ((long long)(rv ? t.z : 0) * ny + (rv ? t.y : 0)) * nx;
    W* const yface = reinterpret_cast<W*>(fr.yface);
    W* const zface = reinterpret_cast<W*>(fr.zface);
    auto yblk = [&](int Y, int Z) { return (long long)(Y * npz + Z) * ybw; };
    auto zblk = [&](int Y, int Z) { return (long long)(Y * npz + Z) * zbw; };
    // faces this lane hands on: row zz = lb of the patch's Y face at word
    // 4 (x + zz) + zz, row zz = la of its Z face at word 8 (x + zz) + zz
    W* const wyp = yface + yblk(t.PYi, t.PZi) + 5 * lb;
    W* const wzp = zface + zblk(t.PYi, t.PZi) + 9 * la;
    const bool wy_ok = rv && la == PY - 1, wz_ok = rv && lb == PZ - 1;
    Faces F;
    F.hY = t.PYi > 0;
    F.hZ = t.PZi > 0;
    F.hC = F.hY && F.hZ;
    F.gY = yface + (F.hY ? yblk(t.PYi - 1, t.PZi) : 0);
    F.gC = yface + (F.hC ? yblk(t.PYi - 1, t.PZi - 1) : 0);
    F.gZ = zface + (F.hZ ? zblk(t.PYi, t.PZi - 1) : 0);
    F.nx = nx; F.ny = ny; F.nz = nz; F.y0 = t.y0; F.z0 = t.z0; F.ybw = ybw; F.zbw = zbw;
    F.ep = epoch;
    F.fst = reinterpret_cast<W*>(wbase + SM::FST_OFF);
    F.fval = reinterpret_cast<double*>(wbase + SM::FVAL_OFF);
    F.lane = lane;
    F.init_mask();
    // face words of a final block leave: Y face by lanes la == 7, Z face by lb == 3
    auto faces_out = [&](int xb, const double (&rj)[BS]) {
#pragma unroll
      for (int j = 0; j < BS; ++j) {
        const bool in = (unsigned)(xb + j) < (unsigned)nx;
        st_face_if(wyp + (long long)(xb + j) * 4, rj[j], epoch, wy_ok && in);
        st_face_if(wzp + (long long)(xb + j) * 8, rj[j], epoch, wz_ok && in);
      }
    };
    Hist3 H = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};

    if (COMPRESS) {
      // ------------------------------------------------------------ compress
      const double inv = 1.0 / two_eb;
      const bool fast_ok = isfinite(inv) && inv > 0.0 && two_eb >= 0x1p-1000 &&
                           inv >= 0x1p-1000 && inv <= 0x1p1000;
      const double guard = fast_ok ? 0.5 - 0x1p-30 : -1.0;
      const T* values = reinterpret_cast<const T*>(fr.values);
      C* const row_out = reinterpret_cast<C*>(fr.codes) + rowi;
      const int nblk = (nx + BS - 1) / BS + WLAST + 2;
      // u8 codes: the code histogram (codec.py:107) is counted here, as the
      // validated codes of a block go to the tile
      unsigned long long* const ghist = sizeof(C) == 1 ? fr.hist : nullptr;
      if (ghist) {
#pragma unroll
        for (int q = 0; q < 8; ++q) whist[lane + 32 * q] = 0u;
        __syncwarp();
      }
      const bool al_in = nx % EP == 0;
      const bool al_out = (nx * (int)sizeof(C)) % 4 == 0;
      // input columns [4j, 4j + 4) of the patch's 32 rows (zeros outside the grid)
      auto load_in = [&](int j) {
        const int x0 = j * BS;
        const int slot = (j & (NCH - 1)) * BS;
        if (al_in) {
          constexpr int G = BS / EP;  // 16-byte groups per row and block
#pragma unroll
          for (int i = 0; i < G; ++i) {
            const int p = lane + 32 * i, r = p / G, g = p % G;
            const int yy = t.y0 + r % PY, zz = t.z0 + r / PY;
            const int xx = x0 + EP * g, rem = nx - xx;
            const int bytes = (yy < ny && zz < nz && rem > 0)
                                  ? (rem >= EP ? 16 : rem * (int)sizeof(T)) : 0;
            const T* src = values + (bytes ? ((long long)zz * ny + yy) * nx + xx : 0);
            cpa16(saddr(f_tile + r * RX + slot + EP * g), src, bytes);
          }
        } else {
#pragma unroll
          for (int i = 0; i < BS; ++i) {
            const int p = lane + 32 * i, r = p / BS, c = p % BS;
            const int yy = t.y0 + r % PY, zz = t.z0 + r / PY;
            const int bytes = (yy < ny && zz < nz && x0 + c < nx) ? (int)sizeof(T) : 0;
            const T* src = values + (bytes ? ((long long)zz * ny + yy) * nx + x0 + c : 0);
            if (sizeof(T) == 4) cpa4(saddr(f_tile + r * RX + slot + c), src, bytes);
            else cpa8(saddr(f_tile + r * RX + slot + c), src, bytes);
          }
        }
        cpa_commit();
      };
      // each lane writes its own row's 4 codes of chunk j
      auto flush_out = [&](int j) {
        const int x0 = j * BS;
        if (j < 0 || x0 >= nx || !rv) return;
        const C* src = c_tile + lane * SM::CODE_STRIDE + (j & (NCH - 1)) * BS;
        if (al_out && x0 + BS <= nx) {
#pragma unroll
          for (int q = 0; q < BS * (int)sizeof(C) / 4; ++q)
            reinterpret_cast<unsigned*>(row_out + x0)[q] = reinterpret_cast<const unsigned*>(src)[q];
        } else {
          const int cnt = nx - x0 < BS ? nx - x0 : BS;
          for (int c = 0; c < cnt; ++c) row_out[x0 + c] = src[c];
        }
      };
      // cp.async groups per block, in order: [faces of block b + 1] [input
      // columns of block b + PD]; the prologue leaves the same pattern behind
#pragma unroll
      for (int j = 0; j < PD - 1; ++j) load_in(j);
      F.issue(0);
      load_in(PD - 1);
      cpa_wait<1>();  // inputs 0 .. PD - 2 and faces 0 have landed
      __syncwarp();
      {
        W w[2];
        F.read(0, w);
        F.settle(0, w);
        F.store(0, w);
      }
      T xv[BS], xn[BS];
#pragma unroll
      for (int j = 0; j < BS; ++j)
        lds_t(a_f + (unsigned)sizeof(T) * (unsigned)((j - sig) & (RX - 1)), xv[j]);
      int cp[BS];  // previous block's codes (validated)
#pragma unroll
      for (int j = 0; j < BS; ++j) cp[j] = 0;
#pragma unroll 1
      for (int b = 0; b < nblk; ++b) {
        const int S0 = b * BS;
        const int xb = S0 - sig;  // this lane's column at the block's first step
        sched_jitter(a.jitter, tk, b + 1);
        F.issue(b + 1);
        load_in(b + PD);
        flush_out(b - (WLAST + 2));
        // groups newer than input b + 1: faces and inputs of blocks b + 2 - PD .. b
        cpa_wait<2 * (PD - 1)>();
        __syncwarp();
        const bool edge = !(S0 >= SMAX && S0 + BS <= nx && t.full_rows);
        const Hist3 Hs = H;  // block-start state (replay)
        const unsigned a_fv = a_fval + 8u * (unsigned)((b & 1) * FW);
        double rj[BS];
        int code[BS];
        bool slow = false;
        auto pass = [&](auto edge_c, auto exact_c) {
          constexpr bool EDGE = decltype(edge_c)::value, EXACT = decltype(exact_c)::value;
#pragma unroll
          for (int j = 0; j < BS; ++j) {
            const double pred = H.predict(a_fv, j, la, lb);
            const double x64 = (double)xv[j];
            const double q = __dmul_rn(__dsub_rn(x64, pred), inv);
            const double tq = __dadd_rn(q, M);
            const double kd = __dsub_rn(tq, M);
            // |k| > center - 1 fails the bound test through a negative bound
            const double ebk = fabs(kd) <= lim ? eb : -1.0;
            // the stored value: RNE float32 cast for float32 elements, none for binary64
            const double rq = (double)Elem<T>::round(__dadd_rn(pred, __dmul_rn(kd, two_eb)));
            const bool safe = fabs(__dsub_rn(q, kd)) < guard;
            const bool good = fabs(__dsub_rn(x64, rq)) <= ebk;
            const long long gm = -(long long)good;
            double r = __longlong_as_double((__double_as_longlong(rq) & gm) |
                                            (__double_as_longlong(x64) & ~gm));
            int c = (center + __double2loint(tq)) & (int)gm;
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
              sts_c<C>(a_c + (unsigned)sizeof(C) * (unsigned)((xb - BS + j) & (RX - 1)), cp[j]);
              if (sizeof(C) == 1) {  // (unconditional: inactive points into the dummy bin)
                const bool actp = ghist != nullptr && rv && (unsigned)(xb - BS + j) < (unsigned)nx;
                asm volatile("red.shared.add.u32 [%0], 1;"
                             ::"r"(a_hist + 4u * (actp ? (unsigned)cp[j] : 256u)) : "memory");
              }
              lds_t(a_f + (unsigned)sizeof(T) * (unsigned)((xb + BS + j) & (RX - 1)), xn[j]);
            }
            if (EDGE) r = act ? r : 0.0;
            rj[j] = r;
            code[j] = c;
            H.L = r;
          }
        };
        typedef std::true_type Yes;
        typedef std::false_type No;
        if (edge) pass(Yes(), No());
        else pass(No(), No());
        // the next block's faces have landed (only this block's input group
        // may still be in flight); one vote: replay, or a late face word
        cpa_wait<1>();
        __syncwarp();
        W w[2];
        F.read(b + 1, w);
        const bool miss = F.missing(w);
        if (__any_sync(EBZ_FULL, slow | miss)) {
          if (__any_sync(EBZ_FULL, slow)) {  // replay the block with the exact quantizer
            H = Hs;
            pass(Yes(), Yes());
          }
          F.settle(b + 1, w);
        }
        F.store(b + 1, w);
        faces_out(xb, rj);  // the block is final
#pragma unroll
        for (int j = 0; j < BS; ++j) {
          xv[j] = xn[j];
          cp[j] = code[j];
        }
      }
      cpa_wait<0>();
      __syncwarp();
      if (ghist) {  // the task's counts into the field's histogram
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const unsigned v = whist[lane + 32 * q];
          if (v) atomicAdd(&ghist[lane + 32 * q], (unsigned long long)v);
        }
        __syncwarp();
      }
    } else {
      // ---------------------------------------------------------- decompress
      T* const row_out = reinterpret_cast<T*>(fr.recon) + rowi;
      const C* const row_in = reinterpret_cast<const C*>(fr.codes) + rowi;
      const T* unpred = reinterpret_cast<const T*>(fr.unpred);
      const unsigned long long n_unpred = fr.info->n_unpred;
      const int nchunks = (nx + SMAX + CH - 1) / CH;
      const bool al_in = (nx * (int)sizeof(C)) % 16 == 0;
      const bool al4_in = (nx * (int)sizeof(C)) % 4 == 0;
      const bool al_out = nx % EP == 0;
      const double c52 = 0x1p52 + (double)a.center;
      unsigned long long ucur = 0, ustart = 0;
      if (rv) {
        const long long R = (long long)t.z * ny + t.y;
        ucur = ustart = fr.rowbase[R] + fr.rowblk[R >> 8];
      }
      unsigned hmax = 0;
      // each lane stages its own row's 16 codes of chunk j (zeros past the row)
      auto load_in = [&](int j) {
        const int x0 = j * CH;
        if (x0 >= nx) return;
        C* dst = c_tile + lane * SM::CODE_STRIDE + (j & 3) * CH;
        const int rem = rv ? nx - x0 : 0;
        const int nb = (rem > CH ? CH : (rem > 0 ? rem : 0)) * (int)sizeof(C);
        if (al_in && rem >= CH) {
#pragma unroll
          for (int v = 0; v < CH * (int)sizeof(C) / 16; ++v)
            cpa16(saddr(dst) + 16u * v, reinterpret_cast<const uint4*>(row_in + x0) + v, 16);
        } else if (al4_in) {
#pragma unroll
          for (int q = 0; q < CH * (int)sizeof(C) / 4; ++q) {
            const int b4 = nb - 4 * q >= 4 ? 4 : 0;
            cpa4(saddr(dst) + 4u * q,
                 b4 ? reinterpret_cast<const unsigned char*>(row_in + x0) + 4 * q
                    : reinterpret_cast<const unsigned char*>(fr.codes), b4);
          }
        } else {
          for (int c = 0; c < CH; ++c) dst[c] = c < rem ? row_in[x0 + c] : (C)0;
        }
      };
      auto flush_out = [&](int j) {
        const int x0 = j * CH;
        if (x0 >= nx || !rv) return;
        const int cnt = nx - x0 < CH ? nx - x0 : CH;
        const T* src = f_tile + lane * RX + (j & 3) * CH;
        if (al_out && cnt == CH) {
#pragma unroll
          for (int v = 0; v < CH / EP; ++v)
            reinterpret_cast<uint4*>(row_out + x0)[v] = reinterpret_cast<const uint4*>(src)[v];
        } else {
          for (int c = 0; c < cnt; ++c) row_out[x0 + c] = src[c];
        }
      };
      // codes and verbatim values of the block starting at step S0
      auto fetch = [&](int S0, int (&cd)[BS], T (&vv)[BS]) {
        const int xb = S0 - sig;
#pragma unroll
        for (int j = 0; j < BS; ++j) {
          const bool act = rv && (unsigned)(xb + j) < (unsigned)nx;
          const int c = lds_c<C>(a_c + (unsigned)sizeof(C) * (unsigned)((xb + j) & (RX - 1)));
          cd[j] = act ? c : -1;
          vv[j] = (T)0;
          const unsigned take = act && c == 0;
          const unsigned ok = take && ucur < n_unpred;
          ldg_nc_if(vv[j], unpred + ucur, ok);
          ucur += take;
        }
      };
      // cp.async groups: [faces of block b + 1] at each block start, [codes of
      // chunk k + 1] behind the first block's faces
      load_in(0);
      cpa_commit();
      F.issue(0);
      cpa_wait<0>();
      __syncwarp();
      {
        W w[2];
        F.read(0, w);
        F.settle(0, w);
        F.store(0, w);
      }
      int cd[BS], cdn[BS];
      T vv[BS], vvn[BS];
      fetch(0, cd, vv);
      for (int k = 0; k < nchunks; ++k) {
#pragma unroll 1
        for (int h = 0; h < CH / BS; ++h) {
          const int S0 = k * CH + h * BS;
          const int xb = S0 - sig;
          const int b = S0 / BS;
          sched_jitter(a.jitter, tk, b + 1);
          F.issue(b + 1);
          if (h == 0) {  // the next chunk's codes, behind this block's faces
            load_in(k + 1);
            cpa_commit();
          }
          if (h + 1 == CH / BS) {  // the next block's codes are in the chunk being staged
            cpa_wait<1>();         // (all but the faces just requested)
            __syncwarp();
          }
          fetch(S0 + BS, cdn, vvn);
          const unsigned a_fv = a_fval + 8u * (unsigned)((b & 1) * FW);
          double rj[BS];
#pragma unroll
          for (int j = 0; j < BS; ++j) {
            const bool act = cd[j] >= 0;
            const double qv = __dmul_rn(__dsub_rn(__hiloint2double(0x43300000, cd[j]), c52), two_eb);
            const double pred = H.predict(a_fv, j, la, lb);
            double r = (double)Elem<T>::round(__dadd_rn(pred, qv));
            r = cd[j] == 0 ? (double)vv[j] : r;
            r = act ? r : 0.0;
            hmax = max(hmax, (unsigned)__double2hiint(r) & 0x7fffffffu);
            sts_t(a_f + (unsigned)sizeof(T) * (unsigned)((xb + j) & (RX - 1)), T(), r);
            rj[j] = r;
            H.L = r;
          }
          faces_out(xb, rj);
          if (h == 0) cpa_wait<1>();  // the faces; the chunk's codes may still be in flight
          else cpa_wait<0>();
          __syncwarp();
          {
            W w[2];
            F.read(b + 1, w);
            F.settle(b + 1, w);
            F.store(b + 1, w);
          }
#pragma unroll
          for (int j = 0; j < BS; ++j) {
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
}

template <typename C, typename T, bool COMPRESS>
cudaError_t launch3b_t(const S3bArgs& fa, const FieldTable& ft, int sms, cudaStream_t s) {
  const size_t smem = (size_t)WPB * Sm3b<C, T>::PER_WARP;
  static KernelAttr attr;
  cudaError_t e = kernel_smem(attr, sweep3b_kernel<C, T, COMPRESS>, smem);
  if (e != cudaSuccess) return e;
  const int per_sm = kernel_occupancy(attr, sweep3b_kernel<C, T, COMPRESS>, 32 * WPB, smem);
  const long long ntasks = (long long)fa.npy * fa.npz * fa.nf;
  // as the one-row kernel: about diag * nx / 14 tasks are runnable at once
  const long long diag = fa.npy < fa.npz ? fa.npy : fa.npz;
  long long active = (diag * ((fa.s.dims[0] + 14) / 14 + 1) + 64) * fa.nf;
  if (active > ntasks) active = ntasks;
  long long blocks = (active + WPB - 1) / WPB;
  if (blocks > (long long)sms * per_sm) blocks = (long long)sms * per_sm;
  if (blocks < 1) blocks = 1;
  sweep3b_kernel<C, T, COMPRESS><<<(unsigned)blocks, 32 * WPB, smem, s>>>(fa, ft);
  return cudaGetLastError();
}

template <typename T>
cudaError_t launch3b_w(const S3bArgs& fa, const FieldTable& ft, bool compress, int sms,
                       cudaStream_t s) {
  const bool wide = fa.s.wide != 0;
  if (compress)
    return wide ? launch3b_t<uint16_t, T, true>(fa, ft, sms, s)
                : launch3b_t<uint8_t, T, true>(fa, ft, sms, s);
  return wide ? launch3b_t<uint16_t, T, false>(fa, ft, sms, s)
              : launch3b_t<uint8_t, T, false>(fa, ft, sms, s);
}

}  // namespace

// 3D, n = 1, without the full-reconstruction output (REC) or the truncated
// coding (TR): every binary64 field; EBZ_NO_SWEEP3B keeps the generic kernel
// (A/B, tests)
bool sweep3b_used(int ndim, int layers, int width, const long long* dims, int nf, bool compress,
                  bool rec, bool trunc) {
  if (getenv("EBZ_NO_SWEEP3B")) return false;
  if (!(ndim == 3 && layers == 1 && !rec && !trunc && dims[0] < (1ll << 26))) return false;
  if (width == 64) return true;
  if (width != 32) return false;
  // float32: compress only, where the time model of the three compress
  // kernels picks it (sweep3.cu sweep3_model_choice) -- lone and few fields;
  // its decompress direction measured no faster than the one-row kernel.
  // EBZ_SWEEP3B32 = "c", "d", "cd" or "" forces it per direction (A/B, tests);
  // a forced EBZ_SWEEP3 keeps it out.
  const char* e = getenv("EBZ_SWEEP3B32");
  if (e) return strchr(e, compress ? 'c' : 'd') != nullptr;
  if (!compress || getenv("EBZ_SWEEP3") || getenv("EBZ_NO_SWEEP3")) return false;
  return sweep3_model_choice(dims, nf) == 2;
}

// face buffer sizes in u64 words (two per 16-byte face word)
void sweep3b_face_words(const long long* dims, long long* ny_words, long long* nz_words) {
  const long long npy = (dims[1] + PY - 1) / PY, npz = (dims[2] + PZ - 1) / PZ;
  *ny_words = 2 * npy * npz * (dims[0] + 4) * 4;
  *nz_words = 2 * npy * npz * (dims[0] + 8) * 8;
}

cudaError_t launch_sweep3b(const SweepArgs& a, const FieldTable& ft, int nf,
                           const unsigned int* d_tasks, int npy, int npz, bool compress, int width,
                           int sms, cudaStream_t s) {
  if (nf < 1 || nf > kBatchMax) return cudaErrorInvalidValue;
  S3bArgs fa;
  fa.s = a;
  fa.tasks = d_tasks;
  fa.npy = npy;
  fa.npz = npz;
  fa.nf = nf;
  return width == 64 ? launch3b_w<double>(fa, ft, compress, sms, s)
                     : launch3b_w<float>(fa, ft, compress, sms, s);
}
