// capi.cu -- C ABI (include/ebz200.h): contexts, per-slot workspaces and the
// compress / decompress pipelines (ebzip/codec.py:92-160 restated on device).
//
// compress(slot):   [range+eb] -> sweep(compress, +histogram, +K) ->
//                   huffman build -> encode count -> scan(+header) -> pack
// decompress(slot): init -> decode tables -> sync -> verify -> write
//                   (-> serial if anomalous) -> row zero ranks -> sweep(decompress)
// Everything between the input copy and the output copy is device work; the
// host only sizes buffers and, in the synchronous one-shots, reads EbzInfo.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "ebz_common.cuh"

namespace {

thread_local std::string g_err;

struct Buf {
  void* p = nullptr;
  size_t cap = 0;
  bool ensure(size_t bytes) {
    if (bytes <= cap && p) return true;
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    size_t want = bytes < 256 ? 256 : bytes;
    if (cudaMalloc(&p, want) != cudaSuccess) {
      p = nullptr;
      return false;
    }
    cap = want;
    return true;
  }
  template <typename T> T* as() const { return reinterpret_cast<T*>(p); }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
};

struct Slot {
  long long task_key[5] = {-1, -1, -1, -1, -1};
  Buf tasks, dctrl, rscratch, yface, zface, dyface, dzface;
  long long bank_key[6] = {-1, -1, -1, -1, -1, -1};
  const long long *bk_deltas = nullptr, *bk_starts = nullptr, *bk_counts = nullptr;
  const double* bk_coeffs = nullptr;
  Buf info, values, codes, recon, hist, head, bits, unpred, agg, progress, ctrl, huff, lengths,
      words, bank;
  // decompress side
  Buf dinfo, dbits, dunpred, dscratch, rowbase, rowtmp, drecon, dlengths, dcodes, dprogress;
  // geometry of the last compress held in this slot
  int width = 32, ndim = 0, layers = 1, m = 8;
  long long dims[4] = {1, 1, 1, 1};
  long long n = 0;
  bool have = false;
  bool hist_done = false;  // the last compress sweep also filled `hist`
  const void* trial_values = nullptr;  // device input of an interval trial (finish)
  int trunc = 0;                       // compress: truncated-mantissa unpredictables (opt-in)
  bool trial = false;                  // holds u16 trial codes, back end not run
  // epoch generation the tagged buffers (faces, progress counters) were
  // last zeroed for: [0] compress, [1] decompress
  unsigned int tag_gen[2] = {0, 0};
  // bytes per face word the buffers last held (8: tagged words of the
  // float32 kernels, 16: {value, epoch} words): a change re-zeroes them, so
  // no stale value bits can pose as a current tag
  int face_width[2] = {0, 0};
  ~Slot() {
    Buf* all[] = {&info, &values, &codes, &recon, &hist, &head, &bits, &unpred, &agg, &progress,
                  &ctrl, &huff, &lengths, &words, &bank, &dinfo, &dbits, &dunpred, &dscratch,
                  &rowbase, &rowtmp, &drecon, &dlengths, &dcodes, &dprogress};
    for (Buf* b : all) b->release();
    tasks.release();
    dctrl.release();
    rscratch.release();
    yface.release();
    zface.release();
    dyface.release();
    dzface.release();
  }
};

}  // namespace

struct EbzCtx {
  int device = 0;
  int sms = 148;
  std::string name;
  std::map<int, Slot*> slots;
  Buf range_scratch;
  Buf an_scratch, an_out;  // analysis entry points
  // launch epochs tag face words and progress counters, in [1, kEpochMax];
  // when the counter wraps the generation advances and each slot re-zeroes
  // its tagged buffers before its next launch, so no stale word can match
  unsigned int epoch = 0, epoch_gen = 0;
  unsigned long long launches = 0;
  std::mutex mu;
  std::mutex an_mu;  // analysis scratch
  std::mutex seam_mu;  // host-buffer seam entry points (private slot)
  bool force_generic = getenv("EBZ_FORCE_GENERIC") != nullptr;
  // in-stream stage timing (CUDA events on the launching stream)
  struct Mark {
    cudaEvent_t a, b;
    int stage;
  };
  bool profiling = false;
  std::vector<Mark> marks;
  std::vector<cudaEvent_t> pool;
  cudaEvent_t take_event() {
    if (!pool.empty()) {
      cudaEvent_t e = pool.back();
      pool.pop_back();
      return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
  }
  int begin(int stage, cudaStream_t s) {
    if (!profiling) return -1;
    std::lock_guard<std::mutex> g(mu);
    Mark mk{take_event(), take_event(), stage};
    cudaEventRecord(mk.a, s);
    marks.push_back(mk);
    return (int)marks.size() - 1;
  }
  void end(int idx, cudaStream_t s) {
    if (idx < 0) return;
    std::lock_guard<std::mutex> g(mu);
    cudaEventRecord(marks[idx].b, s);
  }
  Slot& slot(int i) {
    std::lock_guard<std::mutex> g(mu);
    auto it = slots.find(i);
    if (it != slots.end()) return *it->second;
    Slot* sl = new Slot();
    slots[i] = sl;
    return *sl;
  }
  unsigned int next_epoch(unsigned int* gen) {
    std::lock_guard<std::mutex> g(mu);
    if (++epoch > kEpochMax) {
      epoch = 1;
      ++epoch_gen;
    }
    *gen = epoch_gen;
    return epoch;
  }
};

namespace {

#define EBZ_CUDA(x)                                                                     \
  do {                                                                                  \
    cudaError_t e__ = (x);                                                              \
    if (e__ != cudaSuccess) {                                                           \
      g_err = std::string(#x) + ": " + cudaGetErrorString(e__);                          \
      return EBZ_E_CUDA;                                                                \
    }                                                                                   \
  } while (0)

#define EBZ_ALLOC(buf, bytes)                                                           \
  do {                                                                                  \
    if (!(buf).ensure(bytes)) {                                                         \
      g_err = "cudaMalloc failed (" + std::to_string((size_t)(bytes)) + " bytes)";      \
      return EBZ_E_OOM;                                                                 \
    }                                                                                   \
  } while (0)

bool check_geom(int width, int ndim, const uint64_t* dims, int layers, int m, long long& n) {
  if (width != 32 && width != 64) { g_err = "width must be 32 or 64"; return false; }
  if (ndim < 1 || ndim > 4) { g_err = "ndim must be 1..4"; return false; }
  if (layers < 1 || layers > 255) { g_err = "layers must be 1..255"; return false; }
  if (m < 2 || m > 16) { g_err = "interval exponent must be 2..16"; return false; }
  n = 1;
  for (int a = 0; a < ndim; ++a) {
    if (dims[a] < 1) { g_err = "dims must be positive"; return false; }
    n *= (long long)dims[a];
  }
  return true;
}

// Stencil bank (ebzip/codec.py:54-89): for each non-empty axis mask and each
// effective layer count, the offsets of build_stencil (predictor.py:41-56) in
// itertools.product order, flattened with the scan strides.
struct Bank {
  std::vector<long long> deltas, starts, counts;
  std::vector<double> coeffs;
};

long long choose(int n, int k) {
  long long r = 1;
  for (int i = 1; i <= k; ++i) r = r * (n - k + i) / i;
  return r;
}

Bank make_bank(int ndim, const long long* dims, int layers) {
  Bank b;
  long long stride[4] = {1, 1, 1, 1};
  for (int a = 1; a < ndim; ++a) stride[a] = stride[a - 1] * dims[a - 1];
  const int nslot = ((1 << ndim) - 1) * layers;
  b.starts.assign(nslot, 0);
  b.counts.assign(nslot, 0);
  for (int mask = 1; mask < (1 << ndim); ++mask) {
    int act[4], na = 0;
    for (int a = 0; a < ndim; ++a)
      if ((mask >> a) & 1) act[na++] = a;
    for (int eff = 1; eff <= layers; ++eff) {
      const int slot = (mask - 1) * layers + (eff - 1);
      b.starts[slot] = (long long)b.deltas.size();
      std::vector<int> off(na, 0);
      for (;;) {
        int q = na - 1;  // last position varies fastest
        while (q >= 0 && ++off[q] > eff) off[q--] = 0;
        if (q < 0) break;
        long long coef = 1, delta = 0;
        for (int r = 0; r < na; ++r) {
          const long long c = choose(eff, off[r]);
          coef *= (off[r] & 1) ? -c : c;
          delta += (long long)off[r] * stride[act[r]];
        }
        b.deltas.push_back(delta);
        b.coeffs.push_back((double)(-coef));
      }
      b.counts[slot] = (long long)b.deltas.size() - b.starts[slot];
    }
  }
  return b;
}

// Upload the bank into slot.bank (layout: deltas | coeffs | starts | counts)
int upload_bank(Slot& sl, int ndim, const long long* dims, int layers, cudaStream_t s,
                const long long** d_deltas, const double** d_coeffs, const long long** d_starts,
                const long long** d_counts) {
  const long long key[6] = {ndim, dims[0], dims[1], dims[2], dims[3], layers};
  if (memcmp(key, sl.bank_key, sizeof(key)) == 0) {
    *d_deltas = sl.bk_deltas;
    *d_coeffs = sl.bk_coeffs;
    *d_starts = sl.bk_starts;
    *d_counts = sl.bk_counts;
    return EBZ_OK;
  }
  Bank b = make_bank(ndim, dims, layers);
  const size_t nt = b.deltas.size() ? b.deltas.size() : 1, ns = b.starts.size();
  std::vector<char> host(8 * (2 * nt + 2 * ns));
  char* p = host.data();
  memcpy(p, b.deltas.data(), 8 * b.deltas.size());
  memcpy(p + 8 * nt, b.coeffs.data(), 8 * b.coeffs.size());
  memcpy(p + 16 * nt, b.starts.data(), 8 * ns);
  memcpy(p + 16 * nt + 8 * ns, b.counts.data(), 8 * ns);
  EBZ_ALLOC(sl.bank, host.size());
  // pageable source: staged before the call returns, so `host` may go away
  EBZ_CUDA(cudaMemcpyAsync(sl.bank.p, host.data(), host.size(), cudaMemcpyHostToDevice, s));
  char* d = sl.bank.as<char>();
  sl.bk_deltas = *d_deltas = reinterpret_cast<const long long*>(d);
  sl.bk_coeffs = *d_coeffs = reinterpret_cast<const double*>(d + 8 * nt);
  sl.bk_starts = *d_starts = reinterpret_cast<const long long*>(d + 16 * nt);
  sl.bk_counts = *d_counts = reinterpret_cast<const long long*>(d + 16 * nt + 8 * ns);
  memcpy(sl.bank_key, key, sizeof(key));
  return EBZ_OK;
}


// One field of a sweep launch.
struct FieldIO {
  Slot* sl;
  Info* info;
  const void* values;
  void* recon;
  void* codes;
  const void* unpred;
  const unsigned long long* rowbase;
  const unsigned long long* rowblk;
  unsigned long long* hist;  // compress: zeroed code histogram the sweep may fill
  int center;                // compress: this field's 2^(m-1) (interval trials), 0 = m's
};

// Predict/quantize (or reconstruct) sweep over nf fields of one geometry.
// Fast path: one persistent launch per kBatchMax fields (tickets interleave
// the fields, so every warp always has independent work); generic path: one
// launch per field.
int sweep_run(EbzCtx* ctx, bool compress, int width, int ndim, const long long* dims, int layers,
              int m, const FieldIO* fs, int nf, cudaStream_t s, bool force_wide = false) {
  SweepArgs a;
  memset(&a, 0, sizeof(a));
  a.ndim = ndim;
  a.n = 1;
  for (int i = 0; i < 4; ++i) a.dims[i] = i < ndim ? dims[i] : 1;
  for (int i = 0; i < ndim; ++i) a.n *= dims[i];
  a.nrows = a.n / a.dims[0];
  a.layers = layers;
  a.m = m;
  a.center = 1 << (m - 1);
  a.wide = m > 8 || force_wide;
  a.trunc = compress && nf > 0 && fs[0].sl && fs[0].sl->trunc;
  {  // test hook: schedule perturbation of the wavefront kernels (ns)
    static const unsigned jit = [] {
      const char* e = getenv("EBZ_SCHED_JITTER");
      return e ? (unsigned)atoi(e) : 0u;
    }();
    a.jitter = jit;
  }
  // compress: a field with a recon pointer also receives the full
  // reconstruction (compress_scan's recon output, the C seam); one geometry
  // and one kernel per launch, so the first field decides for the batch
  const bool rec = compress && fs[0].recon != nullptr;
  // binary64 elements have one fast kernel: the 2D block-speculative sweep
  const bool s2 = !ctx->force_generic && sweep2_used(ndim, layers, width, a.dims, rec, a.trunc != 0);
  // ... and the 3D n = 1 patch wavefront with 16-byte face words
  const bool s3b = !ctx->force_generic && sweep3b_used(ndim, layers, width, a.dims, nf, compress, rec, a.trunc != 0);
  bool fast = (width == 32 || s2 || s3b) && !ctx->force_generic &&
              sweep_fast_supported(ndim, layers, a.dims[0]);
  // 3D, n = 1 compress: the z-rows-per-lane kernel (sweep3.cu, 64-bit face offsets)
  const bool s3 = fast && !s3b && sweep3_used(ndim, layers, width, a.dims, nf, compress);
  long long wy = 0, wz = 0;
  if (s3) {
    sweep3_face_words(a.dims, &wy, &wz);
  } else if (s3b) {
    sweep3b_face_words(a.dims, &wy, &wz);
  } else if (fast) {
    // the fast kernel addresses face buffers with 32-bit word offsets
    fast_face_words(ndim, a.dims, layers, compress, &wy, &wz);
    if (width == 64) wy *= 2;  // 16-byte face words {value, epoch} (sweep2.cu)
    fast = wy < (1ll << 31) && wz < (1ll << 31);
  }
  const int mk = ctx->begin(compress ? 1 : 6, s);
  if (fast) {
    int npy = 0, npz = 0;
    if (s3) sweep3_patch_grid(a.dims, &npy, &npz);
    else if (s3b) {  // 8 x 4 row patches in both directions
      npy = (int)((a.dims[1] + 7) / 8);
      npz = (int)((a.dims[2] + 3) / 4);
    }
    else fast_patch_grid(ndim, a.dims, layers, compress, &npy, &npz);
    const size_t by = (size_t)(wy > 0 ? wy : 1) * 8, bz = (size_t)(wz > 0 ? wz : 1) * 8;
    for (int i = 0; i < nf; ++i) {
      // tagged face buffers: fresh memory is zeroed so no word can carry a
      // live epoch tag; afterwards every launch uses a new epoch
      Buf& fy = compress ? fs[i].sl->yface : fs[i].sl->dyface;
      Buf& fz = compress ? fs[i].sl->zface : fs[i].sl->dzface;
      int& fw = fs[i].sl->face_width[compress ? 0 : 1];
      const int fmt = (s3b || width == 64) ? 16 : 8;  // bytes per face word
      const bool sw = fw != 0 && fw != fmt;  // the buffers held the other word format
      fw = fmt;
      const bool gy = by > fy.cap || !fy.p || sw, gz = bz > fz.cap || !fz.p || sw;
      EBZ_ALLOC(fy, by);
      EBZ_ALLOC(fz, bz);
      if (gy) EBZ_CUDA(cudaMemsetAsync(fy.p, 0, fy.cap, s));
      if (gz) EBZ_CUDA(cudaMemsetAsync(fz.p, 0, fz.cap, s));
    }
    Slot& lead = *fs[0].sl;
    // the patch grid depends on the kernel (3D, n = 1 compress: 8 x 8 patches)
    const long long kind = ndim + 16ll * layers +
                           (s3 ? 8192 : s3b ? 16384 : (sweep_r2_used(ndim, layers, compress) ? 4096 : 0));
    const long long key[5] = {kind, a.dims[0], a.dims[1], a.dims[2], a.dims[3]};
    if (memcmp(key, lead.task_key, sizeof(key)) != 0) {
      std::vector<unsigned int> t((size_t)npy * npz);
      // sweep3: a consumer trails its Y producer by ~36 steps, its Z producer
      // by ~9 (sweep3.cu); the other kernels trail both by similar amounts
      if (s3) {
        static int w3[2] = {0, 0};  // EBZ_S3_W="wy,wz": A/B of the ticket order
        if (!w3[0]) {
          const char* e = getenv("EBZ_S3_W");
          if (!e || sscanf(e, "%d,%d", &w3[0], &w3[1]) != 2 || w3[0] < 1 || w3[1] < 1) {
            w3[0] = 4;
            w3[1] = 1;
          }
        }
        fast_task_table(npy, npz, t.data(), w3[0], w3[1]);
      }
      else fast_task_table(npy, npz, t.data(), 1, 1);
      EBZ_ALLOC(lead.tasks, t.size() * 4);
      EBZ_CUDA(cudaMemcpyAsync(lead.tasks.p, t.data(), t.size() * 4, cudaMemcpyHostToDevice, s));
      memcpy(lead.task_key, key, sizeof(key));
    }
    Buf& ctrl = compress ? lead.ctrl : lead.dctrl;
    EBZ_ALLOC(ctrl, 256);
    a.ticket = ctrl.as<unsigned int>();
    FieldTable ft;
    for (int c0 = 0; c0 < nf; c0 += kBatchMax) {
      const int nb = nf - c0 < kBatchMax ? nf - c0 : kBatchMax;
      memset(&ft, 0, sizeof(ft));
      for (int i = 0; i < nb; ++i) {
        const FieldIO& f = fs[c0 + i];
        FieldRef& r = ft.f[i];
        r.values = f.values;
        r.recon = f.recon;
        r.codes = f.codes;
        r.unpred = f.unpred;
        r.rowbase = f.rowbase;
        r.rowblk = f.rowblk;
        r.hist = f.hist;
        ft.center[i] = f.center;
        r.yface = (compress ? f.sl->yface : f.sl->dyface).as<unsigned long long>();
        r.zface = (compress ? f.sl->zface : f.sl->dzface).as<unsigned long long>();
        r.info = f.info;
      }
      unsigned int gen;
      a.epoch = ctx->next_epoch(&gen);
      for (int i = 0; i < nb; ++i) {
        Slot& sl = *fs[c0 + i].sl;
        unsigned int& g = sl.tag_gen[compress ? 0 : 1];
        if (g == gen) continue;
        Buf& fy = compress ? sl.yface : sl.dyface;
        Buf& fz = compress ? sl.zface : sl.dzface;
        EBZ_CUDA(cudaMemsetAsync(fy.p, 0, fy.cap, s));
        EBZ_CUDA(cudaMemsetAsync(fz.p, 0, fz.cap, s));
        g = gen;
      }
      EBZ_CUDA(cudaMemsetAsync(ctrl.p, 0, 256, s));
      if (s3)
        EBZ_CUDA(launch_sweep3(a, ft, nb, lead.tasks.as<unsigned int>(), npy, npz, compress, rec,
                               ctx->sms, s));
      else if (s3b)
        EBZ_CUDA(launch_sweep3b(a, ft, nb, lead.tasks.as<unsigned int>(), npy, npz, compress,
                                width, ctx->sms, s));
      else if (s2)
        EBZ_CUDA(launch_sweep2(a, ft, nb, lead.tasks.as<unsigned int>(), npy, compress, width,
                               ctx->sms, s));
      else
        EBZ_CUDA(launch_sweep_fast(a, ft, nb, lead.tasks.as<unsigned int>(), npy, npz,
                                   compress, rec, ctx->sms, s));
      ctx->launches += 1;
    }
  } else {
    long long ntasks = (a.nrows + 31) / 32 + 64;
    for (int i = 0; i < nf; ++i) {
      const FieldIO& f = fs[i];
      Slot& sl = *f.sl;
      Buf& progress = compress ? sl.progress : sl.dprogress;
      // epoch-tagged counters: fresh memory must start below every epoch tag
      const size_t want = (size_t)ntasks * 8 * kProgPad;
      const bool grow = want > progress.cap || !progress.p;
      EBZ_ALLOC(progress, want);
      if (grow) EBZ_CUDA(cudaMemsetAsync(progress.p, 0, progress.cap, s));
      Buf& ctrl = compress ? sl.ctrl : sl.dctrl;
      EBZ_ALLOC(ctrl, 256);
      a.info = f.info;
      a.info_w = f.info;
      a.center = f.center ? f.center : 1 << (m - 1);
      a.values = f.values;
      a.recon = f.recon;
      if (compress && !a.recon) {
        // the generic kernel predicts from its own stored reconstruction:
        // per-slot scratch when the caller does not want it
        EBZ_ALLOC(sl.recon, (size_t)a.n * (size_t)(width / 8));
        a.recon = sl.recon.p;
      }
      a.codes = f.codes;
      a.hist = nullptr;
      a.unpred = f.unpred;
      a.rowbase = f.rowbase;
      a.rowblk = f.rowblk;
      a.progress = progress.as<unsigned long long>();
      a.ticket = ctrl.as<unsigned int>();
      unsigned int gen;
      a.epoch = ctx->next_epoch(&gen);
      if (sl.tag_gen[compress ? 0 : 1] != gen) {
        EBZ_CUDA(cudaMemsetAsync(progress.p, 0, progress.cap, s));
        sl.tag_gen[compress ? 0 : 1] = gen;
      }
      EBZ_CUDA(cudaMemsetAsync(ctrl.p, 0, 256, s));
      int rc = upload_bank(sl, ndim, a.dims, layers, s, &a.deltas, &a.coeffs, &a.starts, &a.counts);
      if (rc) return rc;
      EBZ_CUDA(launch_sweep_generic(a, width, compress, ctx->sms, s));
      ctx->launches += 1;
    }
  }
  // the two-row compress kernel also histograms u8 codes (sweep_fast.cu)
  // ... as does the 16-byte-face one-row kernel (sweep3b.cu), for either element width
  const bool fused = compress && fast && !a.wide &&
                     (s3b || (width == 32 && (s3 || sweep_r2_used(ndim, layers, compress))));
  for (int i = 0; i < nf; ++i) fs[i].sl->hist_done = fused && fs[i].hist != nullptr;
  ctx->end(mk, s);
  return EBZ_OK;
}

// compress, preparation: buffers, input staging, record reset.  Records the
// geometry in the slot.
int compress_prep(EbzCtx* ctx, int slot, const void* values, int on_host, int width, int ndim,
                  const uint64_t* dims, int layers, int m, int has_abs, int has_rel,
                  cudaStream_t s, const void** d_values_out) {
  long long n;
  if (!check_geom(width, ndim, dims, layers, m, n)) return EBZ_E_ARG;
  if (!has_abs && !has_rel) { g_err = "no bound"; return EBZ_E_ARG; }
  Slot& sl = ctx->slot(slot);
  const size_t ew = (size_t)width / 8;
  const size_t cw = m > 8 ? 2 : 1;
  const long long nsym = 1ll << m;
  const long long nchunks = (n + kEncodeChunk - 1) / kEncodeChunk;
  EBZ_ALLOC(sl.info, sizeof(Info));
  EBZ_ALLOC(sl.codes, (size_t)n * cw + 64);
  EBZ_ALLOC(sl.hist, (size_t)nsym * 8);
  EBZ_ALLOC(sl.head, 36 + 8 * 4 + (size_t)nsym);
  // code stream capacity: generous first guess, regrown on ST_CAPACITY
  size_t bits_cap = (size_t)n * 2 + 4096;
  if (sl.bits.cap > bits_cap) bits_cap = sl.bits.cap;
  EBZ_ALLOC(sl.bits, bits_cap);
  EBZ_ALLOC(sl.unpred, (size_t)n * ew);
  EBZ_ALLOC(sl.agg, (size_t)nchunks * 16);
  EBZ_ALLOC(sl.huff, huffman_scratch_bytes(m));
  EBZ_ALLOC(sl.lengths, (size_t)nsym);
  EBZ_ALLOC(sl.words, (size_t)nsym * 8);
  if (!sl.rscratch.p) {
    // per-slot partials + completion counter (zeroed once, self re-arming)
    EBZ_ALLOC(sl.rscratch, 1184 * 24 + 256);
    EBZ_CUDA(cudaMemsetAsync(sl.rscratch.p, 0, sl.rscratch.cap, s));
  }
  const void* d_values = values;
  if (on_host) {
    EBZ_ALLOC(sl.values, (size_t)n * ew);
    EBZ_CUDA(cudaMemcpyAsync(sl.values.p, values, (size_t)n * ew, cudaMemcpyHostToDevice, s));
    d_values = sl.values.p;
  }
  // the record and the histogram are initialised by the range stage
  sl.width = width;
  sl.ndim = ndim;
  sl.layers = layers;
  sl.m = m;
  for (int a = 0; a < 4; ++a) sl.dims[a] = a < ndim ? (long long)dims[a] : 1;
  sl.n = n;
  sl.have = false;
  sl.trunc = 0;
  *d_values_out = d_values;
  return EBZ_OK;
}

// value range + effective bound (core.py:132-178) of nf prepared slots, one
// launch per kBatchMax fields
int compress_range(EbzCtx* ctx, Slot* const* sls, const void* const* d_values, int nf,
                   int on_host, int has_abs, double abs_bound, int has_rel, double rel_bound,
                   cudaStream_t s) {
  const int mk = ctx->begin(0, s);
  const Slot& s0 = *sls[0];
  for (int c0 = 0; c0 < nf; c0 += kBatchMax) {
    const int nb = nf - c0 < kBatchMax ? nf - c0 : kBatchMax;
    const void* vals[kBatchMax];
    Info* infos[kBatchMax];
    unsigned int* scr[kBatchMax];
    unsigned long long* hists[kBatchMax];
    for (int i = 0; i < nb; ++i) {
      vals[i] = d_values[c0 + i];
      infos[i] = sls[c0 + i]->info.as<Info>();
      scr[i] = sls[c0 + i]->rscratch.as<unsigned int>();
      hists[i] = sls[c0 + i]->hist.as<unsigned long long>();
    }
    EBZ_CUDA(launch_range_batch(vals, infos, scr, hists, 1 << s0.m, nb, s0.width, s0.n, has_abs,
                                abs_bound, has_rel, rel_bound, s));
    ctx->launches += 1;
    if (!on_host && !has_rel)  // device-resident inputs: finiteness (core.py:92-93)
      for (int i = 0; i < nb; ++i) {
        EBZ_CUDA(launch_finite(vals[i], s0.width, s0.n, infos[i], s));
        ctx->launches += 1;
      }
  }
  ctx->end(mk, s);
  return EBZ_OK;
}

FieldIO compress_io(Slot& sl, const void* d_values) {
  FieldIO f;
  memset(&f, 0, sizeof(f));
  f.sl = &sl;
  f.info = sl.info.as<Info>();
  f.values = d_values;
  f.recon = nullptr;  // the pipeline does not keep the compressor's reconstruction
  f.codes = sl.codes.p;
  f.hist = sl.hist.as<unsigned long long>();  // zeroed by the range stage
  return f;
}

EncodeJob encode_job(Slot& sl, const void* d_values) {
  EncodeJob j;
  j.codes = sl.codes.p;
  j.lengths = sl.lengths.as<uint8_t>();
  j.words = sl.words.as<unsigned long long>();
  j.agg = sl.agg.as<unsigned long long>();
  j.info = sl.info.as<Info>();
  j.bits = sl.bits.as<uint8_t>();
  j.bits_cap = sl.bits.cap;
  j.head = sl.head.as<uint8_t>();
  j.values = d_values;
  j.unpred = sl.unpred.p;
  j.trunc = sl.trunc;
  return j;
}

// compress, second half over nf swept slots: histogram (codec.py:107),
// codebooks, encode -- one launch per stage per kBatchMax fields
int compress_back(EbzCtx* ctx, Slot* const* sls, const void* const* d_values, int nf,
                  cudaStream_t s) {
  const Slot& s0 = *sls[0];
  for (int c0 = 0; c0 < nf; c0 += kBatchMax) {
    const int nb = nf - c0 < kBatchMax ? nf - c0 : kBatchMax;
    const void* codes[kBatchMax];
    unsigned long long* hist[kBatchMax];
    Info* info[kBatchMax];
    uint8_t* lens[kBatchMax];
    unsigned long long* words[kBatchMax];
    unsigned long long* scr[kBatchMax];
    EncodeJob jobs[kBatchMax];
    for (int i = 0; i < nb; ++i) {
      Slot& sl = *sls[c0 + i];
      codes[i] = sl.codes.p;
      hist[i] = sl.hist.as<unsigned long long>();
      info[i] = sl.info.as<Info>();
      lens[i] = sl.lengths.as<uint8_t>();
      words[i] = sl.words.as<unsigned long long>();
      scr[i] = sl.huff.as<unsigned long long>();
      jobs[i] = encode_job(sl, d_values[c0 + i]);
    }
    int mk = ctx->begin(2, s);
    // (the fused sweep filled the histograms of every field of the batch:
    // one geometry, one kernel)
    if (!sls[c0]->hist_done) {
      EBZ_CUDA(launch_code_hist_batch(codes, hist, nb, s0.m, s0.n, ctx->sms, s));
      ctx->launches += 1;
    }
    EBZ_CUDA(launch_huffman_batch(hist, info, lens, words, scr, nb, s0.m, s));
    ctx->launches += 1;
    ctx->end(mk, s);
    mk = ctx->begin(3, s);
    EBZ_CUDA(launch_encode_batch(jobs, nb, s0.m, s0.n, s0.width, s0.ndim, s0.dims, s0.layers,
                                 ctx->sms, s));
    ctx->launches += 3;
    ctx->end(mk, s);
  }
  for (int i = 0; i < nf; ++i) sls[i]->have = true;
  return EBZ_OK;
}

int compress_enqueue(EbzCtx* ctx, int slot, const void* values, int on_host, int width, int ndim,
                     const uint64_t* dims, int layers, int m, int has_abs, double abs_bound,
                     int has_rel, double rel_bound, cudaStream_t s, int flags = 0) {
  const void* d_values = nullptr;
  int rc = compress_prep(ctx, slot, values, on_host, width, ndim, dims, layers, m, has_abs,
                         has_rel, s, &d_values);
  if (rc) return rc;
  Slot* sl = &ctx->slot(slot);
  sl->trunc = (flags & EBZ_FLAG_TRUNCATE) ? 1 : 0;
  rc = compress_range(ctx, &sl, &d_values, 1, on_host, has_abs, abs_bound, has_rel, rel_bound, s);
  if (rc) return rc;
  const FieldIO f = compress_io(*sl, d_values);
  rc = sweep_run(ctx, true, width, ndim, sl->dims, layers, m, &f, 1, s);
  if (rc) return rc;
  return compress_back(ctx, &sl, &d_values, 1, s);
}

// regrow the code buffer and re-run the encoder (rare: > 16 bits/value)
int compress_regrow(EbzCtx* ctx, Slot& sl, const void* d_values, unsigned long long need_bits,
                    cudaStream_t s) {
  sl.bits.release();
  EBZ_ALLOC(sl.bits, (size_t)(need_bits / 8) + 4096);
  Info* info = sl.info.as<Info>();
  // clear the capacity bit, recount, rescan, repack
  int st = 0;
  EBZ_CUDA(cudaMemcpyAsync(&st, &info->status, sizeof(int), cudaMemcpyDeviceToHost, s));
  EBZ_CUDA(cudaStreamSynchronize(s));
  st &= ~ST_CAPACITY;
  EBZ_CUDA(cudaMemcpyAsync(&info->status, &st, sizeof(int), cudaMemcpyHostToDevice, s));
  EBZ_CUDA(cudaStreamSynchronize(s));
  const EncodeJob j = encode_job(sl, d_values);
  EBZ_CUDA(launch_encode_batch(&j, 1, sl.m, sl.n, sl.width, sl.ndim, sl.dims, sl.layers,
                               ctx->sms, s));
  ctx->launches += 3;
  return EBZ_OK;
}

// decompress, first half: decode (entropy.py:160-183) + row zero ranks.
// Fills *io for the reconstruction sweep.
// One field's decompress inputs (device pointers).  eb / K come from the
// source compress record when src is set (device-resident round trip: the
// byte budget is then ceil(src->bit_length / 8), read on the device and
// nbytes is only a capacity), else from the host values.
struct DecIn {
  const Info* src;
  double eb;
  unsigned long long k;
  const uint8_t* lengths;
  const uint8_t* bits;
  unsigned long long nbytes;
  const void* unpred;
  void* recon;
};

// decompress, first half over nf fields: decode (entropy.py:160-183) + row
// zero ranks, one launch per stage per kBatchMax fields.  Fills io[] for the
// reconstruction sweep.
int decompress_front(EbzCtx* ctx, Slot* const* sls, const DecIn* in, int nf, int ndim,
                     const long long* dims, int m, cudaStream_t s, FieldIO* io) {
  long long n = 1;
  for (int a = 0; a < ndim; ++a) n *= dims[a];
  const size_t cw = m > 8 ? 2 : 1;
  const long long nrows = n / dims[0];
  for (int i = 0; i < nf; ++i) {
    Slot& sl = *sls[i];
    EBZ_ALLOC(sl.dinfo, sizeof(Info));
    EBZ_ALLOC(sl.dcodes, (size_t)n * cw + 64);
    EBZ_ALLOC(sl.dscratch, decode_scratch_bytes((long long)in[i].nbytes, m));
    EBZ_ALLOC(sl.rowbase, (size_t)nrows * 8);
    EBZ_ALLOC(sl.rowtmp, rowblk_words(nrows) * 8);
  }
  for (int c0 = 0; c0 < nf; c0 += kBatchMax) {
    const int nb = nf - c0 < kBatchMax ? nf - c0 : kBatchMax;
    DecodeJob jobs[kBatchMax];
    const void* codes[kBatchMax];
    unsigned long long* rb[kBatchMax];
    unsigned long long* rk[kBatchMax];
    Info* infos[kBatchMax];
    for (int i = 0; i < nb; ++i) {
      Slot& sl = *sls[c0 + i];
      const DecIn& d = in[c0 + i];
      DecodeJob& j = jobs[i];
      j.bits = d.bits;
      j.nbytes = (long long)d.nbytes;
      j.lengths = d.lengths;
      j.codes = sl.dcodes.p;
      j.info = sl.dinfo.as<Info>();
      j.scratch = sl.dscratch.as<unsigned long long>();
      j.dev_bitlen = d.src ? &d.src->bit_length : nullptr;
      j.src = d.src;
      j.eb = d.eb;
      j.k = d.k;
      codes[i] = sl.dcodes.p;
      rb[i] = sl.rowbase.as<unsigned long long>();
      rk[i] = sl.rowtmp.as<unsigned long long>();
      infos[i] = sl.dinfo.as<Info>();
    }
    int mk = ctx->begin(4, s);
    EBZ_CUDA(launch_decode_batch(jobs, nb, m, n, ctx->sms, s));
    ctx->end(mk, s);
    mk = ctx->begin(5, s);
    EBZ_CUDA(launch_rowbase_batch(codes, rb, rk, infos, nb, m, n, dims[0], s));
    ctx->end(mk, s);
    ctx->launches += 12;  // init, tables, sync, 2 repairs, verify, top, write, serial, 2 ranks
  }
  for (int i = 0; i < nf; ++i) {
    Slot& sl = *sls[i];
    FieldIO& f = io[i];
    memset(&f, 0, sizeof(f));
    f.sl = &sl;
    f.info = sl.dinfo.as<Info>();
    f.recon = in[i].recon;
    f.codes = sl.dcodes.p;
    f.unpred = in[i].unpred;
    f.rowbase = sl.rowbase.as<unsigned long long>();
    f.rowblk = sl.rowtmp.as<unsigned long long>();
  }
  return EBZ_OK;
}

int decompress_enqueue(EbzCtx* ctx, Slot& sl, int width, int ndim, const long long* dims,
                       int layers, int m, const Info* src_info, double eb, unsigned long long k,
                       const uint8_t* d_lengths, const uint8_t* d_bits, unsigned long long nbytes,
                       const void* d_unpred, void* d_recon, cudaStream_t s) {
  FieldIO io;
  Slot* sp = &sl;
  const DecIn d{src_info, eb, k, d_lengths, d_bits, nbytes, d_unpred, d_recon};
  int rc = decompress_front(ctx, &sp, &d, 1, ndim, dims, m, s, &io);
  if (rc) return rc;
  return sweep_run(ctx, false, width, ndim, dims, layers, m, &io, 1, s);
}

}  // namespace

// ============================================================== C ABI ======
extern "C" {

int ebz_abi_version(void) { return EBZ_ABI_VERSION; }

const char* ebz_last_error(void) { return g_err.c_str(); }

EbzCtx* ebz_ctx_create(int device) {
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count <= device) {
    g_err = "no CUDA device";
    return nullptr;
  }
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) {
    g_err = "cudaGetDeviceProperties failed";
    return nullptr;
  }
  if (prop.major != 10) {
    g_err = "libebz200 is built for sm_100a (B200); device is sm_" +
            std::to_string(prop.major) + std::to_string(prop.minor);
    return nullptr;
  }
  if (cudaSetDevice(device) != cudaSuccess) {
    g_err = "cudaSetDevice failed";
    return nullptr;
  }
  EbzCtx* c = new EbzCtx();
  c->device = device;
  c->sms = prop.multiProcessorCount;
  c->name = prop.name;
  return c;
}

void ebz_ctx_destroy(EbzCtx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  for (auto& kv : ctx->slots) delete kv.second;
  ctx->range_scratch.release();
  ctx->an_scratch.release();
  ctx->an_out.release();
  delete ctx;
}

int ebz_ctx_trim(EbzCtx* ctx) {
  if (!ctx) return EBZ_E_ARG;
  cudaSetDevice(ctx->device);
  EBZ_CUDA(cudaDeviceSynchronize());
  std::lock_guard<std::mutex> g(ctx->mu);
  for (auto& kv : ctx->slots) delete kv.second;
  ctx->slots.clear();
  ctx->range_scratch.release();
  ctx->an_scratch.release();
  ctx->an_out.release();
  return EBZ_OK;
}

int ebz_device_info(EbzCtx* ctx, int* sms, char* name, int name_len) {
  if (!ctx) return EBZ_E_ARG;
  if (sms) *sms = ctx->sms;
  if (name && name_len > 0) {
    strncpy(name, ctx->name.c_str(), name_len - 1);
    name[name_len - 1] = 0;
  }
  return EBZ_OK;
}

unsigned long long ebz_launch_count(EbzCtx* ctx) { return ctx ? ctx->launches : 0; }

unsigned int ebz_debug_set_epoch(EbzCtx* ctx, unsigned int epoch) {
  if (!ctx) return 0;
  std::lock_guard<std::mutex> g(ctx->mu);
  const unsigned int old = ctx->epoch;
  ctx->epoch = epoch > kEpochMax ? kEpochMax : epoch;
  return old;
}

unsigned int ebz_epoch_max(void) { return kEpochMax; }

int ebz_sweep_kernel_choice(int width, int ndim, const uint64_t* dims, int layers, int nfields,
                            int compress) {
  if (!dims || ndim < 1 || ndim > 4) return EBZ_E_ARG;
  long long d[4] = {1, 1, 1, 1};
  for (int i = 0; i < ndim; ++i) d[i] = (long long)dims[i];
  if (!sweep_fast_supported(ndim, layers, d[0])) return 0;
  if (sweep2_used(ndim, layers, width, d, false, false)) return 4;
  if (sweep3b_used(ndim, layers, width, d, nfields, compress != 0, false, false)) return 5;
  if (width != 32) return 0;
  if (sweep3_used(ndim, layers, width, d, nfields, compress != 0)) return 3;
  return sweep_r2_used(ndim, layers, compress != 0) ? 2 : 1;
}

int ebz_profile(EbzCtx* ctx, int enable) {
  if (!ctx) return EBZ_E_ARG;
  ctx->profiling = enable != 0;
  return EBZ_OK;
}

int ebz_stage_times(EbzCtx* ctx, double* ms, unsigned long long* counts, int nstages) {
  if (!ctx || !ms || !counts) return EBZ_E_ARG;
  cudaSetDevice(ctx->device);
  for (int i = 0; i < nstages; ++i) {
    ms[i] = 0.0;
    counts[i] = 0;
  }
  std::lock_guard<std::mutex> g(ctx->mu);
  for (auto& mkr : ctx->marks) {
    EBZ_CUDA(cudaEventSynchronize(mkr.b));
    float t = 0.f;
    EBZ_CUDA(cudaEventElapsedTime(&t, mkr.a, mkr.b));
    if (mkr.stage >= 0 && mkr.stage < nstages) {
      ms[mkr.stage] += t;
      counts[mkr.stage] += 1;
    }
    ctx->pool.push_back(mkr.a);
    ctx->pool.push_back(mkr.b);
  }
  ctx->marks.clear();
  return EBZ_OK;
}

int ebz_grid_range(EbzCtx* ctx, const void* d_values, int width, uint64_t n, int has_abs,
                   double abs_bound, int has_rel, double rel_bound, EbzInfo* d_info,
                   void* stream) {
  if (!ctx || !d_values || !d_info || n == 0 || (width != 32 && width != 64)) return EBZ_E_ARG;
  cudaSetDevice(ctx->device);
  cudaStream_t s = (cudaStream_t)stream;
  if (!ctx->range_scratch.p) {
    EBZ_ALLOC(ctx->range_scratch, 1184 * 24 + 256);
    EBZ_CUDA(cudaMemset(ctx->range_scratch.p, 0, ctx->range_scratch.cap));
  }
  // always compute the range here (grid_range semantics); has_abs < 0 forces it
  EBZ_CUDA(launch_range(d_values, width, (long long)n, has_rel ? has_abs : (has_abs ? has_abs : -1),
                        abs_bound, has_rel, rel_bound, d_info,
                        ctx->range_scratch.as<unsigned int>(), s));
  ctx->launches += 1;
  return EBZ_OK;
}

int ebz_compress_scan(EbzCtx* ctx, const void* d_values, int width, int ndim,
                      const uint64_t* dims, int layers, int m, void* d_codes, void* d_recon,
                      unsigned long long* d_hist, EbzInfo* d_info, void* stream) {
  long long n;
  if (!ctx || !check_geom(width, ndim, dims, layers, m, n)) return EBZ_E_ARG;
  cudaSetDevice(ctx->device);
  Slot& sl = ctx->slot(-1);  // seam entry points: private scratch slot
  long long ld[4] = {1, 1, 1, 1};
  for (int a = 0; a < ndim; ++a) ld[a] = (long long)dims[a];
  cudaStream_t s = (cudaStream_t)stream;
  FieldIO f;
  memset(&f, 0, sizeof(f));
  f.sl = &sl;
  f.info = d_info;
  f.values = d_values;
  f.recon = d_recon;
  f.codes = d_codes;
  // the code histogram (caller's, or scratch) gives K = hist[0] either way
  unsigned long long* hist = d_hist;
  if (!hist) {
    EBZ_ALLOC(sl.hist, sizeof(unsigned long long) << m);
    hist = sl.hist.as<unsigned long long>();
  }
  EBZ_CUDA(cudaMemsetAsync(hist, 0, sizeof(unsigned long long) << m, s));
  EBZ_CUDA(cudaMemsetAsync(&d_info->n_unpred, 0, 8, s));
  f.hist = hist;  // the two-row kernel counts u8 codes as it writes them
  int rc = sweep_run(ctx, true, width, ndim, ld, layers, m, &f, 1, s);
  if (rc) return rc;
  if (!sl.hist_done) {
    EBZ_CUDA(launch_code_hist(d_codes, m, n, hist, ctx->sms, s));
    ctx->launches += 1;
  }
  EBZ_CUDA(cudaMemcpyAsync(&d_info->n_unpred, hist, 8, cudaMemcpyDeviceToDevice, s));
  return EBZ_OK;
}

int ebz_decompress_scan(EbzCtx* ctx, const void* d_codes, int width, int ndim,
                        const uint64_t* dims, int layers, int m, const void* d_unpred,
                        uint64_t n_unpred, void* d_recon, EbzInfo* d_info, void* stream) {
  long long n;
  if (!ctx || !check_geom(width, ndim, dims, layers, m, n)) return EBZ_E_ARG;
  cudaSetDevice(ctx->device);
  cudaStream_t s = (cudaStream_t)stream;
  Slot& sl = ctx->slot(-1);  // seam entry points: private scratch slot
  long long ld[4] = {1, 1, 1, 1};
  for (int a = 0; a < ndim; ++a) ld[a] = (long long)dims[a];
  const long long nrows = n / ld[0];
  EBZ_ALLOC(sl.rowbase, (size_t)nrows * 8);
  EBZ_ALLOC(sl.rowtmp, rowblk_words(nrows) * 8);
  // the caller's info carries eb; K is supplied here
  EBZ_CUDA(cudaMemcpyAsync(&d_info->n_unpred, &n_unpred, 8, cudaMemcpyHostToDevice, s));
  EBZ_CUDA(launch_rowbase(d_codes, m, n, ld[0], sl.rowbase.as<unsigned long long>(),
                          sl.rowtmp.as<unsigned long long>(), 0, d_info, s));
  ctx->launches += 2;
  FieldIO f;
  memset(&f, 0, sizeof(f));
  f.sl = &sl;
  f.info = d_info;
  f.recon = d_recon;
  f.codes = (void*)d_codes;
  f.unpred = d_unpred;
  f.rowbase = sl.rowbase.as<unsigned long long>();
  f.rowblk = sl.rowtmp.as<unsigned long long>();
  return sweep_run(ctx, false, width, ndim, ld, layers, m, &f, 1, s);
}

int ebz_build_code(EbzCtx* ctx, const unsigned long long* d_hist, int m, uint8_t* d_lengths,
                   unsigned long long* d_words, EbzInfo* d_info, void* stream) {
  if (!ctx || m < 1 || m > 16) return EBZ_E_ARG;
  cudaSetDevice(ctx->device);
  Slot& sl = ctx->slot(-1);  // seam entry points: private scratch slot
  EBZ_ALLOC(sl.huff, huffman_scratch_bytes(m));
  EBZ_CUDA(launch_huffman_build(d_hist, m, d_info, d_lengths, d_words,
                                sl.huff.as<unsigned long long>(), sl.huff.cap,
                                (cudaStream_t)stream));
  ctx->launches += 1;
  return EBZ_OK;
}

int ebz_pack_bits(EbzCtx* ctx, const void* d_codes, int m, uint64_t n, const void* d_values,
                  int width, const uint8_t* d_lengths, const unsigned long long* d_words,
                  uint8_t* d_bits, size_t bits_cap, void* d_unpred, EbzInfo* d_info,
                  void* stream) {
  if (!ctx || m < 1 || m > 16 || n == 0) return EBZ_E_ARG;
  cudaSetDevice(ctx->device);
  cudaStream_t s = (cudaStream_t)stream;
  Slot& sl = ctx->slot(-1);  // seam entry points: private scratch slot
  const long long nchunks = ((long long)n + kEncodeChunk - 1) / kEncodeChunk;
  EBZ_ALLOC(sl.agg, (size_t)nchunks * 16);
  EBZ_ALLOC(sl.head, 36 + 32 + ((size_t)1 << m));
  long long ld[4] = {(long long)n, 1, 1, 1};
  EncodeJob j;
  j.codes = d_codes;
  j.lengths = d_lengths;
  j.words = d_words;
  j.agg = sl.agg.as<unsigned long long>();
  j.info = d_info;
  j.bits = d_bits;
  j.bits_cap = bits_cap;
  j.head = sl.head.as<uint8_t>();
  j.values = d_values;
  j.unpred = d_unpred;
  j.trunc = 0;
  EBZ_CUDA(launch_encode_batch(&j, 1, m, (long long)n, width, 1, ld, 1, ctx->sms, s));
  ctx->launches += 3;
  return EBZ_OK;
}

int ebz_unpack_bits(EbzCtx* ctx, const uint8_t* d_bits, uint64_t nbytes, const uint8_t* d_lengths,
                    int m, uint64_t n, void* d_codes, EbzInfo* d_info, void* stream) {
  if (!ctx || m < 1 || m > 16) return EBZ_E_ARG;
  cudaSetDevice(ctx->device);
  Slot& sl = ctx->slot(-1);  // seam entry points: private scratch slot
  EBZ_ALLOC(sl.dscratch, decode_scratch_bytes((long long)nbytes, m));
  EBZ_CUDA(launch_decode(d_bits, (long long)nbytes, d_lengths, m, (long long)n, d_codes, d_info,
                         sl.dscratch.as<unsigned long long>(), sl.dscratch.cap, ctx->sms,
                         (cudaStream_t)stream, nullptr));
  ctx->launches += 7;
  return EBZ_OK;
}

int ebz_compress_async(EbzCtx* ctx, int slot, const void* d_values, int width, int ndim,
                       const uint64_t* dims, int layers, int m, int has_abs, double abs_bound,
                       int has_rel, double rel_bound, void* stream) {
  if (!ctx) return EBZ_E_ARG;
  cudaSetDevice(ctx->device);
  return compress_enqueue(ctx, slot, d_values, 0, width, ndim, dims, layers, m, has_abs, abs_bound,
                          has_rel, rel_bound, (cudaStream_t)stream);
}

int ebz_compress_batch(EbzCtx* ctx, int slot0, int nfields, const void* const* d_values,
                       int width, int ndim, const uint64_t* dims, int layers, int m, int has_abs,
                       double abs_bound, int has_rel, double rel_bound, void* stream) {
  if (!ctx || nfields < 1 || !d_values) return EBZ_E_ARG;
  cudaSetDevice(ctx->device);
  cudaStream_t s = (cudaStream_t)stream;
  std::vector<FieldIO> io((size_t)nfields);
  std::vector<Slot*> sls((size_t)nfields);
  std::vector<const void*> dv((size_t)nfields);
  for (int i = 0; i < nfields; ++i) {
    int rc = compress_prep(ctx, slot0 + i, d_values[i], 0, width, ndim, dims, layers, m, has_abs,
                           has_rel, s, &dv[i]);
    if (rc) return rc;
    sls[i] = &ctx->slot(slot0 + i);
    io[i] = compress_io(*sls[i], dv[i]);
  }
  // one launch per stage (per kBatchMax fields): range, sweep, hist, codebooks,
  // encode
  int rc = compress_range(ctx, sls.data(), dv.data(), nfields, 0, has_abs, abs_bound, has_rel,
                          rel_bound, s);
  if (rc) return rc;
  rc = sweep_run(ctx, true, width, ndim, sls[0]->dims, layers, m, io.data(), nfields, s);
  if (rc) return rc;
  return compress_back(ctx, sls.data(), dv.data(), nfields, s);
}

int ebz_decompress_batch(EbzCtx* ctx, int slot0, int src_slot0, int nfields,
                         void* const* d_recon, void* stream) {
  if (!ctx || nfields < 1 || !d_recon) return EBZ_E_ARG;
  cudaSetDevice(ctx->device);
  cudaStream_t s = (cudaStream_t)stream;
  Slot& first = ctx->slot(src_slot0);
  if (!first.have) { g_err = "source slot holds no compressed field"; return EBZ_E_ARG; }
  std::vector<FieldIO> io((size_t)nfields);
  std::vector<Slot*> sls((size_t)nfields);
  std::vector<DecIn> in((size_t)nfields);
  for (int i = 0; i < nfields; ++i) {
    Slot& src = ctx->slot(src_slot0 + i);
    if (!src.have) { g_err = "source slot holds no compressed field"; return EBZ_E_ARG; }
    if (src.width != first.width || src.ndim != first.ndim || src.layers != first.layers ||
        src.m != first.m || memcmp(src.dims, first.dims, sizeof(src.dims)) != 0) {
      g_err = "batched fields must share width, dims, layers and m";
      return EBZ_E_ARG;
    }
    sls[i] = &ctx->slot(slot0 + i);
    in[i] = DecIn{src.info.as<Info>(), 0.0, 0, src.lengths.as<uint8_t>(),
                  src.bits.as<uint8_t>(), src.bits.cap, src.unpred.p, d_recon[i]};
  }
  int rc = decompress_front(ctx, sls.data(), in.data(), nfields, first.ndim, first.dims, first.m,
                            s, io.data());
  if (rc) return rc;
  return sweep_run(ctx, false, first.width, first.ndim, first.dims, first.layers, first.m,
                   io.data(), nfields, s);
}

int ebz_decompress_batch_ptrs(EbzCtx* ctx, int slot0, int nfields, int width, int ndim,
                              const uint64_t* dims, int layers, int m, const double* eb,
                              const uint64_t* n_unpred, const uint8_t* const* d_lengths,
                              const uint8_t* const* d_bits, const uint64_t* nbytes,
                              const void* const* d_unpred, void* const* d_recon, void* stream) {
  long long n;
  if (!ctx || nfields < 1 || !eb || !n_unpred || !d_lengths || !d_bits || !nbytes || !d_unpred ||
      !d_recon || !check_geom(width, ndim, dims, layers, m, n))
    return EBZ_E_ARG;
  cudaSetDevice(ctx->device);
  cudaStream_t s = (cudaStream_t)stream;
  long long ld[4] = {1, 1, 1, 1};
  for (int a = 0; a < ndim; ++a) ld[a] = (long long)dims[a];
  std::vector<FieldIO> io((size_t)nfields);
  std::vector<Slot*> sls((size_t)nfields);
  std::vector<DecIn> in((size_t)nfields);
  for (int i = 0; i < nfields; ++i) {
    sls[i] = &ctx->slot(slot0 + i);
    in[i] = DecIn{nullptr, eb[i], n_unpred[i], d_lengths[i], d_bits[i], nbytes[i], d_unpred[i],
                  d_recon[i]};
  }
  int rc = decompress_front(ctx, sls.data(), in.data(), nfields, ndim, ld, m, s, io.data());
  if (rc) return rc;
  return sweep_run(ctx, false, width, ndim, ld, layers, m, io.data(), nfields, s);
}

int ebz_copy_async(EbzCtx* ctx, void* dst, const void* src, size_t nbytes, void* stream) {
  if (!ctx || (!dst && nbytes) || (!src && nbytes)) return EBZ_E_ARG;
  if (!nbytes) return EBZ_OK;
  cudaSetDevice(ctx->device);
  EBZ_CUDA(cudaMemcpyAsync(dst, src, nbytes, cudaMemcpyDefault, (cudaStream_t)stream));
  return EBZ_OK;
}

int ebz_slot_info_async(EbzCtx* ctx, int slot, int decode_record, EbzInfo* h_info,
                        void* stream) {
  if (!ctx || !h_info) return EBZ_E_ARG;
  cudaSetDevice(ctx->device);
  Slot& sl = ctx->slot(slot);
  Buf& b = decode_record ? sl.dinfo : sl.info;
  if (!b.p) { g_err = "slot holds no record"; return EBZ_E_ARG; }
  EBZ_CUDA(cudaMemcpyAsync(h_info, b.p, sizeof(Info), cudaMemcpyDeviceToHost,
                           (cudaStream_t)stream));
  return EBZ_OK;
}

int ebz_compress_fetch_async(EbzCtx* ctx, int slot, const EbzInfo* h_info, uint8_t* h_head,
                             uint8_t* h_bits, void* h_unpred, void* stream) {
  if (!ctx || !h_info) return EBZ_E_ARG;
  cudaSetDevice(ctx->device);
  cudaStream_t s = (cudaStream_t)stream;
  Slot& sl = ctx->slot(slot);
  if (!sl.have) { g_err = "slot holds no compressed field"; return EBZ_E_ARG; }
  const size_t head = 36 + 8 * (size_t)sl.ndim + ((size_t)1 << sl.m);
  if (h_head) EBZ_CUDA(cudaMemcpyAsync(h_head, sl.head.p, head, cudaMemcpyDeviceToHost, s));
  if (h_bits && h_info->bit_length)
    EBZ_CUDA(cudaMemcpyAsync(h_bits, sl.bits.p, (size_t)((h_info->bit_length + 7) / 8),
                             cudaMemcpyDeviceToHost, s));
  if (h_unpred && h_info->n_unpred)
    EBZ_CUDA(cudaMemcpyAsync(h_unpred, sl.unpred.p, (size_t)h_info->n_unpred * (sl.width / 8),
                             cudaMemcpyDeviceToHost, s));
  return EBZ_OK;
}

int ebz_original_hits(EbzCtx* ctx, const void* d_values, int width, int ndim,
                      const uint64_t* dims, int layers, double bound, uint64_t* h_hits,
                      void* stream) {
  long long n;
  if (!ctx || !d_values || !h_hits || !check_geom(width, ndim, dims, layers, 8, n))
    return EBZ_E_ARG;
  cudaSetDevice(ctx->device);
  cudaStream_t s = (cudaStream_t)stream;
  std::lock_guard<std::mutex> g(ctx->an_mu);
  Slot& sl = ctx->slot(-2);  // analysis scratch slot (stencil bank)
  long long ld[4] = {1, 1, 1, 1};
  for (int a = 0; a < ndim; ++a) ld[a] = (long long)dims[a];
  const long long *deltas, *starts, *counts;
  const double* coeffs;
  int rc = upload_bank(sl, ndim, ld, layers, s, &deltas, &coeffs, &starts, &counts);
  if (rc) return rc;
  EBZ_ALLOC(ctx->an_out, 64);
  EBZ_CUDA(cudaMemsetAsync(ctx->an_out.p, 0, 8, s));
  EBZ_CUDA(launch_original_hits(d_values, width, ndim, ld, layers, bound, deltas, coeffs, starts,
                                counts, ctx->an_out.as<unsigned long long>(), ctx->sms, s));
  ctx->launches += 1;
  EBZ_CUDA(cudaMemcpyAsync(h_hits, ctx->an_out.p, 8, cudaMemcpyDeviceToHost, s));
  EBZ_CUDA(cudaStreamSynchronize(s));
  return EBZ_OK;
}

int ebz_metrics(EbzCtx* ctx, const void* d_a, const void* d_b, int width, uint64_t n, int lags,
                double* h_out, void* stream) {
  if (!ctx || !d_a || !d_b || !h_out || n == 0 || (width != 32 && width != 64) || lags < 0 ||
      lags > EBZ_MAX_LAGS)
    return EBZ_E_ARG;
  cudaSetDevice(ctx->device);
  cudaStream_t s = (cudaStream_t)stream;
  std::lock_guard<std::mutex> g(ctx->an_mu);
  EBZ_ALLOC(ctx->an_scratch, metrics_scratch_bytes(lags));
  EBZ_ALLOC(ctx->an_out, (size_t)(9 + lags) * 8);
  EBZ_CUDA(launch_metrics(d_a, d_b, width, (long long)n, lags, ctx->an_scratch.as<double>(),
                          ctx->an_out.as<double>(), s));
  ctx->launches += 5;
  EBZ_CUDA(cudaMemcpyAsync(h_out, ctx->an_out.p, (size_t)(9 + lags) * 8, cudaMemcpyDeviceToHost,
                           s));
  EBZ_CUDA(cudaStreamSynchronize(s));
  return EBZ_OK;
}

int ebz_slot_info(EbzCtx* ctx, int slot, EbzInfo* h_info, void* stream) {
  if (!ctx || !h_info) return EBZ_E_ARG;
  cudaSetDevice(ctx->device);
  cudaStream_t s = (cudaStream_t)stream;
  Slot& sl = ctx->slot(slot);
  if (!sl.info.p) return EBZ_E_ARG;
  EBZ_CUDA(cudaMemcpyAsync(h_info, sl.info.p, sizeof(Info), cudaMemcpyDeviceToHost, s));
  EBZ_CUDA(cudaStreamSynchronize(s));
  return EBZ_OK;
}

int ebz_slot_decode_info(EbzCtx* ctx, int slot, EbzInfo* h_info, void* stream) {
  if (!ctx || !h_info) return EBZ_E_ARG;
  cudaSetDevice(ctx->device);
  cudaStream_t s = (cudaStream_t)stream;
  Slot& sl = ctx->slot(slot);
  if (!sl.dinfo.p) { g_err = "slot holds no decompress record"; return EBZ_E_ARG; }
  EBZ_CUDA(cudaMemcpyAsync(h_info, sl.dinfo.p, sizeof(Info), cudaMemcpyDeviceToHost, s));
  EBZ_CUDA(cudaStreamSynchronize(s));
  return EBZ_OK;
}

int ebz_compress(EbzCtx* ctx, int slot, const void* values, int on_host, int width, int ndim,
                 const uint64_t* dims, int layers, int m, int has_abs, double abs_bound,
                 int has_rel, double rel_bound, void* stream, EbzInfo* h_info) {
  return ebz_compress_flags(ctx, slot, values, on_host, width, ndim, dims, layers, m, 0, has_abs,
                            abs_bound, has_rel, rel_bound, stream, h_info);
}

int ebz_compress_flags(EbzCtx* ctx, int slot, const void* values, int on_host, int width,
                       int ndim, const uint64_t* dims, int layers, int m, int flags, int has_abs,
                       double abs_bound, int has_rel, double rel_bound, void* stream,
                       EbzInfo* h_info) {
  if (!ctx || !h_info || (flags & ~EBZ_FLAG_TRUNCATE)) return EBZ_E_ARG;
  cudaSetDevice(ctx->device);
  cudaStream_t s = (cudaStream_t)stream;
  int rc = compress_enqueue(ctx, slot, values, on_host, width, ndim, dims, layers, m, has_abs,
                            abs_bound, has_rel, rel_bound, s, flags);
  if (rc) return rc;
  Slot& sl = ctx->slot(slot);
  EBZ_CUDA(cudaMemcpyAsync(h_info, sl.info.p, sizeof(Info), cudaMemcpyDeviceToHost, s));
  EBZ_CUDA(cudaStreamSynchronize(s));
  if (h_info->status & ST_CAPACITY) {
    const void* d_values = on_host ? sl.values.p : values;
    rc = compress_regrow(ctx, sl, d_values, h_info->bit_length, s);
    if (rc) return rc;
    EBZ_CUDA(cudaMemcpyAsync(h_info, sl.info.p, sizeof(Info), cudaMemcpyDeviceToHost, s));
    EBZ_CUDA(cudaStreamSynchronize(s));
  }
  return EBZ_OK;
}

// Interval-count trials (cli.py:146-154 --auto-m): the predict/quantize
// sweeps of every candidate exponent in one batched launch over the same
// input (per-field m; u16 codes for all), then K per trial.  Trial i lives in
// slot slot0 + i; its record (ebz_slot_info) carries eb, status and K.
int ebz_compress_trials(EbzCtx* ctx, int slot0, const void* values, int on_host, int width,
                        int ndim, const uint64_t* dims, int layers, int ntrials, const int* ms,
                        int has_abs, double abs_bound, int has_rel, double rel_bound,
                        void* stream) {
  if (!ctx || !values || !ms || ntrials < 1 || ntrials > kBatchMax) return EBZ_E_ARG;
  cudaSetDevice(ctx->device);
  cudaStream_t s = (cudaStream_t)stream;
  std::vector<Slot*> sls((size_t)ntrials);
  std::vector<const void*> dv((size_t)ntrials);
  std::vector<FieldIO> io((size_t)ntrials);
  const void* d_values = nullptr;
  for (int i = 0; i < ntrials; ++i) {
    // the first trial stages a host input; the others read that copy
    int rc = compress_prep(ctx, slot0 + i, i == 0 ? values : d_values, i == 0 ? on_host : 0,
                           width, ndim, dims, layers, ms[i], has_abs, has_rel, s, &dv[i]);
    if (rc) return rc;
    if (i == 0) d_values = dv[0];
    Slot& sl = ctx->slot(slot0 + i);
    EBZ_ALLOC(sl.codes, (size_t)sl.n * 2 + 64);
    sl.trial_values = d_values;
    sl.trial = true;
    sls[i] = &sl;
    io[i] = compress_io(sl, d_values);
    io[i].hist = nullptr;
    io[i].center = 1 << (ms[i] - 1);
  }
  int rc = compress_range(ctx, sls.data(), dv.data(), ntrials, 0, has_abs, abs_bound, has_rel,
                          rel_bound, s);
  if (rc) return rc;
  rc = sweep_run(ctx, true, width, ndim, sls[0]->dims, layers, ms[0], io.data(), ntrials, s,
                 /*force_wide=*/true);
  if (rc) return rc;
  const uint16_t* codes[kBatchMax];
  unsigned long long* ks[kBatchMax];
  for (int i = 0; i < ntrials; ++i) {
    codes[i] = sls[i]->codes.as<uint16_t>();
    ks[i] = &sls[i]->info.as<Info>()->n_unpred;
    sls[i]->hist_done = false;
  }
  EBZ_CUDA(launch_zero_count_batch(codes, ks, ntrials, sls[0]->n, ctx->sms, s));
  ctx->launches += 1;
  return EBZ_OK;
}

// Finish the chosen trial: histogram, codebook and encoder on its codes (u8
// layout restored for m <= 8); the slot then holds a compressed field like
// ebz_compress's (ebz_compress_fetch / ebz_slot_info), h_info its record.
int ebz_compress_trial_finish(EbzCtx* ctx, int slot, void* stream, EbzInfo* h_info) {
  if (!ctx || !h_info) return EBZ_E_ARG;
  cudaSetDevice(ctx->device);
  cudaStream_t s = (cudaStream_t)stream;
  Slot& sl = ctx->slot(slot);
  if (!sl.trial) { g_err = "slot holds no interval trial"; return EBZ_E_ARG; }
  if (sl.m <= 8) {
    EBZ_ALLOC(sl.dcodes, (size_t)sl.n + 64);
    EBZ_CUDA(launch_narrow_codes(sl.codes.as<uint16_t>(), sl.dcodes.as<uint8_t>(), sl.n,
                                 ctx->sms, s));
    ctx->launches += 1;
    std::swap(sl.codes, sl.dcodes);
  }
  sl.trial = false;
  // the trial batch's range stage zeroed 2^m bins of the first trial's m only
  EBZ_CUDA(cudaMemsetAsync(sl.hist.p, 0, ((size_t)8) << sl.m, s));
  Slot* sp = &sl;
  const void* d_values = sl.trial_values;
  int rc = compress_back(ctx, &sp, &d_values, 1, s);
  if (rc) return rc;
  EBZ_CUDA(cudaMemcpyAsync(h_info, sl.info.p, sizeof(Info), cudaMemcpyDeviceToHost, s));
  EBZ_CUDA(cudaStreamSynchronize(s));
  if (h_info->status & ST_CAPACITY) {
    rc = compress_regrow(ctx, sl, d_values, h_info->bit_length, s);
    if (rc) return rc;
    EBZ_CUDA(cudaMemcpyAsync(h_info, sl.info.p, sizeof(Info), cudaMemcpyDeviceToHost, s));
    EBZ_CUDA(cudaStreamSynchronize(s));
  }
  return EBZ_OK;
}

int ebz_compress_fetch(EbzCtx* ctx, int slot, uint8_t* h_head, uint8_t* h_bits, void* h_unpred,
                       void* stream) {
  if (!ctx) return EBZ_E_ARG;
  cudaSetDevice(ctx->device);
  cudaStream_t s = (cudaStream_t)stream;
  Slot& sl = ctx->slot(slot);
  if (!sl.have) { g_err = "slot holds no compressed field"; return EBZ_E_ARG; }
  Info h;
  EBZ_CUDA(cudaMemcpyAsync(&h, sl.info.p, sizeof(Info), cudaMemcpyDeviceToHost, s));
  EBZ_CUDA(cudaStreamSynchronize(s));
  const size_t head = 36 + 8 * (size_t)sl.ndim + ((size_t)1 << sl.m);
  if (h_head) EBZ_CUDA(cudaMemcpyAsync(h_head, sl.head.p, head, cudaMemcpyDeviceToHost, s));
  if (h_bits && h.bit_length)
    EBZ_CUDA(cudaMemcpyAsync(h_bits, sl.bits.p, (size_t)((h.bit_length + 7) / 8),
                             cudaMemcpyDeviceToHost, s));
  if (h_unpred && h.n_unpred)
    EBZ_CUDA(cudaMemcpyAsync(h_unpred, sl.unpred.p, (size_t)h.n_unpred * (sl.width / 8),
                             cudaMemcpyDeviceToHost, s));
  EBZ_CUDA(cudaStreamSynchronize(s));
  return EBZ_OK;
}

int ebz_compress_outputs(EbzCtx* ctx, int slot, const uint8_t** d_head, const uint8_t** d_bits,
                         const void** d_unpred, const EbzInfo** d_info) {
  if (!ctx) return EBZ_E_ARG;
  Slot& sl = ctx->slot(slot);
  if (d_head) *d_head = sl.head.as<uint8_t>();
  if (d_bits) *d_bits = sl.bits.as<uint8_t>();
  if (d_unpred) *d_unpred = sl.unpred.p;
  if (d_info) *d_info = sl.info.as<EbzInfo>();
  return EBZ_OK;
}

int ebz_decompress(EbzCtx* ctx, int slot, int on_host, int width, int ndim, const uint64_t* dims,
                   int layers, int m, double eb, const uint8_t* lengths, const uint8_t* bits,
                   uint64_t nbytes, const void* unpred, uint64_t n_unpred, void* recon_out,
                   void* stream, EbzInfo* h_info) {
  long long n;
  if (!ctx || !h_info || !check_geom(width, ndim, dims, layers, m, n)) return EBZ_E_ARG;
  cudaSetDevice(ctx->device);
  cudaStream_t s = (cudaStream_t)stream;
  Slot& sl = ctx->slot(slot);
  const size_t ew = (size_t)width / 8;
  long long ld[4] = {1, 1, 1, 1};
  for (int a = 0; a < ndim; ++a) ld[a] = (long long)dims[a];
  const uint8_t* d_lengths = lengths;
  const uint8_t* d_bits = bits;
  const void* d_unpred = unpred;
  void* d_recon = recon_out;
  if (on_host) {
    EBZ_ALLOC(sl.dlengths, (size_t)1 << m);
    EBZ_ALLOC(sl.dbits, (size_t)nbytes + 64);
    EBZ_ALLOC(sl.dunpred, (size_t)n_unpred * ew + 8);
    EBZ_ALLOC(sl.drecon, (size_t)n * ew);
    EBZ_CUDA(cudaMemcpyAsync(sl.dlengths.p, lengths, (size_t)1 << m, cudaMemcpyHostToDevice, s));
    EBZ_CUDA(cudaMemsetAsync(sl.dbits.as<uint8_t>() + nbytes, 0, 64, s));
    if (nbytes)
      EBZ_CUDA(cudaMemcpyAsync(sl.dbits.p, bits, (size_t)nbytes, cudaMemcpyHostToDevice, s));
    if (n_unpred)
      EBZ_CUDA(cudaMemcpyAsync(sl.dunpred.p, unpred, (size_t)n_unpred * ew,
                               cudaMemcpyHostToDevice, s));
    d_lengths = sl.dlengths.as<uint8_t>();
    d_bits = sl.dbits.as<uint8_t>();
    d_unpred = sl.dunpred.p;
    d_recon = sl.drecon.p;
  }
  int rc = decompress_enqueue(ctx, sl, width, ndim, ld, layers, m, nullptr, eb, n_unpred,
                              d_lengths, d_bits, nbytes, d_unpred, d_recon, s);
  if (rc) return rc;
  if (on_host)
    EBZ_CUDA(cudaMemcpyAsync(recon_out, d_recon, (size_t)n * ew, cudaMemcpyDeviceToHost, s));
  EBZ_CUDA(cudaMemcpyAsync(h_info, sl.dinfo.p, sizeof(Info), cudaMemcpyDeviceToHost, s));
  EBZ_CUDA(cudaStreamSynchronize(s));
  return EBZ_OK;
}

int ebz_decompress_async(EbzCtx* ctx, int slot, int src_slot, void* d_recon, void* stream) {
  if (!ctx) return EBZ_E_ARG;
  cudaSetDevice(ctx->device);
  cudaStream_t s = (cudaStream_t)stream;
  Slot& src = ctx->slot(src_slot);
  Slot& sl = ctx->slot(slot);
  if (!src.have) { g_err = "source slot holds no compressed field"; return EBZ_E_ARG; }
  // No host sync: the exact byte budget ceil(bit_length / 8), eb and K are
  // read from the source record on the device; the capacity of the code
  // buffer only bounds the decoder's grid.
  return decompress_enqueue(ctx, sl, src.width, src.ndim, src.dims, src.layers, src.m,
                            src.info.as<Info>(), 0.0, 0, src.lengths.as<uint8_t>(),
                            src.bits.as<uint8_t>(), src.bits.cap, src.unpred.p, d_recon, s);
}

// ---- the reference kernel seam on host buffers (ebzip/_kernels.py) -------
// Each ebz_ref_* entry point takes exactly the arguments of one numba
// kernel (caller-allocated host numpy buffers, filled in place; codes int32
// as codec.py:102), runs it on the device through the kernels above and
// returns the kernel's own result in *result.  The stencil bank the caller
// passes must be codec._stencil_bank(layers, dims) -- the kernels derive
// the same bank from the geometry, so any other bank is rejected.

}  // extern "C"

namespace {

constexpr int kSeamSlot = -3;  // private workspace of the ebz_ref_* entry points

// m of a reference `center` argument (quantizer.py:16-18: center = 2^(m-1))
int seam_m(long long center) {
  if (center < 2 || center > (1 << 15) || (center & (center - 1))) return -1;
  int m = 1;
  while ((1ll << (m - 1)) < center) ++m;
  return m;
}

bool seam_bank_ok(int ndim, const long long* ld, int layers, const int64_t* deltas,
                  const double* coeffs, int64_t nterms, const int64_t* starts,
                  const int64_t* counts, int64_t nslots) {
  if (!deltas || !coeffs || !starts || !counts) return false;
  const Bank b = make_bank(ndim, ld, layers);
  if ((int64_t)b.deltas.size() != nterms || (int64_t)b.starts.size() != nslots) return false;
  for (int64_t t = 0; t < nterms; ++t)
    if (b.deltas[t] != deltas[t] || b.coeffs[t] != coeffs[t]) return false;
  for (int64_t i = 0; i < nslots; ++i)
    if (b.starts[i] != starts[i] || b.counts[i] != counts[i]) return false;
  return true;
}

int seam_geom(const int64_t* dims, int ndim, int64_t layers, long long center, int width,
              uint64_t* ud, long long* ld, int* m, long long* n) {
  if (!dims || ndim < 1 || ndim > 4 || layers < 1 || layers > 255) {
    g_err = "dims must have 1..4 axes and layers must be 1..255";
    return EBZ_E_ARG;
  }
  *m = seam_m(center);
  if (*m < 2 || *m > 16) {
    g_err = "center must be 2^(m-1) with 2 <= m <= 16 (quantizer.center_code)";
    return EBZ_E_ARG;
  }
  for (int a = 0; a < 4; ++a) {
    if (a < ndim && dims[a] < 1) { g_err = "dims must be positive"; return EBZ_E_ARG; }
    ud[a] = a < ndim ? (uint64_t)dims[a] : 1;
    ld[a] = a < ndim ? (long long)dims[a] : 1;
  }
  if (!check_geom(width, ndim, ud, (int)layers, *m, *n)) return EBZ_E_ARG;
  return EBZ_OK;
}

int seam_bank_args(int ndim, const long long* ld, int64_t layers, const int64_t* deltas,
                   const double* coeffs, int64_t nterms, const int64_t* starts,
                   const int64_t* counts, int64_t nslots) {
  if (!seam_bank_ok(ndim, ld, (int)layers, deltas, coeffs, nterms, starts, counts, nslots)) {
    g_err = "stencil bank differs from codec._stencil_bank(layers, dims)";
    return EBZ_E_ARG;
  }
  return EBZ_OK;
}

// canonical codewords of a length table (entropy.py:50-65)
std::vector<unsigned long long> canonical_words(const uint8_t* lens, size_t nsym) {
  std::vector<unsigned long long> w(nsym, 0);
  std::vector<size_t> order;
  for (size_t i = 0; i < nsym; ++i)
    if (lens[i]) order.push_back(i);
  std::stable_sort(order.begin(), order.end(),
                   [&](size_t a, size_t b) { return lens[a] < lens[b]; });
  unsigned long long word = 0;
  int prev = 0;
  for (size_t k = 0; k < order.size(); ++k) {
    const int L = lens[order[k]];
    word <<= (L - prev);
    w[order[k]] = word++;
    prev = L;
  }
  return w;
}

void widen_codes(const std::vector<uint8_t>& hc, size_t cw, uint64_t n, int32_t* out) {
  if (cw == 1)
    for (uint64_t i = 0; i < n; ++i) out[i] = hc[i];
  else
    for (uint64_t i = 0; i < n; ++i) out[i] = reinterpret_cast<const uint16_t*>(hc.data())[i];
}

}  // namespace

extern "C" {

int ebz_ref_compress_scan(EbzCtx* ctx, const void* values, int width, void* recon,
                          int32_t* codes, const int64_t* deltas, const double* coeffs,
                          int64_t nterms, const int64_t* starts, const int64_t* counts,
                          int64_t nslots, const int64_t* dims, int ndim, int64_t layers,
                          int64_t center, double bound, long long* result) {
  if (!ctx || !values || !recon || !codes || !result) return EBZ_E_ARG;
  uint64_t ud[4];
  long long ld[4], n;
  int m;
  int rc = seam_geom(dims, ndim, layers, center, width, ud, ld, &m, &n);
  if (!rc) rc = seam_bank_args(ndim, ld, layers, deltas, coeffs, nterms, starts, counts, nslots);
  if (rc) return rc;
  if (!(bound > 0.0) || !std::isfinite(bound)) {
    g_err = "bound must be positive and finite (core.py:173-177)";
    return EBZ_E_ARG;
  }
  cudaSetDevice(ctx->device);
  std::lock_guard<std::mutex> g(ctx->seam_mu);
  Slot& sl = ctx->slot(kSeamSlot);
  const size_t ew = (size_t)width / 8, cw = m > 8 ? 2 : 1;
  EBZ_ALLOC(sl.values, (size_t)n * ew);
  EBZ_ALLOC(sl.recon, (size_t)n * ew);
  EBZ_ALLOC(sl.codes, (size_t)n * cw + 64);
  EBZ_ALLOC(sl.info, sizeof(Info));
  cudaStream_t s = 0;
  Info h;
  memset(&h, 0, sizeof(h));
  h.eb = bound;
  EBZ_CUDA(cudaMemcpyAsync(sl.info.p, &h, sizeof(h), cudaMemcpyHostToDevice, s));
  EBZ_CUDA(cudaMemcpyAsync(sl.values.p, values, (size_t)n * ew, cudaMemcpyHostToDevice, s));
  rc = ebz_compress_scan(ctx, sl.values.p, width, ndim, ud, (int)layers, m, sl.codes.p,
                         sl.recon.p, nullptr, sl.info.as<EbzInfo>(), s);
  if (rc) return rc;
  std::vector<uint8_t> hc((size_t)n * cw);
  EBZ_CUDA(cudaMemcpyAsync(hc.data(), sl.codes.p, hc.size(), cudaMemcpyDeviceToHost, s));
  EBZ_CUDA(cudaMemcpyAsync(recon, sl.recon.p, (size_t)n * ew, cudaMemcpyDeviceToHost, s));
  EBZ_CUDA(cudaMemcpyAsync(&h, sl.info.p, sizeof(h), cudaMemcpyDeviceToHost, s));
  EBZ_CUDA(cudaStreamSynchronize(s));
  widen_codes(hc, cw, (uint64_t)n, codes);
  *result = (long long)h.n_unpred;
  return EBZ_OK;
}

// Truncated-mantissa block of K unpredictable values (opt-in extension,
// trunc.cu), host buffers, synchronous.  h_out == NULL: size query.
int ebz_tr_pack(EbzCtx* ctx, const void* h_values, uint64_t k, int width, double eb,
                uint8_t* h_out, uint64_t out_cap, uint64_t* out_bits) {
  if (!ctx || !out_bits || (width != 32 && width != 64) || (k && !h_values) ||
      !(eb > 0.0) || !std::isfinite(eb)) {
    g_err = "ebz_tr_pack: bad arguments";
    return EBZ_E_ARG;
  }
  cudaSetDevice(ctx->device);
  std::lock_guard<std::mutex> g(ctx->seam_mu);
  Slot& sl = ctx->slot(kSeamSlot);
  const size_t ew = (size_t)width / 8;
  cudaStream_t s = 0;
  EBZ_ALLOC(sl.values, (size_t)k * ew + 16);
  EBZ_ALLOC(sl.agg, tr_scratch_bytes(k));
  if (k) EBZ_CUDA(cudaMemcpyAsync(sl.values.p, h_values, (size_t)k * ew, cudaMemcpyHostToDevice, s));
  EBZ_CUDA(launch_tr_pack(sl.values.p, width, k, eb, nullptr, sl.agg.as<unsigned long long>(), s,
                          true));
  unsigned long long tot[2] = {0, 0};
  EBZ_CUDA(cudaMemcpyAsync(tot, sl.agg.p, 16, cudaMemcpyDeviceToHost, s));
  EBZ_CUDA(cudaStreamSynchronize(s));
  *out_bits = tot[1];
  if (!h_out) return EBZ_OK;
  const size_t nbytes = (size_t)((tot[1] + 7) / 8);
  if (out_cap < nbytes) {
    g_err = "ebz_tr_pack: output buffer too small";
    return EBZ_E_ARG;
  }
  EBZ_ALLOC(sl.bits, nbytes + 16);
  EBZ_CUDA(cudaMemsetAsync(sl.bits.p, 0, nbytes + 16, s));
  EBZ_CUDA(launch_tr_pack(sl.values.p, width, k, eb, sl.bits.as<uint8_t>(),
                          sl.agg.as<unsigned long long>(), s, false));
  ctx->launches += 3;
  if (nbytes) EBZ_CUDA(cudaMemcpyAsync(h_out, sl.bits.p, nbytes, cudaMemcpyDeviceToHost, s));
  EBZ_CUDA(cudaStreamSynchronize(s));
  return EBZ_OK;
}

int ebz_tr_unpack(EbzCtx* ctx, const uint8_t* h_in, uint64_t nbytes, uint64_t k, int width,
                  double eb, void* h_values) {
  if (!ctx || (width != 32 && width != 64) || (nbytes && !h_in) || (k && !h_values) ||
      !(eb > 0.0) || !std::isfinite(eb)) {
    g_err = "ebz_tr_unpack: bad arguments";
    return EBZ_E_ARG;
  }
  const unsigned long long hb = width == 64 ? 12 : 9;
  if (nbytes * 8 < hb * k) {
    g_err = "truncated-mantissa block too short for its header fields";
    return EBZ_E_ARG;
  }
  cudaSetDevice(ctx->device);
  std::lock_guard<std::mutex> g(ctx->seam_mu);
  Slot& sl = ctx->slot(kSeamSlot);
  const size_t ew = (size_t)width / 8;
  cudaStream_t s = 0;
  EBZ_ALLOC(sl.bits, (size_t)nbytes + 16);
  EBZ_ALLOC(sl.values, (size_t)k * ew + 16);
  EBZ_ALLOC(sl.agg, tr_scratch_bytes(k));
  EBZ_CUDA(cudaMemsetAsync(sl.bits.p, 0, (size_t)nbytes + 16, s));
  if (nbytes) EBZ_CUDA(cudaMemcpyAsync(sl.bits.p, h_in, (size_t)nbytes, cudaMemcpyHostToDevice, s));
  EBZ_CUDA(launch_tr_unpack(sl.bits.as<uint8_t>(), width, k, eb, sl.values.p,
                            sl.agg.as<unsigned long long>(), s));
  ctx->launches += 3;
  unsigned long long tot[2] = {0, 0};
  EBZ_CUDA(cudaMemcpyAsync(tot, sl.agg.p, 16, cudaMemcpyDeviceToHost, s));
  EBZ_CUDA(cudaStreamSynchronize(s));
  if ((tot[1] + 7) / 8 != nbytes) {
    g_err = "truncated-mantissa block size does not match its header fields";
    return EBZ_E_ARG;
  }
  if (k) EBZ_CUDA(cudaMemcpy(h_values, sl.values.p, (size_t)k * ew, cudaMemcpyDeviceToHost));
  return EBZ_OK;
}

int ebz_ref_decompress_scan(EbzCtx* ctx, const int32_t* codes, void* recon, int width,
                            const void* unpred, uint64_t n_unpred, const int64_t* deltas,
                            const double* coeffs, int64_t nterms, const int64_t* starts,
                            const int64_t* counts, int64_t nslots, const int64_t* dims, int ndim,
                            int64_t layers, int64_t center, double bound, long long* result) {
  if (!ctx || !codes || !recon || (!unpred && n_unpred) || !result) return EBZ_E_ARG;
  uint64_t ud[4];
  long long ld[4], n;
  int m;
  int rc = seam_geom(dims, ndim, layers, center, width, ud, ld, &m, &n);
  if (!rc) rc = seam_bank_args(ndim, ld, layers, deltas, coeffs, nterms, starts, counts, nslots);
  if (rc) return rc;
  if (!(bound > 0.0) || !std::isfinite(bound)) {
    g_err = "bound must be positive and finite (core.py:173-177)";
    return EBZ_E_ARG;
  }
  const size_t ew = (size_t)width / 8, cw = m > 8 ? 2 : 1;
  const long long nsym = 1ll << m;
  std::vector<uint8_t> hc((size_t)n * cw);
  for (long long i = 0; i < n; ++i) {
    if (codes[i] < 0 || codes[i] >= nsym) {
      g_err = "code outside [0, 2^m) (the decoder only produces alphabet symbols)";
      return EBZ_E_ARG;
    }
    if (cw == 1) hc[i] = (uint8_t)codes[i];
    else reinterpret_cast<uint16_t*>(hc.data())[i] = (uint16_t)codes[i];
  }
  cudaSetDevice(ctx->device);
  std::lock_guard<std::mutex> g(ctx->seam_mu);
  Slot& sl = ctx->slot(kSeamSlot);
  EBZ_ALLOC(sl.dcodes, (size_t)n * cw + 64);
  EBZ_ALLOC(sl.dunpred, (size_t)(n_unpred ? n_unpred : 1) * ew);
  EBZ_ALLOC(sl.drecon, (size_t)n * ew);
  EBZ_ALLOC(sl.dinfo, sizeof(Info));
  cudaStream_t s = 0;
  Info h;
  memset(&h, 0, sizeof(h));
  h.eb = bound;
  h.n_unpred = n_unpred;
  EBZ_CUDA(cudaMemcpyAsync(sl.dinfo.p, &h, sizeof(h), cudaMemcpyHostToDevice, s));
  EBZ_CUDA(cudaMemcpyAsync(sl.dcodes.p, hc.data(), hc.size(), cudaMemcpyHostToDevice, s));
  if (n_unpred)
    EBZ_CUDA(cudaMemcpyAsync(sl.dunpred.p, unpred, (size_t)n_unpred * ew, cudaMemcpyHostToDevice,
                             s));
  rc = ebz_decompress_scan(ctx, sl.dcodes.p, width, ndim, ud, (int)layers, m, sl.dunpred.p,
                           n_unpred, sl.drecon.p, sl.dinfo.as<EbzInfo>(), s);
  if (rc) return rc;
  EBZ_CUDA(cudaMemcpyAsync(recon, sl.drecon.p, (size_t)n * ew, cudaMemcpyDeviceToHost, s));
  EBZ_CUDA(cudaMemcpyAsync(&h, sl.dinfo.p, sizeof(h), cudaMemcpyDeviceToHost, s));
  EBZ_CUDA(cudaStreamSynchronize(s));
  // _kernels.py:97-99: -1 when the verbatim block runs out, else the count used
  *result = (h.status & ST_UNDERRUN) ? -1 : (long long)h.used;
  return EBZ_OK;
}

int ebz_ref_pack_bits(EbzCtx* ctx, const int32_t* symbols, uint64_t n,
                      const unsigned long long* code_words, const uint8_t* code_lens,
                      uint64_t nsym, uint8_t* out, uint64_t out_bytes, long long* total) {
  if (!ctx || (!symbols && n) || !code_words || !code_lens || !total || nsym == 0 ||
      nsym > 65536)
    return EBZ_E_ARG;
  int m = 2;
  while ((1ull << m) < nsym) ++m;
  const std::vector<unsigned long long> canon = canonical_words(code_lens, (size_t)nsym);
  for (uint64_t i = 0; i < nsym; ++i) {
    if (code_lens[i] > 64 || (code_lens[i] && code_words[i] != canon[i])) {
      g_err = "code_words must be the canonical words of code_lens (entropy.py:50-65)";
      return EBZ_E_ARG;
    }
  }
  const size_t cw = m > 8 ? 2 : 1;
  std::vector<uint8_t> hc((size_t)n * cw + 1);
  unsigned long long bits = 0;
  for (uint64_t i = 0; i < n; ++i) {
    if (symbols[i] < 0 || (uint64_t)symbols[i] >= nsym) {
      g_err = "symbol outside the table's alphabet";
      return EBZ_E_ARG;
    }
    bits += code_lens[symbols[i]];
    if (cw == 1) hc[i] = (uint8_t)symbols[i];
    else reinterpret_cast<uint16_t*>(hc.data())[i] = (uint16_t)symbols[i];
  }
  if ((bits + 7) / 8 > out_bytes) {
    g_err = "out is smaller than ceil(total bits / 8)";
    return EBZ_E_ARG;
  }
  *total = (long long)bits;
  if (n == 0 || bits == 0) return EBZ_OK;
  cudaSetDevice(ctx->device);
  std::lock_guard<std::mutex> g(ctx->seam_mu);
  Slot& sl = ctx->slot(kSeamSlot);
  const size_t asz = (size_t)1 << m;
  std::vector<uint8_t> lens(asz, 0);
  std::vector<unsigned long long> words(asz, 0);
  memcpy(lens.data(), code_lens, (size_t)nsym);
  memcpy(words.data(), code_words, (size_t)nsym * 8);
  EBZ_ALLOC(sl.codes, hc.size() + 64);
  EBZ_ALLOC(sl.lengths, asz);
  EBZ_ALLOC(sl.words, asz * 8);
  EBZ_ALLOC(sl.bits, (size_t)(bits / 8) + 64);
  EBZ_ALLOC(sl.info, sizeof(Info));
  cudaStream_t s = 0;
  EBZ_CUDA(cudaMemsetAsync(sl.info.p, 0, sizeof(Info), s));
  EBZ_CUDA(cudaMemcpyAsync(sl.codes.p, hc.data(), (size_t)n * cw, cudaMemcpyHostToDevice, s));
  EBZ_CUDA(cudaMemcpyAsync(sl.lengths.p, lens.data(), asz, cudaMemcpyHostToDevice, s));
  EBZ_CUDA(cudaMemcpyAsync(sl.words.p, words.data(), asz * 8, cudaMemcpyHostToDevice, s));
  int rc = ebz_pack_bits(ctx, sl.codes.p, m, n, nullptr, 32, sl.lengths.as<uint8_t>(),
                         sl.words.as<unsigned long long>(), sl.bits.as<uint8_t>(), sl.bits.cap,
                         nullptr, sl.info.as<EbzInfo>(), s);
  if (rc) return rc;
  Info h;
  EBZ_CUDA(cudaMemcpyAsync(&h, sl.info.p, sizeof(h), cudaMemcpyDeviceToHost, s));
  EBZ_CUDA(cudaStreamSynchronize(s));
  if (h.bit_length != bits) { g_err = "bit accounting mismatch"; return EBZ_E_CUDA; }
  EBZ_CUDA(cudaMemcpy(out, sl.bits.p, (size_t)((bits + 7) / 8), cudaMemcpyDeviceToHost));
  return EBZ_OK;
}

int ebz_ref_unpack_bits(EbzCtx* ctx, const uint8_t* data, uint64_t nbytes, uint64_t n_bits,
                        const unsigned long long* first_codes, const int64_t* level_counts,
                        const int64_t* level_base, const int32_t* ordered, uint64_t n_ordered,
                        int max_len, int32_t* out, uint64_t count, long long* result) {
  if (!ctx || !first_codes || !level_counts || !level_base || !ordered || !result ||
      (!out && count) || (!data && nbytes) || max_len < 1 || max_len > 64)
    return EBZ_E_ARG;
  if (n_bits != nbytes * 8) {
    g_err = "n_bits must be the whole buffer, 8 * len(data) (entropy.py:171-175)";
    return EBZ_E_ARG;
  }
  // code lengths from the canonical decode tables (entropy.py:67-84)
  int32_t maxsym = -1;
  for (uint64_t i = 0; i < n_ordered; ++i) maxsym = ordered[i] > maxsym ? ordered[i] : maxsym;
  if (maxsym < 0 || maxsym >= 65536) {
    g_err = "ordered symbols outside [0, 65536)";
    return EBZ_E_ARG;
  }
  int m = 2;
  while ((1ll << m) < (long long)maxsym + 1) ++m;
  std::vector<uint8_t> lens((size_t)1 << m, 0);
  for (int L = 1; L <= max_len; ++L)
    for (int64_t j = 0; j < level_counts[L]; ++j) {
      const int64_t k = level_base[L] + j;
      if (k < 0 || (uint64_t)k >= n_ordered || ordered[k] < 0) {
        g_err = "decode tables are inconsistent";
        return EBZ_E_ARG;
      }
      lens[ordered[k]] = (uint8_t)L;
    }
  unsigned long long word = 0;
  for (int L = 1; L <= max_len; ++L) {  // first_codes must be the canonical ones
    word <<= 1;
    if (first_codes[L] != word) {
      g_err = "decode tables are not canonical";
      return EBZ_E_ARG;
    }
    word += (unsigned long long)level_counts[L];
  }
  if (count == 0) {
    *result = 0;
    return EBZ_OK;
  }
  cudaSetDevice(ctx->device);
  std::lock_guard<std::mutex> g(ctx->seam_mu);
  Slot& sl = ctx->slot(kSeamSlot);
  const size_t cw = m > 8 ? 2 : 1;
  EBZ_ALLOC(sl.dbits, (size_t)nbytes + 64);
  EBZ_ALLOC(sl.dlengths, lens.size());
  EBZ_ALLOC(sl.dcodes, (size_t)count * cw + 64);
  EBZ_ALLOC(sl.dinfo, sizeof(Info));
  EBZ_ALLOC(sl.dscratch, decode_scratch_bytes((long long)nbytes, m));
  cudaStream_t s = 0;
  EBZ_CUDA(cudaMemsetAsync(sl.dinfo.p, 0, sizeof(Info), s));
  EBZ_CUDA(cudaMemsetAsync(sl.dbits.as<uint8_t>() + nbytes, 0, 64, s));
  if (nbytes)
    EBZ_CUDA(cudaMemcpyAsync(sl.dbits.p, data, (size_t)nbytes, cudaMemcpyHostToDevice, s));
  EBZ_CUDA(cudaMemcpyAsync(sl.dlengths.p, lens.data(), lens.size(), cudaMemcpyHostToDevice, s));
  int rc = ebz_unpack_bits(ctx, sl.dbits.as<uint8_t>(), nbytes, sl.dlengths.as<uint8_t>(), m,
                           count, sl.dcodes.p, sl.dinfo.as<EbzInfo>(), s);
  if (rc) return rc;
  Info h;
  EBZ_CUDA(cudaMemcpyAsync(&h, sl.dinfo.p, sizeof(h), cudaMemcpyDeviceToHost, s));
  std::vector<uint8_t> hc((size_t)count * cw);
  EBZ_CUDA(cudaMemcpyAsync(hc.data(), sl.dcodes.p, hc.size(), cudaMemcpyDeviceToHost, s));
  EBZ_CUDA(cudaStreamSynchronize(s));
  // _kernels.py:165-183: -2 invalid prefix, -1 exhausted, else the count
  if (h.status & ST_DEC_INVALID) {
    *result = -2;
    return EBZ_OK;
  }
  if (h.status & ST_DEC_EXHAUSTED) {
    *result = -1;
    return EBZ_OK;
  }
  widen_codes(hc, cw, count, out);
  *result = (long long)count;
  return EBZ_OK;
}

int ebz_ref_original_hits(EbzCtx* ctx, const void* values, int width, const int64_t* deltas,
                          const double* coeffs, int64_t nterms, const int64_t* starts,
                          const int64_t* counts, int64_t nslots, const int64_t* dims, int ndim,
                          int64_t layers, double bound, long long* result) {
  if (!ctx || !values || !result) return EBZ_E_ARG;
  uint64_t ud[4];
  long long ld[4], n;
  int m;
  int rc = seam_geom(dims, ndim, layers, 128, width, ud, ld, &m, &n);
  if (!rc) rc = seam_bank_args(ndim, ld, layers, deltas, coeffs, nterms, starts, counts, nslots);
  if (rc) return rc;
  cudaSetDevice(ctx->device);
  std::lock_guard<std::mutex> g(ctx->seam_mu);
  Slot& sl = ctx->slot(kSeamSlot);
  const size_t ew = (size_t)width / 8;
  EBZ_ALLOC(sl.values, (size_t)n * ew);
  EBZ_CUDA(cudaMemcpy(sl.values.p, values, (size_t)n * ew, cudaMemcpyHostToDevice));
  uint64_t hits = 0;
  rc = ebz_original_hits(ctx, sl.values.p, width, ndim, ud, (int)layers, bound, &hits, nullptr);
  if (rc) return rc;
  *result = (long long)hits;
  return EBZ_OK;
}

}  // extern "C"
