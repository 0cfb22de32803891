/*
 * ebz200.h -- C ABI of libebz200.so, the B200 (sm_100a) compress/decompress
 * path of the SZ-1.4-style error-bounded compressor (arXiv 1706.03791).
 *
 * Drop-in boundary.  The reference (`ebzip`, pure Python + numba) has no C
 * FFI; its kernel seam is four numba functions plus numpy reductions called
 * from `ebzip/codec.py`.  Each entry point below replaces one of them
 * (paths relative to /root/reference/pkg/src/ebzip/):
 *
 *   ebz_grid_range       <- core.py:132-136  grid_range (+ core.py:92-93 isfinite,
 *                           core.py:161-178 effective_bound)
 *   ebz_compress_scan    <- _kernels.py:48-80  compress_scan (+ codec.py:107 bincount)
 *   ebz_decompress_scan  <- _kernels.py:83-105 decompress_scan
 *   ebz_build_code       <- entropy.py:87-136  build_code (+ entropy.py:50-65 code_words)
 *   ebz_pack_bits        <- entropy.py:139-157 encode / _kernels.py:124-148 pack_bits
 *                           (+ codec.py:119 unpredictable gather)
 *   ebz_unpack_bits      <- entropy.py:160-183 decode / _kernels.py:151-183 unpack_bits
 *   ebz_compress         <- codec.py:92-136  compress   (one-shot, host or device input)
 *   ebz_decompress       <- codec.py:139-160 decompress (one-shot)
 *
 * Conventions (mirroring the reference seam):
 *  - caller-visible buffers are plain pointers + sizes; no torch types;
 *  - the element width is 32 or 64 (float / double), codes are uint8 for
 *    interval exponent m <= 8 and uint16 for m <= 16;
 *  - every call takes a cudaStream_t (may be 0) and is asynchronous unless
 *    it returns host-visible results (documented per call);
 *  - return value 0 = OK; negative values are EBZ_E_* codes; data-dependent
 *    failures (the reference's ValueErrors) are reported through
 *    EbzInfo.status bits so the host can raise the reference's exception
 *    with the reference's message, in the reference's order.
 *  - there is no CPU fallback: without a usable sm_100 device every entry
 *    point returns EBZ_E_NODEVICE.
 */
#ifndef EBZ200_H
#define EBZ200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define EBZ_ABI_VERSION 1

/* error codes */
#define EBZ_OK 0
#define EBZ_E_ARG -1       /* invalid argument (mirrors reference ValueError on inputs) */
#define EBZ_E_CUDA -2      /* CUDA runtime failure */
#define EBZ_E_NODEVICE -3  /* no CUDA device / not sm_100 */
#define EBZ_E_OOM -4

/* status bits (EbzInfo.status) */
#define EBZ_ST_EB_NONPOSITIVE 0x001   /* core.py:173-177 */
#define EBZ_ST_NONFINITE_IN 0x002     /* core.py:92-93 */
#define EBZ_ST_DEPTH_GT_64 0x004      /* entropy.py:133-134 */
#define EBZ_ST_EMPTY_HIST 0x008
#define EBZ_ST_DEC_EXHAUSTED 0x010    /* entropy.py:176-179 "exhausted" */
#define EBZ_ST_DEC_INVALID 0x020      /* entropy.py:181-182 "invalid" */
#define EBZ_ST_DEC_ANOMALY 0x040      /* parallel decode fell back to serial */
#define EBZ_ST_UNPRED_MISMATCH 0x080  /* codec.py:144-149 "unpredictable" */
#define EBZ_ST_UNDERRUN 0x100         /* codec.py:158-159 */
#define EBZ_ST_NONFINITE_OUT 0x200    /* DataGrid check on the output */
#define EBZ_ST_CAPACITY 0x400         /* internal: output buffer regrown */

/* Per-field result record (device-written, copied back by the one-shots). */
typedef struct EbzInfo {
  double eb;                        /* effective bound (header field) */
  double vmin, vmax;                /* element-precision min / max */
  double range;                     /* float(T(max - min)), core.py:136 */
  unsigned long long n_unpred;      /* K */
  unsigned long long bit_length;    /* code stream length in bits */
  unsigned long long zeros_decoded; /* decompress: count(code == 0) */
  unsigned long long used;          /* decompress: verbatim values consumed */
  long long decoded;                /* decompress: symbols decoded */
  int status;                       /* EBZ_ST_* bits */
  int max_len;                      /* longest codeword */
  unsigned int blocks_done;         /* internal (range reduction) */
  unsigned int pad0;
  unsigned long long total_bytes;   /* container size */
} EbzInfo;

typedef struct EbzCtx EbzCtx;

int ebz_abi_version(void);
/* Creates a context bound to `device` (workspaces grow on demand).
 * Returns NULL if the device is unusable; ebz_last_error() says why. */
EbzCtx* ebz_ctx_create(int device);
void ebz_ctx_destroy(EbzCtx* ctx);
/* Returns every slot's device workspace (and the context scratch) to the
 * driver after synchronising the device; slots re-grow on their next use.
 * For long-running callers: workspaces otherwise stay resident, bounded by
 * the slots in use (compress_many / decompress_many use two groups' worth). */
int ebz_ctx_trim(EbzCtx* ctx);
const char* ebz_last_error(void);
/* number of SMs, device name (for reporting) */
int ebz_device_info(EbzCtx* ctx, int* sms, char* name, int name_len);

/* ---- kernel seam (device pointers) ------------------------------------ */

/* min/max/isfinite over n elements, then eb = min(abs, rel*range).
 * Writes into *d_info (device).  Async.   [core.py:132-178] */
int ebz_grid_range(EbzCtx* ctx, const void* d_values, int width, uint64_t n, int has_abs,
                   double abs_bound, int has_rel, double rel_bound, EbzInfo* d_info,
                   void* stream);

/* Predict + quantize every point in scan order: codes (u8/u16) and, when
 * d_recon != NULL, the reconstruction of every point (T[n], the reference's
 * recon output, _kernels.py:71,77; pass NULL to skip the store).  Always
 * writes K (the code-0 count, the reference's return value) into
 * d_info->n_unpred; the histogram u64[2^m] goes to d_hist when given
 * (zeroed and filled) and to a private scratch otherwise.  eb is read from
 * d_info->eb.  Async.   [_kernels.py:48-80, codec.py:107] */
int ebz_compress_scan(EbzCtx* ctx, const void* d_values, int width, int ndim,
                      const uint64_t* dims, int layers, int m, void* d_codes, void* d_recon,
                      unsigned long long* d_hist, EbzInfo* d_info, void* stream);

/* Mirror scan.  d_rowbase (optional, may be NULL): u64 zero-rank per row;
 * computed internally when NULL.  Async.   [_kernels.py:83-105] */
int ebz_decompress_scan(EbzCtx* ctx, const void* d_codes, int width, int ndim,
                        const uint64_t* dims, int layers, int m, const void* d_unpred,
                        uint64_t n_unpred, void* d_recon, EbzInfo* d_info, void* stream);

/* Huffman lengths (two-queue merge == reference heap order) + canonical
 * words from a u64 histogram.  Async.   [entropy.py:50-136] */
int ebz_build_code(EbzCtx* ctx, const unsigned long long* d_hist, int m, uint8_t* d_lengths,
                   unsigned long long* d_words, EbzInfo* d_info, void* stream);

/* Encode n codes MSB-first into d_bits (capacity bits_cap bytes) and gather
 * the code-0 values of d_values (scan order) into d_unpred.  Sizes in
 * d_info (bit_length, n_unpred).  Async.   [entropy.py:139-157, codec.py:119] */
int ebz_pack_bits(EbzCtx* ctx, const void* d_codes, int m, uint64_t n, const void* d_values,
                  int width, const uint8_t* d_lengths, const unsigned long long* d_words,
                  uint8_t* d_bits, size_t bits_cap, void* d_unpred, EbzInfo* d_info,
                  void* stream);

/* Decode exactly n symbols from nbytes of MSB-first bits (the whole byte
 * buffer is the bit budget, entropy.py:171-175).  Status bits
 * EXHAUSTED / INVALID as the reference.  Async.   [_kernels.py:151-183] */
int ebz_unpack_bits(EbzCtx* ctx, const uint8_t* d_bits, uint64_t nbytes,
                    const uint8_t* d_lengths, int m, uint64_t n, void* d_codes,
                    EbzInfo* d_info, void* stream);

/* ---- reference kernel seam on HOST buffers ------------------------------
 * One entry point per numba kernel of ebzip/_kernels.py, taking exactly that
 * kernel's arguments (caller-allocated host arrays, outputs filled in place;
 * codes / symbols are int32 as in the reference, codec.py:102 /
 * entropy.py:140) plus the array lengths a C signature needs.  The kernel's
 * own return value goes to *result; the int return is EBZ_OK or an EBZ_E_*
 * code (ebz_last_error() says why).  The stencil bank (deltas, coeffs,
 * starts, counts) must be codec._stencil_bank(layers, dims) (codec.py:54-89):
 * the device kernels derive the same bank from the geometry and any other
 * bank is rejected (EBZ_E_ARG).  `center` must be 2^(m-1), 2 <= m <= 16
 * (quantizer.py:16-18).  Synchronous.  Bound from Python by
 * paper_1706_03791_b200/kernels.py. */

/* compress_scan(values, recon, codes, deltas, coeffs, starts, counts, dims,
 * layers, center, bound) -> K          [_kernels.py:48-80] */
int ebz_ref_compress_scan(EbzCtx* ctx, const void* values, int width, void* recon,
                          int32_t* codes, const int64_t* deltas, const double* coeffs,
                          int64_t nterms, const int64_t* starts, const int64_t* counts,
                          int64_t nslots, const int64_t* dims, int ndim, int64_t layers,
                          int64_t center, double bound, long long* result);
/* decompress_scan(codes, recon, unpredictable, deltas, coeffs, starts,
 * counts, dims, layers, center, bound) -> used | -1   [_kernels.py:83-105] */
int ebz_ref_decompress_scan(EbzCtx* ctx, const int32_t* codes, void* recon, int width,
                            const void* unpred, uint64_t n_unpred, const int64_t* deltas,
                            const double* coeffs, int64_t nterms, const int64_t* starts,
                            const int64_t* counts, int64_t nslots, const int64_t* dims, int ndim,
                            int64_t layers, int64_t center, double bound, long long* result);
/* pack_bits(symbols, code_words, code_lens, out) -> total bits; code_words
 * must be the canonical words of code_lens (entropy.py:50-65, the only
 * words the reference passes)            [_kernels.py:124-148] */
int ebz_ref_pack_bits(EbzCtx* ctx, const int32_t* symbols, uint64_t n,
                      const unsigned long long* code_words, const uint8_t* code_lens,
                      uint64_t nsym, uint8_t* out, uint64_t out_bytes, long long* total);
/* unpack_bits(data, n_bits, first_codes, level_counts, level_base,
 * ordered_symbols, max_len, out) -> count | -1 exhausted | -2 invalid; the
 * tables are CodeLengthTable._decode_tables (entropy.py:67-84, 65 entries
 * each), n_bits = 8 * len(data) as entropy.decode passes it
 *                                        [_kernels.py:151-183] */
int ebz_ref_unpack_bits(EbzCtx* ctx, const uint8_t* data, uint64_t nbytes, uint64_t n_bits,
                        const unsigned long long* first_codes, const int64_t* level_counts,
                        const int64_t* level_base, const int32_t* ordered, uint64_t n_ordered,
                        int max_len, int32_t* out, uint64_t count, long long* result);
/* original_hits(values, deltas, coeffs, starts, counts, dims, layers,
 * bound) -> hits                         [_kernels.py:108-121] */
int ebz_ref_original_hits(EbzCtx* ctx, const void* values, int width, const int64_t* deltas,
                          const double* coeffs, int64_t nterms, const int64_t* starts,
                          const int64_t* counts, int64_t nslots, const int64_t* dims, int ndim,
                          int64_t layers, double bound, long long* result);

/* ---- one-shots ---------------------------------------------------------- */

/* Full compress of one grid.  values: host pointer (on_host=1, copied H2D
 * inside) or device pointer.  Results stay in context slot `slot`; this call
 * synchronises the stream and fills *h_info (sizes + status).
 * [codec.py:92-136] */
int ebz_compress(EbzCtx* ctx, int slot, const void* values, int on_host, int width, int ndim,
                 const uint64_t* dims, int layers, int m, int has_abs, double abs_bound,
                 int has_rel, double rel_bound, void* stream, EbzInfo* h_info);
/* ebz_compress with flags.  EBZ_FLAG_TRUNCATE: the opt-in truncated-mantissa
 * coding of unpredictable values (north_star (3); NOT the reference's format:
 * the slot's verbatim values are trunc(v) -- sign, exponent and the top
 * clamp(e(v) - e(eb), 0, M) mantissa bits, |v - trunc(v)| < eb -- and the
 * compressor predicts from them; containers carrying it are version 2,
 * packed by ebz_tr_pack). */
#define EBZ_FLAG_TRUNCATE 1
/* The version-2 verbatim block: K values as sign + exponent fields (9 / 12
 * bits) then their kept mantissa bits, MSB first, byte padded.  Host
 * buffers, synchronous.  ebz_tr_pack with h_out == NULL only sizes it
 * (*out_bits).  ebz_tr_unpack fails (EBZ_E_ARG) unless nbytes is exactly the
 * size the header fields imply. */
int ebz_tr_pack(EbzCtx* ctx, const void* h_values, uint64_t k, int width, double eb,
                uint8_t* h_out, uint64_t out_cap, uint64_t* out_bits);
int ebz_tr_unpack(EbzCtx* ctx, const uint8_t* h_in, uint64_t nbytes, uint64_t k, int width,
                  double eb, void* h_values);
int ebz_compress_flags(EbzCtx* ctx, int slot, const void* values, int on_host, int width,
                       int ndim, const uint64_t* dims, int layers, int m, int flags, int has_abs,
                       double abs_bound, int has_rel, double rel_bound, void* stream,
                       EbzInfo* h_info);

/* Same pipeline, fully asynchronous (no host sync; no size readback).  The
 * device-resident path used for throughput measurement. */
int ebz_compress_async(EbzCtx* ctx, int slot, const void* d_values, int width, int ndim,
                       const uint64_t* dims, int layers, int m, int has_abs, double abs_bound,
                       int has_rel, double rel_bound, void* stream);

/* Copy the products of the last compress in `slot` to host buffers:
 * container head (header + length table, header_bytes = 36 + 8d + 2^m),
 * code bits (ceil(bit_length/8) bytes) and the K verbatim values.
 * Any pointer may be NULL to skip that part.  Synchronous. */
/* Interval-count trials -- replaces the CLI's --auto-m loop of full
 * compressions (ebzip/cli.py:146-154) with ONE batched predict/quantize
 * sweep over the candidate exponents ms[0..ntrials) (per-field m, same
 * input, same bound).  Trial i occupies slot slot0 + i; after the stream is
 * synchronised, ebz_slot_info(slot0 + i) gives its eb, status and K
 * (n_unpred), hence the hitting rate the loop tests.  The caller picks a
 * trial and runs ebz_compress_trial_finish on it; the other trial slots are
 * scratch. */
int ebz_compress_trials(EbzCtx* ctx, int slot0, const void* values, int on_host, int width,
                        int ndim, const uint64_t* dims, int layers, int ntrials, const int* ms,
                        int has_abs, double abs_bound, int has_rel, double rel_bound,
                        void* stream);
/* Histogram, codebook and encoder of the chosen trial (codec.py:107-119):
 * afterwards the slot is a compressed field exactly as ebz_compress at that
 * exponent leaves it (ebz_compress_fetch); h_info receives its record. */
int ebz_compress_trial_finish(EbzCtx* ctx, int slot, void* stream, EbzInfo* h_info);
int ebz_compress_fetch(EbzCtx* ctx, int slot, uint8_t* h_head, uint8_t* h_bits,
                       void* h_unpred, void* stream);

/* Device pointers to the products of the last compress in `slot`. */
int ebz_compress_outputs(EbzCtx* ctx, int slot, const uint8_t** d_head, const uint8_t** d_bits,
                         const void** d_unpred, const EbzInfo** d_info);

/* Full decompress.  Inputs as host pointers (on_host=1) or device pointers.
 * recon_out: host (on_host=1) or device pointer of n elements.  Synchronises
 * and fills *h_info.   [codec.py:139-160] */
int ebz_decompress(EbzCtx* ctx, int slot, int on_host, int width, int ndim, const uint64_t* dims,
                   int layers, int m, double eb, const uint8_t* lengths, const uint8_t* bits,
                   uint64_t nbytes, const void* unpred, uint64_t n_unpred, void* recon_out,
                   void* stream, EbzInfo* h_info);

/* Fully asynchronous decompress of the products held in compress slot
 * `src_slot` into device buffer d_recon (round-trip throughput path). */
int ebz_decompress_async(EbzCtx* ctx, int slot, int src_slot, void* d_recon, void* stream);

/* Batched device-resident pipelines for many fields of one geometry (the
 * reference's cfg5 workload: 64 independent 256^3 fields, each a separate
 * ebzip.codec.compress call, codec.py:92-136 / decompress, codec.py:139-160).
 * d_values / d_recon are HOST arrays of nfields DEVICE pointers.  Field i
 * uses slot slot0 + i (decompress: reads compress slot src_slot0 + i).  The
 * predict/quantize sweeps of all fields run as one persistent launch; the
 * per-field stages run on internal streams joined back to `stream`.
 * Asynchronous; results per slot as for ebz_compress_async. */
int ebz_compress_batch(EbzCtx* ctx, int slot0, int nfields, const void* const* d_values,
                       int width, int ndim, const uint64_t* dims, int layers, int m, int has_abs,
                       double abs_bound, int has_rel, double rel_bound, void* stream);
int ebz_decompress_batch(EbzCtx* ctx, int slot0, int src_slot0, int nfields,
                         void* const* d_recon, void* stream);

/* Batched decompress of caller-supplied device products (one container per
 * field, all of one geometry): per field the code-length table, the code
 * bytes (nbytes, budget 8 * nbytes as entropy.py:171-175), the K verbatim
 * values and eb.  Field i uses slot slot0 + i and writes d_recon[i].  The
 * host arrays eb / n_unpred / nbytes and the pointer arrays are read during
 * the call.  Asynchronous; per-field status via ebz_slot_info_async(.., 1, ..). */
int ebz_decompress_batch_ptrs(EbzCtx* ctx, int slot0, int nfields, int width, int ndim,
                              const uint64_t* dims, int layers, int m, const double* eb,
                              const uint64_t* n_unpred, const uint8_t* const* d_lengths,
                              const uint8_t* const* d_bits, const uint64_t* nbytes,
                              const void* const* d_unpred, void* const* d_recon, void* stream);

/* Stream-ordered copy between any host/device pointers (cudaMemcpyDefault;
 * asynchronous when the host side is pinned). */
int ebz_copy_async(EbzCtx* ctx, void* dst, const void* src, size_t nbytes, void* stream);

/* Asynchronous read-back of a slot's compress record (decode_record = 0) or
 * decompress record (1) into h_info (pinned for true asynchrony). */
int ebz_slot_info_async(EbzCtx* ctx, int slot, int decode_record, EbzInfo* h_info,
                        void* stream);

/* Asynchronous copy of a compressed slot's products to host buffers, sized
 * from a record already read back (ebz_slot_info_async). */
int ebz_compress_fetch_async(EbzCtx* ctx, int slot, const EbzInfo* h_info, uint8_t* h_head,
                             uint8_t* h_bits, void* h_unpred, void* stream);

/* ---- analysis callers of the path -------------------- */

/* Number of points whose prediction from the ORIGINAL neighbours lies within
 * `bound` (ebzip/_kernels.py:108-121, original_hits; used by
 * ebzip/analysis.py:109-141 best_layer_scan).  Device values, synchronous. */
int ebz_original_hits(EbzCtx* ctx, const void* d_values, int width, int ndim,
                      const uint64_t* dims, int layers, double bound, uint64_t* h_hits,
                      void* stream);

/* Fused distortion reductions of an original / reconstructed pair on the
 * device (ebzip/metrics.py:93-137).  h_out receives 9 + lags doubles:
 * [max |a-b|, sum e^2, sum a, sum b, sum e, sum (a-ma)(b-mb), sum (a-ma)^2,
 *  sum (b-mb)^2, sum c^2, sum_i c_i c_{i+1}, ..., sum_i c_i c_{i+lags}] with
 * e = a - b and c = e - mean(e), all in binary64.  Synchronous. */
#define EBZ_MAX_LAGS 1024
int ebz_metrics(EbzCtx* ctx, const void* d_a, const void* d_b, int width, uint64_t n, int lags,
                double* h_out, void* stream);

/* Read back slot info (synchronous): the compress record, or the decompress
 * record (status, verbatim values consumed) of the slot's last decompress. */
int ebz_slot_info(EbzCtx* ctx, int slot, EbzInfo* h_info, void* stream);
int ebz_slot_decode_info(EbzCtx* ctx, int slot, EbzInfo* h_info, void* stream);

/* Kernel launches issued by this context since creation (instrumentation
 * for bench.py's gpu_launches). */
unsigned long long ebz_launch_count(EbzCtx* ctx);

/* Test hook: set the launch-epoch counter (the next sweep launch uses
 * epoch + 1; after kEpochMax = ebz_epoch_max() it wraps to 1 and every slot
 * re-zeroes its epoch-tagged face / progress buffers before its next launch).
 * Lets a test drive the wrap and check the re-zeroing (tests/
 * test_gpu_cfg5.py).  Setting it backwards can make words of earlier launches
 * look current in slots used since: tests use fresh slots.  Returns the old
 * value. */
unsigned int ebz_debug_set_epoch(EbzCtx* ctx, unsigned int epoch);
unsigned int ebz_epoch_max(void);

/* Which predict/quantize sweep kernel a launch of nfields float-width fields
 * of this geometry runs (the dispatch of ebz_compress* / ebz_decompress*; no
 * device work): 0 generic hyperplane kernel, 1 one-row register wavefront
 * (2D / 3D, n <= 2), 2 two-row 8 x 8 patches (3D n = 1 compress, shortest
 * ramp), 3 z-rows 32 x 4 patches (3D n = 1 compress, highest throughput),
 * 4 block-speculative low-latency wavefront (2D n <= 2, float32 and binary64,
 * csrc/sweep2.cu), 5 one-row 3D n = 1 patch wavefront with 16-byte face words
 * (csrc/sweep3b.cu: binary64 fields, and float32 compress of lone fields).
 * Every kernel writes identical bytes; for 3D n = 1 float32 compress a fitted
 * time model picks among kernels 2, 3 and 5 from the shape and the field
 * count (csrc/sweep3.cu sweep3_model_choice). */
int ebz_sweep_kernel_choice(int width, int ndim, const uint64_t* dims, int layers, int nfields,
                            int compress);

/* In-stream stage timing: when enabled, every pipeline stage is bracketed by
 * CUDA events recorded on its launching stream.  Stages: 0 range, 1 compress
 * sweep, 2 Huffman build, 3 encode, 4 decode, 5 zero ranks, 6 decompress
 * sweep.  ebz_stage_times synchronises on the recorded events, returns the
 * summed milliseconds and bracket counts per stage, and clears them. */
int ebz_profile(EbzCtx* ctx, int enable);
int ebz_stage_times(EbzCtx* ctx, double* ms, unsigned long long* counts, int nstages);

#ifdef __cplusplus
}
#endif
#endif /* EBZ200_H */
