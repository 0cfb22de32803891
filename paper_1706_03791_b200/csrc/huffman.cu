// huffman.cu -- canonical Huffman codebook on the device (one CTA).
//
// Reference: entropy.build_code (ebzip/entropy.py:87-136) pops a heap keyed
// by (count, serial) where leaves carry serial = symbol and merged nodes get
// serials 2^m, 2^m+1, ... in creation order; CodeLengthTable.code_words
// (entropy.py:50-65) assigns canonical words by (length, symbol).
//
// Device restatement:
//  1. compact the used symbols into 64-bit keys (count << 16 | symbol) --
//     unique, so any sort is stable enough;
//  2. bitonic-sort the keys (shared memory when they fit, else L2);
//  3. two-queue merge in one thread: sorted leaves vs. a FIFO of merged
//     nodes, the leaf winning ties.  Merged weights are non-decreasing in
//     creation order, so the FIFO front is the minimal merged node and this
//     pops exactly the reference heap's sequence;
//  4. depths by walking parents in reverse creation order; > 64 -> error;
//  5. canonical words: first_code[L] + rank of the symbol among length-L
//     symbols in symbol order (warp-wide match_any ranking).
#include <cstdio>

#include "ebz_common.cuh"

namespace {

constexpr int kThreads = 1024;
constexpr int kSmemKeys = 4096;  // used symbols whose merge state fits in smem
// dynamic smem: keys u64[4096] | wint u64[4096] | parent int[8192] | depth u8[8192]
constexpr size_t kDynSmem = 4096 * 8 + 4096 * 8 + 8192 * 4 + 8192;

// n <= kThreads (every alphabet up to m = 10): one key per thread in a
// register; partners closer than a warp are exchanged by shuffles, farther
// ones through shared memory -- 6 block barriers for 256 keys instead of 36.
// Same network, same result as bitonic_sort.
__device__ void bitonic_sort_reg(unsigned long long* keys, int n /*pow2 <= kThreads*/) {
  const int i = threadIdx.x;
  unsigned long long v = i < n ? keys[i] : ~0ull;
  for (int k = 2; k <= n; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      unsigned long long u;
      if (j >= 32) {
        __syncthreads();
        keys[i] = v;
        __syncthreads();
        u = keys[i ^ j];
      } else {
        u = __shfl_xor_sync(EBZ_FULL, v, j);
      }
      const bool up = (i & k) == 0, lower = (i & j) == 0;
      v = (lower == up) ? (u < v ? u : v) : (u > v ? u : v);
    }
  }
  __syncthreads();
  if (i < n) keys[i] = v;
  __syncthreads();
}

__device__ void bitonic_sort(unsigned long long* keys, int n /*pow2*/) {
  for (int k = 2; k <= n; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const int p = i ^ j;
        if (p > i) {
          const unsigned long long a = keys[i], b = keys[p];
          const bool up = (i & k) == 0;
          if ((a > b) == up) {
            keys[i] = b;
            keys[p] = a;
          }
        }
      }
      __syncthreads();
    }
  }
}

struct HuffTab {  // per-field pointers of a batched launch (one CTA per field)
  const unsigned long long* hist[kBatchMax];
  Info* info[kBatchMax];
  uint8_t* lengths[kBatchMax];
  unsigned long long* words[kBatchMax];
  unsigned long long* scratch[kBatchMax];
};

__global__ void __launch_bounds__(kThreads)
huffman_build_kernel(const __grid_constant__ HuffTab tab, int m) {
  const unsigned long long* __restrict__ hist = tab.hist[blockIdx.x];
  Info* info = tab.info[blockIdx.x];
  uint8_t* __restrict__ lengths = tab.lengths[blockIdx.x];
  unsigned long long* __restrict__ words = tab.words[blockIdx.x];
  unsigned long long* __restrict__ gscratch = tab.scratch[blockIdx.x];
  const int nsym = 1 << m;
#ifdef EBZ_HUFF_CLOCKS
  long long hc[8];
  int hn = 0;
  hc[hn++] = clock64();
#define EBZ_HC() if (hn < 8) hc[hn++] = clock64()
#else
#define EBZ_HC()
#endif
  extern __shared__ unsigned long long s_dyn[];
  unsigned long long* s_keys = s_dyn;
  __shared__ int s_cnt[kThreads];
  __shared__ int s_total;
  __shared__ int s_fail;
  __shared__ unsigned long long s_first[66];
  __shared__ int s_level[66];
  __shared__ int s_maxlen;
  __shared__ int s_run[66];

  // ---- 1. compact used symbols (contiguous segment per thread) -------------
  const int per = (nsym + kThreads - 1) / kThreads;
  const int lo = threadIdx.x * per;
  const int hi = min(lo + per, nsym);
  int mine = 0;
  for (int s = lo; s < hi; ++s) mine += hist[s] > 0;
  {  // block-wide exclusive scan of the per-thread counts (was one thread
     // walking 1024 shared entries: ~15 us of a single-field compress)
    __shared__ int s_wsum[kThreads / 32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int x = mine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(EBZ_FULL, x, o);
      if (lane >= o) x += t;
    }
    if (lane == 31) s_wsum[wid] = x;
    __syncthreads();
    if (wid == 0) {
      int y = s_wsum[lane];  // kThreads / 32 == 32 warps
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(EBZ_FULL, y, o);
        if (lane >= o) y += t;
      }
      s_wsum[lane] = y - s_wsum[lane];  // exclusive warp offsets
      if (lane == 31) s_total = y;
    }
    __syncthreads();
    s_cnt[threadIdx.x] = s_wsum[wid] + x - mine;
    if (threadIdx.x == 0) s_fail = 0;
    static_assert(kThreads == 1024, "one warp scans the 32 warp totals");
  }
  __syncthreads();
  EBZ_HC();
  const int U = s_total;
  int npow = 1;
  while (npow < U) npow <<= 1;
  unsigned long long* keys = npow <= kSmemKeys ? s_keys : gscratch;
  {
    int w = s_cnt[threadIdx.x];
    for (int s = lo; s < hi; ++s)
      if (hist[s] > 0) keys[w++] = (hist[s] << 16) | (unsigned long long)s;
  }
  for (int i = U + threadIdx.x; i < npow; i += kThreads) keys[i] = ~0ull;
  for (int s = threadIdx.x; s < nsym; s += kThreads) lengths[s] = 0;
  __syncthreads();
  if (U == 0) {
    if (threadIdx.x == 0) atomicOr(&info->status, ST_EMPTY_HIST);
    return;
  }
  if (U == 1) {
    // lone symbol: one bit (entropy.py:110-114)
    if (threadIdx.x == 0) {
      const int s = (int)(keys[0] & 0xffff);
      lengths[s] = 1;
    }
    __syncthreads();
  } else {
    // ---- 2. sort ------------------------------------------------------------
    EBZ_HC();
    if (npow <= kThreads) bitonic_sort_reg(keys, npow);
    else bitonic_sort(keys, npow);
    EBZ_HC();
    // ---- 3 + 4. two-queue merge and depths -------------------------------
    if (npow <= kThreads) {
      // (a) merge in one thread with both queue fronts in registers: the
      // next two leaves (prefetched) and the two oldest merged nodes
      // (measured: the smem-resident fronts cost ~320 cycles per merge);
      // (b) depths by pointer jumping over all nodes in parallel (was a
      // dependent walk, ~100 cycles per node); (c) lengths stored in
      // parallel.  Same merge order, same depths, same failure rule.
      unsigned long long* wint = s_dyn + kSmemKeys;
      int* parent = reinterpret_cast<int*>(wint + U);
      int* jb = reinterpret_cast<int*>(s_dyn + kSmemKeys + 3072);  // past the merge state
      int* anc[2] = {jb, jb + 2048};
      int* dd[2] = {jb + 4096, jb + 6144};
      __shared__ int s_root;
      if (threadIdx.x == 0) {
        constexpr unsigned long long INF = ~0ull;  // weights are < 2^48
        auto lw = [&](int i) { return i < U ? (keys[i] >> 16) : INF; };
        int li = 0, ii = 0, ni = 0;
        unsigned long long la = lw(0), la1 = lw(1), ia = INF, ia1 = INF;
        for (int step = 0; step < U - 1; ++step) {
          int pick[2];
          unsigned long long wsum = 0;
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            if (li < U && la <= ia) {  // leaf wins ties; ia = INF: FIFO empty
              wsum += la;
              pick[q] = li++;
              la = la1;
              la1 = lw(li + 1);
            } else {
              wsum += ia;
              pick[q] = U + ii++;
              ia = ia1;
              ia1 = ii + 1 < ni ? wint[ii + 1] : INF;
            }
          }
          parent[pick[0]] = U + ni;
          parent[pick[1]] = U + ni;
          wint[ni] = wsum;
          if (ii == ni) ia = wsum;            // the new node is the FIFO front
          else if (ii + 1 == ni) ia1 = wsum;  // ... or right behind it
          ++ni;
        }
        s_root = U + ni - 1;  // created last
      }
      __syncthreads();
      EBZ_HC();
      const int root = s_root;
      for (int id = threadIdx.x; id <= root; id += kThreads) {
        anc[0][id] = id == root ? root : parent[id];
        dd[0][id] = id == root ? 0 : 1;
      }
      __syncthreads();
      int cur = 0;
      for (int r = 0; r < 7; ++r) {  // distances up to 2^7 > 64
        for (int id = threadIdx.x; id <= root; id += kThreads) {
          const int a = anc[cur][id];
          anc[cur ^ 1][id] = anc[cur][a];
          dd[cur ^ 1][id] = dd[cur][id] + dd[cur][a];
        }
        __syncthreads();
        cur ^= 1;
      }
      bool bad = false;
      for (int id = threadIdx.x; id <= root; id += kThreads)
        bad |= anc[cur][id] != root || dd[cur][id] > 64;
      if (__syncthreads_or(bad)) {
        if (threadIdx.x == 0) {
          s_fail = 1;
          atomicOr(&info->status, ST_DEPTH_GT_64);
        }
      } else {
        for (int li2 = threadIdx.x; li2 < U; li2 += kThreads)
          lengths[keys[li2] & 0xffff] = (uint8_t)dd[cur][li2];
      }
      EBZ_HC();
    } else if (threadIdx.x == 0) {  // large alphabets: one thread, smem or L2
      // merge state: smem when small, else L2 scratch after the keys
      // [wint: U u64][parent: 2U int][depth: 2U uint8]
      unsigned long long* base =
          npow <= kSmemKeys ? s_dyn + kSmemKeys : gscratch + npow;
      unsigned long long* wint = base;
      int* parent = reinterpret_cast<int*>(wint + U);
      uint8_t* depth = reinterpret_cast<uint8_t*>(parent + 2 * U);
      int li = 0, ii = 0, ni = 0;
      for (int step = 0; step < U - 1; ++step) {
        int pick[2];
        unsigned long long wsum = 0;
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const bool take_leaf =
              li < U && (ii >= ni || (keys[li] >> 16) <= wint[ii]);  // leaf wins ties
          if (take_leaf) {
            wsum += keys[li] >> 16;
            pick[q] = li++;
          } else {
            wsum += wint[ii];
            pick[q] = U + ii++;
          }
        }
        parent[pick[0]] = U + ni;
        parent[pick[1]] = U + ni;
        wint[ni++] = wsum;
      }
      EBZ_HC();
      // depths: root = U + ni - 1 (created last), children before parents
      const int root = U + ni - 1;
      int fail = 0;
      depth[root] = 0;
      for (int id = root - 1; id >= 0; --id) {
        const int d = depth[parent[id]] + 1;
        if (d > 64) { fail = 1; depth[id] = 255; continue; }
        depth[id] = (uint8_t)d;
      }
      EBZ_HC();
      if (!fail)
        for (int li2 = 0; li2 < U; ++li2) lengths[keys[li2] & 0xffff] = depth[li2];
      EBZ_HC();
      if (fail) {
        s_fail = 1;
        atomicOr(&info->status, ST_DEPTH_GT_64);
      }
    }
    __syncthreads();
    if (s_fail) return;
  }
  __syncthreads();

  // ---- 5. canonical words -----------------------------------------------
  if (threadIdx.x < 66) { s_level[threadIdx.x] = 0; s_first[threadIdx.x] = 0; }
  if (threadIdx.x == 0) s_maxlen = 0;
  __syncthreads();
  for (int s = threadIdx.x; s < nsym; s += kThreads) {
    const int l = lengths[s];
    if (l) {
      atomicAdd(&s_level[l], 1);
      atomicMax(&s_maxlen, l);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long w = 0;
    for (int l = 1; l <= s_maxlen; ++l) {
      w <<= 1;
      s_first[l] = w;
      w += (unsigned long long)s_level[l];
    }
    info->max_len = s_maxlen;
  }
  __syncthreads();
  // rank within level in symbol order: one warp sweeps the alphabet
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    for (int i = lane; i < 66; i += 32) s_run[i] = 0;
    __syncwarp();
    for (int s0 = 0; s0 < nsym; s0 += 32) {
      const int s = s0 + lane;
      const int l = s < nsym ? lengths[s] : 0;
      const unsigned int peers = __match_any_sync(EBZ_FULL, l);
      const int before = __popc(peers & ((1u << lane) - 1u));
      const int run = s_run[l];
      if (s < nsym) words[s] = l ? s_first[l] + (unsigned long long)(run + before) : 0ull;
      __syncwarp();
      if (l && before == 0) s_run[l] = run + __popc(peers);
      __syncwarp();
    }
  }
#ifdef EBZ_HUFF_CLOCKS
  EBZ_HC();
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    printf("EBZHUFF U-phases:");
    for (int q = 1; q < hn; ++q) printf(" %lld", hc[q] - hc[q - 1]);
    printf(" total %lld\n", hc[hn - 1] - hc[0]);
  }
#endif
}

}  // namespace

size_t huffman_scratch_bytes(int m) {
  const size_t nsym = (size_t)1 << m;
  size_t npow = 1;
  while (npow < nsym) npow <<= 1;
  return npow * 8 + nsym * 8 + nsym * 2 * 4 + nsym * 2 + 64;
}

cudaError_t launch_huffman_batch(const unsigned long long* const* hist, Info* const* info,
                                 uint8_t* const* lengths, unsigned long long* const* words,
                                 unsigned long long* const* scratch, int nf, int m,
                                 cudaStream_t s) {
  if (nf < 1 || nf > kBatchMax) return cudaErrorInvalidValue;
  static KernelAttr attr;
  const cudaError_t e = kernel_smem(attr, huffman_build_kernel, kDynSmem);
  if (e != cudaSuccess) return e;
  HuffTab tab;
  for (int f = 0; f < nf; ++f) {
    tab.hist[f] = hist[f];
    tab.info[f] = info[f];
    tab.lengths[f] = lengths[f];
    tab.words[f] = words[f];
    tab.scratch[f] = scratch[f];
  }
  huffman_build_kernel<<<nf, kThreads, kDynSmem, s>>>(tab, m);
  return cudaGetLastError();
}

cudaError_t launch_huffman_build(const unsigned long long* hist, int m, Info* info,
                                 uint8_t* lengths, unsigned long long* words,
                                 unsigned long long* scratch, size_t scratch_bytes,
                                 cudaStream_t s) {
  (void)scratch_bytes;
  return launch_huffman_batch(&hist, &info, &lengths, &words, &scratch, 1, m, s);
}
