// Snapshot delta fold on the GPU (the step after the recovery remap).
//
// Reference: StandbyInstance.fold (pkg/src/mpssim/recovery.py:83-92) consumes the ring's
// ForwardSnapshots in order; per request (dict insertion order = first appearance) it appends
// the KV-block-id and token deltas, keeps the last progress and a sticky done flag.
// complete_wake (recovery.py:310-363) then restores each request's block table from the fold.
//
// Batch form: S snapshots in consume order as SoA (request id or NO_REQ, delta lengths,
// progress, done) plus the concatenated deltas.  The fold is a stable group-by with
// variable-length payloads.  Every primitive is written here (no library sort or scan).  Id
// spaces up to 2^17 take the bucketed path (further below: one scatter into 256-id buckets,
// then chunk-local work); larger ones this radix path, whose tiles are 8192 snapshots:
//   k_fold_init     clear the per-request tables and the head bitmap
//   k_fold_stats    consume order: per request id first snapshot and sticky done
//                   (fire-and-forget reductions); the block scan of the packed delta lengths
//                   gives each snapshot's source offset inside the tile (meta, with its lengths)
//                   and the tile total
//   k_fold_bits     a request's first snapshot sets its bit in an S-bit head bitmap
//   k_fold_bitcnt   per 8192-bit chunk of the bitmap: word prefixes inside the chunk, chunk total
//   k_fold_scan     one CTA per small array (chunk totals, tile totals): exclusive prefix
//   k_fold_rank     per request: rank = heads before its first snapshot (first-appearance
//                   order); order / done at the rank
//   radix sort      snapshot indices by request rank, stable LSD over the bits min(R, S) needs
//                   (<= 9 bits per pass): k_sort_hist (per-tile digit counts) -> k_sort_hscan
//                   (per-digit prefix over tiles) -> k_sort_scatter (per-warp digit counters,
//                   ballot-matched ranks inside a round of 32, rounds in index order: stable;
//                   the tile is staged in shared memory in digit order and written out as
//                   coalesced runs); the last pass moves each snapshot's meta into fold order
//                   with the tile base added (smeta = source offset + lengths)
//   k_fold_dsum     fold order: tile totals of the live lengths (k_fold_scan: prefix)
//   k_fold_place    fold order: the block scan of the lengths is each snapshot's destination
//                   offset; heads write the CSR start of their request, tails its last progress
//                   (the stable sort puts the request's last snapshot there), the last live snapshot
//                   the CSR end; the deltas move from source to destination warp-cooperatively
//                   (a warp's 256 snapshots have one contiguous destination range, walked 32
//                   words per coalesced store)
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdlib>

#include "mpsf_kernels.h"

namespace mpsf {

constexpr uint32_t NO_REQ = 0xFFFFFFFFu;
constexpr uint32_t FTILE = 8192;              // snapshots per tile (every tiled kernel)
constexpr int SB = 512;                       // sort blocks: 16 warps x 512 consecutive snapshots
constexpr int SIPT = FTILE / SB;
constexpr int SWARPS = SB / 32;
constexpr uint32_t WITEMS = FTILE / SWARPS;
constexpr int CB = 1024;                      // consume / sorted-order tile blocks: 8 per thread
constexpr int CIPT = FTILE / CB;
constexpr int CWARPS = CB / 32;
constexpr int DB_MAX = 9;                     // radix bits per pass
constexpr uint32_t NB_MAX = 1u << DB_MAX;     // digits per pass (<= SB: one per thread)
static_assert(NB_MAX <= (uint32_t)SB, "one digit per thread");
constexpr uint32_t CHUNK_WORDS = 256;         // head-bitmap chunk (8192 bits)

struct FoldDev {            // device-side totals, read back once
  unsigned long long n_requests, n_blocks, n_tokens;
  uint32_t err;             // first snapshot with a request id >= R (NO_REQ: none)
  uint32_t overrun;         // deltas reach past the payload arrays
};

__device__ __forceinline__ unsigned long long pack_len(uint32_t nb, uint32_t nt) {
  return (unsigned long long)nb | ((unsigned long long)nt << 32);
}

template <typename T>
__device__ __forceinline__ T warp_incl_scan(T v) {
  const uint32_t lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const T u = __shfl_up_sync(0xFFFFFFFFu, v, o);
    if (lane >= (uint32_t)o) v += u;
  }
  return v;
}

// Exclusive scan of one value per thread over the block (blockDim.x = 32 * NW); sw holds NW + 1.
template <typename T, int NW>
__device__ __forceinline__ T block_excl_scan(T v, T* sw, T& total) {
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const T inc = warp_incl_scan(v);
  if (lane == 31) sw[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    const T w = lane < (uint32_t)NW ? sw[lane] : T(0);
    const T wi = warp_incl_scan(w);
    if (lane < (uint32_t)NW) sw[lane] = wi - w;
    if (lane == NW - 1) sw[NW] = wi;
  }
  __syncthreads();
  const T ex = sw[warp] + inc - v;
  total = sw[NW];
  __syncthreads();   // sw reusable
  return ex;
}

// Programmatic dependent launch for the bucketed chain: each kernel may be scheduled while its
// predecessor drains, and waits (griddepcontrol.wait) before reading anything it produced; a
// no-op when launched without the attribute (the radix path, kv_reserve).
__device__ __forceinline__ void fold_pdl() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

template <typename... KArgs, typename... Args>
static void launch_pdl(void (*k)(KArgs...), dim3 g, dim3 b, size_t smem, cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = g;
  cfg.blockDim = b;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...);
}

__global__ void k_fold_init(uint32_t R, uint32_t W, uint32_t* __restrict__ first, uint32_t* __restrict__ rdone,
                            uint32_t* __restrict__ bitmap, FoldDev* __restrict__ dev) {
  const uint32_t n = R > W ? R : W;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    if (i < R) {
      first[i] = NO_REQ;
      rdone[i] = 0;
    }
    if (i < W) bitmap[i] = 0;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *dev = FoldDev{0, 0, 0, NO_REQ, 0};
}

// Blocked loads of N consecutive u32 (vectorised when the run is whole and 16-byte aligned).
template <int N>
__device__ __forceinline__ void ldb(const uint32_t* __restrict__ a, uint32_t i0, uint32_t S, uint32_t (&v)[N],
                                    uint32_t dflt) {
  if (i0 + N <= S && ((reinterpret_cast<uintptr_t>(a + i0) & 15u) == 0)) {
    const uint4* p = reinterpret_cast<const uint4*>(a + i0);
#pragma unroll
    for (int q = 0; q < N / 4; ++q) {
      const uint4 x = __ldg(p + q);
      v[4 * q] = x.x; v[4 * q + 1] = x.y; v[4 * q + 2] = x.z; v[4 * q + 3] = x.w;
    }
  } else {
#pragma unroll
    for (int u = 0; u < N; ++u) v[u] = i0 + u < S ? __ldg(a + i0 + u) : dflt;
  }
}

// Consume-order tile, thread t owns [tile * FTILE + 8 t, + 8).
__global__ void __launch_bounds__(CB) k_fold_stats(uint32_t S, uint32_t R, const uint32_t* __restrict__ req,
                                                   const uint8_t* __restrict__ done, const uint32_t* __restrict__ nblk,
                                                   const uint32_t* __restrict__ ntok, uint32_t* __restrict__ first,
                                                   uint32_t* __restrict__ rdone,
                                                   uint4* __restrict__ meta, unsigned long long* __restrict__ tsum,
                                                   FoldDev* __restrict__ dev) {
  __shared__ unsigned long long sw[CWARPS + 1];
  const uint32_t i0 = blockIdx.x * FTILE + threadIdx.x * CIPT;
  uint32_t r[CIPT], nb[CIPT], nt[CIPT];
  ldb(req, i0, S, r, NO_REQ);
  ldb(nblk, i0, S, nb, 0u);
  ldb(ntok, i0, S, nt, 0u);
  unsigned long long s = 0;
#pragma unroll
  for (int u = 0; u < CIPT; ++u) s += pack_len(nb[u], nt[u]);
  unsigned long long total;
  unsigned long long run = block_excl_scan<unsigned long long, CWARPS>(s, sw, total);
  if (threadIdx.x == 0) tsum[blockIdx.x] = total;
  // each snapshot's source offset inside the tile and its lengths (the tile base is added when
  // the sort's last pass moves the word into fold order)
#pragma unroll
  for (int u = 0; u < CIPT; ++u) {
    if (i0 + u < S) __stcg(meta + i0 + u, make_uint4((uint32_t)run, (uint32_t)(run >> 32), nb[u], nt[u]));
    run += pack_len(nb[u], nt[u]);
  }
  uint2 dn = make_uint2(0, 0);
  if (i0 + CIPT <= S && ((reinterpret_cast<uintptr_t>(done + i0) & 7u) == 0)) {
    dn = __ldg(reinterpret_cast<const uint2*>(done + i0));
  } else {
    for (int u = 0; u < CIPT && i0 + u < S; ++u) (u < 4 ? dn.x : dn.y) |= (uint32_t)__ldg(done + i0 + u) << (8 * (u & 3));
  }
#pragma unroll
  for (int u = 0; u < CIPT; ++u) {
    const uint32_t i = i0 + u, rr = r[u];
    if (i >= S || rr == NO_REQ) continue;
    if (rr >= R) {   // request id outside the caller's id space: reported, not folded
      atomicMin(&dev->err, i);
      continue;
    }
    atomicMin(first + rr, i);
    if (((u < 4 ? dn.x : dn.y) >> (8 * (u & 3))) & 0xFFu) atomicOr(rdone + rr, 1u);
  }
}

__global__ void k_fold_bits(uint32_t R, const uint32_t* __restrict__ first, uint32_t* __restrict__ bitmap) {
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < R; r += gridDim.x * blockDim.x) {
    const uint32_t f = first[r];
    if (f != NO_REQ) atomicOr(bitmap + (f >> 5), 1u << (f & 31));
  }
}

// one block of 256 threads per bitmap chunk: heads before each word inside the chunk, the total
__global__ void __launch_bounds__(CHUNK_WORDS) k_fold_bitcnt(uint32_t W, const uint32_t* __restrict__ bitmap,
                                                             uint32_t* __restrict__ wloc,
                                                             unsigned long long* __restrict__ ccount) {
  fold_pdl();
  __shared__ uint32_t sw[CHUNK_WORDS / 32 + 1];
  const uint32_t w = blockIdx.x * CHUNK_WORDS + threadIdx.x;
  const uint32_t c = w < W ? __popc(bitmap[w]) : 0u;
  uint32_t tot;
  const uint32_t ex = block_excl_scan<uint32_t, CHUNK_WORDS / 32>(c, sw, tot);
  if (w < W) wloc[w] = ex;
  if (threadIdx.x == 0) ccount[blockIdx.x] = tot;
}

// One CTA of 1024 threads per small array (<= a few thousand entries): exclusive prefix, total.
__device__ __forceinline__ void scan_small(const unsigned long long* __restrict__ in, unsigned long long* __restrict__ out,
                                           uint32_t n, unsigned long long* total_out) {
  __shared__ unsigned long long sw[33];
  constexpr int K = 4;   // loads issued together
  const uint32_t per = (n + 1023) / 1024, b = threadIdx.x * per, e = min(b + per, n);
  unsigned long long s = 0;
  for (uint32_t i = b; i < e; i += K) {
    unsigned long long x[K];
#pragma unroll
    for (int q = 0; q < K; ++q) x[q] = i + q < e ? in[i + q] : 0ull;
#pragma unroll
    for (int q = 0; q < K; ++q) s += x[q];
  }
  unsigned long long total;
  unsigned long long run = block_excl_scan<unsigned long long, 32>(s, sw, total);
  for (uint32_t i = b; i < e; ++i) {
    const unsigned long long v = in[i];
    out[i] = run;
    run += v;
  }
  if (threadIdx.x == 0 && total_out) *total_out = total;
}

// block j scans array j of up to two
__global__ void __launch_bounds__(1024) k_fold_scan(const unsigned long long* __restrict__ a, unsigned long long* __restrict__ ao,
                                                    uint32_t na, unsigned long long* a_total,
                                                    const unsigned long long* __restrict__ b, unsigned long long* __restrict__ bo,
                                                    uint32_t nb) {
  fold_pdl();
  if (blockIdx.x == 0) scan_small(a, ao, na, a_total);
  else scan_small(b, bo, nb, nullptr);
}

__global__ void k_fold_rank(uint32_t R, const uint32_t* __restrict__ first, const uint32_t* __restrict__ rdone,
                            const uint32_t* __restrict__ bitmap, const uint32_t* __restrict__ wloc,
                            const unsigned long long* __restrict__ cpre, uint32_t* __restrict__ rank,
                            uint32_t* __restrict__ order, uint8_t* __restrict__ done_out) {
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < R; r += gridDim.x * blockDim.x) {
    const uint32_t f = first[r];
    if (f == NO_REQ) continue;
    const uint32_t w = f >> 5;
    const uint32_t k = (uint32_t)cpre[w / CHUNK_WORDS] + wloc[w] + __popc(bitmap[w] & ((1u << (f & 31)) - 1u));
    rank[r] = k;
    order[k] = r;
    done_out[k] = rdone[r] ? 1 : 0;
  }
}

// ---- stable LSD radix sort of snapshot indices by request rank -------------------------------
// Pass 0 reads the request ids and ranks them on the fly (key = rank, or live_bound for
// liveness-only / rejected snapshots, which sort last); its values are the snapshot indices.
__device__ __forceinline__ uint32_t key_of(uint32_t r, uint32_t R, uint32_t live_bound, const uint32_t* rank) {
  return r < R ? __ldg(rank + r) : live_bound;
}

template <bool kFirst>
__global__ void __launch_bounds__(SB) k_sort_hist(uint32_t S, uint32_t R, uint32_t live_bound,
                                                  const uint32_t* __restrict__ kin, const uint32_t* __restrict__ rank,
                                                  uint32_t shift, uint32_t nbk, uint32_t T, uint32_t* __restrict__ hist) {
  __shared__ uint32_t cnt[NB_MAX];
  for (uint32_t d = threadIdx.x; d < nbk; d += SB) cnt[d] = 0;
  __syncthreads();
  uint32_t k[SIPT];
#pragma unroll
  for (int u = 0; u < SIPT; ++u) {
    const uint32_t i = blockIdx.x * FTILE + u * SB + threadIdx.x;
    k[u] = i < S ? __ldg(kin + i) : NO_REQ;
  }
#pragma unroll
  for (int u = 0; u < SIPT; ++u) {
    const uint32_t i = blockIdx.x * FTILE + u * SB + threadIdx.x;
    if (i >= S) break;
    const uint32_t key = kFirst ? key_of(k[u], R, live_bound, rank) : k[u];
    atomicAdd(cnt + ((key >> shift) & (nbk - 1)), 1u);
  }
  __syncthreads();
  for (uint32_t d = threadIdx.x; d < nbk; d += SB) hist[d * T + blockIdx.x] = cnt[d];
}

// one block per digit: exclusive prefix of its row over the tiles, and the row total
__global__ void __launch_bounds__(256) k_sort_hscan(uint32_t T, uint32_t* __restrict__ hist,
                                                    uint32_t* __restrict__ rowtot) {
  __shared__ uint32_t sw[9];
  uint32_t* row = hist + (size_t)blockIdx.x * T;
  uint32_t carry = 0;
  for (uint32_t b = 0; b < T; b += 256) {
    const uint32_t i = b + threadIdx.x;
    const uint32_t v = i < T ? row[i] : 0u;
    uint32_t tot;
    const uint32_t ex = block_excl_scan<uint32_t, 8>(v, sw, tot);
    if (i < T) row[i] = carry + ex;
    carry += tot;
  }
  if (threadIdx.x == 0) rowtot[blockIdx.x] = carry;
}

// lanes of the warp holding the same digit (ballots over its db bits), among the lanes in `valid`
__device__ __forceinline__ uint32_t match_digit(uint32_t d, int db, uint32_t valid) {
  uint32_t peers = valid;
  for (int b = 0; b < db; ++b) {
    const bool bit = (d >> b) & 1u;
    const uint32_t m = __ballot_sync(0xFFFFFFFFu, bit);
    peers &= bit ? m : ~m;
  }
  return peers;
}

// Dynamic shared memory of the scatter: per-warp digit counters / bases, the tile's digit
// offsets and global bases, the tile staged in digit order.
constexpr size_t SCATTER_SMEM = 4 * (SWARPS * NB_MAX + 2 * NB_MAX + 2 * FTILE + SWARPS + 1);

template <bool kFirst, bool kLast>
__global__ void __launch_bounds__(SB) k_sort_scatter(uint32_t S, uint32_t R, uint32_t live_bound,
                                                     const uint32_t* __restrict__ kin, const uint32_t* __restrict__ vin,
                                                     const uint32_t* __restrict__ rank, uint32_t shift, int db,
                                                     uint32_t T, const uint32_t* __restrict__ hist,
                                                     const uint32_t* __restrict__ rowtot, uint32_t* __restrict__ kout,
                                                     uint32_t* __restrict__ vout, const uint4* __restrict__ meta,
                                                     const unsigned long long* __restrict__ tbase,
                                                     uint4* __restrict__ smeta) {
  extern __shared__ __align__(16) uint32_t sm[];
  uint32_t* wc = sm;                              // [SWARPS][NB_MAX]
  uint32_t* tdo = wc + SWARPS * NB_MAX;           // tile-local start of each digit
  uint32_t* gb = tdo + NB_MAX;                    // global start of this tile's run of each digit
  uint32_t* sk = gb + NB_MAX;                     // the tile in digit order
  uint32_t* sv = sk + FTILE;
  uint32_t* sw = sv + FTILE;                      // SWARPS + 1
  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nbk = 1u << db;
  const uint32_t t0 = blockIdx.x * FTILE, nt = min(FTILE, S - t0);
  // global base per digit: digits before it (all tiles) + this digit in earlier tiles
  uint32_t tot;
  const uint32_t dex = block_excl_scan<uint32_t, SWARPS>(tid < nbk ? rowtot[tid] : 0u, sw, tot);
  if (tid < nbk) gb[tid] = dex + hist[tid * T + blockIdx.x];
  for (uint32_t x = tid; x < SWARPS * NB_MAX; x += SB) wc[x] = 0;
  // the warp's WITEMS consecutive snapshots, round u = [.. + 32 u, + 32)
  const uint32_t w0 = t0 + warp * WITEMS;
  uint32_t k[SIPT], v[SIPT];
#pragma unroll
  for (int u = 0; u < SIPT; ++u) {
    const uint32_t i = w0 + u * 32 + lane;
    if (i < S) {
      k[u] = __ldg(kin + i);
      v[u] = kFirst ? i : __ldg(vin + i);
    } else {
      k[u] = 0; v[u] = 0;
    }
  }
  if (kFirst) {
#pragma unroll
    for (int u = 0; u < SIPT; ++u)
      if (w0 + u * 32 + lane < S) k[u] = key_of(k[u], R, live_bound, rank);
  }
  __syncthreads();
#pragma unroll
  for (int u = 0; u < SIPT; ++u)
    if (w0 + u * 32 + lane < S) atomicAdd(&wc[warp * NB_MAX + ((k[u] >> shift) & (nbk - 1))], 1u);
  __syncthreads();
  // tile-local layout: digits in order, inside a digit the warps in order
  uint32_t tc = 0;
  if (tid < nbk) {
#pragma unroll
    for (int w = 0; w < SWARPS; ++w) tc += wc[w * NB_MAX + tid];
  }
  const uint32_t toff = block_excl_scan<uint32_t, SWARPS>(tid < nbk ? tc : 0u, sw, tot);
  if (tid < nbk) {
    tdo[tid] = toff;
    uint32_t run = toff;
#pragma unroll
    for (int w = 0; w < SWARPS; ++w) {
      const uint32_t c = wc[w * NB_MAX + tid];
      wc[w * NB_MAX + tid] = run;
      run += c;
    }
  }
  __syncthreads();
  const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
  for (int u = 0; u < SIPT; ++u) {
    const bool ok = w0 + u * 32 + lane < S;
    const uint32_t valid = __ballot_sync(0xFFFFFFFFu, ok);
    const uint32_t d = (k[u] >> shift) & (nbk - 1);
    const uint32_t peers = match_digit(d, db, valid);
    const uint32_t lr = __popc(peers & lt);
    if (ok) {
      const uint32_t pos = wc[warp * NB_MAX + d] + lr;
      sk[pos] = k[u];
      sv[pos] = v[u];
    }
    __syncwarp();
    if (ok && lr == 0) wc[warp * NB_MAX + d] += __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  // write-out in digit order: consecutive threads write consecutive positions of a digit's run
#pragma unroll 4
  for (uint32_t q = tid; q < nt; q += SB) {
    const uint32_t key = sk[q], val = sv[q], d = (key >> shift) & (nbk - 1);
    const uint32_t gpos = gb[d] + (q - tdo[d]);
    kout[gpos] = key;
    if (kLast) {
      // into fold order: the snapshot's source offset (tile base + in-tile) and lengths
      uint4 m = make_uint4(0, 0, 0, 0);
      if (key < live_bound) {
        m = __ldcg(meta + val);
        const unsigned long long src = tbase[val / FTILE] + ((unsigned long long)m.x | ((unsigned long long)m.y << 32));
        m.x = (uint32_t)src;
        m.y = (uint32_t)(src >> 32);
      }
      smeta[gpos] = m;
    }
    vout[gpos] = val;
  }
}

// sorted order: tile totals of the live lengths (smeta holds zero lengths for the others)
__global__ void __launch_bounds__(CB) k_fold_dsum(uint32_t S, const uint4* __restrict__ smeta,
                                                  unsigned long long* __restrict__ dsum) {
  __shared__ unsigned long long sw[CWARPS + 1];
  unsigned long long s = 0;
#pragma unroll
  for (int u = 0; u < CIPT; ++u) {
    const uint32_t p = blockIdx.x * FTILE + u * CB + threadIdx.x;
    if (p < S) {
      const uint2 m = __ldcg(reinterpret_cast<const uint2*>(smeta + p) + 1);
      s += pack_len(m.x, m.y);
    }
  }
  unsigned long long tot;
  block_excl_scan<unsigned long long, CWARPS>(s, sw, tot);
  if (threadIdx.x == 0) dsum[blockIdx.x] = tot;
}

// Warp-cooperative copy of one payload stream: the warp's 256 snapshots (lane-major, 8 per lane)
// have consecutive destinations, so the warp walks its destination range 32 words at a time
// (one coalesced store per step); each word finds its snapshot by binary search over the staged
// destination starts.  ds / sr: the warp's staged starts and sources (256 each).
__device__ __forceinline__ void warp_copy(const uint32_t* __restrict__ in, unsigned long long n_in,
                                          uint32_t* __restrict__ out, const uint32_t* ds, const uint32_t* sr,
                                          uint32_t lo, uint32_t hi) {
  const uint32_t lane = threadIdx.x & 31;
  for (uint32_t o = lo + lane; o < hi; o += 32) {
    uint32_t j = 0;
#pragma unroll
    for (uint32_t step = 128; step; step >>= 1)
      if (ds[j + step] <= o) j += step;   // last snapshot starting at or before o
    const unsigned long long src = (unsigned long long)sr[j] + (o - ds[j]);
    if (src < n_in && o < n_in) out[o] = __ldg(in + src);
  }
}

// Fold-order tile, thread t owns sorted positions [tile * FTILE + 8 t, + 8): the block scan of
// the lengths is each snapshot's destination offset; heads write the CSR start of their request,
// the last live snapshot the CSR end; the deltas move from their source offsets (smeta) with
// the warp-cooperative copy (a snapshot's deltas reaching past the payload arrays set overrun).
constexpr size_t PLACE_SMEM = (size_t)CWARPS * 2 * 256 * 4;

__global__ void __launch_bounds__(CB) k_fold_place(uint32_t S, uint32_t live_bound, const uint32_t* __restrict__ skey,
                                                   const uint32_t* __restrict__ sval, const uint32_t* __restrict__ progress,
                                                   uint32_t* __restrict__ prog_out, const uint4* __restrict__ smeta,
                                                   const unsigned long long* __restrict__ dbase,
                                                   const uint32_t* __restrict__ blocks, unsigned long long n_blocks_in,
                                                   const uint32_t* __restrict__ tokens, unsigned long long n_tokens_in,
                                                   unsigned long long* __restrict__ blk_off,
                                                   unsigned long long* __restrict__ tok_off,
                                                   uint32_t* __restrict__ blocks_out, uint32_t* __restrict__ tokens_out,
                                                   FoldDev* __restrict__ dev) {
  __shared__ unsigned long long sw[CWARPS + 1];
  extern __shared__ __align__(16) uint32_t psm[];
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t* ds = psm + warp * 512;   // [256] destination starts, [256] sources
  uint32_t* sr = ds + 256;
  const uint32_t p0 = blockIdx.x * FTILE + threadIdx.x * CIPT;
  uint32_t k[CIPT];
  ldb(skey, p0, S, k, live_bound);
  uint4 m[CIPT];
#pragma unroll
  for (int u = 0; u < CIPT; ++u) m[u] = p0 + u < S ? __ldg(smeta + p0 + u) : make_uint4(0, 0, 0, 0);
  unsigned long long s = 0;
#pragma unroll
  for (int u = 0; u < CIPT; ++u) s += pack_len(m[u].z, m[u].w);
  unsigned long long tot;
  const unsigned long long d0 = dbase[blockIdx.x] + block_excl_scan<unsigned long long, CWARPS>(s, sw, tot);
  unsigned long long d = d0;
  uint32_t prev = p0 && p0 < S ? __ldg(skey + p0 - 1) : 0xFFFFFFFFu;
  bool over = false;
#pragma unroll
  for (int u = 0; u < CIPT; ++u) {
    const uint32_t p = p0 + u, key = k[u];
    const unsigned long long len = pack_len(m[u].z, m[u].w);
    if (p < S && key < live_bound) {
      if (key != prev) {   // the request's first snapshot in fold order: its CSR start
        blk_off[key] = (uint32_t)d;
        tok_off[key] = (uint32_t)(d >> 32);
      }
      const uint32_t nxt = u + 1 < CIPT ? k[u + 1] : (p + 1 < S ? __ldg(skey + p + 1) : live_bound);
      if (nxt != key) prog_out[key] = __ldg(progress + __ldg(sval + p));   // the request's last snapshot
      if (nxt >= live_bound) {   // the last live snapshot: the CSR ends
        const unsigned long long e = d + len;
        blk_off[key + 1] = (uint32_t)e;
        tok_off[key + 1] = (uint32_t)(e >> 32);
        dev->n_blocks = (uint32_t)e;
        dev->n_tokens = (uint32_t)(e >> 32);
      }
      over |= (unsigned long long)m[u].x + m[u].z > n_blocks_in || (unsigned long long)m[u].y + m[u].w > n_tokens_in ||
              (unsigned long long)(uint32_t)d + m[u].z > n_blocks_in ||
              (unsigned long long)(uint32_t)(d >> 32) + m[u].w > n_tokens_in;
    }
    prev = key;
    d += len;
  }
  if (over) atomicOr(&dev->overrun, 1u);
  // the warp's destination ranges: [lane 0's first start, lane 31's end) per stream
  const unsigned long long wlo = __shfl_sync(0xFFFFFFFFu, d0, 0), whi = __shfl_sync(0xFFFFFFFFu, d, 31);
  // tokens, then blocks (the staging buffers are reused)
#pragma unroll
  for (int stream = 0; stream < 2; ++stream) {
    const int sh = stream == 0 ? 32 : 0;
    unsigned long long dd = d0;
#pragma unroll
    for (int u = 0; u < CIPT; ++u) {
      ds[lane * CIPT + u] = (uint32_t)(dd >> sh);
      sr[lane * CIPT + u] = stream == 0 ? m[u].y : m[u].x;
      dd += pack_len(m[u].z, m[u].w);
    }
    __syncwarp();
    if (stream == 0) warp_copy(tokens, n_tokens_in, tokens_out, ds, sr, (uint32_t)(wlo >> 32), (uint32_t)(whi >> 32));
    else warp_copy(blocks, n_blocks_in, blocks_out, ds, sr, (uint32_t)wlo, (uint32_t)whi);
    __syncwarp();
  }
}

// ---- bucketed fold (id spaces up to BK_MAX * BK_IDS) -------------------------------------
// One consume-order pass scatters the live snapshots into buckets of 256 consecutive request
// ids (stable: a bucket holds its snapshots in consume order), as 16-B records {snapshot index,
// id & 255 | done << 31, lengths} plus their 8-B source offsets.  Each bucket is then cut into
// chunks of 8192 records that are independent of each other:
//   k_fb_count    consume-order tiles of 4096: per-tile bucket counts, exact per-tile delta
//                 sums (blocks, tokens), rejected ids; clears the head bitmap
//   k_fb_scan     per-bucket prefix over the tiles; the tiles' source offsets
//   k_fb_scatter  per-warp bucket counters, ballot-matched ranks (stable), the tile staged in
//                 bucket order in shared memory and written out as coalesced runs; block 0
//                 publishes the bucket and chunk bases
//   k_fb_stats    per chunk and id: delta sums, first / last snapshot, sticky done
//   k_fb_mid      one cooperative kernel, grid barriers between its phases: per id, the chunk
//                 sums become each chunk's prefix inside the request, first / last / done /
//                 totals, the head bit of the first snapshot; the head-bitmap prefix; the
//                 first-appearance ranks, order, done, progress; the CSR offsets
//   k_fb_place    per chunk: per-warp per-id running sums give each record its place among its
//                 request's deltas (stable); the chunk's deltas are gathered into shared memory
//                 grouped by request and written out as one contiguous run per request
constexpr uint32_t BK_SH = 8, BK_IDS = 1u << BK_SH;   // request ids per bucket
constexpr uint32_t BK_MAX = NB_MAX;                   // buckets (one ranking pass of <= 9 bits)
constexpr uint32_t BT = 4096;                         // consume-order tile of the scatter
constexpr int BTN = 512, BT_WARPS = BTN / 32;
constexpr uint32_t BT_WITEMS = BT / BT_WARPS;         // 256 consecutive snapshots per warp
constexpr int BT_ROUNDS = BT_WITEMS / 32;
constexpr uint32_t CH = 4096;                         // records per bucket chunk
constexpr int SCN = 1024, SC_ROUNDS = CH / SCN;       // k_fb_stats: 4 records per thread
constexpr int CHN = 512, CH_WARPS = CHN / 32;         // k_fb_place: two CTAs per SM
constexpr int CH_ROUNDS = CH / CHN;                   // 8 records per thread
constexpr uint32_t STAGE_CAP = 14336;                 // delta words staged per chunk
constexpr uint32_t CSR_TILE = 8192;

struct FoldDevB {           // zeroed by one memset per fold
  unsigned long long n_requests, n_blocks, n_tokens;
  uint32_t err_enc;         // max of ~i over rejected snapshots (0: none)
  uint32_t overrun;
  uint32_t barrier;         // k_fb_mid's grid barrier count
  uint32_t pad;
  uint32_t flag[BK_MAX * BK_IDS / CSR_TILE];
  unsigned long long incl[BK_MAX * BK_IDS / CSR_TILE];
};

__global__ void __launch_bounds__(BTN) k_fb_count(uint32_t S, uint32_t R, uint32_t nbk, uint32_t T, uint32_t W,
                                                  const uint32_t* __restrict__ req, const uint32_t* __restrict__ nblk,
                                                  const uint32_t* __restrict__ ntok, uint32_t* __restrict__ hist,
                                                  unsigned long long* __restrict__ tsb,
                                                  unsigned long long* __restrict__ tst, uint32_t* __restrict__ bitmap,
                                                  FoldDevB* __restrict__ dev) {
  __shared__ uint32_t cnt[BK_MAX];
  __shared__ unsigned long long red[2][BT_WARPS];
  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (uint32_t d = tid; d < nbk; d += BTN) cnt[d] = 0;
  const uint32_t wb = blockIdx.x * (BT / 32), we = blockIdx.x + 1 == gridDim.x ? W : wb + BT / 32;
  for (uint32_t w = wb + tid; w < we; w += BTN) bitmap[w] = 0;
  __syncthreads();
  constexpr int IPT = BT / BTN;
  const uint32_t i0 = blockIdx.x * BT + tid * IPT;
  uint32_t r[IPT], nb[IPT], nt[IPT];
  ldb(req, i0, S, r, NO_REQ);
  ldb(nblk, i0, S, nb, 0u);
  ldb(ntok, i0, S, nt, 0u);
  unsigned long long sb = 0, st = 0;
  uint32_t bad = NO_REQ;
#pragma unroll
  for (int u = 0; u < IPT; ++u) {
    sb += nb[u];
    st += nt[u];
    if (r[u] < R) atomicAdd(cnt + (r[u] >> BK_SH), 1u);
    else if (r[u] != NO_REQ && i0 + u < S) bad = min(bad, i0 + u);
  }
  if (bad != NO_REQ) atomicMax(&dev->err_enc, ~bad);
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    sb += __shfl_xor_sync(0xFFFFFFFFu, sb, o);
    st += __shfl_xor_sync(0xFFFFFFFFu, st, o);
  }
  if (lane == 0) {
    red[0][warp] = sb;
    red[1][warp] = st;
  }
  __syncthreads();
  for (uint32_t d = tid; d < nbk; d += BTN) hist[d * T + blockIdx.x] = cnt[d];
  if (tid < 2) {
    unsigned long long s = 0;
#pragma unroll
    for (int w = 0; w < BT_WARPS; ++w) s += red[tid][w];
    (tid ? tst : tsb)[blockIdx.x] = s;
  }
}

// blocks [0, nbk): one bucket's row of tile counts -> exclusive prefix, row total; block nbk:
// the tiles' consume-order delta offsets (exact 64-bit prefixes, packed blocks | tokens << 32;
// totals that do not fit 32 bits are an overrun)
__global__ void __launch_bounds__(256) k_fb_scan(uint32_t T, uint32_t nbk, uint32_t* __restrict__ hist,
                                                 uint32_t* __restrict__ rowtot, const unsigned long long* __restrict__ tsb,
                                                 const unsigned long long* __restrict__ tst,
                                                 unsigned long long* __restrict__ tbase, FoldDevB* __restrict__ dev) {
  fold_pdl();
  __shared__ unsigned long long sw[9];
  // thread t owns the P consecutive tiles [t P, t P + P): its loads are independent, one block
  // scan per array
  const uint32_t P = (T + 255) / 256, i0 = threadIdx.x * P, i1 = min(i0 + P, T);
  if (blockIdx.x < nbk) {
    __shared__ uint32_t sw32[9];
    uint32_t* row = hist + (size_t)blockIdx.x * T;
    uint32_t s = 0;
    for (uint32_t i = i0; i < i1; ++i) s += row[i];
    uint32_t tot;
    uint32_t run = block_excl_scan<uint32_t, 8>(s, sw32, tot);
    for (uint32_t i = i0; i < i1; ++i) {
      const uint32_t v = row[i];
      row[i] = run;
      run += v;
    }
    if (threadIdx.x == 0) rowtot[blockIdx.x] = tot;
    return;
  }
  unsigned long long sb = 0, st = 0;
  for (uint32_t i = i0; i < i1; ++i) {
    sb += tsb[i];
    st += tst[i];
  }
  unsigned long long tb, tt;
  unsigned long long rb = block_excl_scan<unsigned long long, 8>(sb, sw, tb);
  unsigned long long rt = block_excl_scan<unsigned long long, 8>(st, sw, tt);
  for (uint32_t i = i0; i < i1; ++i) {
    tbase[i] = rb | (rt << 32);
    rb += tsb[i];
    rt += tst[i];
  }
  if (threadIdx.x == 0 && ((tb >> 32) || (tt >> 32))) dev->overrun = 1;
}

constexpr size_t FB_SCATTER_SMEM = 4 * (BT_WARPS * BK_MAX + 2 * BK_MAX) + 2 * BT + 16 * BT;

__global__ void __launch_bounds__(BTN, 2) k_fb_scatter(uint32_t S, uint32_t R, uint32_t nbk, int db, uint32_t T,
                                                       const uint32_t* __restrict__ req, const uint32_t* __restrict__ nblk,
                                                       const uint32_t* __restrict__ ntok, const uint8_t* __restrict__ done,
                                                       const uint32_t* __restrict__ hist, const uint32_t* __restrict__ rowtot,
                                                       const unsigned long long* __restrict__ tbase, uint64_t n_blocks_in,
                                                       uint64_t n_tokens_in, uint4* __restrict__ rec,
                                                       uint2* __restrict__ src, uint32_t* __restrict__ bbase,
                                                       uint32_t* __restrict__ cbase, FoldDevB* __restrict__ dev) {
  fold_pdl();
  extern __shared__ __align__(16) uint32_t sm[];
  uint32_t* wc = sm;                                    // [BT_WARPS][BK_MAX]
  uint32_t* tdo = wc + BT_WARPS * BK_MAX;               // tile-local start of each bucket
  uint32_t* gb = tdo + BK_MAX;                          // global start of this tile's run
  uint4* stg = reinterpret_cast<uint4*>(gb + BK_MAX);   // the tile in bucket order
  uint16_t* sd = reinterpret_cast<uint16_t*>(stg + BT); // its bucket
  __shared__ uint32_t sw[BT_WARPS + 1];
  __shared__ unsigned long long swl[BT_WARPS + 1];
  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  uint32_t tot;
  const uint32_t rt = tid < nbk ? rowtot[tid] : 0u;
  const uint32_t dex = block_excl_scan<uint32_t, BT_WARPS>(rt, sw, tot);
  if (tid < nbk) gb[tid] = dex + hist[tid * T + blockIdx.x];
  if (blockIdx.x == 0) {   // bucket bases and chunk bases for the per-chunk kernels
    if (tid < nbk) bbase[tid] = dex;
    if (tid == 0) bbase[nbk] = tot;
    uint32_t ctot;
    const uint32_t cex = block_excl_scan<uint32_t, BT_WARPS>((rt + CH - 1) / CH, sw, ctot);
    if (tid < nbk) cbase[tid] = cex;
    if (tid == 0) cbase[nbk] = ctot;
  }
  for (uint32_t x = tid; x < BT_WARPS * BK_MAX; x += BTN) wc[x] = 0;
  const uint32_t w0 = blockIdx.x * BT + warp * BT_WITEMS;
  uint32_t r[BT_ROUNDS], nb[BT_ROUNDS], nt[BT_ROUNDS], dn = 0;
#pragma unroll
  for (int u = 0; u < BT_ROUNDS; ++u) {
    const uint32_t i = w0 + u * 32 + lane;
    if (i < S) {
      r[u] = __ldg(req + i);
      nb[u] = __ldg(nblk + i);
      nt[u] = __ldg(ntok + i);
      dn |= (__ldg(done + i) ? 1u : 0u) << u;
    } else {
      r[u] = NO_REQ; nb[u] = 0; nt[u] = 0;
    }
  }
  // consume-order source offsets inside the tile: per-round warp scans, then across the warps
  unsigned long long pre[BT_ROUNDS], run = 0;
#pragma unroll
  for (int u = 0; u < BT_ROUNDS; ++u) {
    const unsigned long long len = pack_len(nb[u], nt[u]);
    const unsigned long long inc = warp_incl_scan(len);
    pre[u] = run + inc - len;
    run += __shfl_sync(0xFFFFFFFFu, inc, 31);
  }
  if (lane == 0) swl[warp] = run;
  __syncthreads();
  if (warp == 0) {
    const unsigned long long w = lane < (uint32_t)BT_WARPS ? swl[lane] : 0ull;
    const unsigned long long wi = warp_incl_scan(w);
    if (lane < (uint32_t)BT_WARPS) swl[lane] = wi - w;
  }
#pragma unroll
  for (int u = 0; u < BT_ROUNDS; ++u)
    if (r[u] < R) atomicAdd(&wc[warp * BK_MAX + (r[u] >> BK_SH)], 1u);
  __syncthreads();
  const unsigned long long base = tbase[blockIdx.x] + swl[warp];
  // tile-local layout: buckets in order, inside a bucket the warps in order
  uint32_t tc = 0;
  if (tid < nbk) {
#pragma unroll
    for (int w = 0; w < BT_WARPS; ++w) tc += wc[w * BK_MAX + tid];
  }
  uint32_t ntl;
  const uint32_t toff = block_excl_scan<uint32_t, BT_WARPS>(tc, sw, ntl);
  if (tid < nbk) {
    tdo[tid] = toff;
    uint32_t o = toff;
#pragma unroll
    for (int w = 0; w < BT_WARPS; ++w) {
      const uint32_t c = wc[w * BK_MAX + tid];
      wc[w * BK_MAX + tid] = o;
      o += c;
    }
  }
  __syncthreads();
  const uint32_t lt = (1u << lane) - 1u;
  uint32_t pos[BT_ROUNDS];
  bool over = false;
#pragma unroll
  for (int u = 0; u < BT_ROUNDS; ++u) {
    const bool ok = r[u] < R;
    const uint32_t valid = __ballot_sync(0xFFFFFFFFu, ok);
    const uint32_t d = ok ? r[u] >> BK_SH : 0u;
    const uint32_t peers = match_digit(d, db, valid);
    const uint32_t lr = __popc(peers & lt);
    pos[u] = 0;
    if (ok) {
      const uint32_t p = wc[warp * BK_MAX + d] + lr;
      pos[u] = p;
      stg[p] = make_uint4(w0 + u * 32 + lane, (r[u] & (BK_IDS - 1)) | (((dn >> u) & 1u) << 31), nb[u], nt[u]);
      sd[p] = (uint16_t)d;
      const unsigned long long s = base + pre[u];
      over |= (s & 0xFFFFFFFFull) + nb[u] > n_blocks_in || (s >> 32) + nt[u] > n_tokens_in;
    }
    __syncwarp();
    if (ok && lr == 0) wc[warp * BK_MAX + d] += __popc(peers);
    __syncwarp();
  }
  if (over) atomicOr(&dev->overrun, 1u);
  __syncthreads();
  for (uint32_t q = tid; q < ntl; q += BTN) {
    const uint32_t d = sd[q];
    rec[gb[d] + (q - tdo[d])] = stg[q];
  }
  __syncthreads();
  uint2* stg2 = reinterpret_cast<uint2*>(stg);
#pragma unroll
  for (int u = 0; u < BT_ROUNDS; ++u)
    if (r[u] < R) {
      const unsigned long long s = base + pre[u];
      stg2[pos[u]] = make_uint2((uint32_t)s, (uint32_t)(s >> 32));
    }
  __syncthreads();
  for (uint32_t q = tid; q < ntl; q += BTN) {
    const uint32_t d = sd[q];
    src[gb[d] + (q - tdo[d])] = stg2[q];
  }
}

// L2 residency for the delta gathers of k_fb_place: the payload arrays are prefetched with
// evict_last while the chunk kernels stream their records with evict_first
__device__ __forceinline__ void prefetch_l2_last(const void* p) {
  asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(p));
}
__device__ __forceinline__ void prefetch_slice(const uint32_t* a, uint64_t n, uint32_t part, uint32_t parts) {
  const uint64_t lines = (n * 4 + 127) / 128, b = lines * part / parts, e = lines * (part + 1) / parts;
  for (uint64_t x = b + threadIdx.x; x < e; x += blockDim.x) prefetch_l2_last(reinterpret_cast<const char*>(a) + x * 128);
}
__device__ __forceinline__ unsigned long long evict_first_policy() {
  unsigned long long pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint4 ld_stream16(const uint4* p, unsigned long long pol) {
  uint4 v;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
      : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ uint2 ld_stream8(const uint2* p, unsigned long long pol) {
  uint2 v;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.u32 {%0,%1}, [%2], %3;" : "=r"(v.x), "=r"(v.y) : "l"(p), "l"(pol));
  return v;
}

// chunk c of the bucket layout: its bucket and record range (scb: chunk bases in shared memory)
__device__ __forceinline__ bool chunk_of(uint32_t c, uint32_t nbk, const uint32_t* scb,
                                         const uint32_t* __restrict__ bbase, uint32_t& d, uint32_t& p0,
                                         uint32_t& p1) {
  if (c >= scb[nbk]) return false;
  uint32_t lo = 0;
  for (uint32_t step = BK_MAX / 2; step; step >>= 1)
    if (lo + step < nbk && scb[lo + step] <= c) lo += step;
  d = lo;
  p0 = __ldg(bbase + d) + (c - scb[d]) * CH;
  p1 = min(p0 + CH, __ldg(bbase + d + 1));
  return true;
}

__global__ void __launch_bounds__(SCN) k_fb_stats(uint32_t nbk, const uint32_t* __restrict__ bbase,
                                                  const uint32_t* __restrict__ cbase, const uint4* __restrict__ rec,
                                                  uint4* __restrict__ cstat, const uint32_t* __restrict__ blocks,
                                                  uint64_t nbin, const uint32_t* __restrict__ tokens, uint64_t ntin) {
  fold_pdl();
  prefetch_slice(tokens, ntin, blockIdx.x, gridDim.x);
  prefetch_slice(blocks, nbin, blockIdx.x, gridDim.x);
  __shared__ uint32_t scb[BK_MAX + 1];
  __shared__ uint32_t first[BK_IDS], last[BK_IDS], dn[BK_IDS], lb[BK_IDS], lt[BK_IDS];
  const uint32_t tid = threadIdx.x;
  for (uint32_t x = tid; x <= nbk; x += SCN) scb[x] = __ldg(cbase + x);
  if (tid < BK_IDS) {
    first[tid] = NO_REQ;
    last[tid] = 0;
    dn[tid] = 0;
    lb[tid] = 0;
    lt[tid] = 0;
  }
  __syncthreads();
  uint32_t d, p0, p1;
  if (!chunk_of(blockIdx.x, nbk, scb, bbase, d, p0, p1)) return;
  uint4 x[SC_ROUNDS];
#pragma unroll
  for (int u = 0; u < SC_ROUNDS; ++u) {
    const uint32_t p = p0 + u * SCN + tid;
    x[u] = p < p1 ? __ldg(rec + p) : make_uint4(0, 0, 0, 0);
  }
#pragma unroll
  for (int u = 0; u < SC_ROUNDS; ++u) {
    if (p0 + u * SCN + tid < p1) {
      const uint32_t l = x[u].y & (BK_IDS - 1);
      atomicMin(first + l, x[u].x);
      atomicMax(last + l, x[u].x);
      if (x[u].z) atomicAdd(lb + l, x[u].z);   // (chunk sums fit: the fold's totals are < 2^32)
      atomicAdd(lt + l, x[u].w);
      if (x[u].y >> 31) dn[l] = 1;
    }
  }
  __syncthreads();
  if (tid < BK_IDS)
    cstat[(size_t)blockIdx.x * BK_IDS + tid] = make_uint4(lb[tid], lt[tid], first[tid] | (dn[tid] << 31), last[tid]);
}




// The id / rank / CSR steps between the chunk statistics and the placement, as one cooperative
// kernel (one CTA per SM, grid-wide barriers between the phases) instead of five dependent
// launches: per id, chunk prefixes, totals and the head bit | per bitmap chunk, a warp's word
// prefixes | the chunk prefix (CTA 0) | ranks, order, done, progress, per-rank sums | per
// 8192-rank tile totals, then each tile's offsets after its predecessors' totals.
__device__ __forceinline__ void grid_barrier(unsigned int* bar, unsigned int& gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned int target = (gen + 1) * gridDim.x;
    __threadfence();
    atomicAdd(bar, 1u);
    while (*reinterpret_cast<volatile unsigned int*>(bar) < target) {}
    __threadfence();
  }
  ++gen;
  __syncthreads();
}

__global__ void __launch_bounds__(1024, 1) k_fb_mid(uint32_t R, uint32_t W, uint32_t C, const uint32_t* __restrict__ cbase,
                                                    uint4* __restrict__ cstat, uint32_t* __restrict__ first,
                                                    uint32_t* __restrict__ lastx, uint32_t* __restrict__ rdone,
                                                    unsigned long long* __restrict__ lensr, uint32_t* __restrict__ bitmap,
                                                    uint32_t* __restrict__ wloc, unsigned long long* __restrict__ ccount,
                                                    unsigned long long* __restrict__ cpre,
                                                    const uint32_t* __restrict__ progress, uint32_t* __restrict__ rank,
                                                    uint32_t* __restrict__ order, uint8_t* __restrict__ done_out,
                                                    uint32_t* __restrict__ prog_out, unsigned long long* __restrict__ rl,
                                                    unsigned long long* __restrict__ blk_off,
                                                    unsigned long long* __restrict__ tok_off, FoldDevB* dev) {
  fold_pdl();
  __shared__ unsigned long long sw[33];
  unsigned int gen = 0;
  unsigned int* bar = &dev->barrier;
  const uint32_t tid = threadIdx.x, lane = tid & 31, gtid = blockIdx.x * 1024 + tid, gthreads = gridDim.x * 1024;
  // ids
  for (uint32_t r = gtid; r < R; r += gthreads) {
    const uint32_t d = r >> BK_SH, l = r & (BK_IDS - 1);
    const uint32_t c0 = __ldg(cbase + d), c1 = __ldg(cbase + d + 1);
    uint32_t f = NO_REQ, la = 0, dn = 0;
    unsigned long long run = 0;
    for (uint32_t c = c0; c < c1; ++c) {
      uint4* sp = cstat + (size_t)c * BK_IDS + l;
      const uint4 sv = *sp;
      if (sv.z != NO_REQ) {
        if (f == NO_REQ) f = sv.z & 0x7FFFFFFFu;
        dn |= sv.z >> 31;
        la = sv.w;
        *reinterpret_cast<uint2*>(sp) = make_uint2((uint32_t)run, (uint32_t)(run >> 32));
        run += (unsigned long long)sv.x | ((unsigned long long)sv.y << 32);
      }
    }
    first[r] = f;
    lastx[r] = la;
    rdone[r] = dn;
    lensr[r] = run;
    if (f != NO_REQ) atomicOr(bitmap + (f >> 5), 1u << (f & 31));
  }
  grid_barrier(bar, gen);
  // bitmap chunks: a warp each
  for (uint32_t c = gtid >> 5; c < C; c += gthreads >> 5) {
    constexpr int WPL = CHUNK_WORDS / 32;
    const uint32_t w0 = c * CHUNK_WORDS + lane * WPL;
    uint32_t cnt[WPL], t = 0;
#pragma unroll
    for (int u = 0; u < WPL; ++u) {
      cnt[u] = w0 + u < W ? __popc(bitmap[w0 + u]) : 0u;
      t += cnt[u];
    }
    const uint32_t inc = warp_incl_scan(t);
    uint32_t ex = inc - t;
#pragma unroll
    for (int u = 0; u < WPL; ++u) {
      if (w0 + u < W) wloc[w0 + u] = ex;
      ex += cnt[u];
    }
    if (lane == 31) ccount[c] = inc;
  }
  grid_barrier(bar, gen);
  if (blockIdx.x == 0) scan_small(ccount, cpre, C, &dev->n_requests);
  grid_barrier(bar, gen);
  const uint32_t n = (uint32_t)*reinterpret_cast<volatile unsigned long long*>(&dev->n_requests);
  for (uint32_t r = gtid; r < R; r += gthreads) {
    const uint32_t f = first[r];
    if (f == NO_REQ) continue;
    const uint32_t w = f >> 5;
    const uint32_t k = (uint32_t)cpre[w / CHUNK_WORDS] + wloc[w] + __popc(bitmap[w] & ((1u << (f & 31)) - 1u));
    rank[r] = k;
    order[k] = r;
    done_out[k] = rdone[r] ? 1 : 0;
    prog_out[k] = __ldg(progress + lastx[r]);
    rl[k] = lensr[r];
  }
  grid_barrier(bar, gen);
  // CSR over ranks: tiles of 8192 (CTA t takes tile t), totals published, then offsets.  The tile
  // goes through shared memory so both the loads and the two output arrays are coalesced
  // (thread-blocked global accesses cost one sector request per 8 bytes).
  constexpr int IPT = CSR_TILE / 1024;
  extern __shared__ __align__(16) unsigned long long csr_s[];   // [CSR_TILE]
  const uint32_t ntile = (n + CSR_TILE - 1) / CSR_TILE;
  const uint32_t k0 = blockIdx.x * CSR_TILE;
  const bool mine = blockIdx.x < ntile;
  unsigned long long run = 0, tot = 0;
  if (mine) {
#pragma unroll
    for (int u = 0; u < IPT; ++u) {
      const uint32_t k = k0 + u * 1024 + tid;
      csr_s[u * 1024 + tid] = k < n ? rl[k] : 0ull;
    }
    __syncthreads();
    unsigned long long s = 0;
#pragma unroll
    for (int u = 0; u < IPT; ++u) s += csr_s[tid * IPT + u];
    run = block_excl_scan<unsigned long long, 32>(s, sw, tot);
    if (tid == 0) dev->incl[blockIdx.x] = tot;
  }
  grid_barrier(bar, gen);
  if (mine) {
    if (tid < 32) {
      unsigned long long pre = tid < blockIdx.x ? *reinterpret_cast<volatile unsigned long long*>(dev->incl + tid) : 0ull;
#pragma unroll
      for (int o = 16; o; o >>= 1) pre += __shfl_xor_sync(0xFFFFFFFFu, pre, o);
      if (tid == 0) sw[32] = pre;
    }
    __syncthreads();
    run += sw[32];
#pragma unroll
    for (int u = 0; u < IPT; ++u) {   // exclusive offsets in place
      const unsigned long long v = csr_s[tid * IPT + u];
      csr_s[tid * IPT + u] = run;
      run += v;
    }
    if (k0 + (tid + 1) * IPT >= n && k0 + tid * IPT < n) {   // the thread holding rank n - 1: the CSR end
      blk_off[n] = run & 0xFFFFFFFFull;
      tok_off[n] = run >> 32;
      dev->n_blocks = run & 0xFFFFFFFFull;
      dev->n_tokens = run >> 32;
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < IPT; ++u) {
      const uint32_t k = k0 + u * 1024 + tid;
      if (k < n) {
        const unsigned long long o = csr_s[u * 1024 + tid];
        blk_off[k] = o & 0xFFFFFFFFull;
        tok_off[k] = o >> 32;
      }
    }
  }
}

constexpr size_t FB_PLACE_SMEM = 8 * (CH_WARPS * BK_IDS + CH_WARPS * 32 + 2 * BK_IDS) + 4 * (2 * (BK_IDS + 1)) +
                                 4 * (BK_MAX + 1) + 4 * STAGE_CAP;


__global__ void __launch_bounds__(CHN, 2) k_fb_place(uint32_t R, uint32_t nbk, const uint32_t* __restrict__ bbase,
                                                     const uint32_t* __restrict__ cbase, const uint4* __restrict__ rec,
                                                     const uint2* __restrict__ src, const uint4* __restrict__ cstat,
                                                     const uint32_t* __restrict__ rank,
                                                     const unsigned long long* __restrict__ blk_off,
                                                     const unsigned long long* __restrict__ tok_off,
                                                     const uint32_t* __restrict__ blocks, uint64_t nbin,
                                                     const uint32_t* __restrict__ tokens, uint64_t ntin,
                                                     uint32_t* __restrict__ blocks_out, uint32_t* __restrict__ tokens_out) {
  fold_pdl();
  extern __shared__ __align__(16) unsigned long long psm64[];
  unsigned long long* wl = psm64;                       // [CH_WARPS][BK_IDS] per-warp running sums
  unsigned long long* lbuf = wl + CH_WARPS * BK_IDS;    // [CH_WARPS][32] the round's lengths
  unsigned long long* curb = lbuf + CH_WARPS * 32;      // [BK_IDS] destination of the id's first block word
  unsigned long long* curt = curb + BK_IDS;             // [BK_IDS] ... token word
  uint32_t* lbb = reinterpret_cast<uint32_t*>(curt + BK_IDS);   // [BK_IDS + 1] the id's start in the staged blocks
  uint32_t* lbt = lbb + BK_IDS + 1;                     // [BK_IDS + 1] ... tokens
  uint32_t* scb = lbt + BK_IDS + 1;                     // [BK_MAX + 1]
  uint32_t* stage = scb + BK_MAX + 1;                   // [STAGE_CAP]
  __shared__ unsigned long long sw[CH_WARPS + 1];
  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (uint32_t x = tid; x <= nbk; x += CHN) scb[x] = __ldg(cbase + x);
  __syncthreads();
  uint32_t d, p0, p1;
  if (!chunk_of(blockIdx.x, nbk, scb, bbase, d, p0, p1)) return;
  // the warp's records (256 consecutive), loaded up front; lanes past the chunk get a private id
  const uint32_t pw = p0 + warp * (CH / CH_WARPS);
  const unsigned long long pol = evict_first_policy();
  uint32_t lv[CH_ROUNDS];
  unsigned long long len[CH_ROUNDS];
#pragma unroll
  for (int u = 0; u < CH_ROUNDS; ++u) {
    const uint32_t p = pw + u * 32 + lane;
    if (p < p1) {
      const uint4 x = ld_stream16(rec + p, pol);
      lv[u] = x.y & (BK_IDS - 1);
      len[u] = pack_len(x.z, x.w);
    } else {
      lv[u] = BK_IDS + lane;
      len[u] = 0;
    }
  }
  for (uint32_t x = tid; x < CH_WARPS * BK_IDS; x += CHN) wl[x] = 0;
  if (tid < BK_IDS) {
    const uint32_t r = d * BK_IDS + tid;
    unsigned long long cb = 0, ct = 0;
    if (r < R) {
      const uint4 s = __ldg(cstat + (size_t)blockIdx.x * BK_IDS + tid);
      if (s.z != NO_REQ) {
        const uint32_t k = __ldg(rank + r);
        cb = __ldg(blk_off + k) + s.x;
        ct = __ldg(tok_off + k) + s.y;
      }
    }
    curb[tid] = cb;
    curt[tid] = ct;
  }
  __syncthreads();
  // per warp, rounds of 32 records in order: the record's offset among its request's deltas
  // inside the warp (earlier rounds + lower peer lanes)
  const uint32_t lt = (1u << lane) - 1u;
  unsigned long long wpre[CH_ROUNDS];
#pragma unroll
  for (int u = 0; u < CH_ROUNDS; ++u) {
    const bool ok = lv[u] < BK_IDS;
    const uint32_t peers = match_digit(lv[u], BK_SH, __ballot_sync(0xFFFFFFFFu, ok));
    lbuf[warp * 32 + lane] = len[u];
    __syncwarp();
    const unsigned long long old = ok ? wl[warp * BK_IDS + lv[u]] : 0ull;
    unsigned long long pre = 0;
    for (uint32_t m = peers & lt; m; m &= m - 1) pre += lbuf[warp * 32 + __ffs(m) - 1];
    wpre[u] = old + pre;
    __syncwarp();
    if (ok && (peers >> lane) == 1u) wl[warp * BK_IDS + lv[u]] = old + pre + len[u];
    __syncwarp();
  }
  __syncthreads();
  // across warps: exclusive per id; the chunk's ids grouped in id order in the staging area
  unsigned long long idt = 0;
  if (tid < BK_IDS) {
#pragma unroll
    for (int w = 0; w < CH_WARPS; ++w) {
      const unsigned long long t = wl[w * BK_IDS + tid];
      wl[w * BK_IDS + tid] = idt;
      idt += t;
    }
  }
  unsigned long long ctot;
  const unsigned long long lb = block_excl_scan<unsigned long long, CH_WARPS>(idt, sw, ctot);
  if (tid < BK_IDS) {
    lbb[tid] = (uint32_t)lb;
    lbt[tid] = (uint32_t)(lb >> 32);
  }
  if (tid == 0) {
    lbb[BK_IDS] = (uint32_t)ctot;
    lbt[BK_IDS] = (uint32_t)(ctot >> 32);
  }
  __syncthreads();
  const uint32_t totb = (uint32_t)ctot, tott = (uint32_t)(ctot >> 32);
  const bool staged = (unsigned long long)totb + tott <= STAGE_CAP;
  uint32_t* stok = stage + totb;
#pragma unroll
  for (int u = 0; u < CH_ROUNDS; ++u) {
    const uint32_t l = lv[u];
    if (l >= BK_IDS) continue;
    const uint2 s = ld_stream8(src + pw + u * 32 + lane, pol);
    const unsigned long long o = wl[warp * BK_IDS + l] + wpre[u];   // offset inside the id's group
    const uint32_t nb = (uint32_t)len[u], nt = (uint32_t)(len[u] >> 32);
    if (staged) {
      uint32_t* bd = stage + lbb[l] + (uint32_t)o;
      uint32_t* td = stok + lbt[l] + (uint32_t)(o >> 32);
#pragma unroll
      for (uint32_t j = 0; j < 4; ++j)   // the common short deltas: independent loads
        if (j < nt && s.y + j < ntin) td[j] = __ldg(tokens + s.y + j);
      if (nb && s.x < nbin) bd[0] = __ldg(blocks + s.x);
      for (uint32_t j = 4; j < nt; ++j)
        if (s.y + j < ntin) td[j] = __ldg(tokens + s.y + j);
      for (uint32_t j = 1; j < nb; ++j)
        if (s.x + j < nbin) bd[j] = __ldg(blocks + s.x + j);
    } else {   // too many deltas to stage: straight to the destination
      const unsigned long long db0 = curb[l] + (uint32_t)o, dt0 = curt[l] + (uint32_t)(o >> 32);
      for (uint32_t j = 0; j < nb; ++j)
        if (s.x + j < nbin && db0 + j < nbin) blocks_out[db0 + j] = __ldg(blocks + s.x + j);
      for (uint32_t j = 0; j < nt; ++j)
        if (s.y + j < ntin && dt0 + j < ntin) tokens_out[dt0 + j] = __ldg(tokens + s.y + j);
    }
  }
  if (!staged) return;
  __syncthreads();
  // one contiguous destination run per request: a warp per id
  for (uint32_t l = warp; l < BK_IDS; l += CH_WARPS) {
    const uint32_t b0 = lbb[l], b1 = lbb[l + 1], t0 = lbt[l], t1 = lbt[l + 1];
    const unsigned long long ob = curb[l] - b0, ot = curt[l] - t0;
    for (uint32_t q = b0 + lane; q < b1; q += 32)
      if (ob + q < nbin) blocks_out[ob + q] = stage[q];
    for (uint32_t q = t0 + lane; q < t1; q += 32)
      if (ot + q < ntin) tokens_out[ot + q] = stok[q];
  }
}

static size_t al256(size_t x) { return (x + 255) & ~size_t(255); }

static int key_bits(uint32_t live_bound) {   // bits for keys in [0, live_bound]
  int b = 1;
  while (b < 32 && (1ull << b) <= live_bound) ++b;
  return b;
}

static uint32_t tiles(uint64_t S) { return (uint32_t)((S + FTILE - 1) / FTILE); }

// scratch layout for S snapshots and R request ids (the larger of the two paths)
static size_t radix_scratch_bytes(uint64_t S, uint64_t R) {
  const uint64_t T = tiles(S), W = S / 32 + 1, C = (W + CHUNK_WORDS - 1) / CHUNK_WORDS;
  size_t o = al256(64) + al256(4 * R) * 3;                 // dev, first, rdone, rank
  o += al256(4 * W) * 2 + al256(8 * C) * 2;                // bitmap, wloc, chunk counts / prefix
  o += al256(8 * T) * 4;                                   // tsum, tbase, dsum, dbase
  o += al256(4 * S) * 4;                                   // sort keys / values, two buffers
  o += al256(16 * S) * 2;                                  // meta in consume order, in fold order
  o += al256(4ull * NB_MAX * T) + al256(4 * NB_MAX);       // hist, rowtot
  return o + 256;
}

static bool bucketed(uint64_t R) { return R <= (uint64_t)BK_MAX * BK_IDS; }
static uint32_t n_buckets(uint64_t R) { return (uint32_t)((R + BK_IDS - 1) / BK_IDS); }
static uint32_t max_chunks(uint64_t S, uint64_t R) { return (uint32_t)((S + CH - 1) / CH + n_buckets(R)); }

static size_t bucket_scratch_bytes(uint64_t S, uint64_t R) {
  const uint64_t T = (S + BT - 1) / BT, W = S / 32 + 1, C = (W + CHUNK_WORDS - 1) / CHUNK_WORDS, NB = n_buckets(R);
  size_t o = al256(sizeof(FoldDevB)) + al256(4 * R) * 4 + al256(8 * R) * 2;   // dev; first, rdone, rank, last; lens, rl
  o += al256(4 * W) * 2 + al256(8 * C) * 2;                // bitmap, wloc, chunk counts / prefix
  o += al256(8 * T) * 3;                                   // tile delta sums, source bases
  o += al256(4 * NB * T) + al256(4 * NB) + al256(4 * (NB + 1)) * 2;   // hist, rowtot, bucket / chunk bases
  o += al256(16 * S) + al256(8 * S);                       // records, source offsets
  o += al256(16ull * BK_IDS * max_chunks(S, R));           // per-chunk id stats
  return o + 256;
}

size_t fold_scratch_bytes(uint64_t S, uint64_t R) {
  const size_t a = radix_scratch_bytes(S, R);
  return bucketed(R) ? std::max(a, bucket_scratch_bytes(S, R)) : a;
}

static int sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  }
  return n;
}

// MPSF_FOLD_RADIX=1 forces the radix path at any id space (tests and A/Bs)
static bool force_radix() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("MPSF_FOLD_RADIX");
    v = e && e[0] == '1' ? 1 : 0;
  }
  return v == 1;
}

static int launch_fold_bucket(uint8_t* scratch, uint32_t S, uint32_t R, const uint32_t* req, const uint32_t* nblk,
                              const uint32_t* ntok, const uint32_t* progress, const uint8_t* done,
                              const uint32_t* blocks, uint64_t n_blocks_in, const uint32_t* tokens,
                              uint64_t n_tokens_in, uint32_t* order, uint64_t* blk_off, uint32_t* blocks_out,
                              uint64_t* tok_off, uint32_t* tokens_out, uint32_t* prog_out, uint8_t* done_out,
                              FoldTotals* tot, cudaStream_t st, const Marker& mk) {
  const uint32_t T = (S + BT - 1) / BT, W = S / 32 + 1, C = (W + CHUNK_WORDS - 1) / CHUNK_WORDS, NB = n_buckets(R);
  const uint32_t NC = max_chunks(S, R);
  uint8_t* p = scratch;
  auto take = [&](size_t bytes) { uint8_t* r = p; p += al256(bytes); return r; };
  auto u32 = [&](size_t n) { return reinterpret_cast<uint32_t*>(take(4 * n)); };
  auto u64 = [&](size_t n) { return reinterpret_cast<unsigned long long*>(take(8 * n)); };
  FoldDevB* dev = reinterpret_cast<FoldDevB*>(take(sizeof(FoldDevB)));
  uint32_t *first = u32(R), *rdone = u32(R), *rank = u32(R), *lastx = u32(R);
  unsigned long long *lensr = u64(R), *rl = u64(R);
  uint32_t *bitmap = u32(W), *wloc = u32(W);
  unsigned long long *ccount = u64(C), *cpre = u64(C);
  unsigned long long *tsb = u64(T), *tst = u64(T), *tbase = u64(T);
  uint32_t *hist = u32((size_t)NB * T), *rowtot = u32(NB), *bbase = u32(NB + 1), *cbase = u32(NB + 1);
  uint4* rec = reinterpret_cast<uint4*>(take(16ull * S));
  uint2* src = reinterpret_cast<uint2*>(take(8ull * S));
  uint4* cstat = reinterpret_cast<uint4*>(take(16ull * BK_IDS * NC));
  const uint32_t gR = (uint32_t)std::min<uint64_t>((R + 255) / 256, (uint64_t)sms() * 8);
  int launches = 0;
  auto done_launch = [&](const char* name) { mk.mark(name); ++launches; };
  if (cudaMemsetAsync(dev, 0, sizeof(FoldDevB), st) != cudaSuccess) return -1;
  k_fb_count<<<T, BTN, 0, st>>>(S, R, NB, T, W, req, nblk, ntok, hist, tsb, tst, bitmap, dev);
  done_launch("k_fb_count");
  launch_pdl(k_fb_scan, NB + 1, 256, 0, st, T, NB, hist, rowtot, tsb, tst, tbase, dev);
  done_launch("k_fb_scan");
  if (cudaFuncSetAttribute(k_fb_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)FB_SCATTER_SMEM) !=
          cudaSuccess ||
      cudaFuncSetAttribute(k_fb_place, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)FB_PLACE_SMEM) != cudaSuccess)
    return -1;
  const int db = NB > 1 ? key_bits(NB - 1) : 1;
  launch_pdl(k_fb_scatter, T, BTN, FB_SCATTER_SMEM, st, S, R, NB, db, T, req, nblk, ntok, done, hist, rowtot, tbase,
             n_blocks_in, n_tokens_in, rec, src, bbase, cbase, dev);
  done_launch("k_fb_scatter");
  launch_pdl(k_fb_stats, NC, SCN, 0, st, NB, bbase, cbase, rec, cstat, blocks, n_blocks_in, tokens, n_tokens_in);
  done_launch("k_fb_stats");
  {   // one CTA per SM, all resident (the grid barrier needs every CTA running)
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)sms());   // >= the 16 CSR tiles an id space of 2^17 needs
    cfg.blockDim = dim3(1024);
    cfg.dynamicSmemBytes = 8 * CSR_TILE;
    cfg.stream = st;
    if (cudaFuncSetAttribute(k_fb_mid, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * CSR_TILE) != cudaSuccess)
      return -1;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    if (cudaLaunchKernelEx(&cfg, k_fb_mid, R, W, C, (const uint32_t*)cbase, cstat, first, lastx, rdone, lensr, bitmap,
                           wloc, ccount, cpre, progress, rank, order, done_out, prog_out, rl,
                           reinterpret_cast<unsigned long long*>(blk_off), reinterpret_cast<unsigned long long*>(tok_off),
                           dev) != cudaSuccess)
      return -1;
    done_launch("k_fb_mid");
  }
  launch_pdl(k_fb_place, NC, CHN, FB_PLACE_SMEM, st, R, NB, bbase, cbase, rec, src, cstat, rank,
             reinterpret_cast<const unsigned long long*>(blk_off), reinterpret_cast<const unsigned long long*>(tok_off),
             blocks, n_blocks_in, tokens, n_tokens_in, blocks_out, tokens_out);
  done_launch("k_fb_place");
  FoldDevB h{};
  if (cudaMemcpyAsync(&h, dev, 40, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess)
    return -1;
  if (!h.n_requests) {   // no live request: the CSR is the single zero offset
    const unsigned long long z = 0;
    if (cudaMemcpyAsync(blk_off, &z, 8, cudaMemcpyHostToDevice, st) != cudaSuccess ||
        cudaMemcpyAsync(tok_off, &z, 8, cudaMemcpyHostToDevice, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
      return -1;
  }
  tot->n_requests = h.n_requests;
  tot->n_blocks = h.n_blocks;
  tot->n_tokens = h.n_tokens;
  tot->error_index = h.err_enc ? (uint64_t)(uint32_t)~h.err_enc : ~0ull;
  tot->overrun = h.overrun;
  tot->launches = (uint32_t)launches;
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

int launch_fold(uint8_t* scratch, size_t scratch_bytes, uint32_t S, uint32_t R, const uint32_t* req,
                const uint32_t* nblk, const uint32_t* ntok, const uint32_t* progress, const uint8_t* done,
                const uint32_t* blocks, uint64_t n_blocks_in, const uint32_t* tokens, uint64_t n_tokens_in,
                uint32_t* order, uint64_t* blk_off, uint32_t* blocks_out, uint64_t* tok_off, uint32_t* tokens_out,
                uint32_t* prog_out, uint8_t* done_out, FoldTotals* tot, cudaStream_t st, const Marker& mk) {
  if (scratch_bytes < fold_scratch_bytes(S, R)) return -1;
  if (bucketed(R) && !force_radix())
    return launch_fold_bucket(scratch, S, R, req, nblk, ntok, progress, done, blocks, n_blocks_in, tokens, n_tokens_in,
                              order, blk_off, blocks_out, tok_off, tokens_out, prog_out, done_out, tot, st, mk);
  const uint32_t T = tiles(S), W = S / 32 + 1, C = (W + CHUNK_WORDS - 1) / CHUNK_WORDS;
  uint8_t* p = scratch;
  auto take = [&](size_t bytes) { uint8_t* r = p; p += al256(bytes); return r; };
  auto u32 = [&](size_t n) { return reinterpret_cast<uint32_t*>(take(4 * n)); };
  auto u64 = [&](size_t n) { return reinterpret_cast<unsigned long long*>(take(8 * n)); };
  FoldDev* dev = reinterpret_cast<FoldDev*>(take(64));
  uint32_t *first = u32(R), *rdone = u32(R), *rank = u32(R);
  uint32_t *bitmap = u32(W), *wloc = u32(W);
  unsigned long long *ccount = u64(C), *cpre = u64(C);
  unsigned long long *tsum = u64(T), *tbase = u64(T), *dsum = u64(T), *dbase = u64(T);
  uint32_t *kA = u32(S), *vA = u32(S), *kB = u32(S), *vB = u32(S);
  uint4* meta = reinterpret_cast<uint4*>(take(16ull * S));
  uint4* smeta = reinterpret_cast<uint4*>(take(16ull * S));
  uint32_t* hist = u32((size_t)NB_MAX * T);
  uint32_t* rowtot = u32(NB_MAX);
  const uint32_t live_bound = R < S ? R : S;   // ranks < min(R, S)
  const uint32_t gR = (uint32_t)std::min<uint64_t>((std::max(R, W) + 255) / 256, (uint64_t)sms() * 8);
  int launches = 0;
  auto done_launch = [&](const char* name) { mk.mark(name); ++launches; };

  k_fold_init<<<gR, 256, 0, st>>>(R, W, first, rdone, bitmap, dev);
  done_launch("k_fold_init");
  k_fold_stats<<<T, CB, 0, st>>>(S, R, req, done, nblk, ntok, first, rdone, meta, tsum, dev);
  done_launch("k_fold_stats");
  k_fold_bits<<<gR, 256, 0, st>>>(R, first, bitmap);
  done_launch("k_fold_bits");
  k_fold_bitcnt<<<C, CHUNK_WORDS, 0, st>>>(W, bitmap, wloc, ccount);
  done_launch("k_fold_bitcnt");
  k_fold_scan<<<2, 1024, 0, st>>>(ccount, cpre, C, &dev->n_requests, tsum, tbase, T);
  done_launch("k_fold_scan");
  k_fold_rank<<<gR, 256, 0, st>>>(R, first, rdone, bitmap, wloc, cpre, rank, order, done_out);
  done_launch("k_fold_rank");
  // radix sort by rank: passes of <= DB_MAX bits over the bits live_bound needs
  const int bits = key_bits(live_bound);
  const int passes = (bits + DB_MAX - 1) / DB_MAX, db = (bits + passes - 1) / passes;
  const uint32_t nbk = 1u << db;
  const uint32_t* kin = req;
  const uint32_t* vin = nullptr;
  uint32_t* ko = kA;
  uint32_t* vo = vA;
  for (int ps = 0; ps < passes; ++ps) {
    const uint32_t shift = (uint32_t)(ps * db);
    const bool f = ps == 0, l = ps == passes - 1;
    if (f) k_sort_hist<true><<<T, SB, 0, st>>>(S, R, live_bound, kin, rank, shift, nbk, T, hist);
    else k_sort_hist<false><<<T, SB, 0, st>>>(S, R, live_bound, kin, rank, shift, nbk, T, hist);
    done_launch("k_sort_hist");
    k_sort_hscan<<<nbk, 256, 0, st>>>(T, hist, rowtot);
    done_launch("k_sort_hscan");
    auto* kern = f ? (l ? k_sort_scatter<true, true> : k_sort_scatter<true, false>)
                   : (l ? k_sort_scatter<false, true> : k_sort_scatter<false, false>);
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SCATTER_SMEM) != cudaSuccess)
      return -1;

    kern<<<T, SB, SCATTER_SMEM, st>>>(S, R, live_bound, kin, vin, rank, shift, db, T, hist, rowtot, ko, vo, meta, tbase,
                                      smeta);
    done_launch("k_sort_scatter");
    kin = ko;
    vin = vo;
    ko = ko == kA ? kB : kA;
    vo = vo == vA ? vB : vA;
  }
  k_fold_dsum<<<T, CB, 0, st>>>(S, smeta, dsum);
  done_launch("k_fold_dsum");
  k_fold_scan<<<1, 1024, 0, st>>>(dsum, dbase, T, nullptr, nullptr, nullptr, 0);
  done_launch("k_fold_scan");
  if (cudaFuncSetAttribute(k_fold_place, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)PLACE_SMEM) != cudaSuccess)
    return -1;
  k_fold_place<<<T, CB, PLACE_SMEM, st>>>(S, live_bound, kin, vin, progress, prog_out, smeta, dbase, blocks, n_blocks_in, tokens, n_tokens_in,
                                 reinterpret_cast<unsigned long long*>(blk_off),
                                 reinterpret_cast<unsigned long long*>(tok_off), blocks_out, tokens_out, dev);
  done_launch("k_fold_place");
  FoldDev h{};
  if (cudaMemcpyAsync(&h, dev, sizeof(h), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess)
    return -1;
  if (!h.n_requests) {   // no live request: the CSR is the single zero offset
    const unsigned long long z = 0;
    if (cudaMemcpyAsync(blk_off, &z, 8, cudaMemcpyHostToDevice, st) != cudaSuccess ||
        cudaMemcpyAsync(tok_off, &z, 8, cudaMemcpyHostToDevice, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
      return -1;
  }
  tot->n_requests = h.n_requests;
  tot->n_blocks = h.n_blocks;
  tot->n_tokens = h.n_tokens;
  tot->error_index = h.err == NO_REQ ? ~0ull : h.err;
  tot->overrun = h.overrun;
  tot->launches = (uint32_t)launches;
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

// ---- KV pool restore: BlockPool.reserve (workload.py:77-80) of the folded block ids ----------
// complete_wake reserves every folded request's block ids in the standby's pool
// (recovery.py:356-357); the pool's free list is then the unreserved ids, popped smallest
// first.  Output: the reserved mask (the remap's valid mask over KV pages) and the free ids
// ascending (the heap's pop order): a stream compaction of the mask -- per-tile free counts,
// their prefix (one CTA), then each tile writes its free ids at its base.  Ids >= total are not
// pool blocks: they mark nothing.

__global__ void k_kv_mark(const uint32_t* __restrict__ blocks, uint64_t nb, uint32_t total,
                          uint8_t* __restrict__ reserved) {
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < nb; j += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t b = __ldcs(blocks + j);
    if (b < total) reserved[b] = 1;
  }
}

// thread t of tile b owns ids [b * FTILE + 8 t, + 8): its free mask as 8 bits
__device__ __forceinline__ uint32_t free_bits(const uint8_t* __restrict__ reserved, uint32_t i0, uint32_t total) {
  uint32_t m = 0;
  if (i0 + CIPT <= total && ((reinterpret_cast<uintptr_t>(reserved + i0) & 7u) == 0)) {
    const uint2 x = __ldg(reinterpret_cast<const uint2*>(reserved + i0));
#pragma unroll
    for (int b = 0; b < 8; ++b) m |= ((((b < 4 ? x.x : x.y) >> (8 * (b & 3))) & 0xFFu) == 0 ? 1u : 0u) << b;
  } else {
    for (uint32_t u = 0; u < CIPT && i0 + u < total; ++u) m |= (reserved[i0 + u] == 0 ? 1u : 0u) << u;
  }
  return m;
}

__global__ void __launch_bounds__(CB) k_kv_count(const uint8_t* __restrict__ reserved, uint32_t total,
                                                 unsigned long long* __restrict__ tcnt) {
  __shared__ unsigned long long sw[CWARPS + 1];
  const uint32_t m = free_bits(reserved, blockIdx.x * FTILE + threadIdx.x * CIPT, total);
  unsigned long long tot;
  block_excl_scan<unsigned long long, CWARPS>((unsigned long long)__popc(m), sw, tot);
  if (threadIdx.x == 0) tcnt[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(CB) k_kv_emit(const uint8_t* __restrict__ reserved, uint32_t total,
                                                const unsigned long long* __restrict__ tbase,
                                                uint32_t* __restrict__ free_ids) {
  __shared__ unsigned long long sw[CWARPS + 1];
  const uint32_t i0 = blockIdx.x * FTILE + threadIdx.x * CIPT;
  uint32_t m = free_bits(reserved, i0, total);
  unsigned long long tot;
  unsigned long long o = tbase[blockIdx.x] + block_excl_scan<unsigned long long, CWARPS>((unsigned long long)__popc(m), sw, tot);
  while (m) {
    const int b = __ffs(m) - 1;
    free_ids[o++] = i0 + b;
    m &= m - 1;
  }
}

size_t kv_reserve_scratch_bytes(uint32_t total) {
  const uint64_t T = tiles(total);
  return al256(8) + al256(8 * T) * 2 + 256;
}

int launch_kv_reserve(uint8_t* scratch, size_t scratch_bytes, uint32_t total, const uint32_t* blocks, uint64_t nb,
                      uint8_t* reserved, uint32_t* free_ids, uint64_t* n_free, cudaStream_t st) {
  if (scratch_bytes < kv_reserve_scratch_bytes(total)) return -1;
  const uint32_t T = tiles(total);
  unsigned long long* d_nfree = reinterpret_cast<unsigned long long*>(scratch);
  unsigned long long* tcnt = reinterpret_cast<unsigned long long*>(scratch + al256(8));
  unsigned long long* tb = reinterpret_cast<unsigned long long*>(scratch + al256(8) + al256(8ull * T));
  if (cudaMemsetAsync(reserved, 0, total, st) != cudaSuccess) return -1;
  if (nb) {
    const uint64_t g = std::min<uint64_t>((nb + 255) / 256, (uint64_t)sms() * 16);
    k_kv_mark<<<(uint32_t)g, 256, 0, st>>>(blocks, nb, total, reserved);
  }
  k_kv_count<<<T, CB, 0, st>>>(reserved, total, tcnt);
  k_fold_scan<<<1, 1024, 0, st>>>(tcnt, tb, T, d_nfree, nullptr, nullptr, 0);
  k_kv_emit<<<T, CB, 0, st>>>(reserved, total, tb, free_ids);
  unsigned long long h = 0;
  if (cudaMemcpyAsync(&h, d_nfree, 8, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess)
    return -1;
  *n_free = h;
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

}  // namespace mpsf
