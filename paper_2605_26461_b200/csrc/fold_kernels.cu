// Snapshot delta fold on the GPU (the step after the recovery remap).
//
// Reference: StandbyInstance.fold (pkg/src/mpssim/recovery.py:83-92) consumes the ring's
// ForwardSnapshots in order; per request (dict insertion order = first appearance) it appends
// the KV-block-id and token deltas, keeps the last progress and a sticky done flag.
// complete_wake (recovery.py:310-363) then restores each request's block table from the fold.
//
// Batch form: S snapshots in consume order as SoA (request id or NO_REQ, delta lengths,
// progress, done) plus the concatenated deltas.  The fold is a stable group-by with
// variable-length payloads:
//   k_fold_stats   per request id: first / last snapshot (atomicMin/Max), sticky done (atomicOr)
//   head scan      heads (a request's first snapshot) counted in consume order, fed by an
//                  iterator: ranks the requests in first-appearance order
//   k_fold_rank    per head: rank, order, last progress, done, request count
//   src scan       (blocks | tokens << 32) in consume order: each snapshot's source offsets
//   sort           snapshot indices by request rank, stable (CUB onesweep radix sort over
//                  only the bits min(R, S) needs; liveness-only snapshots sort last)
//   dst scan       packed lengths in sorted order, scattered back to consume order through a
//                  permutation output iterator: each snapshot's destination offsets
//   k_fold_copy    thread per snapshot in consume order (coalesced reads of the SoA, the
//                  offsets and the payload): its deltas to their destination; heads write
//                  their request's CSR start, the last live snapshot in fold order the ends
// CUB supplies the scans and the radix sort (library primitives, like cuBLAS for a GEMM).
#include <cub/cub.cuh>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <thrust/iterator/counting_iterator.h>
#include <thrust/iterator/permutation_iterator.h>
#include <thrust/iterator/transform_iterator.h>

#include "mpsf_kernels.h"

namespace mpsf {

constexpr uint32_t NO_REQ = 0xFFFFFFFFu;

struct FoldDev {            // device-side totals, read back once
  unsigned long long n_requests, n_blocks, n_tokens;
  uint32_t err;             // first snapshot with a request id >= R (NO_REQ: none)
  uint32_t overrun;         // deltas reach past the payload arrays
};

__device__ __forceinline__ unsigned long long pack_len(uint32_t nb, uint32_t nt) {
  return (unsigned long long)nb | ((unsigned long long)nt << 32);
}

// The gather kernels (rank, keys) and the stats take FI snapshots per thread (block-strided, so every load stays
// coalesced) and issue all of their loads before the dependent gathers / atomics: one
// snapshot per thread left them latency-bound at 10-20 % issue activity.
constexpr int FI = 4;
__device__ __forceinline__ uint32_t fi_index(int u) { return blockIdx.x * (blockDim.x * FI) + u * blockDim.x + threadIdx.x; }

__global__ void k_fold_stats(uint32_t S, uint32_t R, const uint32_t* __restrict__ req,
                             const uint8_t* __restrict__ done, uint32_t* __restrict__ first,
                             uint32_t* __restrict__ last, uint32_t* __restrict__ rdone, FoldDev* __restrict__ dev) {
  uint32_t r[FI];
  uint8_t dn[FI];
#pragma unroll
  for (int u = 0; u < FI; ++u) {
    const uint32_t i = fi_index(u);
    r[u] = i < S ? req[i] : NO_REQ;
    dn[u] = i < S ? done[i] : 0;
  }
#pragma unroll
  for (int u = 0; u < FI; ++u) {
    const uint32_t i = fi_index(u);
    if (r[u] == NO_REQ) continue;
    if (r[u] >= R) {   // request id outside the caller's id space: reported, not folded
      atomicMin(&dev->err, i);
      continue;
    }
    atomicMin(first + r[u], i);
    atomicMax(last + r[u], i);
    if (dn[u]) atomicOr(rdone + r[u], 1u);
  }
}

struct HeadFlag {           // snapshot i is its request's first
  const uint32_t* req;
  const uint32_t* first;
  uint32_t R;
  __device__ uint32_t operator()(uint32_t i) const {
    const uint32_t r = req[i];
    return (r < R && first[r] == i) ? 1u : 0u;
  }
};

struct PackLen {            // packed lengths of snapshot i, consume order (every snapshot)
  const uint32_t* nblk;
  const uint32_t* ntok;
  __device__ unsigned long long operator()(uint32_t i) const { return pack_len(nblk[i], ntok[i]); }
};

struct PackLenSorted {      // packed lengths at sorted position p (liveness-only snapshots: 0)
  const uint32_t* sidx;
  const uint32_t* skey;
  const uint32_t* nblk;
  const uint32_t* ntok;
  uint32_t live_bound;
  __device__ unsigned long long operator()(uint32_t p) const {
    if (skey[p] >= live_bound) return 0ull;
    const uint32_t i = sidx[p];
    return pack_len(nblk[i], ntok[i]);
  }
};

// heads: rank, the request's order entry, its last progress and sticky done; the count
__global__ void k_fold_rank(uint32_t S, uint32_t R, const uint32_t* __restrict__ req,
                            const uint32_t* __restrict__ first, const uint32_t* __restrict__ last,
                            const uint32_t* __restrict__ rdone, const uint32_t* __restrict__ progress,
                            const uint32_t* __restrict__ head_pos, uint32_t* __restrict__ rank,
                            uint32_t* __restrict__ order, uint32_t* __restrict__ prog_out,
                            uint8_t* __restrict__ done_out, FoldDev* __restrict__ dev) {
  uint32_t r[FI], f[FI];
#pragma unroll
  for (int u = 0; u < FI; ++u) {
    const uint32_t i = fi_index(u);
    r[u] = i < S ? req[i] : NO_REQ;
  }
#pragma unroll
  for (int u = 0; u < FI; ++u) f[u] = r[u] < R ? first[r[u]] : NO_REQ;
#pragma unroll
  for (int u = 0; u < FI; ++u) {
    const uint32_t i = fi_index(u);
    if (i >= S) break;
    const bool head = r[u] < R && f[u] == i;
    if (head) {
      const uint32_t k = head_pos[i];
      rank[r[u]] = k;
      order[k] = r[u];
      prog_out[k] = progress[last[r[u]]];
      done_out[k] = rdone[r[u]] ? 1 : 0;
    }
    if (i == S - 1) dev->n_requests = head_pos[i] + (head ? 1u : 0u);
  }
}

// sort keys: the request's rank; liveness-only (and rejected) snapshots key past every rank
__global__ void k_fold_keys(uint32_t S, uint32_t R, uint32_t live_bound, const uint32_t* __restrict__ req,
                            const uint32_t* __restrict__ rank, uint32_t* __restrict__ key,
                            uint32_t* __restrict__ idx) {
  uint32_t r[FI], k[FI];
#pragma unroll
  for (int u = 0; u < FI; ++u) {
    const uint32_t i = fi_index(u);
    r[u] = i < S ? req[i] : NO_REQ;
  }
#pragma unroll
  for (int u = 0; u < FI; ++u) k[u] = r[u] < R ? rank[r[u]] : live_bound;
#pragma unroll
  for (int u = 0; u < FI; ++u) {
    const uint32_t i = fi_index(u);
    if (i < S) {
      key[i] = k[u];
      idx[i] = i;
    }
  }
}

// thread per snapshot in consume order: coalesced reads of the SoA, offsets and payload
__global__ void k_fold_copy(uint32_t S, uint32_t R, const uint32_t* __restrict__ req,
                            const uint32_t* __restrict__ nblk, const uint32_t* __restrict__ ntok,
                            const uint32_t* __restrict__ first, const uint32_t* __restrict__ last,
                            const uint32_t* __restrict__ rank, const unsigned long long* __restrict__ src,
                            const unsigned long long* __restrict__ dst, const uint32_t* __restrict__ blocks,
                            const uint32_t* __restrict__ tokens, unsigned long long n_blocks_in,
                            unsigned long long n_tokens_in, unsigned long long* __restrict__ blk_off,
                            unsigned long long* __restrict__ tok_off, uint32_t* __restrict__ blocks_out,
                            uint32_t* __restrict__ tokens_out, FoldDev* __restrict__ dev) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= S) return;
  const uint32_t r = req[i];
  if (r >= R) return;                        // liveness-only / rejected
  const unsigned long long s = src[i], d = dst[i];
  const uint32_t sb = (uint32_t)s, st = (uint32_t)(s >> 32), db = (uint32_t)d, dt = (uint32_t)(d >> 32);
  const uint32_t nb = nblk[i], nt = ntok[i];
  if ((unsigned long long)sb + nb > n_blocks_in || (unsigned long long)st + nt > n_tokens_in ||
      (unsigned long long)db + nb > n_blocks_in || (unsigned long long)dt + nt > n_tokens_in) {
    atomicOr(&dev->overrun, 1u);
  } else {
    for (uint32_t j = 0; j < nb; ++j) blocks_out[db + j] = blocks[sb + j];
    for (uint32_t j = 0; j < nt; ++j) tokens_out[dt + j] = tokens[st + j];
  }
  const bool head = first[r] == i, tail = last[r] == i;
  if (head || tail) {
    const uint32_t k = rank[r];
    if (head) {                              // the request's CSR start
      blk_off[k] = db;
      tok_off[k] = dt;
    }
    if (tail && k + 1ull == dev->n_requests) {   // the last live snapshot in fold order: the CSR ends
      blk_off[k + 1] = (unsigned long long)db + nb;
      tok_off[k + 1] = (unsigned long long)dt + nt;
      dev->n_blocks = (unsigned long long)db + nb;
      dev->n_tokens = (unsigned long long)dt + nt;
    }
  }
}

static size_t al256(size_t x) { return (x + 255) & ~size_t(255); }

static int key_bits(uint32_t live_bound) {   // bits for keys in [0, live_bound]
  int b = 1;
  while (b < 32 && (1ull << b) <= live_bound) ++b;
  return b;
}

// scratch layout for S snapshots and R request ids
size_t fold_scratch_bytes(uint64_t S, uint64_t R) {
  size_t o = al256(sizeof(FoldDev)) + al256(4 * R) * 4;   // dev, first, last, rdone, rank
  o += al256(4 * S) * 5;                                   // head_pos, key, idx, skey, sidx
  o += al256(8 * S) * 2;                                   // src, dst
  size_t cub_bytes = 0, t = 0;
  thrust::counting_iterator<uint32_t> c0(0);
  cub::DeviceScan::ExclusiveSum(nullptr, t, thrust::make_transform_iterator(c0, HeadFlag{}), (uint32_t*)nullptr,
                                (int)S);
  cub_bytes = t > cub_bytes ? t : cub_bytes;
  cub::DeviceScan::ExclusiveSum(nullptr, t, thrust::make_transform_iterator(c0, PackLen{}),
                                (unsigned long long*)nullptr, (int)S);
  cub_bytes = t > cub_bytes ? t : cub_bytes;
  cub::DeviceScan::ExclusiveSum(nullptr, t, thrust::make_transform_iterator(c0, PackLenSorted{}),
                                thrust::make_permutation_iterator((unsigned long long*)nullptr, (const uint32_t*)nullptr),
                                (int)S);
  cub_bytes = t > cub_bytes ? t : cub_bytes;
  cub::DeviceRadixSort::SortPairs(nullptr, t, (const uint32_t*)nullptr, (uint32_t*)nullptr,
                                  (const uint32_t*)nullptr, (uint32_t*)nullptr, (int)S);
  cub_bytes = t > cub_bytes ? t : cub_bytes;
  return o + al256(cub_bytes) + 256;
}

int launch_fold(uint8_t* scratch, size_t scratch_bytes, uint32_t S, uint32_t R, const uint32_t* req,
                const uint32_t* nblk, const uint32_t* ntok, const uint32_t* progress, const uint8_t* done,
                const uint32_t* blocks, uint64_t n_blocks_in, const uint32_t* tokens, uint64_t n_tokens_in,
                uint32_t* order, uint64_t* blk_off, uint32_t* blocks_out, uint64_t* tok_off, uint32_t* tokens_out,
                uint32_t* prog_out, uint8_t* done_out, FoldTotals* tot, cudaStream_t st) {
  uint8_t* p = scratch;
  auto take = [&](size_t bytes) { uint8_t* r = p; p += al256(bytes); return r; };
  FoldDev* dev = reinterpret_cast<FoldDev*>(take(sizeof(FoldDev)));
  uint32_t* first = reinterpret_cast<uint32_t*>(take(4ull * R));
  uint32_t* last = reinterpret_cast<uint32_t*>(take(4ull * R));
  uint32_t* rdone = reinterpret_cast<uint32_t*>(take(4ull * R));
  uint32_t* rank = reinterpret_cast<uint32_t*>(take(4ull * R));
  uint32_t* head_pos = reinterpret_cast<uint32_t*>(take(4ull * S));
  uint32_t* key = reinterpret_cast<uint32_t*>(take(4ull * S));
  uint32_t* idx = reinterpret_cast<uint32_t*>(take(4ull * S));
  uint32_t* skey = reinterpret_cast<uint32_t*>(take(4ull * S));
  uint32_t* sidx = reinterpret_cast<uint32_t*>(take(4ull * S));
  unsigned long long* src = reinterpret_cast<unsigned long long*>(take(8ull * S));
  unsigned long long* dst = reinterpret_cast<unsigned long long*>(take(8ull * S));
  uint8_t* cub_tmp = p;
  const size_t cub_bytes = scratch_bytes - (size_t)(p - scratch);
  const uint32_t live_bound = R < S ? R : S;   // ranks < min(R, S)
  const FoldDev init{0, 0, 0, NO_REQ, 0};
  if (cudaMemcpyAsync(dev, &init, sizeof(init), cudaMemcpyHostToDevice, st) != cudaSuccess ||
      cudaMemsetAsync(first, 0xFF, 4ull * R, st) != cudaSuccess ||
      cudaMemsetAsync(last, 0, 4ull * R, st) != cudaSuccess || cudaMemsetAsync(rdone, 0, 4ull * R, st) != cudaSuccess)
    return -1;
  const uint32_t b = 256, g = (S + b * FI - 1) / (b * FI);
  k_fold_stats<<<g, b, 0, st>>>(S, R, req, done, first, last, rdone, dev);
  thrust::counting_iterator<uint32_t> c0(0);
  size_t t = cub_bytes;
  if (cub::DeviceScan::ExclusiveSum(cub_tmp, t, thrust::make_transform_iterator(c0, HeadFlag{req, first, R}),
                                    head_pos, (int)S, st) != cudaSuccess)
    return -1;
  k_fold_rank<<<g, b, 0, st>>>(S, R, req, first, last, rdone, progress, head_pos, rank, order, prog_out, done_out,
                               dev);
  k_fold_keys<<<g, b, 0, st>>>(S, R, live_bound, req, rank, key, idx);
  t = cub_bytes;
  if (cub::DeviceRadixSort::SortPairs(cub_tmp, t, key, skey, idx, sidx, (int)S, 0, key_bits(live_bound), st) !=
      cudaSuccess)
    return -1;
  t = cub_bytes;
  if (cub::DeviceScan::ExclusiveSum(cub_tmp, t, thrust::make_transform_iterator(c0, PackLen{nblk, ntok}), src,
                                    (int)S, st) != cudaSuccess)
    return -1;
  t = cub_bytes;
  if (cub::DeviceScan::ExclusiveSum(
          cub_tmp, t, thrust::make_transform_iterator(c0, PackLenSorted{sidx, skey, nblk, ntok, live_bound}),
          thrust::make_permutation_iterator(dst, sidx), (int)S, st) != cudaSuccess)
    return -1;
  k_fold_copy<<<(S + b - 1) / b, b, 0, st>>>(S, R, req, nblk, ntok, first, last, rank, src, dst, blocks, tokens, n_blocks_in,
                               n_tokens_in, reinterpret_cast<unsigned long long*>(blk_off),
                               reinterpret_cast<unsigned long long*>(tok_off), blocks_out, tokens_out, dev);
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
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

// ---- KV pool restore: BlockPool.reserve (workload.py:77-80) of the folded block ids ----------
// complete_wake reserves every folded request's block ids in the standby's pool
// (recovery.py:356-357); the pool's free list is then the unreserved ids, popped smallest
// first.  Output: the reserved mask (the remap's valid mask over KV pages) and the free ids
// ascending (the heap's pop order).  Ids >= total are not pool blocks: they mark nothing.

__global__ void k_kv_mark(const uint32_t* __restrict__ blocks, uint64_t nb, uint32_t total,
                          uint8_t* __restrict__ reserved) {
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < nb; j += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t b = __ldcs(blocks + j);
    if (b < total) reserved[b] = 1;
  }
}

struct IsFree {
  const uint8_t* reserved;
  __device__ bool operator()(uint32_t b) const { return reserved[b] == 0; }
};

size_t kv_reserve_scratch_bytes(uint32_t total) {
  size_t t = 0;
  thrust::counting_iterator<uint32_t> c0(0);
  cub::DeviceSelect::If(nullptr, t, c0, (uint32_t*)nullptr, (unsigned long long*)nullptr, (int64_t)total, IsFree{});
  return al256(8) + al256(t) + 256;
}

int launch_kv_reserve(uint8_t* scratch, size_t scratch_bytes, uint32_t total, const uint32_t* blocks, uint64_t nb,
                      uint8_t* reserved, uint32_t* free_ids, uint64_t* n_free, cudaStream_t st) {
  unsigned long long* d_nsel = reinterpret_cast<unsigned long long*>(scratch);
  uint8_t* cub_tmp = scratch + al256(8);
  size_t t = scratch_bytes - al256(8);
  if (cudaMemsetAsync(reserved, 0, total, st) != cudaSuccess) return -1;
  if (nb) {
    const uint64_t g = std::min<uint64_t>((nb + 255) / 256, 148ull * 16);
    k_kv_mark<<<(uint32_t)g, 256, 0, st>>>(blocks, nb, total, reserved);
  }
  thrust::counting_iterator<uint32_t> c0(0);
  if (cub::DeviceSelect::If(cub_tmp, t, c0, free_ids, d_nsel, (int64_t)total, IsFree{reserved}, st) != cudaSuccess)
    return -1;
  unsigned long long h = 0;
  if (cudaMemcpyAsync(&h, d_nsel, 8, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess)
    return -1;
  *n_free = h;
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

}  // namespace mpsf
