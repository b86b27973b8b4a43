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
//   k_fold_stats   per request: first / last snapshot, delta totals, done (atomics)
//   heads          a snapshot is its request's head iff it is the request's first; the heads'
//                  exclusive scan ranks the requests in first-appearance order
//   sort           snapshots by request rank, stable (CUB radix sort keeps index order)
//   scans          source offsets (consume order) and destination offsets (sorted order)
//   k_fold_copy    one warp per snapshot copies its deltas to their destination
// CUB supplies the scan and the radix sort (library primitives, like cuBLAS for a GEMM).
#include <cub/cub.cuh>
#include <cuda_runtime.h>
#include <stdint.h>

#include "mpsf_kernels.h"

namespace mpsf {

constexpr uint32_t NO_REQ = 0xFFFFFFFFu;

__global__ void k_fold_stats(uint32_t S, const uint32_t* __restrict__ req, const uint32_t* __restrict__ nblk,
                             const uint32_t* __restrict__ ntok, const uint8_t* __restrict__ done,
                             uint32_t* __restrict__ first, uint32_t* __restrict__ last,
                             unsigned long long* __restrict__ cblk, unsigned long long* __restrict__ ctok,
                             uint32_t* __restrict__ rdone, uint32_t R, uint32_t* __restrict__ err) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < S; i += gridDim.x * blockDim.x) {
    const uint32_t r = req[i];
    if (r == NO_REQ) continue;
    if (r >= R) {   // request id outside the caller's id space: reported, nothing folded for it
      atomicMin(err, i);
      continue;
    }
    atomicMin(first + r, i);
    atomicMax(last + r, i);
    if (nblk[i]) atomicAdd(cblk + r, (unsigned long long)nblk[i]);
    if (ntok[i]) atomicAdd(ctok + r, (unsigned long long)ntok[i]);
    if (done[i]) atomicOr(rdone + r, 1u);
  }
}

__global__ void k_fold_heads(uint32_t S, const uint32_t* __restrict__ req, const uint32_t* __restrict__ first,
                             uint32_t* __restrict__ head) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < S; i += gridDim.x * blockDim.x) {
    const uint32_t r = req[i];
    head[i] = (r != NO_REQ && first[r] == i) ? 1u : 0u;
  }
}

// rank per request, the order list, per-rank outputs; sort keys (rank, liveness snapshots last)
__global__ void k_fold_rank(uint32_t S, const uint32_t* __restrict__ req, const uint32_t* __restrict__ head,
                            const uint32_t* __restrict__ head_pos, const uint32_t* __restrict__ last,
                            const unsigned long long* __restrict__ cblk, const unsigned long long* __restrict__ ctok,
                            const uint32_t* __restrict__ rdone, const uint32_t* __restrict__ progress,
                            uint32_t* __restrict__ rank, uint32_t* __restrict__ order,
                            unsigned long long* __restrict__ blk_cnt, unsigned long long* __restrict__ tok_cnt,
                            uint32_t* __restrict__ prog_out, uint8_t* __restrict__ done_out) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < S; i += gridDim.x * blockDim.x) {
    if (!head[i]) continue;
    const uint32_t r = req[i], k = head_pos[i];
    rank[r] = k;
    order[k] = r;
    blk_cnt[k] = cblk[r];
    tok_cnt[k] = ctok[r];
    prog_out[k] = progress[last[r]];
    done_out[k] = rdone[r] ? 1 : 0;
  }
}

__global__ void k_fold_keys(uint32_t S, const uint32_t* __restrict__ req, const uint32_t* __restrict__ rank,
                            uint32_t* __restrict__ key, uint32_t* __restrict__ idx) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < S; i += gridDim.x * blockDim.x) {
    const uint32_t r = req[i];
    key[i] = r == NO_REQ ? NO_REQ : rank[r];
    idx[i] = i;
  }
}

// position p -> snapshot i: the delta lengths in that order (key == nullptr: every snapshot, for
// the source offsets -- a liveness snapshot's deltas still occupy the input; else liveness
// snapshots count zero, for the destination offsets in sorted order)
__global__ void k_fold_gather(uint32_t S, const uint32_t* __restrict__ sidx, const uint32_t* __restrict__ key,
                              const uint32_t* __restrict__ nblk, const uint32_t* __restrict__ ntok,
                              unsigned long long* __restrict__ sb, unsigned long long* __restrict__ st) {
  for (uint32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < S; p += gridDim.x * blockDim.x) {
    const uint32_t i = sidx[p];
    const bool live = key == nullptr || key[p] != NO_REQ;
    sb[p] = live ? nblk[i] : 0;
    st[p] = live ? ntok[i] : 0;
  }
}

// one warp per sorted snapshot: its deltas from their consume-order offsets to the fold
__global__ void k_fold_copy(uint32_t S, const uint32_t* __restrict__ sidx, const uint32_t* __restrict__ key,
                            const uint32_t* __restrict__ nblk, const uint32_t* __restrict__ ntok,
                            const unsigned long long* __restrict__ src_b, const unsigned long long* __restrict__ src_t,
                            const unsigned long long* __restrict__ dst_b, const unsigned long long* __restrict__ dst_t,
                            const uint32_t* __restrict__ blocks, const uint32_t* __restrict__ tokens,
                            uint32_t* __restrict__ blocks_out, uint32_t* __restrict__ tokens_out) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t W = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t p = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; p < S; p += W) {
    if (key[p] == NO_REQ) continue;
    const uint32_t i = sidx[p];
    for (uint32_t k = lane; k < nblk[i]; k += 32) blocks_out[dst_b[p] + k] = blocks[src_b[i] + k];
    for (uint32_t k = lane; k < ntok[i]; k += 32) tokens_out[dst_t[p] + k] = tokens[src_t[i] + k];
  }
}

static size_t al256(size_t x) { return (x + 255) & ~size_t(255); }

// scratch layout for S snapshots and R request ids
size_t fold_scratch_bytes(uint64_t S, uint64_t R) {
  size_t o = 0;
  o += al256(4 * R) * 3;            // first, last, rdone
  o += al256(8 * R) * 2;            // cblk, ctok
  o += al256(4 * R);                // rank
  o += al256(4 * S) * 6;            // head, head_pos, key, idx, skey, sidx
  o += al256(8 * S) * 6;            // src_b, src_t, sb, st, dst_b, dst_t
  o += al256(8 * (S + 1)) * 2;      // blk_cnt / tok_cnt by rank (+1 for the totals)
  o += al256(4);                    // err
  size_t cub_bytes = 0, t = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, t, (const unsigned long long*)nullptr, (unsigned long long*)nullptr,
                                (int)(S + 1));
  cub_bytes = t > cub_bytes ? t : cub_bytes;
  cub::DeviceScan::ExclusiveSum(nullptr, t, (const uint32_t*)nullptr, (uint32_t*)nullptr, (int)S);
  cub_bytes = t > cub_bytes ? t : cub_bytes;
  cub::DeviceRadixSort::SortPairs(nullptr, t, (const uint32_t*)nullptr, (uint32_t*)nullptr,
                                  (const uint32_t*)nullptr, (uint32_t*)nullptr, (int)S);
  cub_bytes = t > cub_bytes ? t : cub_bytes;
  return o + al256(cub_bytes) + 256;
}

int launch_fold(uint8_t* scratch, size_t scratch_bytes, uint32_t S, uint32_t R, const uint32_t* req,
                const uint32_t* nblk, const uint32_t* ntok, const uint32_t* progress, const uint8_t* done,
                const uint32_t* blocks, const uint32_t* tokens, uint32_t* order, uint64_t* blk_off,
                uint32_t* blocks_out, uint64_t* tok_off, uint32_t* tokens_out, uint32_t* prog_out,
                uint8_t* done_out, FoldTotals* tot, cudaStream_t st) {
  uint8_t* p = scratch;
  auto take = [&](size_t bytes) { uint8_t* r = p; p += al256(bytes); return r; };
  uint32_t* first = reinterpret_cast<uint32_t*>(take(4ull * R));
  uint32_t* last = reinterpret_cast<uint32_t*>(take(4ull * R));
  uint32_t* rdone = reinterpret_cast<uint32_t*>(take(4ull * R));
  unsigned long long* cblk = reinterpret_cast<unsigned long long*>(take(8ull * R));
  unsigned long long* ctok = reinterpret_cast<unsigned long long*>(take(8ull * R));
  uint32_t* rank = reinterpret_cast<uint32_t*>(take(4ull * R));
  uint32_t* head = reinterpret_cast<uint32_t*>(take(4ull * S));
  uint32_t* head_pos = reinterpret_cast<uint32_t*>(take(4ull * S));
  uint32_t* key = reinterpret_cast<uint32_t*>(take(4ull * S));
  uint32_t* idx = reinterpret_cast<uint32_t*>(take(4ull * S));
  uint32_t* skey = reinterpret_cast<uint32_t*>(take(4ull * S));
  uint32_t* sidx = reinterpret_cast<uint32_t*>(take(4ull * S));
  unsigned long long* src_b = reinterpret_cast<unsigned long long*>(take(8ull * S));
  unsigned long long* src_t = reinterpret_cast<unsigned long long*>(take(8ull * S));
  unsigned long long* sb = reinterpret_cast<unsigned long long*>(take(8ull * S));
  unsigned long long* stk = reinterpret_cast<unsigned long long*>(take(8ull * S));
  unsigned long long* dst_b = reinterpret_cast<unsigned long long*>(take(8ull * S));
  unsigned long long* dst_t = reinterpret_cast<unsigned long long*>(take(8ull * S));
  unsigned long long* bcnt = reinterpret_cast<unsigned long long*>(take(8ull * (S + 1)));
  unsigned long long* tcnt = reinterpret_cast<unsigned long long*>(take(8ull * (S + 1)));
  uint32_t* err = reinterpret_cast<uint32_t*>(take(4));
  uint8_t* cub_tmp = p;
  size_t cub_bytes = scratch_bytes - (size_t)(p - scratch);
  if (cudaMemsetAsync(first, 0xFF, 4ull * R, st) != cudaSuccess || cudaMemsetAsync(last, 0, 4ull * R, st) ||
      cudaMemsetAsync(rdone, 0, 4ull * R, st) || cudaMemsetAsync(cblk, 0, 8ull * R, st) ||
      cudaMemsetAsync(ctok, 0, 8ull * R, st) || cudaMemsetAsync(bcnt, 0, 8ull * (S + 1), st) ||
      cudaMemsetAsync(tcnt, 0, 8ull * (S + 1), st) || cudaMemsetAsync(err, 0xFF, 4, st))
    return -1;
  const int g = 296, b = 256;
  k_fold_stats<<<g, b, 0, st>>>(S, req, nblk, ntok, done, first, last, cblk, ctok, rdone, R, err);
  k_fold_heads<<<g, b, 0, st>>>(S, req, first, head);
  size_t t = cub_bytes;
  if (cub::DeviceScan::ExclusiveSum(cub_tmp, t, head, head_pos, (int)S, st) != cudaSuccess) return -1;
  k_fold_rank<<<g, b, 0, st>>>(S, req, head, head_pos, last, cblk, ctok, rdone, progress, rank, order, bcnt, tcnt,
                               prog_out, done_out);
  k_fold_keys<<<g, b, 0, st>>>(S, req, rank, key, idx);
  t = cub_bytes;
  if (cub::DeviceRadixSort::SortPairs(cub_tmp, t, key, skey, idx, sidx, (int)S, 0, 32, st) != cudaSuccess) return -1;
  // source offsets: consume order
  t = cub_bytes;
  k_fold_gather<<<g, b, 0, st>>>(S, idx, nullptr, nblk, ntok, sb, stk);   // identity order, all lengths
  if (cub::DeviceScan::ExclusiveSum(cub_tmp, t, sb, src_b, (int)S, st) != cudaSuccess) return -1;
  t = cub_bytes;
  if (cub::DeviceScan::ExclusiveSum(cub_tmp, t, stk, src_t, (int)S, st) != cudaSuccess) return -1;
  // destination offsets: sorted order (liveness snapshots carry no payload)
  k_fold_gather<<<g, b, 0, st>>>(S, sidx, skey, nblk, ntok, sb, stk);
  t = cub_bytes;
  if (cub::DeviceScan::ExclusiveSum(cub_tmp, t, sb, dst_b, (int)S, st) != cudaSuccess) return -1;
  t = cub_bytes;
  if (cub::DeviceScan::ExclusiveSum(cub_tmp, t, stk, dst_t, (int)S, st) != cudaSuccess) return -1;
  // per-request CSR offsets (ranks beyond the request count carry zero counts)
  t = cub_bytes;
  if (cub::DeviceScan::ExclusiveSum(cub_tmp, t, bcnt, reinterpret_cast<unsigned long long*>(blk_off), (int)(S + 1),
                                    st) != cudaSuccess)
    return -1;
  t = cub_bytes;
  if (cub::DeviceScan::ExclusiveSum(cub_tmp, t, tcnt, reinterpret_cast<unsigned long long*>(tok_off), (int)(S + 1),
                                    st) != cudaSuccess)
    return -1;
  k_fold_copy<<<g, b, 0, st>>>(S, sidx, skey, nblk, ntok, src_b, src_t, dst_b, dst_t, blocks, tokens, blocks_out,
                               tokens_out);
  // request count = number of heads = head_pos[S-1] + head[S-1]; totals = the CSR ends
  uint32_t hp = 0, hd = 0, e = NO_REQ;
  if (S && (cudaMemcpyAsync(&hp, head_pos + S - 1, 4, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
            cudaMemcpyAsync(&hd, head + S - 1, 4, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
            cudaMemcpyAsync(&e, err, 4, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
            cudaStreamSynchronize(st) != cudaSuccess))
    return -1;
  tot->n_requests = hp + hd;
  tot->error_index = e == NO_REQ ? ~0ull : e;
  tot->n_blocks = tot->n_tokens = 0;
  if (tot->n_requests && (cudaMemcpyAsync(&tot->n_blocks, blk_off + tot->n_requests, 8, cudaMemcpyDeviceToHost,
                                          st) != cudaSuccess ||
                          cudaMemcpyAsync(&tot->n_tokens, tok_off + tot->n_requests, 8, cudaMemcpyDeviceToHost,
                                          st) != cudaSuccess ||
                          cudaStreamSynchronize(st) != cudaSuccess))
    return -1;
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

}  // namespace mpsf
