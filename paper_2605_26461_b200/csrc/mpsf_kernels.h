// Host-side launch entry points of the sm_100a kernels (called by mpsf_abi.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "mpsf.h"
#include "mpsf_device.cuh"

namespace mpsf {

// Optional per-kernel timing hook: called right after each launch on the same stream
// (mpsf_abi.cu records a CUDA event there when profiling is on).
struct Marker {
  void (*fn)(void* ctx, const char* name) = nullptr;
  void* ctx = nullptr;
  void mark(const char* name) const {
    if (fn) fn(ctx, name);
  }
};

// pass 1 (counts accumulate across the launches of a chunked batch; k_init zeroes them)
int launch_scan(const World& W, const Scratch& S, const mpsf_fault_entry* in, uint64_t n, const Params& P,
                unsigned long long* counts, cudaStream_t st, const Marker& mk);
int launch_resolve(const World& W, const Scratch& S, const Params& P, mpsf_client_verdict* verdict,
                   cudaStream_t st, const Marker& mk);
int launch_general(const World& W, const Scratch& S, const mpsf_fault_entry* in, uint64_t n, const Params& P,
                   int stage, cudaStream_t st, const Marker& mk);
int launch_resolve2(const World& W, const Scratch& S, const Params& P, cudaStream_t st, const Marker& mk);
// single-GPU batches on the fixed layout: k_resolve + k_general stage 1 in one launch; pass 2 then
// folds in what k_resolve2 would (so neither separate launch is needed)
bool resolve_fused_fits(const World& W);
int launch_resolve_general(const World& W, const Scratch& S, const mpsf_fault_entry* in, uint64_t n, const Params& P,
                           mpsf_client_verdict* verdict, cudaStream_t st, const Marker& mk);
// pass 2 over entries [0, n) of `in`, a chunk of the batch starting at batch chunk q_base (the
// chunk's first entry is batch entry 64 * q_base); then, once per batch, the ordered lists
int launch_finalize(const World& W, const Scratch& S, const mpsf_fault_entry* in, uint64_t n, const Params& P,
                    mpsf_out_record* out, uint64_t q_base, cudaStream_t st, const Marker& mk);
int launch_lists(const Scratch& S, const mpsf_fault_entry* in, const mpsf_out_record* out, uint64_t n,
                 uint64_t base_index, unsigned long long* dkeys, uint32_t* didx, uint32_t* cancel, DevSummary* sum,
                 cudaStream_t st, const Marker& mk);
int launch_copyout(const Scratch& S, uint64_t n, const unsigned long long* d_dk, const uint32_t* d_di,
                   const uint32_t* d_ca, unsigned long long* h_dk, uint32_t* h_di, uint32_t* h_ca, cudaStream_t st);
// batched translation (MemoryModel.resolve_va over an access stream): hit bytes, the misses as
// fault entries in order, the populating prefetches; summary n_cancel = misses, n_dedup = pops
int launch_translate(const World& W, const Scratch& S, const mpsf_fault_entry* in, uint64_t n, const Params& P,
                     uint8_t* hit, mpsf_fault_entry* faults, uint32_t* fault_idx, uint32_t* pop_idx, DevSummary* sum,
                     cudaStream_t st, const Marker& mk);
int launch_translate_prefetch(const World& W, const Scratch& S, const mpsf_fault_entry* in, uint64_t n,
                              const Params& P, cudaStream_t st, const Marker& mk);
int launch_translate_finish(const World& W, const Scratch& S, const mpsf_fault_entry* in, uint64_t n,
                            const Params& P, uint8_t* hit, mpsf_fault_entry* faults, uint32_t* fault_idx,
                            uint32_t* pop_idx, DevSummary* sum, cudaStream_t st, const Marker& mk);
// batched top half: scenario id (0xFF skipped) and rid (NO_RID) per entry, then the summary
int launch_classify(const World& W, const Scratch& S, const mpsf_fault_entry* in, uint64_t n, const Params& P,
                    uint8_t* sid, uint32_t* rid, DevSummary* sum, cudaStream_t st, const Marker& mk);
uint32_t chunk_entries();   // entries per chunk (host chunk boundaries must be multiples)
uint64_t chunks_for(uint64_t n);
uint64_t segments_for(uint64_t n);
int launch_hash_export(const Hash& h, uint64_t cap, unsigned long long* keys, uint32_t* vals, uint32_t* counter,
                       uint64_t out_cap, cudaStream_t st);
int launch_hash_merge(const Hash& h, uint32_t* ctrl, const unsigned long long* keys, const uint32_t* vals,
                      uint64_t count, cudaStream_t st);
// sparse exchange of a u32 minima table: compact the non-EMPTY words / MIN-merge (index, value) pairs
int launch_sparse_export(const uint32_t* buf, uint64_t count, uint32_t* idx, uint32_t* val, uint32_t* counter,
                         uint64_t cap, cudaStream_t st);
int launch_sparse_merge(uint32_t* buf, uint64_t count, const uint32_t* idx, const uint32_t* val, uint64_t n,
                        cudaStream_t st);

int launch_remap(uint64_t va_base, const uint64_t* phys, uint64_t npages4k, uint32_t gran_log2,
                 mpsf_remap_entry* out, cudaStream_t st);
int launch_remap_blocks(uint64_t va_base, const uint64_t* phys, uint64_t npages4k,
                        const uint32_t* blocks, uint64_t nblocks, mpsf_remap_entry* out,
                        uint32_t* err_flag, cudaStream_t st);
// snapshot delta fold (StandbyInstance.fold over a batch of snapshots); synchronous on st; every
// primitive hand-written (fold_kernels.cu), each launch marked for the per-kernel profile
struct FoldTotals {
  uint64_t n_requests, n_blocks, n_tokens, error_index;
  uint32_t overrun;   // the delta lengths reach past the payload arrays
  uint32_t launches;  // kernels launched
};
size_t fold_scratch_bytes(uint64_t S, uint64_t R);
int launch_fold(uint8_t* scratch, size_t scratch_bytes, uint32_t S, uint32_t R, const uint32_t* req,
                const uint32_t* nblk, const uint32_t* ntok, const uint32_t* progress, const uint8_t* done,
                const uint32_t* blocks, uint64_t n_blocks_in, const uint32_t* tokens, uint64_t n_tokens_in,
                uint32_t* order, uint64_t* blk_off, uint32_t* blocks_out, uint64_t* tok_off, uint32_t* tokens_out,
                uint32_t* prog_out, uint8_t* done_out, FoldTotals* tot, cudaStream_t st, const Marker& mk);
// KV pool restore (BlockPool.reserve of folded block ids): reserved mask + free ids ascending
size_t kv_reserve_scratch_bytes(uint32_t total);
int launch_kv_reserve(uint8_t* scratch, size_t scratch_bytes, uint32_t total, const uint32_t* blocks, uint64_t nb,
                      uint8_t* reserved, uint32_t* free_ids, uint64_t* n_free, cudaStream_t st);
}  // namespace mpsf
