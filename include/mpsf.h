/*
 * mpsf.h -- C ABI of libmpsf.so, the B200 (sm_100a) batched MMU-fault-buffer
 * processing path and recovery remap for the fault-resilient MPS design
 * (arxiv/paper_2605_26461; reference package `mpssim`, paths below are relative
 * to the reference's pkg/src/mpssim/).
 *
 * Plain C: fixed-layout structs, device pointers + sizes, a cudaStream_t passed
 * as void*.  No exceptions cross this boundary: every call returns 0 or a
 * negative MPSF_E_* code (see mpsf_strerror).  The Python host side
 * (paper_2605_26461_b200/engine.py) binds it with ctypes; INTEGRATION.md shows
 * the binding a maintainer would add to the reference.
 *
 * What each entry point replaces in the reference:
 *   mpsf_upload_world  -- the state classify/range_at read: MemoryModel.ranges
 *                         (memory.py:122-237), UvmHandler.channel_to_pid
 *                         (pipeline.py:73,89-91), client/TSG wiring (execmodel.py:164-204)
 *   mpsf_process       -- per batch: raise_mmu_fault's classify (pipeline.py:96-129,
 *                         faults.py:134-171, range_at memory.py:233-237) for every entry,
 *                         then service_bottom_half (pipeline.py:160-183) with
 *                         intercept_and_isolate (270-304), _report_fatal/rc_recovery
 *                         (224-265, execmodel.py:345-374), benign completion drop
 *                         (pipeline.py:198-200) and raise_sm_trap (151-155), evaluated
 *                         with the batch rules C0-C9 of SURVEY.md Appendix C
 *   mpsf_remap         -- MemoryModel.vmm_map's per-page mapping (memory.py:269-283) as
 *                         called from recovery.deploy_pair (recovery.py:175-184)
 *   mpsf_remap_blocks  -- complete_wake's block-table restore (recovery.py:342-344)
 */
#ifndef MPSF_H
#define MPSF_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MPSF_ABI_VERSION 1

/* ---- packed fault-buffer entry (16 B; FaultSeed memory.py:104-109 + record kind) ---- */
typedef struct {
  uint64_t va;        /* faulting virtual address (translation entries)                 */
  uint32_t channel;   /* channel index into the uploaded channel table                  */
  uint8_t engine;     /* 0 SM, 1 CE, 2 PBDMA (EngineClass, execmodel.py:19-22)          */
  uint8_t access;     /* 0 read, 1 write, 2 prefetch (AccessType, memory.py:50-53)      */
  uint8_t kind;       /* 0 translation; 1..5 parse-time category (faults.py:289-292);
                         8..12 SM trap EXC_2/4/5/6/7 (faults.py:116-122)                */
  uint8_t flags;      /* bit0 valid; entries without it are skipped                     */
} mpsf_fault_entry;

/* ---- interval table row (32 B; VaRange memory.py:83-101), sorted by (client, base) ---- */
typedef struct {
  uint64_t base, end; /* [base, end), 4 KiB aligned                                      */
  uint32_t client;    /* client index                                                    */
  uint32_t page_off;  /* first page-state slot; the range owns npages+1 slots (last = guard) */
  uint8_t kind;       /* 0 managed, 1 external (RangeKind)                               */
  uint8_t lifecycle;  /* 0 live, 1 zombie                                                */
  uint8_t migratable; /* 0/1                                                             */
  uint8_t state;      /* uniform page-state byte, or 0xFF = read page_state[]           */
  uint32_t rid;       /* reference VaRange.rid                                           */
} mpsf_range_entry;

typedef struct { uint32_t client; uint8_t engine; uint8_t pad[3]; } mpsf_channel_entry;
/* mode: 0 MPS client, 1 standalone.  flags: bit0 alive, bit1 CE TSG already destroyed */
typedef struct { uint8_t mode, flags; uint16_t pad; } mpsf_client_entry;

/* ---- per-entry result (8 B) ----
 * verdict bits: [1:0] outcome 0 none (trap/invalid) 1 serviced 2 isolated 3 fatal
 *               [3:2] mechanism 0 none 1 M1 2 M2 3 M3
 *               [4] cancelled  [5] dup (coalesced, C2)  [6] replayable buffer          */
typedef struct { uint32_t rid; uint8_t scenario; uint8_t verdict; uint16_t client; } mpsf_out_record;

/* ---- per-client fate (4 B): state 0 running 1 terminated; reason 0 '-' 1 isolation
 * 2 fault-propagation 3 unchanged (dead before the batch); notifier: scenario id,
 * 0xFF none, 0xFE unchanged                                                             */
typedef struct { uint8_t state, reason, notifier, flags; } mpsf_client_verdict;

typedef struct { uint64_t va; uint64_t phys; } mpsf_remap_entry;

#define MPSF_PF_ISOLATION 0x1u
#define MPSF_WF_GR_DEAD 0x1u

typedef struct {
  uint32_t flags;      /* MPSF_PF_ISOLATION = uvm.isolation_enabled                     */
  uint32_t benign_us;  /* SimParams latencies (kernel.py:34-37)                          */
  uint32_t m1_us, m2_us, m3_us;
  uint32_t reserved;
  uint64_t base_index; /* global index of entry 0 (sharded runs); base_index+n <= 2^29   */
} mpsf_params;

typedef struct {
  int32_t status;           /* 0 or MPSF_E_*                                              */
  uint32_t path;            /* bit0: general (release-aware) path ran                     */
  uint64_t n_dedup;         /* dedup-set size U                                           */
  uint64_t n_cancel;        /* cancel-list size C                                         */
  uint64_t error_index;     /* first offending entry for entry errors                     */
  uint64_t hash_used;       /* wild-page hash slots claimed                               */
} mpsf_summary;

#define MPSF_OK 0
#define MPSF_E_CUDA (-1)
#define MPSF_E_ARG (-2)
#define MPSF_E_NO_CHANNEL (-3)      /* NoChannelAttribution (errors.py:59-60)             */
#define MPSF_E_BAD_ENTRY (-4)
#define MPSF_E_ENGINE_MISMATCH (-5)
#define MPSF_E_VA_RANGE (-6)
#define MPSF_E_WORLD (-7)           /* overlapping / unsorted / unaligned interval table   */
#define MPSF_E_OVERFLOW (-8)        /* wild-page hash table full: call again (it grows)    */
#define MPSF_E_NO_WORLD (-9)
#define MPSF_E_TOO_LARGE (-10)

typedef struct mpsf_ctx mpsf_ctx;

int mpsf_version(void);
const char* mpsf_strerror(int code);

/* One context per device; owns the uploaded world tables and its scratch. */
int mpsf_create(mpsf_ctx** out, int device);
void mpsf_destroy(mpsf_ctx* ctx);

/* Host pointers; synchronous copy into HBM.  Validates sortedness/overlap/alignment. */
int mpsf_upload_world(mpsf_ctx* ctx, const mpsf_range_entry* ranges, uint32_t n_ranges,
                      const uint8_t* page_state, uint64_t n_pages,
                      const mpsf_channel_entry* channels, uint32_t n_channels,
                      const mpsf_client_entry* clients, uint32_t n_clients,
                      uint32_t world_flags);

/* Device pointers, asynchronous on `stream`.  Output capacities: out[n],
 * verdict[n_clients], counts[n_clients*28], dedup_keys/dedup_idx/cancel[n].
 * dedup key = client<<48 | engine<<46 | scenario<<41 | page.
 * Lists are in entry-index order and hold global indices (base_index + i).
 * Call mpsf_get_summary to wait and read the status and list lengths. */
int mpsf_process(mpsf_ctx* ctx, const mpsf_fault_entry* d_entries, uint64_t n,
                 const mpsf_params* params, mpsf_out_record* d_out,
                 mpsf_client_verdict* d_verdict, uint64_t* d_counts,
                 uint64_t* d_dedup_keys, uint32_t* d_dedup_idx, uint32_t* d_cancel,
                 void* stream);

/* Waits for the last mpsf_process on this context and reports it. */
int mpsf_get_summary(mpsf_ctx* ctx, mpsf_summary* out);

/* End-to-end form with HOST buffers (pinned for full speed): chunked H2D of the
 * entries overlapped with the first pass, D2H of every output; synchronous. */
int mpsf_process_host(mpsf_ctx* ctx, const mpsf_fault_entry* h_entries, uint64_t n,
                      const mpsf_params* params, mpsf_out_record* h_out,
                      mpsf_client_verdict* h_verdict, uint64_t* h_counts,
                      uint64_t* h_dedup_keys, uint32_t* h_dedup_idx, uint32_t* h_cancel,
                      mpsf_summary* summary);

/* Remap table of one shared allocation: entry k = (va_base + k*G, phys[k*G/4096]),
 * G = 1<<gran_log2 (12..30), ceil(npages4k*4096/G) entries.  Device pointers, async. */
int mpsf_remap(mpsf_ctx* ctx, uint64_t va_base, const uint64_t* d_phys_pages,
               uint64_t npages4k, uint32_t gran_log2, mpsf_remap_entry* d_out, void* stream);

/* Live-KV remap from folded block ids: entry j = (va_base + b_j*4096, phys[b_j]). */
int mpsf_remap_blocks(mpsf_ctx* ctx, uint64_t va_base, const uint64_t* d_phys_pages,
                      uint64_t npages4k, const uint32_t* d_block_ids, uint64_t nblocks,
                      mpsf_remap_entry* d_out, void* stream);

/* Asynchronous host-buffer form (the same work as mpsf_process_host): mpsf_submit_host
 * enqueues one batch into slot 0 .. MPSF_HOST_SLOTS-1 and returns; mpsf_collect_host waits for that slot and
 * reports it (and re-runs the batch if the wild-page hash overflowed).  Batches execute in
 * submission order; the H2D of one overlaps the passes and the D2H of the other.  Output
 * buffers must stay valid until collected; with pinned (device-accessible) list buffers the
 * lists are written by the device without a host round trip.  mpsf_process_host = submit
 * (slot 0) + collect. */
#define MPSF_HOST_SLOTS 3   /* batches the asynchronous host form can hold in flight */
int mpsf_submit_host(mpsf_ctx* ctx, int slot, const mpsf_fault_entry* h_entries, uint64_t n,
                     const mpsf_params* params, mpsf_out_record* h_out,
                     mpsf_client_verdict* h_verdict, uint64_t* h_counts, uint64_t* h_dedup_keys,
                     uint32_t* h_dedup_idx, uint32_t* h_cancel);
int mpsf_collect_host(mpsf_ctx* ctx, int slot, mpsf_summary* summary);

/* ---- batched top half: faults.classify + MemoryModel.range_at of every entry ----
 * What raise_mmu_fault computes per record before queueing it (pipeline.py:103-104;
 * faults.py:134-171; memory.py:233-237): d_scenario[i] = the scenario id (position in
 * faults.py:79-108; 0xFF for an entry without the valid flag), d_rid[i] = the rid of the range
 * holding the VA (0xFFFFFFFF: none).  Parse-time / SM-trap entries get their scenario.  Device
 * pointers, asynchronous; mpsf_get_summary reports entry errors like mpsf_process. */
int mpsf_classify(mpsf_ctx* ctx, const mpsf_fault_entry* d_entries, uint64_t n, uint64_t base_index,
                  uint8_t* d_scenario, uint32_t* d_rid, void* stream);

/* ---- batched translation: MemoryModel.resolve_va (memory.py:339-364) over an access stream ----
 * The step before the fault path: each access (a kind-0 entry: va, access,
 * engine, channel) is translated in stream order against the uploaded page tables plus the
 * one mutation translation makes -- a PREFETCH into a managed range populates its page
 * (populate_page, memory.py:368-380), so later accesses to that page see it GPU-resident.
 * Outputs: d_hit[n] (1 Hit, 0 Miss, 0xFF entry skipped), the misses in order as fault-buffer
 * entries d_faults[] (the seeds mpsf_process consumes) with their indices d_fault_idx[], and
 * d_pop_idx[] = the prefetches that populated a page.  Entry errors as mpsf_process.  Do not
 * interleave with the phase calls of an unfinished mpsf_process batch (shared scratch). */
typedef struct {
  int32_t status;
  uint32_t pad;
  uint64_t n_miss;        /* fault entries written                                          */
  uint64_t n_populated;   /* pages populated by prefetches                                  */
  uint64_t error_index;
} mpsf_translate_summary;
int mpsf_translate(mpsf_ctx* ctx, const mpsf_fault_entry* d_accesses, uint64_t n, uint64_t base_index,
                   uint8_t* d_hit, mpsf_fault_entry* d_faults, uint32_t* d_fault_idx, uint32_t* d_pop_idx,
                   void* stream);
int mpsf_get_translate_summary(mpsf_ctx* ctx, mpsf_translate_summary* out);
/* The same as two phases, for sharded streams (one process per GPU, contiguous index ranges
 * base_index .. base_index+n): mpsf_translate_prefetch records the first PREFETCH per
 * managed page (global indices) in the table mpsf_exchange_buffers(ctx, 4, ...) exposes;
 * after the shards combine it with a MIN, mpsf_translate_finish classifies and compacts this
 * shard (same n / base_index).  mpsf_translate = prefetch + finish. */
int mpsf_translate_prefetch(mpsf_ctx* ctx, const mpsf_fault_entry* d_accesses, uint64_t n, uint64_t base_index,
                            void* stream);
int mpsf_translate_finish(mpsf_ctx* ctx, const mpsf_fault_entry* d_accesses, uint64_t n, uint64_t base_index,
                          uint8_t* d_hit, mpsf_fault_entry* d_faults, uint32_t* d_fault_idx, uint32_t* d_pop_idx,
                          void* stream);

/* ---- snapshot delta fold: StandbyInstance.fold (recovery.py:83-92) over a batch ----
 * The step after the recovery remap.  n_snap ForwardSnapshots
 * (recovery.py:30-41) in consume order, as device arrays: d_req[i] the request id (< n_req_ids)
 * or 0xFFFFFFFF for a liveness-only snapshot; d_nblk[i] / d_ntok[i] the lengths of its
 * KV-block and token deltas, concatenated in consume order in d_blocks / d_tokens;
 * d_progress[i]; d_done[i] (0/1).  Output per request, in first-appearance order (the
 * fold dict's insertion order): d_order[k] its id, the CSR offsets d_blk_off[k..k+1] /
 * d_tok_off[k..k+1] into d_blocks_out / d_tokens_out (the deltas appended in consume order),
 * d_progress_out[k] (the last snapshot's), d_done_out[k] (sticky OR).  Capacities: n_snap
 * for the per-request arrays, n_snap+1 for the offsets, n_blocks / n_tokens (the payload
 * lengths, each < 2^32) for the payloads.  Deltas reaching past the payloads: MPSF_E_ARG.
 * last_consumed_seq is the last snapshot's seq (the caller holds it); n_req_ids <= 2^30.  A request id >= n_req_ids
 * returns MPSF_E_BAD_ENTRY with the first such snapshot in error_index (its snapshot is not
 * folded).  Synchronous on `stream` (the summary needs the counts). */
typedef struct {
  int32_t status;
  uint32_t pad;
  uint64_t n_requests;
  uint64_t n_blocks;
  uint64_t n_tokens;
  uint64_t error_index;
} mpsf_fold_summary;
int mpsf_fold(mpsf_ctx* ctx, uint64_t n_snap, uint32_t n_req_ids, const uint32_t* d_req,
              const uint32_t* d_nblk, const uint32_t* d_ntok, const uint32_t* d_progress,
              const uint8_t* d_done, const uint32_t* d_blocks, uint64_t n_blocks,
              const uint32_t* d_tokens, uint64_t n_tokens, uint32_t* d_order, uint64_t* d_blk_off, uint32_t* d_blocks_out, uint64_t* d_tok_off,
              uint32_t* d_tokens_out, uint32_t* d_progress_out, uint8_t* d_done_out,
              mpsf_fold_summary* summary, void* stream);

/* ---- KV pool restore: BlockPool.reserve (workload.py:77-80) of folded block ids ----
 * complete_wake reserves every folded request's blocks in the standby's pool
 * (recovery.py:356-357).  d_reserved[total_blocks] = 1 for every id in d_block_ids[n] (ids >=
 * total_blocks are not pool blocks and mark nothing) -- the valid mask of the live-KV remap;
 * d_free[total_blocks] = the unreserved ids ascending (the pool heap's pop order), *n_free
 * of them.  Synchronous on `stream`. */
int mpsf_kv_reserve(mpsf_ctx* ctx, uint32_t total_blocks, const uint32_t* d_block_ids, uint64_t n,
                    uint8_t* d_reserved, uint32_t* d_free, uint64_t* n_free, void* stream);

/* ---- Trace-line rendering of a processed batch (host only) ----
 * Trace.render_record (kernel.py:127-132) lines for `n` entries and the OutRecords
 * mpsf_process produced for them: MPSF_RENDER_TOP = the top half per entry in index (raise)
 * order (fault_raised, shadow_copy; pipeline.py:113-143), MPSF_RENDER_DRAIN = the bottom half
 * in drain order as the batch verdicts apply (bh_service, parse_fatal, tlb_invalidate,
 * fatal_report, isolate_begin; pipeline.py:160-183, 224-230, 296-298).  SM traps and skipped
 * entries render nothing.  Writes at most `cap` bytes of '\n'-terminated lines into buf and
 * returns the total length (> cap, or buf NULL: nothing written, call again with that
 * capacity), or a negative MPSF_E_* code.  Needs no device. */
#define MPSF_RENDER_TOP 1u
#define MPSF_RENDER_DRAIN 2u
typedef struct {
  uint64_t t_drain;                  /* world.clock.now at the drain                        */
  const uint64_t* t_raise;           /* per-entry raise time (top half), NULL: t_drain       */
  uint32_t m1_us, m2_us, m3_us;      /* SimParams mechanism latencies (isolate_begin)        */
  uint32_t parts;                    /* MPSF_RENDER_TOP | MPSF_RENDER_DRAIN                  */
  const char* const* channel_names;  /* reference channel ids ("c1.sm"), by channel index    */
  uint32_t n_channels;
  uint32_t n_clients;
  const char* const* client_names;   /* reference pids ("c1"), by client index               */
  uint32_t threads;                  /* host threads (0: all)                                */
  uint32_t pad;
} mpsf_render_params;
int64_t mpsf_render_trace(const mpsf_fault_entry* entries, const mpsf_out_record* out, uint64_t n,
                          const mpsf_render_params* params, char* buf, uint64_t cap);

/* Number of kernel launches the last mpsf_process / mpsf_remap enqueued. */
int mpsf_last_launches(mpsf_ctx* ctx);

/* Per-kernel device time: with profiling on, a CUDA event is recorded on the launching
 * stream after every kernel; mpsf_get_profile waits for them and returns the accumulated
 * per-kernel launches and milliseconds since profiling was (re)enabled. */
typedef struct {
  char name[32];
  uint64_t launches;
  double total_ms;
} mpsf_kernel_time;

int mpsf_set_profiling(mpsf_ctx* ctx, int on);
int mpsf_get_profile(mpsf_ctx* ctx, mpsf_kernel_time* out, int cap);

/* ---- phase entry points (sharded multi-GPU runs; mpsf_process == their composition) ----
 * Each rank runs mpsf_scan on its shard (params->base_index = first global index), then the
 * caller combines the exchange buffers across ranks (MIN on the unsigned values, SUM for
 * counts) and merges the sparse hash tables, then runs mpsf_resolve; with isolation on, the
 * general stages follow (exchange stage 2 after stage 1, stage 3 after stage 2); finally
 * mpsf_finalize writes this shard's outputs.  Because every cross-entry dependency is a
 * group minimum, the concatenated per-rank outputs equal a single-GPU run bit for bit. */
/* Dedup-slot layout, before upload: on > 0 one dense slot per (page, group) (sharded runs);
 * on < 0 one claimed slot per page, other groups through the hash, no per-page first-eligible
 * keys (the layout large worlds get; forcing it lets small worlds test that path); 0 by size. */
int mpsf_set_dense_dedup(mpsf_ctx* ctx, int on);
int mpsf_scan(mpsf_ctx* ctx, const mpsf_fault_entry* d_entries, uint64_t n, const mpsf_params* params,
              uint64_t* d_counts, void* stream);
int mpsf_resolve(mpsf_ctx* ctx, const mpsf_params* params, mpsf_client_verdict* d_verdict,
                 uint64_t* d_counts, void* stream);
int mpsf_general(mpsf_ctx* ctx, const mpsf_fault_entry* d_entries, uint64_t n, const mpsf_params* params,
                 int stage, void* stream);
int mpsf_resolve2(mpsf_ctx* ctx, const mpsf_params* params, void* stream);
int mpsf_finalize(mpsf_ctx* ctx, const mpsf_fault_entry* d_entries, uint64_t n, const mpsf_params* params,
                  mpsf_out_record* d_out, uint64_t* d_dedup_keys, uint32_t* d_dedup_idx,
                  uint32_t* d_cancel, void* stream);

#define MPSF_XOP_MIN 0u
#define MPSF_XOP_SUM 1u
typedef struct {
  void* ptr;            /* device pointer                                   */
  uint64_t count;       /* elements                                         */
  uint32_t elem_bytes;  /* 4 or 8 (unsigned)                                */
  uint32_t op;          /* MPSF_XOP_MIN / MPSF_XOP_SUM                      */
} mpsf_xbuf;
/* stage 1: after mpsf_scan; 2: after mpsf_general(stage 1); 3: after stage 2;
 * 4: after mpsf_translate_prefetch (the first-PREFETCH page table, MIN) */
int mpsf_exchange_buffers(mpsf_ctx* ctx, int stage, mpsf_xbuf* out, int cap);
/* which: 0 dedup hash, 1 first-isolation (NR) hash.  Export compacts the non-empty slots
 * (returns the count, waits on the stream); merge inserts keys with atomic-min values. */
int64_t mpsf_hash_export(mpsf_ctx* ctx, int which, uint64_t* d_keys, uint32_t* d_vals, uint64_t cap,
                         void* stream);
int mpsf_hash_merge(mpsf_ctx* ctx, int which, const uint64_t* d_keys, const uint32_t* d_vals,
                    uint64_t count, void* stream);

/* Sparse form of a MIN exchange buffer of 4-byte words (the page-sized dedup slots and
 * first-eligible keys of a large world are mostly empty): export compacts the words that are
 * not 0xFFFFFFFF into (index, value) pairs (returns the count, MPSF_E_OVERFLOW beyond cap;
 * waits on the stream); merge applies pairs gathered from the other ranks with an atomic MIN.
 * Export + all-gather + merge on every rank == a MIN all-reduce of the buffer. */
int64_t mpsf_sparse_export(mpsf_ctx* ctx, const uint32_t* d_buf, uint64_t count, uint32_t* d_idx, uint32_t* d_val,
                           uint64_t cap, void* stream);
int mpsf_sparse_merge(mpsf_ctx* ctx, uint32_t* d_buf, uint64_t count, const uint32_t* d_idx, const uint32_t* d_val,
                      uint64_t n, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* MPSF_H */
