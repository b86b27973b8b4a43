// Device-side building blocks of the batched fault path (sm_100a).
//
// Reference semantics restated here (paths relative to the reference's pkg/src/mpssim/):
//   classify()   -- faults.classify, faults.py:134-171 (priority order 145-171)
//   range_at     -- MemoryModel.range_at, memory.py:233-237: the (client, base)-sorted,
//                   page-granular interval table plus per-client skip tables (World below),
//                   used by decode_fast in fault_kernels.cu instead of a linear scan
//   scenario predicates -- the 28-row table faults.py:79-108 (ids = list position)
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "mpsf.h"

namespace mpsf {

constexpr uint32_t EMPTY32 = 0xFFFFFFFFu;
constexpr unsigned long long EMPTY64 = 0xFFFFFFFFFFFFFFFFull;
constexpr long long REL_NONE = 0x7FFFFFFFFFFFFFFFll;  // client never released in this batch
constexpr long long REL_PRE = -1;                      // released before the drain (trap / dead)
constexpr int NSCEN = 28;
constexpr uint32_t NO_RID = 0xFFFFFFFFu;
constexpr uint32_t MAX_GIDX = 1u << 29;
constexpr uint64_t VA_LIMIT = 1ull << 53;
constexpr int HASH_MAX_PROBE = 256;
constexpr uint32_t MPSF_ENTRY_VALID = 1u;

// error bits in ctrl[C_ERR]
constexpr uint32_t EB_NO_CHANNEL = 1u, EB_BAD_ENTRY = 2u, EB_MISMATCH = 4u, EB_VA = 8u;

// ctrl word slots
enum : int {
  C_ERR = 0, C_PATH = 1, C_HASH_DD = 2, C_HASH_NR = 3, C_OVF = 4,
  C_TILE_FIN = 5, C_NCTRL = 16
};

// per-client derived state written by k_resolve, read by the finalize pass
enum : uint32_t {
  CS_ALIVE0 = 1u, CS_SA = 2u, CS_CE_ALIVE0 = 4u, CS_CE_TORN = 8u, CS_KILL_ALL = 16u,
  CS_TRAPPED = 32u, CS_ELIG = 64u
};
struct CState {
  long long rel;          // release key: REL_PRE, REL_NONE or the ok32 of the teardown record
  uint32_t ft_ce_ok;      // first CE-TSG fatal (ok32) or EMPTY32
  uint32_t ft_sa_ok;      // first standalone-TSG fatal (ok32) or EMPTY32
  uint32_t trap_sa_idx;   // first standalone trap (global idx) or EMPTY32
  uint32_t kill_tie;      // benign records with ok32 > kill_tie are cancelled (EMPTY32: none)
  uint32_t flags;
  uint32_t pad;
};
static_assert(sizeof(CState) == 32, "CState layout");

// scalars shared by every client
struct Globals {
  uint32_t ft_gr_ok;            // applied GR teardown record (ok32) or EMPTY32
  uint32_t trap_mps_idx;        // applied MPS trap (idx) or EMPTY32
  uint32_t gr_alive0;
  uint32_t has_elig;
};

// Per-client decision table of pass 2, folded from CState + Globals so an
// entry's verdict is a few compares (rules C4-C7 of SURVEY.md Appendix C):
//   trap records: applied iff idx == trap_ok (a second trap on a destroyed TSG is cancelled)
//   fatal reports: applied iff the representative's ok32 == ft[channel is CE] (C4)
//   benign completions: cancelled iff bflags[channel is CE] or ok32 > tie (C5/C6)
//   isolation: epoch 1 iff rel < ok32 (C3); pre_nrall: epoch-1 keys are pass 1's first-record keys
struct FinClient {
  long long rel;
  uint32_t trap_ok, ft0, ft1, tie;
  uint32_t bflags;      // bit0: benign always cancelled; bit1: same for a CE channel
  uint32_t pre_nrall;
};
static_assert(sizeof(FinClient) == 32, "FinClient layout");

__device__ __forceinline__ FinClient fin_client(const CState& cs, const Globals& G, bool has_nrall) {
  FinClient f;
  f.rel = cs.rel;
  const bool sa = cs.flags & CS_SA, alive0 = cs.flags & CS_ALIVE0;
  if (sa) {
    f.trap_ok = alive0 ? cs.trap_sa_idx : EMPTY32;
    f.ft0 = (alive0 && !(cs.flags & CS_TRAPPED)) ? cs.ft_sa_ok : EMPTY32;
    f.ft1 = f.ft0;
  } else {
    f.trap_ok = G.gr_alive0 ? G.trap_mps_idx : EMPTY32;
    f.ft0 = G.ft_gr_ok;
    f.ft1 = ((cs.flags & CS_CE_ALIVE0) && cs.ft_ce_ok != EMPTY32 && !(cs.rel < (long long)cs.ft_ce_ok))
                ? cs.ft_ce_ok : EMPTY32;
  }
  const bool b0 = cs.rel != REL_NONE || (cs.flags & CS_KILL_ALL);
  const bool b1 = b0 || (cs.flags & CS_CE_TORN);
  f.bflags = (b0 ? 1u : 0u) | (b1 ? 2u : 0u);
  f.tie = cs.kill_tie;
  f.pre_nrall = (cs.rel == REL_PRE && has_nrall) ? 1u : 0u;
  return f;
}

constexpr uint32_t SKIP_MAX = 256;       // skip-table slots per client (cap)
constexpr uint64_t VA_TABLE_LIMIT = (1ull << 44) - 8192;   // range ends: guard page numbers stay below 2^32 - 1

// Device form of the interval table, built by mpsf_upload_world (page-granular SoA so a warp's
// random lookups touch 4-byte words: no 32-byte-row bank conflicts).  Per client, a skip table
// maps (page - span) >> shift to the last range whose base is <= the slot start; the shift is
// chosen so that a slot holds at most one range base (exact1: attribution takes <= 1 step).
struct World {
  const mpsf_range_entry* ranges;   // original rows (host order)
  const uint32_t* client_off;
  const uint8_t* page_state;
  const mpsf_channel_entry* channels;
  const mpsf_client_entry* clients;
  const uint32_t* pg_base;          // [R + 1] base >> 12 (row R = 0xFFFFFFFF)
  const uint32_t* pg_end;           // [R + 1] end >> 12
  const uint32_t* poff;             // [R + 1] first page-state slot
  const uint32_t* rattr;            // [R + 1] kind | lifecycle << 8 | migratable << 16 | state << 24
  const uint32_t* rrid;             // [R + 1] reference rid
  const uint16_t* skip;             // [n_skip + 1] per-client skip tables, concatenated
  const uint32_t* chan;             // [nch + 1] client | engine << 16 | standalone << 18 | valid << 31
  const uint4* cinfo4;              // [C] (lo | hi << 16, span, shift | (slots - 1) << 8, skip offset)
  uint32_t n_ranges, n_clients, n_channels, world_flags;
  uint64_t n_pages;
  uint32_t has_mps;
  uint32_t dd_groups;   // 5: one dense dedup slot per (page, group); 1: one claimed slot per page
  uint32_t n_skip;
  uint32_t exact1;      // every skip slot holds at most one range base
  // row form of the same tables for the streaming passes (one 16- or 8-byte shared load per step):
  const uint4* chan4;   // [nch + 1] {channel word, client span start page, skip shift, skip offset | jmax << 16}
  const uint2* skip2;   // [n_skip + 1] {range index at the slot start, base page of the next range if it
                        //  starts inside the slot else 0xFFFFFFFF}
  const uint4* row4;    // [R + 1] {base page, end page, first page-state slot, attr}; attr = uniform state
                        //  [2:0] | range class (kind | zombie << 1 | migratable << 2) [5:3] | per-page state [7]
};

constexpr uint32_t ROW_PERPAGE = 0x80u;

constexpr uint32_t CH_VALID = 1u << 31;

struct Hash {
  unsigned long long* keys;   // 16-byte slots: [2s] key, [2s+1] = min value | generation << 32
  uint32_t mask;
  uint32_t used_slot;  // ctrl index counting claimed slots
  uint32_t gen;        // this batch's generation: a slot of another generation is free (so the
                       //  tables need no clearing between batches; never 0, fresh tables are zeroed)
};

struct Scratch {
  uint32_t* dd;        // [n_pages] dense dedup slots: (gidx << 3 | group), EMPTY32
  uint32_t* nr0;       // [n_ranges] guard-page first-isolation key, epoch 0
  uint32_t* nr1;       // [n_pages] first-isolation key per page, epoch 1 (general path)
  uint32_t* nrall;     // [n_pages] first eligible record per in-range page (dense worlds), or null
  uint32_t* pf;        // [n_pages] first PREFETCH per managed page (batched translation)
  Hash hdd;            // dedup keys of pages outside every range's slot span
  Hash hnr;            // NR keys (client, page, epoch) of such pages
  uint32_t* ext;       // [n_ranges] first isolation-eligible record per external range
  unsigned long long* ft_ce;    // [C]
  unsigned long long* ft_sa;    // [C]
  unsigned long long* trap_sa;  // [C]
  unsigned long long* ft_gr;    // min (ok32 << 8 | sid) over fatal GR-TSG records
  unsigned long long* trap_mps; // min (idx << 8 | sid) over traps raised by MPS clients
  uint32_t* iso1;      // [C] snapshot-unmapped eligible (M1 candidates)
  uint32_t* iso2;      // [C] managed-range eligible (M2)
  uint32_t* iso3;      // [C] external-range eligible (M3 candidates)
  uint32_t* giso;      // [3*C] exact per-mechanism minima, general path
  CState* cstate;      // [C]
  FinClient* fclient;  // [C] pass-2 decision table (k_resolve / k_resolve2)
  Globals* glob;
  uint32_t* ctrl;      // [C_NCTRL]
  unsigned long long* err_idx;
  uint4* cmask;                // [chunks] ballots: cancelled entries 2l / 2l+1, representatives 2l / 2l+1
  unsigned long long* segcnt;  // [segments] cancel count | dedup count << 32
  unsigned long long* segbase; // [segments] exclusive prefix of segcnt (large batches: k_seg_scan)
  uint4* trstage;              // [chunks][64] translation: each chunk's miss entries compacted in
                               //  access order (k_tr_classify -> k_tr_lists)
  unsigned long long* dstage;  // [chunks][KSTAGE] first dedup keys of each chunk (k_finalize -> k_lists)
  unsigned long long* drec;    // [n] pass-1 records (fixed-layout worlds), entry drec_base first
  uint64_t drec_base;          // global index of drec[0] (params.base_index of the batch)
};

// What mpsf_get_summary reads back after a batch.
struct DevSummary {
  uint32_t ctrl[C_NCTRL];
  unsigned long long err_idx;
  unsigned long long n_cancel;
  unsigned long long n_dedup;
};

struct Params {
  uint32_t flags, benign_us, m1_us, m2_us, m3_us;
  uint64_t base_index;
};

// ---- scenario table predicates (faults.py:79-108) ----
__device__ __forceinline__ bool s_serviceable(int s) { return s >= 14 && s <= 17; }
__device__ __forceinline__ bool s_parse(int s) { return s >= 23; }
__device__ __forceinline__ bool s_trap(int s) { return s >= 18 && s <= 22; }
__device__ __forceinline__ bool s_replayable(int s) { return s <= 5 || s == 14 || s == 15 || s >= 23; }

// faults.classify, faults.py:134-171.  eng: 0 SM 1 CE 2 PBDMA; acc: 0 R 1 W 2 PREFETCH.
__device__ __forceinline__ int classify(int eng, int acc, bool has, int kind, int lifecycle,
                                        int migratable, uint32_t st) {
  if (acc == 2) return 15;                                   // invalid prefetch, any engine
  const int oob = eng == 0 ? 0 : 2 + 4 * eng;                // 0 / 6 / 10
  if (!has) return oob;
  if (lifecycle == 1) return 4 + 4 * eng;                    // zombie 4 / 8 / 12
  const int res = st & 3;
  const bool ro = (st & 4) != 0;
  if (!migratable && res == 1) return 5 + 4 * eng;           // non-migratable 5 / 9 / 13
  if (acc == 1 && ro) {
    if (eng == 0) return kind == 1 ? 3 : (res == 2 ? 2 : 1); // am_vmm / am_gpu / am_cpu
    return 3 + 4 * eng;                                      // am.ce 7 / am.pbdma 11
  }
  if (kind == 0 && res <= 1) return eng == 0 ? 14 : 15 + eng; // benign 14 / 16 / 17
  return oob;                                                 // would-hit fallthrough
}

// ---- classification LUT ---------------------------------------------------------------------
// Every decode outcome of an entry maps to one 32-bit word built once per CTA from classify():
// translation entries index ((eng * 3 + acc) * 16 + rcls) * 8 + st with rcls = kind |
// lifecycle << 1 | migratable << 2 for an attributed range (8: none, st = 0); the other entry
// kinds index LUT_XK + kind.  The word carries the scenario id, the dedup group and every
// predicate the passes branch on, so the per-entry path is one lookup instead of a tree.
constexpr int LUT_XK = 9 * 16 * 8;
constexpr int LUT_N = LUT_XK + 16;
enum : uint32_t {
  LF_S = 31u,                 // scenario id bits [4:0]
  LF_GROUP_SH = 5,            // dedup group bits [7:5]
  LF_REPL = 1u << 8,          // replayable buffer (faults.py:48, pipeline.py:116-123)
  LF_DD = 1u << 9,            // replayable translation record: dedup candidate (rule C2)
  LF_SERV = 1u << 10,         // serviceable (benign)
  LF_ELIG = 1u << 11,         // isolation-eligible (isolation on, not serviceable)
  LF_FATAL = 1u << 12,        // fatal report (parse-time, or not serviceable with isolation off)
  LF_TRAP = 1u << 13,         // SM trap (raise_sm_trap, pipeline.py:151-155)
  LF_BAD = 1u << 14,          // not a known entry kind
  LF_M_SH = 15,               // bits [16:15]: 0 no range, 1 managed range, 2 external range
  LF_XKIND = 1u << 17,        // not a translation entry
  LF_VALID = 1u << 31
};

__device__ __forceinline__ uint32_t lut_word(int idx, bool isolation) {
  if (idx >= LUT_XK) {
    const int k = idx - LUT_XK;
    if (k >= 1 && k <= 5) return LF_VALID | LF_XKIND | (uint32_t)(23 + k - 1) | LF_REPL | LF_FATAL;
    if (k >= 8 && k <= 12) return LF_VALID | LF_XKIND | (uint32_t)(18 + k - 8) | LF_TRAP;
    return LF_VALID | LF_XKIND | LF_BAD;
  }
  const int st = idx & 7, rcls = (idx >> 3) & 15, ea = idx >> 7;
  const int eng = ea / 3, acc = ea % 3;
  if (rcls > 8) return LF_VALID | LF_BAD;
  const bool has = rcls < 8;
  const int kind = rcls & 1, lc = (rcls >> 1) & 1, mig = (rcls >> 2) & 1;
  const int s = classify(eng, acc, has, kind, lc, mig, has ? (uint32_t)st : 0u);
  uint32_t group;
  if (eng == 0 && acc != 2) group = (acc == 1 && s >= 1 && s <= 3) ? 1u : 0u;
  else group = eng == 0 ? 2u : (uint32_t)(2 + eng);
  const bool repl = s_replayable(s), serv = s_serviceable(s);
  const uint32_t m = !has ? 0u : (kind == 0 ? 1u : 2u);
  return LF_VALID | (uint32_t)s | (group << LF_GROUP_SH) | (repl ? (LF_REPL | LF_DD) : 0u) |
         (serv ? LF_SERV : (isolation ? LF_ELIG : LF_FATAL)) | (m << LF_M_SH);
}

// Tables a lookup reads (shared memory when staged, else global).  The per-client words and
// the channel table may be replicated 32x ([i][lane]) so a warp's lookups are bank-conflict free.
struct Tables {
  const uint32_t *pg_base, *pg_end, *poff, *rattr, *rrid;
  const uint16_t* skip;
  const uint32_t* chan;
  uint32_t rep_client, rep_chan;   // 32 when replicated per lane, else 0
  const uint4* cinfo;              // [C] or [C][32] client rows (World::cinfo4)
  const uint32_t* lut;             // [LUT_N] classification words (always shared memory)
  uint32_t n_channels, exact1;
};

// Decoded entry of the lean path (decode_fast).
struct Dec {
  uint32_t f;       // LUT word; 0 when the entry is skipped (valid flag clear) or an error was raised
  uint32_t c, cw;   // client, channel word
  uint32_t slot;    // page slot (in range or the guard page)
  uint32_t ridx;    // range index (in range / guard owner), NO_RID when wild
  bool inr, guard;
  uint64_t va;
};

__device__ __forceinline__ uint32_t rep_load(const uint32_t* a, uint32_t i, uint32_t rep, uint32_t lane) {
  return rep ? a[i * 32 + lane] : a[i];
}

__device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdull;
  x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull;
  x ^= x >> 33;
  return x;
}

// Open addressing, linear probing over 16-byte slots {u64 key, u32 value, u32 generation}: one
// load reads the whole slot; value = atomic min.  A slot whose generation is not the batch's is
// free: it is claimed with one 128-bit CAS of the whole slot.  Returns false on overflow.
__device__ __forceinline__ uint32_t* hash_val(const Hash& h, uint32_t s) {
  return reinterpret_cast<uint32_t*>(h.keys + 2ull * s + 1);
}

__device__ __forceinline__ ulonglong2 cas128(ulonglong2* a, ulonglong2 cmp, ulonglong2 val) {
  ulonglong2 old;
  asm volatile("{ .reg .b128 c, n, d;\n\t"
               "mov.b128 c, {%2, %3};\n\t"
               "mov.b128 n, {%4, %5};\n\t"
               "atom.global.cas.b128 d, [%6], c, n;\n\t"
               "mov.b128 {%0, %1}, d; }"
               : "=l"(old.x), "=l"(old.y)
               : "l"(cmp.x), "l"(cmp.y), "l"(val.x), "l"(val.y), "l"(a)
               : "memory");
  return old;
}

// `used` counts claimed slots (a block-local smem counter in the scan, flushed once per block).
__device__ __forceinline__ bool hash_min(const Hash& h, uint32_t* used, uint64_t key, uint32_t v) {
  uint32_t s = (uint32_t)mix64(key) & h.mask;
  for (int p = 0; p < HASH_MAX_PROBE; ++p) {
    ulonglong2* a = reinterpret_cast<ulonglong2*>(h.keys) + s;
    ulonglong2 slot = __ldcg(a);
    while ((uint32_t)(slot.y >> 32) != h.gen) {          // free in this batch: claim it whole
      const ulonglong2 want = make_ulonglong2(key, (unsigned long long)v | ((unsigned long long)h.gen << 32));
      const ulonglong2 old = cas128(a, slot, want);
      if (old.x == slot.x && old.y == slot.y) {
        atomicAdd(used, 1u);
        return true;
      }
      slot = old;                                         // claimed meanwhile: look at it again
    }
    if (slot.x == key) {
      if ((uint32_t)slot.y > v) atomicMin(hash_val(h, s), v);
      return true;
    }
    s = (s + 1) & h.mask;
  }
  return false;
}

__device__ __forceinline__ uint32_t hash_get(const Hash& h, uint64_t key) {
  uint32_t s = (uint32_t)mix64(key) & h.mask;
  for (int p = 0; p < HASH_MAX_PROBE; ++p) {
    const ulonglong2 slot = __ldcg(reinterpret_cast<const ulonglong2*>(h.keys) + s);
    if ((uint32_t)(slot.y >> 32) != h.gen) return EMPTY32;   // a free slot ends the probe run
    if (slot.x == key) return (uint32_t)slot.y;
    s = (s + 1) & h.mask;
  }
  return EMPTY32;
}

// global minimum with a load pre-check (used where nothing filters the calls first)
__device__ __forceinline__ void min32(uint32_t* g, uint32_t v) {
  if (__ldcg(g) > v) atomicMin(g, v);
}
__device__ __forceinline__ void min64(unsigned long long* g, unsigned long long v) {
  if (__ldcg(g) > v) atomicMin(g, v);
}
// block-local minima in shared memory: the scan keeps per-client / per-range minima here and
// flushes them to global once per block (no same-address global atomics inside the loop)
__device__ __forceinline__ void smin32(uint32_t* c, uint32_t v) {
  if (*c > v) atomicMin(c, v);
}
__device__ __forceinline__ void smin64(unsigned long long* c, unsigned long long v) {
  if (*c > v) atomicMin(c, v);
}

// dedup key (SURVEY.md Appendix C rule C2)
__device__ __forceinline__ uint64_t dedup_key(uint32_t c, int eng, int s, uint64_t page) {
  return ((uint64_t)c << 48) | ((uint64_t)eng << 46) | ((uint64_t)s << 41) | page;
}
__device__ __forceinline__ uint64_t nr_key(uint32_t c, int epoch, uint64_t page) {
  return ((uint64_t)c << 42) | ((uint64_t)epoch << 41) | page;
}

// Dedup group of a replayable translation record inside one page: SM read-class,
// SM write-class (merged with read when both classify alike), and PREFETCH per engine.
__device__ __forceinline__ uint32_t dedup_group(int eng, int acc, int s_read, int s_write) {
  if (eng == 0) {
    if (acc == 2) return 2;
    return (acc == 1 && s_write != s_read) ? 1 : 0;
  }
  return eng == 1 ? 3 : 4;
}

}  // namespace mpsf
