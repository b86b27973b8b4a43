// Batched MMU-fault-buffer processing for sm_100a.
//
// One batch = N packed 16-byte fault-buffer entries resident in HBM.  The reference
// (pkg/src/mpssim/) handles them one record at a time: raise_mmu_fault classifies each
// (pipeline.py:96-129), service_bottom_half drains replayable-then-non-replayable and
// acts per record on the evolving world (pipeline.py:160-183).  Here the same result is
// computed with the parallel recipe C9 of SURVEY.md Appendix C -- every cross-record
// dependency is a first-in-group minimum over the drain key:
//
//   k_init      clear the per-batch scratch (dedup slots, minima, hash tables, counters)
//   k_scan      pass 1: decode (channel word, skip-table attribution in the smem interval
//               table, one smem LUT word = faults.classify), per-block (client, scenario)
//               counts, group minima (fatal TSG teardowns, traps, first isolation per
//               external range / guard page / client, first record per dedup key; wild
//               pages through L2 hash tables), and an 8-byte pass-1 record per entry
//   k_resolve   block 0: per-client release keys, kill thresholds, fates, fast/general
//               path, the per-client decision table
//   k_general   [general path: a client with isolation-eligible records is released
//               inside the batch, or m2 <= benign] release-aware first-isolation keys
//               (rule C3 epochs) and exact per-client mechanism minima
//   k_resolve2  [general path] kill thresholds from the exact minima
//   k_finalize  pass 2 over the records: dup / mechanism / cancel per entry, the 8-byte
//               OutRecord, per-chunk ballot masks and segment counters, staged dedup keys
//   k_lists     the cancel list and the dedup set in index order (block per segment)
//
// The streaming passes are persistent grids of 1024-thread CTAs with the world tables at
// fixed shared-memory offsets; each lane reads two adjacent entries with one 32-byte
// non-allocating load (or two 8-byte records with one 16-byte load) and requests the next
// chunk before working on the current one.  Kernel boundaries use programmatic dependent
// launch.  DESIGN.md §4 has the measured bound of each.
#include <cuda_runtime.h>
#include <stdint.h>

#include "mpsf_device.cuh"
#include "mpsf_kernels.h"


namespace mpsf {

// Streaming passes: persistent grid of 1024-thread CTAs (one per SM, shared memory holds the
// world tables); every warp owns 64-entry chunks (two adjacent entries per lane).
#ifndef MPSF_BLOCK
#define MPSF_BLOCK 1024   // threads per persistent CTA (experiments override)
#endif
constexpr int BLOCK = MPSF_BLOCK;
constexpr int WARPS = BLOCK / 32;
constexpr int QCAP = 64;                   // per-warp deferred hash-op stack (scan)

// ---- batched translation LUT (MemoryModel.resolve_va, memory.py:339-364) --------------------
// The same index space as lut_word; the word says what an access decides on the batch-start
// page state: TR_HIT, TR_HIT_POP (the outcome once an earlier PREFETCH populated the page),
// TR_PF (a PREFETCH into a managed range: Hit, populates the page, memory.py:344-349) and TR_POP
// (... and the page was not GPU-resident, so populate_page changes it, memory.py:368-380).
enum : uint32_t { TR_HIT = 1u, TR_HIT_POP = 2u, TR_PF = 4u, TR_POP = 8u };

__device__ __forceinline__ uint32_t tr_word(int idx) {
  if (idx >= LUT_XK) return LF_VALID | LF_XKIND | LF_BAD;     // translation streams: kind 0 only
  const int st = idx & 7, rcls = (idx >> 3) & 15, ea = idx >> 7;
  const int acc = ea % 3;
  if (rcls > 8) return LF_VALID | LF_BAD;
  const bool has = rcls < 8;
  const int kind = rcls & 1, lc = (rcls >> 1) & 1, mig = (rcls >> 2) & 1;
  const int res = st & 3;
  const bool ro = (st & 4) != 0;
  uint32_t w = 0;
  if (acc == 2) {                                   // PREFETCH: Hit iff a managed range
    if (has && kind == 0) w = TR_HIT | TR_HIT_POP | TR_PF | (res != 2 ? TR_POP : 0u);
  } else if (has && lc == 0) {                      // zombie / no range: Miss
    const bool am = acc == 1 && ro;
    if (!(!mig && res == 1) && !am && res == 2) w |= TR_HIT;
    if (!am) w |= TR_HIT_POP;                       // populated: GPU-resident, protection kept
  }
  return LF_VALID | w;
}

// ---- shared-memory layout ---------------------------------------------------------------
__host__ __device__ inline uint32_t al16(uint64_t x) { return (uint32_t)((x + 15) & ~uint64_t(15)); }

struct Layout {
  uint32_t lut, slut, fclient, cinfo, queue;
  uint32_t pg_base, pg_end, poff, rattr, rrid, skip, chan;
  uint32_t c64, iso, r32, counts, used, cstate, total;
  uint32_t rep_chan;
};

// kStaged: the interval table (page-granular SoA + skip tables, the client rows and the
// channel table replicated per bank) and the pass-1 caches live in smem at FIXED offsets
// sized for the FX_* limits, so every table access is an immediate-offset LDS.  Worlds beyond
// the limits run the global-table variant.  The LUT always lives in smem.
constexpr uint32_t FX_C = 64, FX_R = 2048, FX_CH = 256, FX_SKIP = 4096;

__host__ __device__ inline bool fits_fixed(const World& W) {
  return W.n_clients <= FX_C && W.n_ranges + 1 <= FX_R && W.n_channels <= FX_CH && W.n_skip + 1 <= FX_SKIP;
}

__host__ __device__ inline Layout make_layout(const World& W, bool staged, bool fin) {
  const uint32_t nr = staged ? FX_R : W.n_ranges + 1, nc = staged ? FX_C : W.n_clients;
  const uint32_t nch = staged ? FX_CH + 1 : W.n_channels + 1;
  const uint32_t nskip = staged ? FX_SKIP : W.n_skip + 1;
  Layout L;
  uint32_t o = 0;
  L.rep_chan = staged ? 32u : 0u;
  L.lut = o; o += 4 * LUT_N;
  L.slut = o; o += 4 * 32;
  L.fclient = o; if (fin && staged) o += al16(32ull * nc);
  L.queue = o; if (!fin) o += WARPS * QCAP * 16;
  L.cinfo = o; if (staged) o += al16(512ull * nc);
  L.pg_base = o; if (staged) o += al16(4ull * nr);
  L.pg_end = o; if (staged) o += al16(4ull * nr);
  L.poff = o; if (staged) o += al16(4ull * nr);
  L.rattr = o; if (staged) o += al16(4ull * nr);
  L.rrid = o; if (staged && fin) o += al16(4ull * nr);
  L.skip = o; if (staged) o += al16(2ull * nskip);
  L.chan = o; if (staged) o += al16(4ull * nch * (L.rep_chan ? 32 : 1));
  L.c64 = o; if (staged && !fin) o += al16(24ull * nc + 16);
  L.iso = o; if (staged && !fin) o += al16(3ull * 128 * nc);
  L.r32 = o; if (staged && !fin) o += al16(8ull * nr);
  L.counts = o; if (staged && !fin) o += al16(4ull * NSCEN * nc);
  L.used = o; if (staged && !fin) o += 16;
  L.cstate = o; if (staged && fin) o += al16(32ull * nc);
  L.total = o;
  return L;
}

// Block-wide view of the world tables (smem when staged, else global) and pass-1 caches.
struct View {
  Tables T;
  unsigned long long *ft_ce, *ft_sa, *trap_sa;   // pass-1 caches (or the global minima)
  unsigned long long *ft_gr, *trap_mps;
  uint32_t* iso;                                  // [3][C][32] per-warp copies (or null)
  uint32_t *ext, *nr0, *counts;
  uint32_t* used;                                 // [2] claimed hash slots (dd, nr)
  const CState* cst;
};

template <bool kStaged>
__device__ View setup(uint8_t* sm, const Layout& L, const World& W, const Scratch& S, bool scan, bool fin,
                      bool isolation_flag, bool translation = false) {
  View v;
  const uint32_t tid = threadIdx.x, nb = blockDim.x;
  const uint32_t R1 = W.n_ranges + 1, C = W.n_clients;
  if (kStaged) {
    uint32_t* pb = reinterpret_cast<uint32_t*>(sm + L.pg_base);
    uint32_t* pe = reinterpret_cast<uint32_t*>(sm + L.pg_end);
    uint32_t* po = reinterpret_cast<uint32_t*>(sm + L.poff);
    uint32_t* ra = reinterpret_cast<uint32_t*>(sm + L.rattr);
    uint32_t* rr = reinterpret_cast<uint32_t*>(sm + L.rrid);
    for (uint32_t i = tid; i < R1; i += nb) {
      pb[i] = __ldg(W.pg_base + i); pe[i] = __ldg(W.pg_end + i);
      po[i] = __ldg(W.poff + i); ra[i] = __ldg(W.rattr + i);
      if (fin) rr[i] = __ldg(W.rrid + i);
    }
    uint16_t* sk = reinterpret_cast<uint16_t*>(sm + L.skip);
    for (uint32_t i = tid; i <= W.n_skip; i += nb) sk[i] = __ldg(W.skip + i);
    uint32_t* cn = reinterpret_cast<uint32_t*>(sm + L.chan);
    const uint32_t rc = L.rep_chan ? 32u : 1u;
    for (uint32_t i = tid; i < rc * (W.n_channels + 1); i += nb) cn[i] = __ldg(W.chan + i / rc);
    uint4* ci = reinterpret_cast<uint4*>(sm + L.cinfo);
    for (uint32_t i = tid; i < 32 * C; i += nb) ci[i] = __ldg(W.cinfo4 + i / 32);
    v.T.cinfo = ci;
    v.T.pg_base = pb; v.T.pg_end = pe; v.T.poff = po; v.T.rattr = ra; v.T.rrid = fin ? rr : W.rrid;
    v.T.skip = sk; v.T.chan = cn;
    v.T.rep_client = 32; v.T.rep_chan = L.rep_chan;
  } else {
    v.T.pg_base = W.pg_base; v.T.pg_end = W.pg_end; v.T.poff = W.poff; v.T.rattr = W.rattr; v.T.rrid = W.rrid;
    v.T.skip = W.skip; v.T.chan = W.chan;
    v.T.rep_client = 0; v.T.rep_chan = 0;
    v.T.cinfo = W.cinfo4;
  }
  uint32_t* lut = reinterpret_cast<uint32_t*>(sm + L.lut);
  for (uint32_t i = tid; i < (uint32_t)LUT_N; i += nb)
    lut[i] = translation ? tr_word((int)i) : lut_word((int)i, isolation_flag);
  v.T.lut = lut;
  v.T.n_channels = W.n_channels;
  v.T.exact1 = W.exact1;
  v.ft_ce = S.ft_ce; v.ft_sa = S.ft_sa; v.trap_sa = S.trap_sa;
  v.ft_gr = S.ft_gr; v.trap_mps = S.trap_mps;
  v.iso = nullptr;
  v.ext = S.ext; v.nr0 = S.nr0; v.counts = nullptr;
  v.used = S.ctrl + C_HASH_DD;                    // C_HASH_NR follows it
  v.cst = S.cstate;
  if (kStaged && scan) {
    unsigned long long* c64 = reinterpret_cast<unsigned long long*>(sm + L.c64);
    for (uint32_t i = tid; i < 3 * C + 2; i += nb) c64[i] = EMPTY64;
    v.ft_ce = c64; v.ft_sa = c64 + C; v.trap_sa = c64 + 2 * C;
    v.ft_gr = c64 + 3 * C; v.trap_mps = c64 + 3 * C + 1;
    uint32_t* iso = reinterpret_cast<uint32_t*>(sm + L.iso);
    for (uint32_t i = tid; i < 3 * 32 * C; i += nb) iso[i] = EMPTY32;
    v.iso = iso;
    uint32_t* r32 = reinterpret_cast<uint32_t*>(sm + L.r32);
    for (uint32_t i = tid; i < 2 * R1; i += nb) r32[i] = EMPTY32;
    v.ext = r32; v.nr0 = r32 + R1;
    uint32_t* cnt = reinterpret_cast<uint32_t*>(sm + L.counts);
    for (uint32_t i = tid; i < NSCEN * C; i += nb) cnt[i] = 0;
    v.counts = cnt;
    uint32_t* used = reinterpret_cast<uint32_t*>(sm + L.used);
    if (tid < 2) used[tid] = 0;
    v.used = used;
  }
  return v;
}

// Programmatic dependent launch: a kernel launched with programmatic stream serialization may
// start while its predecessor drains -- it stages its world tables first, then waits here for
// the predecessor's results (griddepcontrol.wait); pdl_trigger lets the successor start early.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// Branch-free conditional reductions (one predicated RED, no divergent block): the hot per-entry
// minima and counters.  The address must be valid whatever p is.
__device__ __forceinline__ void red_add_s(bool p, uint32_t* a) {
  asm volatile("{.reg .pred q; setp.ne.u32 q, %0, 0; @q red.shared.add.u32 [%1], 1;}" ::"r"((uint32_t)p),
               "r"((uint32_t)__cvta_generic_to_shared(a)) : "memory");
}
__device__ __forceinline__ void min_s_if(bool p, uint32_t* a, uint32_t v) {   // shared: load, compare, reduce
  const uint32_t sa = (uint32_t)__cvta_generic_to_shared(a);
  asm volatile("{.reg .pred q, r; .reg .u32 cur; ld.shared.u32 cur, [%1]; setp.ne.u32 q, %0, 0;"
               " setp.gt.and.u32 r, cur, %2, q; @r red.shared.min.u32 [%1], %2;}" ::"r"((uint32_t)p), "r"(sa), "r"(v)
               : "memory");
}
__device__ __forceinline__ void min_g_if(bool p, uint32_t cur, uint32_t* a, uint32_t v) {   // global, pre-loaded
  asm volatile("{.reg .pred q, r; setp.ne.u32 q, %0, 0; setp.gt.and.u32 r, %1, %2, q; @r red.relaxed.gpu.global.min.u32 [%3], %2;}"
               ::"r"((uint32_t)p), "r"(cur), "r"(v), "l"(a) : "memory");
}

__device__ __forceinline__ void raise_err(const Scratch& S, uint32_t bit, uint64_t gidx) {
  atomicOr(S.ctrl + C_ERR, bit);
  atomicMin(S.err_idx, (unsigned long long)gidx);
}

// Lean decode shared by the passes: channel word, client row, skip-table attribution
// (MemoryModel.range_at, memory.py:233-237: the unique range of the client with
// base <= va < end, plus the guard page right after it) and one LUT word
// (faults.classify, faults.py:134-171).  Entries with the valid flag clear decode to f = 0;
// malformed entries raise the error bits the host maps onto the reference's exceptions and
// also give 0: no channel (NoChannelAttribution, errors.py:59-60), engine / access out of
// range, engine not the channel's (KindMismatch, errors.py:36-37), VA beyond 2^53, unknown
// entry kind.
__device__ __forceinline__ Dec decode_fast(const Tables& T, const uint8_t* __restrict__ page_state,
                                           const Scratch& S, uint4 e, uint32_t gidx, uint32_t lane) {
  Dec d;
  d.va = (uint64_t)e.x | ((uint64_t)e.y << 32);
  const uint32_t w3 = e.w;
  const uint32_t eng = w3 & 0xFF, acc = (w3 >> 8) & 0xFF, ek = (w3 >> 16) & 0xFF;
  const bool valid = (w3 >> 24) & MPSF_ENTRY_VALID;
  const bool chok = e.z < T.n_channels;
  const uint32_t cw = rep_load(T.chan, chok ? e.z : T.n_channels, T.rep_chan, lane);   // row nch: invalid
  const uint32_t c = cw & 0xFFFFu, ceng = (cw >> 16) & 3u;
  const bool k0 = ek == 0;
  const uint4 ci = T.rep_client ? T.cinfo[c * 32 + lane] : T.cinfo[c];
  const uint32_t lo = ci.x & 0xFFFFu, hi = ci.x >> 16;
  const uint32_t page = (uint32_t)(d.va >> 12);
  const bool look = k0 && lo != hi && d.va < VA_TABLE_LIMIT && page >= ci.y;
  uint32_t j = (page - ci.y) >> (ci.z & 31u);
  const uint32_t jmax = ci.z >> 8;
  j = j < jmax ? j : jmax;
  uint32_t k = T.skip[ci.w + j];
  k += (k + 1 < hi && T.pg_base[k + 1] <= page) ? 1u : 0u;
  if (!T.exact1) {
    while (k + 1 < hi && T.pg_base[k + 1] <= page) ++k;
  }
  const uint32_t end = T.pg_end[k], base = T.pg_base[k];
  d.inr = look && page < end;
  d.guard = look && page == end;
  d.slot = T.poff[k] + (page - base);
  d.ridx = (d.inr || d.guard) ? k : NO_RID;
  const uint32_t a = T.rattr[k];
  const uint32_t ust = a >> 24;
  uint32_t st = ust;
  if (d.inr && ust == 0xFF) st = page_state[d.slot];
  const uint32_t rcls = d.inr ? ((a & 1u) | ((a >> 7) & 2u) | ((a >> 14) & 4u)) : 8u;
  st = d.inr ? (st & 7u) : 0u;
  const uint32_t e3 = eng < 3 ? eng : 2u, a3 = acc < 3 ? acc : 2u;
  const uint32_t idx = k0 ? ((e3 * 3 + a3) * 16 + rcls) * 8 + st : (uint32_t)LUT_XK + (ek < 16 ? ek : 15u);
  const uint32_t f = T.lut[idx];
  const bool bad = !(cw & CH_VALID) ||
                   (k0 ? (eng > 2 || acc > 2 || eng != ceng || d.va >= VA_LIMIT) : (f & LF_BAD) != 0);
  if (valid && bad) {
    const uint32_t bit = !(cw & CH_VALID) ? EB_NO_CHANNEL
                         : (!k0 || eng > 2 || acc > 2) ? EB_BAD_ENTRY
                         : (eng != ceng ? EB_MISMATCH : EB_VA);
    raise_err(S, bit, gidx);
  }
  d.f = (valid && !bad) ? f : 0u;
  d.c = c;
  d.cw = cw;
  return d;
}

// Decoded + classified view of one entry (the general and finalize passes).
struct Rec {
  bool valid;
  uint32_t c;       // client
  int ceng;         // channel engine
  int eng, kind;
  int s;            // scenario id
  uint64_t va;
  bool repl;        // replayable buffer
  uint32_t group;   // dedup group (replayable translation)
  bool sa;          // client is standalone
  struct { int ridx; bool in_range, guard; uint32_t slot; int kind; } at;
};

__device__ __forceinline__ Rec to_rec(const Dec& d, uint4 e) {
  Rec r;
  r.valid = d.f != 0;
  r.va = d.va;
  r.c = d.c;
  r.ceng = (int)((d.cw >> 16) & 3u);
  r.sa = (d.cw >> 18) & 1u;
  r.eng = (int)(e.w & 0xFF);
  r.kind = (int)((e.w >> 16) & 0xFF);
  r.s = (int)(d.f & LF_S);
  r.repl = (d.f & LF_REPL) != 0;
  r.group = (d.f >> LF_GROUP_SH) & 7u;
  r.at.ridx = d.ridx == NO_RID ? -1 : (int)d.ridx;
  r.at.in_range = d.inr;
  r.at.guard = d.guard;
  r.at.slot = d.slot;
  r.at.kind = ((d.f >> LF_M_SH) & 3u) == 2u ? 1 : 0;
  return r;
}

__device__ __forceinline__ uint32_t ok32_of(bool repl, uint64_t gidx) {
  return (repl ? 0u : 0x80000000u) | (uint32_t)gidx;
}

__device__ __forceinline__ uint32_t dd_slot(const World& W, const Rec& r) {
  return W.dd_groups == 1 ? r.at.slot : r.at.slot * W.dd_groups + r.group;
}

// Stream for the order-free passes (scan, general): warp w of the grid owns 64-entry chunks
// w, w + W, w + 2W, ...; each lane reads its two adjacent entries with one 32-byte
// non-allocating load (L2 evict-first) and the next chunk's pair is requested before the
// current one is processed, so a chunk's HBM latency hides behind the previous chunk's work.
constexpr int WCHUNK = 64;

__device__ __forceinline__ void ld_pair(const mpsf_fault_entry* in, uint32_t n, uint32_t i0, bool a32, uint4& a,
                                        uint4& b) {
  const uint4* p = reinterpret_cast<const uint4*>(in) + i0;
  if (a32 && i0 + 1 < n) {
    asm("ld.global.nc.L1::no_allocate.L2::evict_first.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w), "=r"(b.x), "=r"(b.y), "=r"(b.z), "=r"(b.w)
                 : "l"(p));
  } else {
    a = i0 < n ? __ldcs(p) : make_uint4(0, 0, 0, 0);
    b = i0 + 1 < n ? __ldcs(p + 1) : make_uint4(0, 0, 0, 0);
  }
}

template <typename F>
__device__ __forceinline__ void ldg_stream(const mpsf_fault_entry* in, uint64_t n64, F&& fn) {
  // batch indices stay below MAX_GIDX (2^29): chunk and entry indices are 32-bit
  const uint32_t n = (uint32_t)n64;
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t gw = blockIdx.x * (blockDim.x >> 5) + warp, GW = gridDim.x * (blockDim.x >> 5);
  const uint32_t nch = (n + WCHUNK - 1) / WCHUNK;
  const bool a32 = ((uintptr_t)in & 31u) == 0;
  uint4 na = make_uint4(0, 0, 0, 0), nb = na;
  if (gw < nch) ld_pair(in, n, gw * WCHUNK + 2 * lane, a32, na, nb);
  for (uint32_t c = gw; c < nch; c += GW) {
    const uint4 e0 = na, e1 = nb;
    if (c + GW < nch) ld_pair(in, n, (c + GW) * WCHUNK + 2 * lane, a32, na, nb);
    const uint32_t i0 = c * WCHUNK + 2 * lane;
    fn(e0, i0, i0 < n, e1, i0 + 1, i0 + 1 < n);
  }
}

// Flags of a scenario id alone (the pass-1 record keeps the scenario, not the LUT index): the
// lut_word bits that do not depend on the range or the access.
__device__ __forceinline__ uint32_t scen_word(int sid, bool isolation) {
  if (sid >= 28) return 0u;
  if (sid >= 23) return LF_VALID | LF_XKIND | (uint32_t)sid | LF_REPL | LF_FATAL;
  if (sid >= 18) return LF_VALID | LF_XKIND | (uint32_t)sid | LF_TRAP;
  const bool repl = s_replayable(sid), serv = s_serviceable(sid);
  return LF_VALID | (uint32_t)sid | (repl ? (LF_REPL | LF_DD) : 0u) |
         (serv ? LF_SERV : (isolation ? LF_ELIG : LF_FATAL));
}

// The pass-1 record stream: lane l of a warp-chunk reads records 2l, 2l+1 with one 16-byte
// load, the next chunk's pair requested before the current one is processed.
template <typename F>
__device__ __forceinline__ void rec_stream(const unsigned long long* rec, uint64_t n64, F&& fn) {
  const uint32_t n = (uint32_t)n64;   // < MAX_GIDX
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t gw = blockIdx.x * (blockDim.x >> 5) + warp, GW = gridDim.x * (blockDim.x >> 5);
  const uint32_t nch = (n + WCHUNK - 1) / WCHUNK;
  const bool a16 = ((uintptr_t)rec & 15u) == 0;
  auto ld = [&](uint32_t i0) {
    if (a16 && i0 + 1 < n) return __ldcs(reinterpret_cast<const ulonglong2*>(rec + i0));
    return make_ulonglong2(i0 < n ? __ldcs(rec + i0) : 0ull, i0 + 1 < n ? __ldcs(rec + i0 + 1) : 0ull);
  };
  ulonglong2 nx = make_ulonglong2(0, 0);
  if (gw < nch) nx = ld(gw * WCHUNK + 2 * lane);
  for (uint32_t c = gw; c < nch; c += GW) {
    const ulonglong2 r = nx;
    if (c + GW < nch) nx = ld((c + GW) * WCHUNK + 2 * lane);
    const uint32_t i0 = c * WCHUNK + 2 * lane;
    fn(r, i0, i0 < n, i0 + 1 < n);
  }
}

// ---- pass 1 ---------------------------------------------------------------------------------
// After its block-local part (counts and per-client / per-range minima in shared memory) an
// entry leaves at most two first-in-group minima on global tables: its dedup key (rule C2,
// a dense (page, group) slot or a claimed page slot) and the first eligible record of its page
// (nrall).  Both entries of a lane issue their L2 loads together and resolve afterwards.
// Wild pages (no range, no guard) go to a per-warp stack of deferred hash operations that is
// drained 32 at a time, so their CAS round trips never sit on the common path.
struct QOp { unsigned long long key; uint32_t val, tab; };

struct ScanOut {
  uint32_t* pa; uint32_t va;     // nrall precheck-min
  uint32_t* pd; uint32_t vd;     // dedup slot precheck-min / claim
  bool qn, qd;                   // deferred hash ops: NR key (hnr), dedup key (hdd)
  uint32_t c, eng, sid;          // key material (hash ops, claim fallback)
  uint64_t page;
  unsigned long long rec;        // pass-1 record (fixed-layout worlds)
};

// ---- pass-1 record (worlds within the FX limits) ----------------------------------------------
// k_scan leaves every entry's decode in one 8-byte record so pass 2 reads 8 bytes instead of
// the 16-byte entry and skips the decode:
//   [4:0] scenario  [10:5] client  [21:11] range index  [23:22] loc (0 skipped, 1 in range,
//   2 guard page, 3 no range / not a translation)  [25:24] channel engine  [26] standalone
//   [28:27] mechanism class m  [29] page >= 2^32 (pass 2 re-reads the entry)
//   [63:32] page slot (in range / guard) or the page number (no range)
constexpr uint32_t LOC_SKIP = 0, LOC_IN = 1, LOC_GUARD = 2, LOC_NONE = 3;

__device__ __forceinline__ unsigned long long pack_rec(const Dec& d) {
  if (!d.f) return 0ull;
  const uint32_t loc = d.inr ? LOC_IN : (d.guard ? LOC_GUARD : LOC_NONE);
  const uint64_t page = d.va >> 12;
  const bool inw = d.inr || d.guard;
  const uint32_t lo = (d.f & LF_S) | ((d.c & 63u) << 5) | ((inw ? d.ridx & 0x7FFu : 0u) << 11) | (loc << 22) |
                      (((d.cw >> 16) & 3u) << 24) | (((d.cw >> 18) & 1u) << 26) | (((d.f >> LF_M_SH) & 3u) << 27) |
                      ((!inw && (page >> 32)) ? (1u << 29) : 0u);
  const uint32_t hi = inw ? d.slot : (uint32_t)page;
  return (unsigned long long)lo | ((unsigned long long)hi << 32);
}

// Rebuilds the Dec of a record (the LUT word from the scenario, the page of in-world entries
// from the range row).  Returns false for a skipped entry.
__device__ __forceinline__ bool unpack_rec(const View& v, const uint32_t* slut, unsigned long long r,
                                           const mpsf_fault_entry* in, uint64_t i, Dec& d) {
  const uint32_t lo = (uint32_t)r, hi = (uint32_t)(r >> 32);
  const uint32_t loc = (lo >> 22) & 3u;
  d.f = 0; d.c = 0; d.cw = 0; d.inr = false; d.guard = false; d.ridx = NO_RID; d.slot = 0; d.va = 0;
  if (loc == LOC_SKIP) return false;
  const uint32_t sid = lo & 31u, ceng = (lo >> 24) & 3u;
  d.c = (lo >> 5) & 63u;
  d.cw = d.c | (ceng << 16) | (((lo >> 26) & 1u) << 18) | CH_VALID;
  uint32_t group;
  if (ceng == 0) group = sid == 15 ? 2u : ((sid >= 1 && sid <= 3) ? 1u : 0u);
  else group = 2u + ceng;
  d.f = slut[sid] | (((lo >> 27) & 3u) << LF_M_SH) | (group << LF_GROUP_SH);
  d.inr = loc == LOC_IN;
  d.guard = loc == LOC_GUARD;
  if (d.inr || d.guard) {
    d.ridx = (lo >> 11) & 0x7FFu;
    d.slot = hi;
    d.va = (uint64_t)(v.T.pg_base[d.ridx] + (hi - v.T.poff[d.ridx])) << 12;
  } else if (lo & (1u << 29)) {
    const uint4 e = __ldcs(reinterpret_cast<const uint4*>(in) + i);   // page beyond 32 bits: re-read
    d.va = (uint64_t)e.x | ((uint64_t)e.y << 32);
  } else {
    d.va = (uint64_t)hi << 12;
  }
  return true;
}

__device__ __forceinline__ unsigned long long scan_dkey(const ScanOut& o) {
  return dedup_key(o.c, (int)o.eng, (int)o.sid, o.page);
}

// Rare part of pass 1: SM traps and fatal reports (parse-time, or isolation off).  Inlined:
// as a call it cost a 176-byte stack frame and 1.5 % of k_scan.
template <bool kStaged>
__device__ __forceinline__ void scan_fatal(const View& v, const Scratch& S, uint32_t f, uint32_t c, uint32_t cw,
                                        uint64_t gidx) {
  const uint32_t sid = f & LF_S;
  const bool sa = (cw >> 18) & 1u;
  if (f & LF_TRAP) {
    const unsigned long long t = (gidx << 8) | (unsigned long long)sid;
    if (kStaged) smin64(sa ? v.trap_sa + c : v.trap_mps, t);
    else min64(sa ? S.trap_sa + c : S.trap_mps, t);
    return;
  }
  // fatal report (pipeline.py:168-182): keyed by its drain position
  const uint32_t ok = ((f & LF_REPL) ? 0u : 0x80000000u) | (uint32_t)gidx;
  const unsigned long long t = ((unsigned long long)ok << 8) | (unsigned long long)sid;
  const uint32_t ceng = (cw >> 16) & 3u;
  if (kStaged) smin64(sa ? v.ft_sa + c : (ceng == 1 ? v.ft_ce + c : v.ft_gr), t);
  else min64(sa ? S.ft_sa + c : (ceng == 1 ? S.ft_ce + c : S.ft_gr), t);
}

template <bool kStaged>
__device__ __forceinline__ void scan_fast(const World& W, const View& v, const Scratch& S, uint4 e, uint32_t gidx,
                                          unsigned long long* counts, ScanOut& o) {
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const Dec d = decode_fast(v.T, W.page_state, S, e, gidx, lane);
  const uint32_t f = d.f, c = d.c, sid = f & LF_S;
  if (kStaged) red_add_s(f != 0, v.counts + (f ? c * NSCEN + sid : 0u));
  else if (f) atomicAdd(counts + (uint64_t)c * NSCEN + sid, 1ull);
  if (f & (LF_TRAP | LF_FATAL)) scan_fatal<kStaged>(v, S, f, c, d.cw, gidx);
  const uint32_t ok = ((f & LF_REPL) ? 0u : 0x80000000u) | (uint32_t)gidx;
  // isolation-eligible (pipeline.py:177-179): per-client minimum per mechanism class (iso1
  // unmapped / iso2 managed / iso3 external; per-warp smem copies: a warp's indices only grow),
  // first record per guard page (nr0) and per external range (ext)
  const bool elig = (f & LF_ELIG) && !(f & LF_TRAP);
  const uint32_t m = (f >> LF_M_SH) & 3u;
  const bool inw = d.inr || d.guard;
  const bool rr = elig && (d.guard || (d.inr && m == 2));
  if (kStaged) {
    uint32_t* pi = v.iso + (m * W.n_clients + c) * 32 + warp;
    min_s_if(elig, pi, ok);
    uint32_t* pr = (d.guard ? v.nr0 : v.ext) + (inw ? d.ridx : 0u);
    min_s_if(rr, pr, ok);
  } else {
    if (elig) min32((m == 0 ? S.iso1 : (m == 1 ? S.iso2 : S.iso3)) + c, ok);
    if (rr) min32((d.guard ? S.nr0 : S.ext) + d.ridx, ok);
  }
  // first eligible record per in-range page: the epoch-1 first-isolation key of a client
  // released before the drain (trap / dead at start), so that case needs no extra pass
  o.pa = (elig && d.inr && S.nrall) ? S.nrall + d.slot : nullptr;
  o.va = ok;
  // dedup insert (rule C2): dense (page, group) slot or claimed page slot; wild pages hash
  const bool dd = (f & LF_DD) != 0;
  const uint32_t group = (f >> LF_GROUP_SH) & 7u;
  o.pd = (dd && inw) ? S.dd + (W.dd_groups == 1 ? d.slot : d.slot * W.dd_groups + group) : nullptr;
  o.vd = ((uint32_t)gidx << 3) | group;
  o.qn = elig && !inw;
  o.qd = dd && !inw;
  o.c = c; o.eng = e.w & 0xFF; o.sid = sid; o.page = d.va >> 12;
  o.rec = pack_rec(d);
}

// Claimed-slot dedup (sparse worlds): first claim wins the page for its group; a record of
// another group of the same page goes to the hash.
__device__ __forceinline__ void claim_resolve(const Scratch& S, uint32_t* used, uint32_t* slot, uint32_t val,
                                              uint32_t cur, unsigned long long key) {
  while (true) {
    if (cur == EMPTY32) {
      const uint32_t prev = atomicCAS(slot, EMPTY32, val);
      if (prev == EMPTY32) return;
      cur = prev;
      continue;
    }
    if ((cur & 7u) == (val & 7u)) { if (cur > val) atomicMin(slot, val); return; }
    if (!hash_min(S.hdd, used, key, val >> 3)) atomicOr(S.ctrl + C_OVF, 1u);
    return;
  }
}

// Deferred hash ops: push (warp-collective), drained 32 at a time.
__device__ __forceinline__ void q_push(QOp* q, uint32_t& cnt, bool has, unsigned long long key, uint32_t val,
                                       uint32_t tab, const Scratch& S, uint32_t* used) {
  const uint32_t lane = threadIdx.x & 31;
  const unsigned m = __ballot_sync(0xFFFFFFFFu, has);
  if (!m) return;
  if (has) {
    QOp x; x.key = key; x.val = val; x.tab = tab;
    q[cnt + __popc(m & ((1u << lane) - 1u))] = x;
  }
  cnt += __popc(m);
  if (cnt >= 32) {
    __syncwarp();
    const QOp x = q[cnt - 32 + lane];
    const Hash& h = x.tab ? S.hnr : S.hdd;
    if (!hash_min(h, used + x.tab, x.key, x.val)) atomicOr(S.ctrl + C_OVF, 1u);
    cnt -= 32;
    __syncwarp();
  }
}

__device__ __forceinline__ void q_drain(QOp* q, uint32_t cnt, const Scratch& S, uint32_t* used) {
  __syncwarp();
  const uint32_t lane = threadIdx.x & 31;
  if (lane < cnt) {
    const QOp x = q[lane];
    const Hash& h = x.tab ? S.hnr : S.hdd;
    if (!hash_min(h, used + x.tab, x.key, x.val)) atomicOr(S.ctrl + C_OVF, 1u);
  }
}

// End of a staged scan block: fold the block-local minima into the global ones (fire-and-forget
// reductions, one per touched slot).
__device__ __forceinline__ void flush_minima(const World& W, const Scratch& S, const View& v) {
  const uint32_t C = W.n_clients, R = W.n_ranges;
  for (uint32_t i = threadIdx.x; i < 3 * C; i += blockDim.x) {
    const uint32_t* w = v.iso + i * 32;
    uint32_t m = EMPTY32;
#pragma unroll 8
    for (int k = 0; k < 32; ++k) m = min(m, w[k]);
    uint32_t* g = (i < C ? S.iso1 : (i < 2 * C ? S.iso2 : S.iso3)) + (i % C);
    if (m != EMPTY32) atomicMin(g, m);
    const unsigned long long t = v.ft_ce[i];      // c64 = [ft_ce | ft_sa | trap_sa | ft_gr | trap_mps]
    if (t != EMPTY64) atomicMin(i < C ? S.ft_ce + i : (i < 2 * C ? S.ft_sa + (i - C) : S.trap_sa + (i - 2 * C)), t);
  }
  if (threadIdx.x < 2) {
    const unsigned long long t = v.ft_ce[3 * C + threadIdx.x];
    if (t != EMPTY64) atomicMin(threadIdx.x ? S.trap_mps : S.ft_gr, t);
  }
  for (uint32_t i = threadIdx.x; i < R; i += blockDim.x) {
    if (v.ext[i] != EMPTY32) atomicMin(S.ext + i, v.ext[i]);
    if (v.nr0[i] != EMPTY32) atomicMin(S.nr0 + i, v.nr0[i]);
  }
  if (threadIdx.x < 2 && v.used[threadIdx.x]) atomicAdd(S.ctrl + C_HASH_DD + threadIdx.x, v.used[threadIdx.x]);
}

// Pass 1 over entries [0, n) of `in` (global index P.base_index + i) by the calling CTA of a
// persistent grid: stream, flush the block-local minima and counts.
template <bool kStaged>
__device__ __forceinline__ void scan_phase(const World& W, const Scratch& S, const View& v, const Layout& L,
                                           uint8_t* smem, const mpsf_fault_entry* __restrict__ in, uint64_t n,
                                           const Params& P, unsigned long long* __restrict__ counts) {
  QOp* q = reinterpret_cast<QOp*>(smem + L.queue) + (threadIdx.x >> 5) * QCAP;
  uint32_t qn = 0;
  const bool sparse = W.dd_groups == 1;
  const uint32_t base = (uint32_t)P.base_index;                          // < MAX_GIDX
  unsigned long long* const drec = kStaged ? S.drec + (P.base_index - S.drec_base) : nullptr;
  ldg_stream(in, n, [&](uint4 e0, uint32_t i0, bool ok0, uint4 e1, uint32_t i1, bool ok1) {
    ScanOut o0, o1;
    if (!ok0) e0.w = 0;                       // past the end: decodes as a skipped entry
    if (!ok1) e1.w = 0;
    scan_fast<kStaged>(W, v, S, e0, base + i0, counts, o0);
    // entry 0's L2 pre-check loads go out before entry 1 is decoded, entry 1's right after:
    // the decode of entry 1 and the record store cover entry 0's L2 round trip
    const uint32_t ra0 = o0.pa ? __ldcg(o0.pa) : 0u, rd0 = o0.pd ? __ldcg(o0.pd) : 0u;
    scan_fast<kStaged>(W, v, S, e1, base + i1, counts, o1);
    const uint32_t ra1 = o1.pa ? __ldcg(o1.pa) : 0u, rd1 = o1.pd ? __ldcg(o1.pd) : 0u;
    if (kStaged) {                                     // pass-1 records, two per lane (16 bytes)
      unsigned long long* rp = drec + i0;
      // streaming stores (evict-first): the records must not push the dedup slots out of the L2
      if (ok1 && (((uintptr_t)rp & 15u) == 0)) __stcs(reinterpret_cast<ulonglong2*>(rp), make_ulonglong2(o0.rec, o1.rec));
      else {
        if (ok0) __stcs(rp, o0.rec);
        if (ok1) __stcs(rp + 1, o1.rec);
      }
    }
    min_g_if(o0.pa != nullptr, ra0, o0.pa, o0.va);
    min_g_if(o1.pa != nullptr, ra1, o1.pa, o1.va);
    if (!sparse) {
      min_g_if(o0.pd != nullptr, rd0, o0.pd, o0.vd);
      min_g_if(o1.pd != nullptr, rd1, o1.pd, o1.vd);
    } else {
      if (o0.pd) claim_resolve(S, v.used, o0.pd, o0.vd, rd0, scan_dkey(o0));
      if (o1.pd) claim_resolve(S, v.used, o1.pd, o1.vd, rd1, scan_dkey(o1));
    }
    if (__any_sync(0xFFFFFFFFu, o0.qn || o0.qd || o1.qn || o1.qd)) {
      q_push(q, qn, o0.qn, nr_key(o0.c, 0, o0.page), o0.va, 1, S, v.used);
      q_push(q, qn, o0.qd, scan_dkey(o0), (uint32_t)(o0.vd >> 3), 0, S, v.used);
      q_push(q, qn, o1.qn, nr_key(o1.c, 0, o1.page), o1.va, 1, S, v.used);
      q_push(q, qn, o1.qd, scan_dkey(o1), (uint32_t)(o1.vd >> 3), 0, S, v.used);
    }
  });
  q_drain(q, qn, S, v.used);
  if (kStaged) {
    __syncthreads();
    // fold the block's (client, scenario) counts into the batch counts (accumulates across the
    // launches of a chunked batch)
    for (uint32_t i = threadIdx.x; i < NSCEN * W.n_clients; i += blockDim.x)
      if (v.counts[i]) atomicAdd(counts + i, (unsigned long long)v.counts[i]);
    flush_minima(W, S, v);
  }
}

template <bool kStaged>
__global__ void __launch_bounds__(BLOCK, 1) k_scan(World W, Scratch S, const mpsf_fault_entry* __restrict__ in,
                                                   uint64_t n, Params P, unsigned long long* __restrict__ counts) {
  extern __shared__ __align__(128) uint8_t smem[];
  pdl_trigger();
  const Layout L = make_layout(W, kStaged, false);
  const View v = setup<kStaged>(smem, L, W, S, true, false, P.flags & MPSF_PF_ISOLATION);
  __syncthreads();
  pdl_wait();
  scan_phase<kStaged>(W, S, v, L, smem, in, n, P, counts);
}

// ---- per-client resolution ------------------------------------------------------------------
// Rules C4-C7 of SURVEY.md Appendix C (C9 "ROUND 1" + fate).  Block 0; blocks 1.. reduce counts.
__device__ inline void kill_thresholds(const Params& P, uint32_t m1, uint32_t m2, uint32_t m3,
                                       bool use_m2, bool& kill_all, uint32_t& tie) {
  kill_all = false;
  tie = EMPTY32;
  const uint32_t lat[3] = {P.m1_us, P.m2_us, P.m3_us};
  const uint32_t v[3] = {m1, m2, m3};
#pragma unroll
  for (int m = 0; m < 3; ++m) {
    if (m == 1 && !use_m2) continue;
    if (v[m] == EMPTY32) continue;
    if (lat[m] < P.benign_us) kill_all = true;
    else if (lat[m] == P.benign_us && v[m] < tie) tie = v[m];
  }
}

// Rules C4-C7 (C9 "ROUND 1" + fate) for every client, by the calling block: the client states go
// to cs (global or the CTA's shared copy), the shared scalars to gl; with `outputs` the block
// also writes the per-client verdicts, the global copies and the path word.  Returns whether
// the release-aware (general) path is needed -- the same on every block that calls it.
__device__ __forceinline__ bool resolve_phase(const World& W, const Scratch& S, const Params& P, CState* cs_out,
                                              Globals* gl, mpsf_client_verdict* __restrict__ verdict,
                                              bool outputs, int* s_general) {
  if (threadIdx.x == 0) *s_general = 0;
  __syncthreads();
  const bool iso = P.flags & MPSF_PF_ISOLATION;
  const bool gr_alive0 = W.has_mps && !(W.world_flags & MPSF_WF_GR_DEAD);
  const unsigned long long trap_mps = __ldcg(S.trap_mps), ft_gr = __ldcg(S.ft_gr);
  const bool trapped_mps = gr_alive0 && trap_mps != EMPTY64;
  const bool gr_applied = gr_alive0 && !trapped_mps && ft_gr != EMPTY64;
  const long long gr_rel = (!gr_alive0 || trapped_mps) ? REL_PRE
                           : (gr_applied ? (long long)(ft_gr >> 8) : REL_NONE);
  int general = 0;
  for (uint32_t c = threadIdx.x; c < W.n_clients; c += blockDim.x) {
    const mpsf_client_entry ce = W.clients[c];
    const bool sa = ce.mode == 1;
    const bool alive0 = ce.flags & 1;
    const bool ce_alive0 = !sa && alive0 && !(ce.flags & 2);
    const unsigned long long tsa = __ldcg(S.trap_sa + c), fsa = __ldcg(S.ft_sa + c), fce = __ldcg(S.ft_ce + c);
    const bool trapped = sa ? (alive0 && tsa != EMPTY64) : trapped_mps;
    const bool sa_applied = sa && alive0 && !trapped && fsa != EMPTY64;
    long long rel;
    if (!alive0) rel = REL_PRE;
    else if (sa) rel = trapped ? REL_PRE : (sa_applied ? (long long)(fsa >> 8) : REL_NONE);
    else rel = gr_rel;
    const bool ce_applied = ce_alive0 && fce != EMPTY64 && !(rel < (long long)(fce >> 8));
    const uint32_t i1 = __ldcg(S.iso1 + c), i2 = __ldcg(S.iso2 + c), i3 = __ldcg(S.iso3 + c);
    const bool elig = (i1 & i2 & i3) != EMPTY32;
    CState cs;
    cs.rel = rel;
    cs.ft_ce_ok = fce == EMPTY64 ? EMPTY32 : (uint32_t)(fce >> 8);
    cs.ft_sa_ok = fsa == EMPTY64 ? EMPTY32 : (uint32_t)(fsa >> 8);
    cs.trap_sa_idx = tsa == EMPTY64 ? EMPTY32 : (uint32_t)(tsa >> 8);
    bool kill_all;
    uint32_t tie;
    kill_thresholds(P, i1, i2, i3, false, kill_all, tie);
    cs.kill_tie = tie;
    cs.flags = (alive0 ? CS_ALIVE0 : 0u) | (sa ? CS_SA : 0u) | (ce_alive0 ? CS_CE_ALIVE0 : 0u) |
               ((!sa && (!ce_alive0 || ce_applied)) ? CS_CE_TORN : 0u) | (kill_all ? CS_KILL_ALL : 0u) |
               (trapped ? CS_TRAPPED : 0u) | (elig ? CS_ELIG : 0u);
    cs.pad = 0;
    cs_out[c] = cs;
    if (outputs) {
      if (cs_out != S.cstate) S.cstate[c] = cs;
      mpsf_client_verdict v;
      v.flags = 0;
      if (alive0) {
        if (trapped) { v.state = 1; v.reason = 2; v.notifier = (uint8_t)((sa ? tsa : trap_mps) & 0xFF); }
        else if (!sa && gr_applied) { v.state = 1; v.reason = 2; v.notifier = (uint8_t)(ft_gr & 0xFF); }
        else if (sa_applied) { v.state = 1; v.reason = 2; v.notifier = (uint8_t)(fsa & 0xFF); }
        else if (elig) { v.state = 1; v.reason = 1; v.notifier = ce_applied ? (uint8_t)(fce & 0xFF) : 0xFF; }
        else if (ce_applied) { v.state = 0; v.reason = 0; v.notifier = (uint8_t)(fce & 0xFF); }
        else { v.state = 0; v.reason = 0; v.notifier = 0xFF; }
      } else {
        v.state = 1; v.reason = 3;
        v.notifier = (!sa && trapped_mps) ? (uint8_t)(trap_mps & 0xFF)
                     : ((!sa && gr_applied) ? (uint8_t)(ft_gr & 0xFF) : 0xFE);
      }
      verdict[c] = v;
    }
    // release-aware pass needed: a client released inside the drain (C3 epochs), a client
    // released before it when pass 1 kept no per-page keys, or exact M2 minima (m2 <= benign)
    if (iso && elig &&
        ((rel != REL_NONE && !(rel == REL_PRE && S.nrall)) || (rel == REL_NONE && P.m2_us <= P.benign_us)))
      general = 1;
  }
  if (general) atomicOr(s_general, 1);
  __syncthreads();
  if (threadIdx.x == 0) {
    Globals g;
    g.ft_gr_ok = gr_applied ? (uint32_t)(ft_gr >> 8) : EMPTY32;
    g.trap_mps_idx = trapped_mps ? (uint32_t)(trap_mps >> 8) : EMPTY32;
    g.gr_alive0 = gr_alive0;
    g.has_elig = 0;
    *gl = g;
    if (outputs) {
      if (gl != S.glob) *S.glob = g;
      S.ctrl[C_PATH] = *s_general;
    }
  }
  __syncthreads();
  if (outputs)   // the global decision table (worlds beyond the fixed layout read it in pass 2)
    for (uint32_t c = threadIdx.x; c < W.n_clients; c += blockDim.x)
      S.fclient[c] = fin_client(cs_out[c], *gl, S.nrall != nullptr);
  return *s_general != 0;
}

__global__ void k_resolve(World W, Scratch S, Params P, mpsf_client_verdict* __restrict__ verdict) {
  pdl_wait();
  pdl_trigger();
  if (blockIdx.x > 0) return;
  __shared__ int s_general;
  if (__ldcg(S.ctrl + C_ERR) != 0) return;
  resolve_phase(W, S, P, S.cstate, S.glob, verdict, true, &s_general);
}

// ---- general path (rule C3 epochs) ----------------------------------------------------------
__device__ __forceinline__ uint32_t dedup_rep(const World& W, const Scratch& S, const Rec& r) {
  // smallest global index among records of r's dedup key
  if (r.at.in_range || r.at.guard) {
    const uint32_t cur = __ldcg(S.dd + dd_slot(W, r));
    if (cur != EMPTY32 && (cur & 7u) == r.group) return cur >> 3;
  }
  return hash_get(S.hdd, dedup_key(r.c, r.eng, r.s, r.va >> 12));
}

// First isolation-eligible record of r's (client, page, epoch).  A client released before the
// drain (rel == REL_PRE) has only epoch-1 records, all seeing an empty address space, so its
// key is the first eligible record of the page: pass 1's nrall / nr0 / epoch-0 hash entries.
__device__ __forceinline__ uint32_t nr_lookup(const Scratch& S, const Rec& r, bool epoch1, bool pre) {
  if (epoch1 && !(pre && S.nrall)) {
    if (r.at.in_range || r.at.guard) return __ldcg(S.nr1 + r.at.slot);
    return hash_get(S.hnr, nr_key(r.c, 1, r.va >> 12));
  }
  if (r.at.in_range) return __ldcg(S.nrall + r.at.slot);
  if (r.at.guard) return __ldcg(S.nr0 + r.at.ridx);
  return hash_get(S.hnr, nr_key(r.c, 0, r.va >> 12));
}

// stage 1: epoch-1 NR keys, exact M1 / M3 / direct-M2 minima (giso[3*c + m-1])
// stage 2: noRange non-first records -> M2 minima (needs NR complete)
template <bool kStaged, int kStage>
__device__ __forceinline__ void general_entry(const World& W, const View& v, const Scratch& S, const Params& P,
                                              uint4 e, uint64_t gidx) {
  const Rec r = to_rec(decode_fast(v.T, W.page_state, S, e, gidx, threadIdx.x & 31), e);
  if (!r.valid || r.kind != 0 || s_serviceable(r.s)) return;      // eligible translation records only
  const long long rel = v.cst[r.c].rel;
  const uint32_t ok = ok32_of(r.repl, gidx);
  if (rel == REL_NONE && P.m2_us > P.benign_us) return;           // pass-1 minima already exact
  if (rel == REL_PRE && S.nrall) return;                          // keys from pass 1; fates fixed
  if (r.repl && dedup_rep(W, S, r) != (uint32_t)gidx) return;       // dups excluded (C2)
  const bool epoch1 = rel < (long long)ok;
  const bool no_range = !r.at.in_range || epoch1;
  uint32_t* giso = S.giso + 3 * r.c;
  if (kStage == 1) {
    if (no_range) {
      min32(giso + 0, ok);
      if (epoch1) {
        if (r.at.in_range || r.at.guard) min32(S.nr1 + r.at.slot, ok);
        else if (!hash_min(S.hnr, S.ctrl + C_HASH_NR, nr_key(r.c, 1, r.va >> 12), ok)) atomicOr(S.ctrl + C_OVF, 1u);
      }
    } else if (r.at.kind == 0) {
      min32(giso + 1, ok);
    } else {
      const uint32_t ext = __ldcg(S.ext + r.at.ridx);
      if (ok == ext && (long long)ext < rel) min32(giso + 2, ok);
      else min32(giso + 1, ok);
    }
  } else {
    if (no_range && nr_lookup(S, r, epoch1, false) != ok) min32(giso + 1, ok);
  }
}

template <bool kStaged, int kStage>
__device__ __forceinline__ void general_phase(const World& W, const Scratch& S, const View& v,
                                              const mpsf_fault_entry* __restrict__ in, uint64_t n, const Params& P) {
  ldg_stream(in, n, [&](uint4 e0, uint64_t i0, bool ok0, uint4 e1, uint64_t i1, bool ok1) {
    if (ok0) general_entry<kStaged, kStage>(W, v, S, P, e0, P.base_index + i0);
    if (ok1) general_entry<kStaged, kStage>(W, v, S, P, e1, P.base_index + i1);
  });
}

template <bool kStaged, int kStage>
__global__ void __launch_bounds__(BLOCK, 1) k_general(World W, Scratch S, const mpsf_fault_entry* __restrict__ in,
                                                      uint64_t n, Params P) {
  pdl_trigger();
  pdl_wait();
  if (__ldcg(S.ctrl + C_PATH) == 0) return;
  extern __shared__ __align__(128) uint8_t smem[];
  const Layout L = make_layout(W, kStaged, true);
  View v = setup<kStaged>(smem, L, W, S, false, true, P.flags & MPSF_PF_ISOLATION);
  if (kStaged) {                                 // the client states k_resolve wrote
    CState* cs = reinterpret_cast<CState*>(smem + L.cstate);
    for (uint32_t i = threadIdx.x; i < W.n_clients; i += blockDim.x) cs[i] = S.cstate[i];
    v.cst = cs;
  }
  __syncthreads();
  general_phase<kStaged, kStage>(W, S, v, in, n, P);
}

// k_resolve and k_general (stage 1) in one launch (single-GPU batches on the fixed layout): every
// CTA resolves the client states itself into its shared copy -- O(clients), the same on every CTA;
// CTA 0 writes the outputs k_resolve writes -- and runs the release-aware pass only when a client
// needs it (otherwise the launch ends there: no separate k_resolve / k_general round trips).
__global__ void __launch_bounds__(BLOCK, 1) k_resolve_general(World W, Scratch S, const mpsf_fault_entry* __restrict__ in,
                                                              uint64_t n, Params P,
                                                              mpsf_client_verdict* __restrict__ verdict) {
  pdl_trigger();
  extern __shared__ __align__(128) uint8_t smem[];
  const Layout L = make_layout(W, true, true);
  CState* cs = reinterpret_cast<CState*>(smem + L.cstate);
  // (the layout is at the shared-memory limit: the resolution's scalars go into the decision-table
  // region, which the release-aware pass does not use)
  Globals* s_gl = reinterpret_cast<Globals*>(smem + L.fclient);
  int* s_general = reinterpret_cast<int*>(smem + L.fclient + sizeof(Globals));
  pdl_wait();
  if (__ldcg(S.ctrl + C_ERR) != 0) return;
  if (!resolve_phase(W, S, P, cs, s_gl, verdict, blockIdx.x == 0, s_general)) return;
  // the tables of the release-aware pass only when it runs (setup leaves the client states alone)
  View v = setup<true>(smem, L, W, S, false, true, P.flags & MPSF_PF_ISOLATION);
  v.cst = cs;
  __syncthreads();
  general_phase<true, 1>(W, S, v, in, n, P);
}

// Kill thresholds from the exact minima of the general path, one client (idempotent: a client
// state recomputed from the same minima is the same).
__device__ __forceinline__ void resolve2_client(const Scratch& S, const Params& P, uint32_t c, CState& cs) {
  if (cs.rel == REL_NONE && P.m2_us > P.benign_us) return;       // pass-1 minima are exact
  bool kill_all;
  uint32_t tie;
  uint32_t g0 = __ldcg(S.giso + 3 * c), g1 = __ldcg(S.giso + 3 * c + 1), g2 = __ldcg(S.giso + 3 * c + 2);
  if (cs.rel == REL_NONE) {                 // only M2 needed recomputing: keep exact M1 / M3
    g0 = __ldcg(S.iso1 + c);
    g2 = __ldcg(S.iso3 + c);
  }
  kill_thresholds(P, g0, g1, g2, true, kill_all, tie);
  cs.kill_tie = tie;
  cs.flags = (cs.flags & ~CS_KILL_ALL) | (kill_all ? CS_KILL_ALL : 0u);
}

// Kill thresholds from the exact minima of the general path (cs: global or the CTA's copy).
__device__ __forceinline__ void resolve2_phase(const World& W, const Scratch& S, const Params& P, CState* cs_arr) {
  for (uint32_t c = threadIdx.x; c < W.n_clients; c += blockDim.x) {
    CState cs = cs_arr[c];
    resolve2_client(S, P, c, cs);
    cs_arr[c] = cs;
  }
}

__global__ void k_resolve2(World W, Scratch S, Params P) {
  pdl_wait();
  pdl_trigger();
  if (__ldcg(S.ctrl + C_PATH) == 0) return;
  resolve2_phase(W, S, P, S.cstate);
  __syncthreads();
  for (uint32_t c = threadIdx.x; c < W.n_clients; c += blockDim.x)
    S.fclient[c] = fin_client(S.cstate[c], *S.glob, S.nrall != nullptr);
}

// ---- pass 2 -----------------------------------------------------------------------------
// k_finalize writes every OutRecord and, per 64-entry chunk, the bitmasks of cancelled entries
// and of dedup representatives, and adds the chunk's two counts to its segment counter
// (SEG_CHUNKS chunks per segment).  k_lists then writes the cancel list and the dedup set in
// index order: a block per segment sums the counters of the earlier segments for its base and
// scans its own chunks' popcounts -- no serial look-back between tiles.
constexpr uint32_t SEG_CHUNKS = 256;
constexpr uint32_t KSTAGE = WCHUNK;   // dedup keys staged per chunk by k_finalize, in index order
#ifndef LIST_KEYS
#define LIST_KEYS 8                    // dedup keys in flight per lane in k_lists
#endif

// Pass 2 per entry, in two halves so both entries of a lane issue their L2 lookups together:
// fin_addr decodes and picks the words the verdict depends on (the dedup slot of its key,
// the first-isolation word of its (client, page, epoch), its external range's first
// isolation); fin_resolve turns the loaded words into the OutRecord, the cancel flag and the
// dedup-set membership.  Wild pages (no range, no guard) look their keys up in the hashes.
struct FinA {
  Dec d;
  uint32_t ok;
  const uint32_t* pd;   // dedup slot word (in-world dedup candidates)
  const uint32_t* pn;   // first-isolation word (nrall / nr1 / nr0)
  const uint32_t* pe;   // external range's first isolation (ext)
  bool needs_nr, e1keys;
};

template <bool kStaged>
__device__ __forceinline__ void fin_addr(const World& W, const View& v, const Scratch& S, const FinClient* fct,
                                         const Dec& dd, uint32_t gidx, FinA& a) {
  a.d = dd;
  const Dec& d = a.d;
  const uint32_t f = d.f;
  const bool inw = d.inr || d.guard;
  a.ok = ((f & LF_REPL) ? 0u : 0x80000000u) | (uint32_t)gidx;
  a.pd = ((f & LF_DD) && inw)
             ? S.dd + (W.dd_groups == 1 ? d.slot : d.slot * W.dd_groups + ((f >> LF_GROUP_SH) & 7u)) : nullptr;
  const bool elig = (f & LF_ELIG) != 0;
  const long long rel = fct[d.c].rel;
  const bool epoch1 = rel < (long long)a.ok;
  a.needs_nr = elig && (!d.inr || epoch1);
  a.e1keys = epoch1 && !fct[d.c].pre_nrall;
  const uint32_t* pn = a.e1keys ? (inw ? S.nr1 + d.slot : nullptr)
                                : (d.inr ? S.nrall + d.slot : (d.guard ? S.nr0 + d.ridx : nullptr));
  a.pn = a.needs_nr ? pn : nullptr;
  a.pe = (elig && d.inr && !epoch1 && ((f >> LF_M_SH) & 3u) == 2u) ? S.ext + d.ridx : nullptr;
}

template <bool kStaged>
__device__ __forceinline__ void fin_resolve(const World& W, const View& v, const Scratch& S, const FinClient* fct,
                                            uint32_t gidx, const FinA& a, uint32_t wd, uint32_t wn,
                                            uint32_t we, unsigned long long& o8, bool& canc, bool& rep,
                                            unsigned long long& key) {
  const Dec& d = a.d;
  const uint32_t f = d.f;
  canc = false; rep = false; key = 0;
  if (!f) {
    o8 = 0xFFFF000000000000ull | (0xFFull << 32) | NO_RID;     // rid NO_RID, scenario 0xFF, client 0xFFFF
    return;
  }
  const uint32_t sid = f & LF_S, c = d.c, ceng = (d.cw >> 16) & 3u;
  const FinClient& fc = fct[c];
  const bool inw = d.inr || d.guard;
  const uint32_t ok = a.ok;
  const bool dd = f & LF_DD, trap = f & LF_TRAP, elig = f & LF_ELIG, serv = f & LF_SERV;
  // rule C2: the smallest index of the entry's dedup key
  uint32_t rep_ok = ok;
  bool dup = false;
  if (dd) {
    const uint32_t group = (f >> LF_GROUP_SH) & 7u;
    key = dedup_key(c, (int)ceng, (int)sid, d.va >> 12);      // translation: engine == channel's
    uint32_t ri = wd >> 3;
    if (!(inw && wd != EMPTY32 && (wd & 7u) == group))
      ri = hash_get(S.hdd, key);
    dup = ri != (uint32_t)gidx;
    rep_ok = ri;                                                 // replayable: ok32 == idx
    rep = !dup;
    if (!rep) key = 0;
  }
  const bool ce = ceng == 1;
  if (trap) canc = (uint32_t)gidx != fc.trap_ok;
  else if (serv) canc = ((fc.bflags >> (ce ? 1 : 0)) & 1u) || rep_ok > fc.tie;
  else if (!elig) canc = rep_ok != (ce ? fc.ft1 : fc.ft0);
  uint32_t mech = 0;
  if (elig && !dup) {                                            // isolation mechanism (C3)
    if (a.needs_nr) {
      uint32_t nr = wn;
      if (!inw) nr = hash_get(S.hnr, nr_key(c, a.e1keys ? 1 : 0, d.va >> 12));
      mech = nr == ok ? 1u : 2u;
    } else {
      mech = (a.pe && we == ok) ? 3u : 2u;
    }
  }
  const uint32_t outcome = trap ? 0u : (elig ? 2u : (serv ? 1u : 3u));
  const uint32_t verdict = outcome | (mech << 2) | (canc ? 0x10u : 0u) | (dup ? 0x20u : 0u) |
                           ((f & LF_REPL) ? 0x40u : 0u);
  const uint32_t rid = d.inr ? v.T.rrid[d.ridx] : NO_RID;
  o8 = (unsigned long long)rid | ((unsigned long long)sid << 32) | ((unsigned long long)verdict << 40) |
       ((unsigned long long)c << 48);
}

// Staged dedup key (re-read by k_lists): an L2-allocating store with the default policy (an
// evict-last policy here pinned up to 80 MB of keys at config 3 and pushed the dedup slots out).
__device__ __forceinline__ void st_keep(unsigned long long* p, unsigned long long v) { __stcg(p, v); }

// Spread the 32 bits of x to the even bits of a 64-bit word (bit i -> bit 2i).
__device__ __forceinline__ unsigned long long spread2(uint32_t x) {
  unsigned long long v = x;
  v = (v | (v << 16)) & 0x0000FFFF0000FFFFull;
  v = (v | (v << 8)) & 0x00FF00FF00FF00FFull;
  v = (v | (v << 4)) & 0x0F0F0F0F0F0F0F0Full;
  v = (v | (v << 2)) & 0x3333333333333333ull;
  v = (v | (v << 1)) & 0x5555555555555555ull;
  return v;
}

// Pass 2 (OutRecords, per-chunk masks, segment counts) by the calling CTA of a persistent grid over entries [0, n) of `in` (batch chunk q_base
// on): fct / slut are the CTA's client decision table and scenario flags (shared memory).
template <bool kStaged>
__device__ __forceinline__ void finalize_phase(const World& W, const Scratch& S, const View& v,
                                               const FinClient* fct, const uint32_t* slut,
                                               const mpsf_fault_entry* __restrict__ in, uint64_t n, const Params& P,
                                               mpsf_out_record* __restrict__ out, uint64_t q_base) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t base = (uint32_t)P.base_index;   // < MAX_GIDX
  auto body = [&](const Dec& d0, const Dec& d1, uint32_t i0, bool ok0, bool ok1) {
    const uint32_t i1 = i0 + 1;
    FinA a0, a1;
    fin_addr<kStaged>(W, v, S, fct, d0, base + i0, a0);
    fin_addr<kStaged>(W, v, S, fct, d1, base + i1, a1);
    const uint32_t wd0 = a0.pd ? __ldcg(a0.pd) : EMPTY32, wn0 = a0.pn ? __ldcg(a0.pn) : EMPTY32;
    const uint32_t we0 = a0.pe ? __ldcg(a0.pe) : EMPTY32;
    const uint32_t wd1 = a1.pd ? __ldcg(a1.pd) : EMPTY32, wn1 = a1.pn ? __ldcg(a1.pn) : EMPTY32;
    const uint32_t we1 = a1.pe ? __ldcg(a1.pe) : EMPTY32;
    unsigned long long o0, o1, k0, k1;
    bool c0, c1, r0, r1;
    fin_resolve<kStaged>(W, v, S, fct, base + i0, a0, wd0, wn0, we0, o0, c0, r0, k0);
    fin_resolve<kStaged>(W, v, S, fct, base + i1, a1, wd1, wn1, we1, o1, c1, r1, k1);
    unsigned long long* o = reinterpret_cast<unsigned long long*>(out) + i0;
    if (ok1 && (((uintptr_t)o & 15u) == 0)) __stcs(reinterpret_cast<ulonglong2*>(o), make_ulonglong2(o0, o1));
    else {
      if (ok0) __stcs(o, o0);
      if (ok1) __stcs(o + 1, o1);
    }
    const uint32_t bc0 = __ballot_sync(0xFFFFFFFFu, ok0 && c0), bc1 = __ballot_sync(0xFFFFFFFFu, ok1 && c1);
    const uint32_t bd0 = __ballot_sync(0xFFFFFFFFu, ok0 && r0), bd1 = __ballot_sync(0xFFFFFFFFu, ok1 && r1);
    const uint64_t qq = q_base + i0 / WCHUNK;
    // representative keys staged at their entry's position in the chunk
    if (ok0 && r0) st_keep(S.dstage + qq * KSTAGE + 2 * lane, k0);
    if (ok1 && r1) st_keep(S.dstage + qq * KSTAGE + 2 * lane + 1, k1);
    if (lane == 0) {
      // raw ballots (bit l of .x/.y: entry 2l / 2l + 1 cancelled; .z/.w: representatives)
      S.cmask[qq] = make_uint4(bc0, bc1, bd0, bd1);
      const uint32_t nc = __popc(bc0) + __popc(bc1), nd = __popc(bd0) + __popc(bd1);
      if (nc | nd) atomicAdd(S.segcnt + qq / SEG_CHUNKS, (unsigned long long)nc | ((unsigned long long)nd << 32));
    }
  };
  if (kStaged) {
    // staged worlds stream the pass-1 records: one 16-byte load = this lane's two records
    const unsigned long long* rec = S.drec + (P.base_index - S.drec_base);
    rec_stream(rec, n, [&](ulonglong2 r, uint32_t i0, bool ok0, bool ok1) {
      Dec d0, d1;
      unpack_rec(v, slut, ok0 ? r.x : 0ull, in, i0, d0);
      unpack_rec(v, slut, ok1 ? r.y : 0ull, in, i0 + 1, d1);
      body(d0, d1, i0, ok0, ok1);
    });
  } else {
    ldg_stream(in, n, [&](uint4 e0, uint32_t i0, bool ok0, uint4 e1, uint32_t i1, bool ok1) {
      if (!ok0) e0.w = 0;                     // past the end: decodes as a skipped entry
      if (!ok1) e1.w = 0;
      const Dec d0 = decode_fast(v.T, W.page_state, S, e0, base + i0, lane);
      const Dec d1 = decode_fast(v.T, W.page_state, S, e1, base + i1, lane);
      body(d0, d1, i0, ok0, ok1);
    });
  }
}

// The CTA's copies of the client decision table and the scenario flags.
__device__ __forceinline__ void fin_tables(const World& W, const Scratch& S, const Params& P, const CState* cs,
                                           const Globals& G, FinClient* fct, uint32_t* slut) {
  if (fct)
    for (uint32_t k = threadIdx.x; k < W.n_clients; k += blockDim.x) fct[k] = fin_client(cs[k], G, S.nrall != nullptr);
  for (uint32_t k = threadIdx.x; k < 32; k += blockDim.x) slut[k] = scen_word((int)k, P.flags & MPSF_PF_ISOLATION);
}

template <bool kStaged>
__global__ void __launch_bounds__(BLOCK, 1) k_finalize(World W, Scratch S, const mpsf_fault_entry* __restrict__ in,
                                                       uint64_t n, Params P, mpsf_out_record* __restrict__ out,
                                                       uint64_t q_base) {
  extern __shared__ __align__(128) uint8_t smem[];
  pdl_trigger();
  const Layout L = make_layout(W, kStaged, true);
  const View v = setup<kStaged>(smem, L, W, S, false, true, P.flags & MPSF_PF_ISOLATION);
  pdl_wait();
  if (__ldcg(S.ctrl + C_ERR) != 0) return;
  // the client decision table: the CTA's copy (fixed-layout worlds) or the global one k_resolve /
  // k_resolve2 wrote (any number of clients)
  FinClient* fct = kStaged ? reinterpret_cast<FinClient*>(smem + L.fclient) : S.fclient;
  uint32_t* slut = reinterpret_cast<uint32_t*>(smem + L.slut);
  if (kStaged) fin_tables(W, S, P, S.cstate, *S.glob, fct, slut);
  else fin_tables(W, S, P, S.cstate, *S.glob, nullptr, slut);
  __syncthreads();
  finalize_phase<kStaged>(W, S, v, fct, slut, in, n, P, out, q_base);
}

// Cancel list + dedup set in index order.  Block = one segment of SEG_CHUNKS chunks, one
// thread per chunk: a block-wide scan of the chunks' popcounts gives every chunk its offsets,
// then each thread writes its own chunk's entries (the L2 merges the short runs).  `in` /
// `out` / the masks cover the whole batch (nq chunks).
// The summary usually lives in mapped pinned host memory: one thread gathers it in registers
// and writes it with 16-byte stores (no read-back of host memory -- each one is a PCIe round
// trip).
__device__ __forceinline__ void write_summary(const Scratch& S, unsigned long long tot, DevSummary* out) {
  static_assert(sizeof(DevSummary) == 4 * C_NCTRL + 24 && C_NCTRL % 4 == 0, "summary layout");
  uint32_t c[C_NCTRL];
#pragma unroll
  for (int i = 0; i < C_NCTRL; ++i) c[i] = __ldcg(S.ctrl + i);
  const unsigned long long e = __ldcg(S.err_idx);
  const bool err = c[C_ERR] != 0;
  uint4* o4 = reinterpret_cast<uint4*>(out);
#pragma unroll
  for (int i = 0; i < C_NCTRL / 4; ++i) o4[i] = make_uint4(c[4 * i], c[4 * i + 1], c[4 * i + 2], c[4 * i + 3]);
  unsigned long long* t = reinterpret_cast<unsigned long long*>(out->ctrl + C_NCTRL);
  t[0] = e;
  t[1] = err ? 0ull : (tot & 0xFFFFFFFFull);
  t[2] = err ? 0ull : (tot >> 32);
}

__global__ void __launch_bounds__(SEG_CHUNKS) k_lists(Scratch S, const mpsf_fault_entry* __restrict__ in,
                                                   const mpsf_out_record* __restrict__ out, uint64_t nq,
                                                   uint64_t base_index, unsigned long long* __restrict__ dkeys,
                                                   uint32_t* __restrict__ didx, uint32_t* __restrict__ cancel,
                                                   DevSummary* __restrict__ sum, bool prescan) {
  static_assert(SEG_CHUNKS % 32 == 0 && SEG_CHUNKS <= 1024, "one thread per chunk");
  pdl_wait();
  const bool last = blockIdx.x == gridDim.x - 1;
  if (__ldcg(S.ctrl + C_ERR) != 0) {
    if (last && threadIdx.x == 0) write_summary(S, 0, sum);
    return;
  }
  __shared__ unsigned long long s_base;
  __shared__ unsigned long long s_w[32];
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t seg = blockIdx.x;
  // base: counts of all earlier segments (prescanned by k_seg_scan for large batches, where the
  // per-block sums would read O(segments^2) counters)
  if (prescan) {
    if (threadIdx.x == 0) s_base = __ldcg(S.segbase + seg);
  } else {
    unsigned long long acc = 0;
    for (uint64_t i = threadIdx.x; i < seg; i += blockDim.x) acc += __ldcg(S.segcnt + i);
    if (threadIdx.x == 0) s_base = 0;
    __syncthreads();
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xFFFFFFFFu, acc, o);
    if (lane == 0 && acc) atomicAdd(&s_base, acc);
  }
  const uint64_t q = seg * SEG_CHUNKS + threadIdx.x;
  ulonglong2 mk = make_ulonglong2(0, 0);
  if (q < nq) {
    const uint4 b = __ldcg(S.cmask + q);
    mk = make_ulonglong2(spread2(b.x) | (spread2(b.y) << 1), spread2(b.z) | (spread2(b.w) << 1));
  }
  const unsigned long long mine = (unsigned long long)__popcll(mk.x) | ((unsigned long long)__popcll(mk.y) << 32);
  unsigned long long x = mine;   // inclusive warp scan (both counts packed)
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long u = __shfl_up_sync(0xFFFFFFFFu, x, o);
    if (lane >= o) x += u;
  }
  if (lane == 31) s_w[warp] = x;
  __syncthreads();
  unsigned long long pre = s_base;
  for (uint32_t w = 0; w < warp; ++w) pre += s_w[w];
  if (last && threadIdx.x == blockDim.x - 1) write_summary(S, pre + x, sum);   // batch totals
  pre += x - mine;
  const uint64_t pc = pre & 0xFFFFFFFFull;
  uint64_t pd = pre >> 32;
  const uint32_t g0 = (uint32_t)(base_index + q * WCHUNK);
  // cancel list: each lane lists its chunk's cancelled entries (ascending) into the warp's shared
  // buffer from its offset in the warp (a warp scan of the counts), then the warp copies the
  // buffer out with coalesced stores -- the warp's chunks are consecutive, so are their cancels
  __shared__ uint16_t s_code[SEG_CHUNKS / 32][32 * WCHUNK];   // per warp: its 32 chunks' entries
  {
    uint16_t* buf = s_code[warp];            // (chunk in the warp << 6 | entry)
    const uint32_t cnt = (uint32_t)__popcll(mk.x);
    uint32_t inc = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t u = __shfl_up_sync(0xFFFFFFFFu, inc, o);
      if (lane >= o) inc += u;
    }
    const uint32_t tot = __shfl_sync(0xFFFFFFFFu, inc, 31);
    uint32_t pos = inc - cnt;
    for (unsigned long long m = mk.x; m; m &= m - 1)
      buf[pos++] = (uint16_t)((lane << 6) | (uint32_t)(__ffsll((long long)m) - 1));
    __syncwarp();
    const uint64_t cb0 = __shfl_sync(0xFFFFFFFFu, pc, 0);
    const uint32_t gw0 = __shfl_sync(0xFFFFFFFFu, g0, 0);   // the warp's first entry
    for (uint32_t t = lane; t < tot; t += 32) cancel[cb0 + t] = gw0 + buf[t];
    __syncwarp();
  }
  // dedup set: the warp's representatives occupy consecutive positions from its first chunk's
  // offset on.  Each lane lists its chunk's representatives (chunk << 6 | entry) at their flat
  // ranks in a per-warp shared table, then lane l writes ranks l, l + 32, ... (coalesced) with
  // one table read each.  Keys were staged by k_finalize.
  {
    uint16_t* code = s_code[warp];
    unsigned long long dm_l = mk.y;
    const uint32_t cnt = (uint32_t)__popcll(dm_l);
    uint32_t inc = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t u = __shfl_up_sync(0xFFFFFFFFu, inc, o);
      if (lane >= o) inc += u;
    }
    const uint32_t R = __shfl_sync(0xFFFFFFFFu, inc, 31);
    const uint64_t pd0 = __shfl_sync(0xFFFFFFFFu, pd, 0);
    const uint64_t q0w = q - lane;
    for (uint32_t pos = inc - cnt; dm_l; dm_l &= dm_l - 1)
      code[pos++] = (uint16_t)((lane << 6) | (uint32_t)(__ffsll((long long)dm_l) - 1));
    __syncwarp();
    for (uint32_t r0 = 0; r0 < R; r0 += 32 * LIST_KEYS) {
      unsigned long long key[LIST_KEYS];
      uint32_t gix[LIST_KEYS];
#pragma unroll
      for (int h = 0; h < LIST_KEYS; ++h) {
        const uint32_t f = r0 + 32 * h + lane;
        const uint32_t c = f < R ? code[f] : 0u;
        const uint64_t qj = q0w + (c >> 6);
        key[h] = f < R ? __ldcg(S.dstage + qj * KSTAGE + (c & 63u)) : 0ull;
        gix[h] = (uint32_t)(base_index + qj * WCHUNK) + (c & 63u);
      }
#pragma unroll
      for (int h = 0; h < LIST_KEYS; ++h) {
        const uint32_t f = r0 + 32 * h + lane;
        if (f < R) {
          dkeys[pd0 + f] = key[h];
          didx[pd0 + f] = gix[h];
        }
      }
    }
  }
}

// Exclusive prefix of the segment counters (one CTA; thread t owns a contiguous run).
__global__ void __launch_bounds__(1024) k_seg_scan(const Scratch S, uint64_t nseg) {
  pdl_wait();
  pdl_trigger();
  __shared__ unsigned long long sw[33];
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t per = (nseg + 1023) / 1024, b = threadIdx.x * per, e = min(b + per, nseg);
  unsigned long long s = 0;
  for (uint64_t i0 = b; i0 < e; i0 += 8) {   // eight loads in flight
    unsigned long long v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = i0 + k < e ? __ldcg(S.segcnt + i0 + k) : 0ull;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += v[k];
  }
  unsigned long long inc = s;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long u = __shfl_up_sync(0xFFFFFFFFu, inc, o);
    if (lane >= (uint32_t)o) inc += u;
  }
  if (lane == 31) sw[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    const unsigned long long w = sw[lane];
    unsigned long long wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long u = __shfl_up_sync(0xFFFFFFFFu, wi, o);
      if (lane >= (uint32_t)o) wi += u;
    }
    sw[lane] = wi - w;
  }
  __syncthreads();
  unsigned long long run = sw[warp] + inc - s;
  for (uint64_t i0 = b; i0 < e; i0 += 8) {
    unsigned long long v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = i0 + k < e ? __ldcg(S.segcnt + i0 + k) : 0ull;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (i0 + k < e) S.segbase[i0 + k] = run;
      run += v[k];
    }
  }
}

// Batch summary: error / overflow words and the list lengths (sum of the segment counters).
__global__ void k_summary(const Scratch S, uint64_t nseg, DevSummary* out) {
  pdl_wait();
  __shared__ unsigned long long s_tot;
  if (threadIdx.x == 0) s_tot = 0;
  __syncthreads();
  unsigned long long acc = 0;
  for (uint64_t i = threadIdx.x; i < nseg; i += blockDim.x) acc += __ldcg(S.segcnt + i);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xFFFFFFFFu, acc, o);
  if ((threadIdx.x & 31) == 0 && acc) atomicAdd(&s_tot, acc);
  __syncthreads();
  if (threadIdx.x == 0) write_summary(S, s_tot, out);
}

#include "fx_passes.cuh"

// ---- batched translation kernels ------------------------------------------------------------
// T1: the first PREFETCH index per managed page (the only in-batch dependency of resolve_va).
// Only PREFETCH translations matter here (~1 in 10 accesses), so a warp stacks its candidates
// (entry + index) in shared memory and decodes them 32 at a time: one decode per 32 prefetches
// instead of one per access.  (Malformed entries are reported by k_tr_classify, which decodes
// every access.)  Without room for the stacks (use_q false) every access is decoded.
constexpr uint32_t PFQ = 96;                       // per-warp stack: < 32 kept + 64 per chunk
constexpr uint32_t PFQ_BYTES = WARPS * PFQ * 20;   // uint4 entry + u32 index

template <bool kStaged>
__global__ void __launch_bounds__(BLOCK, 1) k_tr_prefetch(World W, Scratch S, const mpsf_fault_entry* __restrict__ in,
                                                          uint64_t n, Params P, uint32_t use_q) {
  extern __shared__ __align__(128) uint8_t smem[];
  pdl_trigger();
  const Layout L = make_layout(W, kStaged, true);
  const View v = setup<kStaged>(smem, L, W, S, false, true, false, true);
  __syncthreads();
  pdl_wait();
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t base = (uint32_t)P.base_index;
  if (!use_q) {
    ldg_stream(in, n, [&](uint4 e0, uint32_t i0, bool ok0, uint4 e1, uint32_t i1, bool ok1) {
      if (!ok0) e0.w = 0;
      if (!ok1) e1.w = 0;
      const Dec d0 = decode_fast(v.T, W.page_state, S, e0, base + i0, lane);
      const Dec d1 = decode_fast(v.T, W.page_state, S, e1, base + i1, lane);
      if ((d0.f & TR_PF) && d0.inr) min32(S.pf + d0.slot, base + i0);
      if ((d1.f & TR_PF) && d1.inr) min32(S.pf + d1.slot, base + i1);
    });
    return;
  }
  uint4* qe = reinterpret_cast<uint4*>(smem + L.total) + warp * PFQ;
  uint32_t* qi = reinterpret_cast<uint32_t*>(smem + L.total + WARPS * PFQ * 16) + warp * PFQ;
  uint32_t qn = 0;
  auto drain = [&](uint32_t k) {   // decode stack entries [qn - k, qn) by lanes 0..k-1
    __syncwarp();
    if (lane < k) {
      const uint32_t g = qi[qn - k + lane];
      const Dec d = decode_fast(v.T, W.page_state, S, qe[qn - k + lane], g, lane);
      if ((d.f & TR_PF) && d.inr) min32(S.pf + d.slot, g);
    }
    qn -= k;
    __syncwarp();
  };
  const uint32_t lt = (1u << lane) - 1u;
  ldg_stream(in, n, [&](uint4 e0, uint32_t i0, bool ok0, uint4 e1, uint32_t i1, bool ok1) {
    // candidates: valid translation entries with access PREFETCH
    const bool c0 = ok0 && (e0.w & 0x01FFFF00u) == (0x01000000u | (2u << 8));
    const bool c1 = ok1 && (e1.w & 0x01FFFF00u) == (0x01000000u | (2u << 8));
    const uint32_t b0 = __ballot_sync(0xFFFFFFFFu, c0), b1 = __ballot_sync(0xFFFFFFFFu, c1);
    if (!(b0 | b1)) return;
    if (c0) {
      const uint32_t p = qn + __popc(b0 & lt);
      qe[p] = e0;
      qi[p] = base + i0;
    }
    qn += __popc(b0);
    if (c1) {
      const uint32_t p = qn + __popc(b1 & lt);
      qe[p] = e1;
      qi[p] = base + i1;
    }
    qn += __popc(b1);
    while (qn >= 32) drain(32);
  });
  if (qn) drain(qn);
}

// T2: Hit / Miss per access (the page state an earlier prefetch left), per-chunk ballots of
// the misses (.x/.y) and of the populating prefetches (.z/.w), segment counters.
template <bool kStaged>
__global__ void __launch_bounds__(BLOCK, 1) k_tr_classify(World W, Scratch S, const mpsf_fault_entry* __restrict__ in,
                                                          uint64_t n, Params P, uint8_t* __restrict__ hit) {
  extern __shared__ __align__(128) uint8_t smem[];
  pdl_trigger();
  const Layout L = make_layout(W, kStaged, true);
  const View v = setup<kStaged>(smem, L, W, S, false, true, false, true);
  __syncthreads();
  pdl_wait();
  if (__ldcg(S.ctrl + C_ERR) != 0) return;
  const uint32_t lane = threadIdx.x & 31;
  ldg_stream(in, n, [&](uint4 e0, uint64_t i0, bool ok0, uint4 e1, uint64_t i1, bool ok1) {
    if (!ok0) e0.w = 0;
    if (!ok1) e1.w = 0;
    const uint32_t g0 = (uint32_t)(P.base_index + i0), g1 = (uint32_t)(P.base_index + i1);
    const Dec d0 = decode_fast(v.T, W.page_state, S, e0, g0, lane);
    const Dec d1 = decode_fast(v.T, W.page_state, S, e1, g1, lane);
    const uint32_t pf0 = d0.inr ? __ldcg(S.pf + d0.slot) : EMPTY32;
    const uint32_t pf1 = d1.inr ? __ldcg(S.pf + d1.slot) : EMPTY32;
    const bool h0 = (d0.f & (pf0 < g0 ? TR_HIT_POP : TR_HIT)) != 0;
    const bool h1 = (d1.f & (pf1 < g1 ? TR_HIT_POP : TR_HIT)) != 0;
    const bool m0 = d0.f && !h0, m1 = d1.f && !h1;
    const bool p0 = (d0.f & TR_POP) && pf0 == g0, p1 = (d1.f & TR_POP) && pf1 == g1;
    const uint32_t b0 = d0.f ? (h0 ? 1u : 0u) : 0xFFu, b1 = d1.f ? (h1 ? 1u : 0u) : 0xFFu;
    uint8_t* hp = hit + i0;
    if (ok1 && (((uintptr_t)hp & 1u) == 0)) *reinterpret_cast<uint16_t*>(hp) = (uint16_t)(b0 | (b1 << 8));
    else {
      if (ok0) hp[0] = (uint8_t)b0;
      if (ok1) hp[1] = (uint8_t)b1;
    }
    const uint32_t bm0 = __ballot_sync(0xFFFFFFFFu, ok0 && m0), bm1 = __ballot_sync(0xFFFFFFFFu, ok1 && m1);
    const uint32_t bp0 = __ballot_sync(0xFFFFFFFFu, ok0 && p0), bp1 = __ballot_sync(0xFFFFFFFFu, ok1 && p1);
    {   // the chunk's misses compacted in access order: k_tr_lists copies them out without
        // re-reading the stream (which its scattered reads would pull in nearly whole)
      const uint32_t below = (1u << lane) - 1u;
      uint4* stg = S.trstage + (i0 / WCHUNK) * WCHUNK + __popc(bm0 & below) + __popc(bm1 & below);
      if (ok0 && m0) __stcg(stg, e0);
      if (ok1 && m1) __stcg(stg + ((ok0 && m0) ? 1 : 0), e1);
    }
    if (lane == 0) {
      const uint64_t q = i0 / WCHUNK;
      S.cmask[q] = make_uint4(bm0, bm1, bp0, bp1);
      const uint32_t nm = __popc(bm0) + __popc(bm1), np_ = __popc(bp0) + __popc(bp1);
      if (nm | np_) atomicAdd(S.segcnt + q / SEG_CHUNKS, (unsigned long long)nm | ((unsigned long long)np_ << 32));
    }
  });
}

// T3: the misses in access order as fault-buffer entries (+ their indices), the populating
// prefetches' indices; one SEG_CHUNKS-thread block per segment (as k_lists).
__global__ void __launch_bounds__(SEG_CHUNKS) k_tr_lists(Scratch S, const mpsf_fault_entry* __restrict__ in,
                                                      uint64_t nq, uint64_t base_index,
                                                      mpsf_fault_entry* __restrict__ faults,
                                                      uint32_t* __restrict__ fault_idx, uint32_t* __restrict__ pop_idx,
                                                      DevSummary* __restrict__ sum) {
  pdl_wait();
  const bool last = blockIdx.x == gridDim.x - 1;
  if (__ldcg(S.ctrl + C_ERR) != 0) {
    if (last && threadIdx.x == 0) write_summary(S, 0, sum);
    return;
  }
  __shared__ unsigned long long s_base;
  __shared__ unsigned long long s_w[32];
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t seg = blockIdx.x;
  unsigned long long acc = 0;
  for (uint64_t i = threadIdx.x; i < seg; i += blockDim.x) acc += __ldcg(S.segcnt + i);
  if (threadIdx.x == 0) s_base = 0;
  __syncthreads();
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xFFFFFFFFu, acc, o);
  if (lane == 0 && acc) atomicAdd(&s_base, acc);
  const uint64_t q = seg * SEG_CHUNKS + threadIdx.x;
  ulonglong2 mk = make_ulonglong2(0, 0);
  if (q < nq) {
    const uint4 b = __ldcg(S.cmask + q);
    mk = make_ulonglong2(spread2(b.x) | (spread2(b.y) << 1), spread2(b.z) | (spread2(b.w) << 1));
  }
  const unsigned long long mine = (unsigned long long)__popcll(mk.x) | ((unsigned long long)__popcll(mk.y) << 32);
  unsigned long long x = mine;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long u = __shfl_up_sync(0xFFFFFFFFu, x, o);
    if (lane >= o) x += u;
  }
  if (lane == 31) s_w[warp] = x;
  __syncthreads();
  unsigned long long pre = s_base;
  for (uint32_t w = 0; w < warp; ++w) pre += s_w[w];
  if (last && threadIdx.x == blockDim.x - 1) write_summary(S, pre + x, sum);
  pre += x - mine;
  const uint64_t pm = pre & 0xFFFFFFFFull, pp = pre >> 32;
  const uint32_t g0 = (uint32_t)(base_index + q * WCHUNK);
  // misses: each lane lists its chunk's misses (chunk in the warp << 6 | entry, ascending) at
  // their flat ranks in the warp's shared table and notes its chunk's first rank; the warp then
  // copies ranks l, l + 32, ... with TR_KEYS staged entries in flight per lane and coalesced
  // stores (as k_lists: the warp's chunks are consecutive, so are their misses)
  constexpr int TR_KEYS = 8;
  __shared__ uint16_t s_code[SEG_CHUNKS / 32][32 * WCHUNK];
  __shared__ uint32_t s_cst[SEG_CHUNKS / 32][32];
  uint16_t* code = s_code[warp];
  const uint64_t q0w = q - lane;
  const uint32_t gw0 = __shfl_sync(0xFFFFFFFFu, g0, 0);   // the warp's first access
  {
    unsigned long long m = mk.x;
    const uint32_t cnt = (uint32_t)__popcll(m);
    uint32_t inc = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t u = __shfl_up_sync(0xFFFFFFFFu, inc, o);
      if (lane >= o) inc += u;
    }
    const uint32_t R = __shfl_sync(0xFFFFFFFFu, inc, 31);
    const uint64_t pm0 = __shfl_sync(0xFFFFFFFFu, pm, 0);
    s_cst[warp][lane] = inc - cnt;
    for (uint32_t pos = inc - cnt; m; m &= m - 1)
      code[pos++] = (uint16_t)((lane << 6) | (uint32_t)(__ffsll((long long)m) - 1));
    __syncwarp();
    uint4* const faults4 = reinterpret_cast<uint4*>(faults);
    for (uint32_t r0 = 0; r0 < R; r0 += 32 * TR_KEYS) {
      uint4 v[TR_KEYS];
      uint32_t gi[TR_KEYS];
#pragma unroll
      for (int h = 0; h < TR_KEYS; ++h) {
        const uint32_t f = r0 + 32 * h + lane;
        const uint32_t c = f < R ? code[f] : 0u, ch = c >> 6;
        v[h] = f < R ? __ldcs(S.trstage + (q0w + ch) * WCHUNK + (f - s_cst[warp][ch])) : make_uint4(0u, 0u, 0u, 0u);
        gi[h] = gw0 + ch * WCHUNK + (c & 63u);
      }
#pragma unroll
      for (int h = 0; h < TR_KEYS; ++h) {
        const uint32_t f = r0 + 32 * h + lane;
        if (f < R) {
          faults4[pm0 + f] = v[h];
          fault_idx[pm0 + f] = gi[h];
        }
      }
    }
    __syncwarp();
  }
  // populating prefetches: the same listing, indices only
  {
    unsigned long long m = mk.y;
    const uint32_t cnt = (uint32_t)__popcll(m);
    uint32_t inc = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t u = __shfl_up_sync(0xFFFFFFFFu, inc, o);
      if (lane >= o) inc += u;
    }
    const uint32_t R = __shfl_sync(0xFFFFFFFFu, inc, 31);
    const uint64_t pp0 = __shfl_sync(0xFFFFFFFFu, pp, 0);
    for (uint32_t pos = inc - cnt; m; m &= m - 1)
      code[pos++] = (uint16_t)((lane << 6) | (uint32_t)(__ffsll((long long)m) - 1));
    __syncwarp();
    for (uint32_t f = lane; f < R; f += 32) {
      const uint32_t c = code[f];
      pop_idx[pp0 + f] = gw0 + (c >> 6) * WCHUNK + (c & 63u);
    }
  }
}

// ---- sparse hash exchange (multi-GPU) ------------------------------------------------------
__global__ void k_hash_export(Hash h, uint64_t cap, unsigned long long* __restrict__ keys, uint32_t* __restrict__ vals,
                              uint32_t* __restrict__ counter, uint64_t out_cap) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < cap; i += (uint64_t)gridDim.x * blockDim.x) {
    const unsigned long long k = h.keys[2 * i];
    if ((uint32_t)(h.keys[2 * i + 1] >> 32) != h.gen) continue;   // free in this batch
    const uint32_t o = atomicAdd(counter, 1u);
    if (o < out_cap) { keys[o] = k; vals[o] = *hash_val(h, (uint32_t)i); }
  }
}

__global__ void k_hash_merge(Hash h, uint32_t* ctrl, const unsigned long long* __restrict__ keys,
                             const uint32_t* __restrict__ vals, uint64_t count) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count; i += (uint64_t)gridDim.x * blockDim.x) {
    const unsigned long long k = keys[i];
    if (k == EMPTY64) continue;
    if (!hash_min(h, ctrl + h.used_slot, k, vals[i])) atomicOr(ctrl + C_OVF, 1u);
  }
}

// ---- launch helpers (host) ----------------------------------------------------------------
static int g_sms = 0;

static int sm_count() {
  if (!g_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev);
  }
  return g_sms;
}

template <typename K>
static int grid_for(K kernel, size_t smem) {
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, BLOCK, smem);
  if (per_sm < 1) per_sm = 1;
  return per_sm * sm_count();
}

constexpr int SMEM_MAX = 227 * 1024;

static bool staged_fits(const World& W) {
  return fits_fixed(W) && make_layout(W, true, false).total <= (uint32_t)SMEM_MAX &&
         make_layout(W, true, true).total <= (uint32_t)SMEM_MAX;
}

// the row-table passes (fx_passes.cuh): fixed layout and at most one range base per skip slot
static bool fx_fits(const World& W) {
  return staged_fits(W) && W.exact1 && W.n_skip + 1 <= FX_SKIP && W.n_pages < (1ull << 30);
}

template <bool kStaged>
static void set_attrs() {
  static bool done = false;
  if (done) return;
  const int mx = SMEM_MAX;
  cudaFuncSetAttribute(k_scan<kStaged>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
  cudaFuncSetAttribute(k_general<kStaged, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
  cudaFuncSetAttribute(k_general<kStaged, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
  cudaFuncSetAttribute(k_finalize<kStaged>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
  cudaFuncSetAttribute(k_resolve_general, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
  cudaFuncSetAttribute(fx::k_scan_fx<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
  cudaFuncSetAttribute(fx::k_scan_fx<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
  cudaFuncSetAttribute(fx::k_finalize_fx<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
  cudaFuncSetAttribute(fx::k_finalize_fx<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
  done = true;
}

static int ok_or_err() { return cudaGetLastError() == cudaSuccess ? 0 : -1; }

// Launch with programmatic stream serialization (the kernel may start while the previous one
// on the stream drains; it waits with griddepcontrol.wait before reading its inputs).
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
  cudaLaunchKernelEx(&cfg, k, args...);
}

// at least one 64-entry chunk per warp
static int clamp_grid(int g, uint64_t n) {
  const uint64_t per_block = (uint64_t)WCHUNK * WARPS;
  const uint64_t need = (n + per_block - 1) / per_block;
  return (uint64_t)g > need ? (int)need : g;
}



template <bool kStaged>
static int scan_t(const World& W, const Scratch& S, const mpsf_fault_entry* in, uint64_t n, const Params& P,
                  unsigned long long* counts, cudaStream_t st, const Marker& mk) {
  set_attrs<kStaged>();
  if (n == 0) return 0;
  if (kStaged && fx_fits(W)) {
    auto* k = W.dd_groups == 1 ? fx::k_scan_fx<true> : fx::k_scan_fx<false>;
    const int g = clamp_grid(grid_for(k, fx::SCAN_BYTES), n);
    launch_pdl(k, dim3(g), dim3(BLOCK), fx::SCAN_BYTES, st, W, S, in, n, P, counts);
    mk.mark("k_scan");
    return ok_or_err();
  }
  const uint32_t smem = make_layout(W, kStaged, false).total;
  int g = grid_for(k_scan<kStaged>, smem);
  if (kStaged && g > (int)(2 * sm_count())) g = 2 * sm_count();
  g = clamp_grid(g, n);
  launch_pdl(k_scan<kStaged>, dim3(g), dim3(BLOCK), smem, st, W, S, in, n, P, counts);
  mk.mark("k_scan");
  return ok_or_err();
}

template <bool kStaged>
static int general_t(const World& W, const Scratch& S, const mpsf_fault_entry* in, uint64_t n, const Params& P,
                     int stage, cudaStream_t st, const Marker& mk) {
  set_attrs<kStaged>();
  if (n == 0) return 0;
  const uint32_t smem = make_layout(W, kStaged, true).total;
  int g = clamp_grid(grid_for(k_general<kStaged, 1>, smem), n);
  if (stage == 1) {
    launch_pdl(k_general<kStaged, 1>, dim3(g), dim3(BLOCK), smem, st, W, S, in, n, P);
    mk.mark("k_general1");
  } else {
    launch_pdl(k_general<kStaged, 2>, dim3(g), dim3(BLOCK), smem, st, W, S, in, n, P);
    mk.mark("k_general2");
  }
  return ok_or_err();
}

template <bool kStaged>
static int finalize_t(const World& W, const Scratch& S, const mpsf_fault_entry* in, uint64_t n, const Params& P,
                      mpsf_out_record* out, uint64_t q_base, cudaStream_t st, const Marker& mk) {
  set_attrs<kStaged>();
  if (n == 0) return 0;
  if (kStaged && fx_fits(W)) {
    auto* k = W.dd_groups == 1 ? fx::k_finalize_fx<true> : fx::k_finalize_fx<false>;
    const int g = clamp_grid(grid_for(k, fx::FIN_BYTES), n);
    launch_pdl(k, dim3(g), dim3(BLOCK), fx::FIN_BYTES, st, W, S, n, P, out, q_base);
    mk.mark("k_finalize");
    return ok_or_err();
  }
  const uint32_t smem = make_layout(W, kStaged, true).total;
  const int g = clamp_grid(grid_for(k_finalize<kStaged>, smem), n);
  launch_pdl(k_finalize<kStaged>, dim3(g), dim3(BLOCK), smem, st, W, S, in, n, P, out, q_base);
  mk.mark("k_finalize");
  return ok_or_err();
}

uint32_t chunk_entries() { return (uint32_t)WCHUNK; }
uint64_t chunks_for(uint64_t n) { return (n + WCHUNK - 1) / WCHUNK; }
uint64_t segments_for(uint64_t n) { return (chunks_for(n) + SEG_CHUNKS - 1) / SEG_CHUNKS; }

int launch_scan(const World& W, const Scratch& S, const mpsf_fault_entry* in, uint64_t n, const Params& P,
                unsigned long long* counts, cudaStream_t st, const Marker& mk) {
  return staged_fits(W) ? scan_t<true>(W, S, in, n, P, counts, st, mk)
                        : scan_t<false>(W, S, in, n, P, counts, st, mk);
}

int launch_resolve(const World& W, const Scratch& S, const Params& P, mpsf_client_verdict* verdict,
                   cudaStream_t st, const Marker& mk) {
  launch_pdl(k_resolve, dim3(1), dim3(256), 0, st, W, S, P, verdict);
  mk.mark("k_resolve");
  return ok_or_err();
}

int launch_general(const World& W, const Scratch& S, const mpsf_fault_entry* in, uint64_t n, const Params& P,
                   int stage, cudaStream_t st, const Marker& mk) {
  return staged_fits(W) ? general_t<true>(W, S, in, n, P, stage, st, mk)
                        : general_t<false>(W, S, in, n, P, stage, st, mk);
}

bool resolve_fused_fits(const World& W) { return fx_fits(W); }

int launch_resolve_general(const World& W, const Scratch& S, const mpsf_fault_entry* in, uint64_t n, const Params& P,
                           mpsf_client_verdict* verdict, cudaStream_t st, const Marker& mk) {
  set_attrs<true>();
  const uint32_t smem = make_layout(W, true, true).total;
  const int g = clamp_grid(grid_for(k_resolve_general, smem), n);
  launch_pdl(k_resolve_general, dim3(g), dim3(BLOCK), smem, st, W, S, in, n, P, verdict);
  mk.mark("k_resolve_general");
  return ok_or_err();
}

int launch_resolve2(const World& W, const Scratch& S, const Params& P, cudaStream_t st, const Marker& mk) {
  launch_pdl(k_resolve2, dim3(1), dim3(256), 0, st, W, S, P);
  mk.mark("k_resolve2");
  return ok_or_err();
}

int launch_finalize(const World& W, const Scratch& S, const mpsf_fault_entry* in, uint64_t n, const Params& P,
                    mpsf_out_record* out, uint64_t q_base, cudaStream_t st, const Marker& mk) {
  return staged_fits(W) ? finalize_t<true>(W, S, in, n, P, out, q_base, st, mk)
                        : finalize_t<false>(W, S, in, n, P, out, q_base, st, mk);
}

// cancel list + dedup set + the batch summary (k_summary alone when there is nothing to list)
int launch_lists(const Scratch& S, const mpsf_fault_entry* in, const mpsf_out_record* out, uint64_t n,
                 uint64_t base_index, unsigned long long* dkeys, uint32_t* didx, uint32_t* cancel, DevSummary* sum,
                 cudaStream_t st, const Marker& mk) {
  const uint64_t nseg = segments_for(n);
  if (nseg == 0) {
    launch_pdl(k_summary, dim3(1), dim3(1024), 0, st, S, (uint64_t)0, sum);
    mk.mark("k_summary");
    return ok_or_err();
  }
  const bool prescan = nseg > 2048;
  if (prescan) {
    launch_pdl(k_seg_scan, dim3(1), dim3(1024), 0, st, S, nseg);
    mk.mark("k_seg_scan");
  }
  launch_pdl(k_lists, dim3((unsigned)nseg), dim3(SEG_CHUNKS), 0, st, S, in, out, chunks_for(n), base_index, dkeys,
             didx, cancel, sum, prescan);
  mk.mark("k_lists");
  return ok_or_err();
}

// The lists of a batch straight into (device-mapped) pinned host buffers; the lengths are read
// from the segment counters on the device, so the host never waits for them.
__global__ void k_copyout(Scratch S, uint64_t nseg, const unsigned long long* __restrict__ d_dk,
                          const uint32_t* __restrict__ d_di, const uint32_t* __restrict__ d_ca,
                          unsigned long long* h_dk, uint32_t* h_di, uint32_t* h_ca) {
  pdl_wait();
  __shared__ unsigned long long s_tot;
  if (threadIdx.x == 0) s_tot = 0;
  __syncthreads();
  if (__ldcg(S.ctrl + C_ERR) != 0) return;
  unsigned long long acc = 0;
  for (uint64_t i = threadIdx.x; i < nseg; i += blockDim.x) acc += __ldcg(S.segcnt + i);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xFFFFFFFFu, acc, o);
  if ((threadIdx.x & 31) == 0 && acc) atomicAdd(&s_tot, acc);
  __syncthreads();
  const uint64_t nc = s_tot & 0xFFFFFFFFull, nd = s_tot >> 32;
  const uint64_t T = (uint64_t)gridDim.x * blockDim.x, t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (uint64_t i = t; i < nd; i += T) { h_dk[i] = __ldcs(d_dk + i); h_di[i] = __ldcs(d_di + i); }
  for (uint64_t i = t; i < nc; i += T) h_ca[i] = __ldcs(d_ca + i);
}

int launch_copyout(const Scratch& S, uint64_t n, const unsigned long long* d_dk, const uint32_t* d_di,
                   const uint32_t* d_ca, unsigned long long* h_dk, uint32_t* h_di, uint32_t* h_ca, cudaStream_t st) {
  launch_pdl(k_copyout, dim3(2 * sm_count()), dim3(512), 0, st, S, segments_for(n), d_dk, d_di, d_ca, h_dk, h_di,
             h_ca);
  return ok_or_err();
}

// ---- sparse exchange of page-sized minima tables (multi-GPU round 1b) ---------------------
// The dense dedup slots / first-eligible page keys of a large world are mostly EMPTY: a rank
// compacts its non-empty words to (index, value) pairs (warp-aggregated append), the ranks
// all-gather the pairs and each merges the others' with an atomic MIN -- the same minima as a
// dense all-reduce, moving O(keys) instead of O(pages) bytes.
__global__ void k_sparse_export(const uint32_t* __restrict__ buf, uint64_t count, uint32_t* __restrict__ idx,
                                uint32_t* __restrict__ val, uint32_t* __restrict__ counter, uint64_t cap) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i0 = (uint64_t)blockIdx.x * blockDim.x; i0 < count; i0 += stride) {
    const uint64_t i = i0 + threadIdx.x;
    const uint32_t v = i < count ? __ldcs(buf + i) : EMPTY32;
    const bool has = v != EMPTY32;
    const unsigned m = __ballot_sync(0xFFFFFFFFu, has);
    if (!m) continue;
    uint32_t base = 0;
    if (lane == 0) base = atomicAdd(counter, (uint32_t)__popc(m));
    base = __shfl_sync(0xFFFFFFFFu, base, 0);
    if (has) {
      const uint64_t o = base + __popc(m & ((1u << lane) - 1u));
      if (o < cap) { idx[o] = (uint32_t)i; val[o] = v; }
    }
  }
}

__global__ void k_sparse_merge(uint32_t* __restrict__ buf, uint64_t count, const uint32_t* __restrict__ idx,
                               const uint32_t* __restrict__ val, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t k = idx[i];
    if (k < count) min32(buf + k, val[i]);
  }
}

int launch_sparse_export(const uint32_t* buf, uint64_t count, uint32_t* idx, uint32_t* val, uint32_t* counter,
                         uint64_t cap, cudaStream_t st) {
  if (count == 0) return 0;
  k_sparse_export<<<4 * sm_count(), 512, 0, st>>>(buf, count, idx, val, counter, cap);
  return ok_or_err();
}

int launch_sparse_merge(uint32_t* buf, uint64_t count, const uint32_t* idx, const uint32_t* val, uint64_t n,
                        cudaStream_t st) {
  if (n == 0) return 0;
  k_sparse_merge<<<4 * sm_count(), 512, 0, st>>>(buf, count, idx, val, n);
  return ok_or_err();
}

template <bool kStaged>
static void translate_attrs() {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_tr_prefetch<kStaged>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_MAX);
    cudaFuncSetAttribute(k_tr_classify<kStaged>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_MAX);
    attr = true;
  }
}

template <bool kStaged>
static int translate_prefetch_t(const World& W, const Scratch& S, const mpsf_fault_entry* in, uint64_t n,
                                const Params& P, cudaStream_t st, const Marker& mk) {
  translate_attrs<kStaged>();
  const uint32_t smem = make_layout(W, kStaged, true).total;
  const int g = clamp_grid(grid_for(k_tr_classify<kStaged>, smem), n);
  const uint32_t use_q = smem + PFQ_BYTES <= (uint32_t)SMEM_MAX ? 1u : 0u;
  launch_pdl(k_tr_prefetch<kStaged>, dim3(g), dim3(BLOCK), smem + (use_q ? PFQ_BYTES : 0u), st, W, S, in, n, P,
             use_q);
  mk.mark("k_tr_prefetch");
  return ok_or_err();
}

template <bool kStaged>
static int translate_finish_t(const World& W, const Scratch& S, const mpsf_fault_entry* in, uint64_t n,
                              const Params& P, uint8_t* hit, mpsf_fault_entry* faults, uint32_t* fault_idx,
                              uint32_t* pop_idx, DevSummary* sum, cudaStream_t st, const Marker& mk) {
  translate_attrs<kStaged>();
  const uint32_t smem = make_layout(W, kStaged, true).total;
  const int g = clamp_grid(grid_for(k_tr_classify<kStaged>, smem), n);
  launch_pdl(k_tr_classify<kStaged>, dim3(g), dim3(BLOCK), smem, st, W, S, in, n, P, hit);
  mk.mark("k_tr_classify");
  const uint64_t nseg = segments_for(n);
  launch_pdl(k_tr_lists, dim3((unsigned)nseg), dim3(SEG_CHUNKS), 0, st, S, in, chunks_for(n), (uint64_t)P.base_index,
             faults, fault_idx, pop_idx, sum);
  mk.mark("k_tr_lists");
  return ok_or_err();
}

// Phase 1 of a batched translation: the first PREFETCH per managed page (S.pf, global
// indices -- shards combine it with a MIN before phase 2).
int launch_translate_prefetch(const World& W, const Scratch& S, const mpsf_fault_entry* in, uint64_t n,
                              const Params& P, cudaStream_t st, const Marker& mk) {
  if (n == 0) return 0;
  return staged_fits(W) ? translate_prefetch_t<true>(W, S, in, n, P, st, mk)
                        : translate_prefetch_t<false>(W, S, in, n, P, st, mk);
}

// Phase 2: hit / miss per access against S.pf, the ordered miss and population lists.
int launch_translate_finish(const World& W, const Scratch& S, const mpsf_fault_entry* in, uint64_t n,
                            const Params& P, uint8_t* hit, mpsf_fault_entry* faults, uint32_t* fault_idx,
                            uint32_t* pop_idx, DevSummary* sum, cudaStream_t st, const Marker& mk) {
  if (n == 0) {
    launch_pdl(k_summary, dim3(1), dim3(1024), 0, st, S, (uint64_t)0, sum);
    return ok_or_err();
  }
  return staged_fits(W) ? translate_finish_t<true>(W, S, in, n, P, hit, faults, fault_idx, pop_idx, sum, st, mk)
                        : translate_finish_t<false>(W, S, in, n, P, hit, faults, fault_idx, pop_idx, sum, st, mk);
}

// ---- batched top half: faults.classify + MemoryModel.range_at per entry -----------------------
// raise_mmu_fault's classification of every entry (pipeline.py:103-104, faults.py:134-171,
// memory.py:233-237): the scenario id (0xFF: entry skipped) and the rid of the range the VA is in
// (NO_RID: none).  The same decode and LUT as the fault path; errors raise the same status bits.
template <bool kStaged>
__global__ void __launch_bounds__(BLOCK, 1) k_classify(World W, Scratch S, const mpsf_fault_entry* __restrict__ in,
                                                       uint64_t n, Params P, uint8_t* __restrict__ sid_out,
                                                       uint32_t* __restrict__ rid_out) {
  extern __shared__ __align__(128) uint8_t smem[];
  pdl_trigger();
  const Layout L = make_layout(W, kStaged, true);
  const View v = setup<kStaged>(smem, L, W, S, false, true, true);
  __syncthreads();
  pdl_wait();
  const uint32_t lane = threadIdx.x & 31, base = (uint32_t)P.base_index;
  ldg_stream(in, n, [&](uint4 e0, uint32_t i0, bool ok0, uint4 e1, uint32_t i1, bool ok1) {
    if (!ok0) e0.w = 0;
    if (!ok1) e1.w = 0;
    const Dec d0 = decode_fast(v.T, W.page_state, S, e0, base + i0, lane);
    const Dec d1 = decode_fast(v.T, W.page_state, S, e1, base + i1, lane);
    const uint32_t s0 = d0.f ? (d0.f & LF_S) : 0xFFu, s1 = d1.f ? (d1.f & LF_S) : 0xFFu;
    const uint32_t r0 = (d0.f && d0.inr) ? v.T.rrid[d0.ridx] : NO_RID, r1 = (d1.f && d1.inr) ? v.T.rrid[d1.ridx] : NO_RID;
    if (ok1 && ((i0 & 1u) == 0)) {
      *reinterpret_cast<uint16_t*>(sid_out + i0) = (uint16_t)(s0 | (s1 << 8));
      __stcs(reinterpret_cast<uint2*>(rid_out + i0), make_uint2(r0, r1));
    } else {
      if (ok0) { sid_out[i0] = (uint8_t)s0; rid_out[i0] = r0; }
      if (ok1) { sid_out[i1] = (uint8_t)s1; rid_out[i1] = r1; }
    }
  });
}

template <bool kStaged>
static int classify_t(const World& W, const Scratch& S, const mpsf_fault_entry* in, uint64_t n, const Params& P,
                      uint8_t* sid, uint32_t* rid, DevSummary* sum, cudaStream_t st, const Marker& mk) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_classify<kStaged>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_MAX);
    attr = true;
  }
  if (n) {
    const uint32_t smem = make_layout(W, kStaged, true).total;
    const int g = clamp_grid(grid_for(k_classify<kStaged>, smem), n);
    launch_pdl(k_classify<kStaged>, dim3(g), dim3(BLOCK), smem, st, W, S, in, n, P, sid, rid);
    mk.mark("k_classify");
  }
  launch_pdl(k_summary, dim3(1), dim3(1024), 0, st, S, (uint64_t)0, sum);
  return ok_or_err();
}

int launch_classify(const World& W, const Scratch& S, const mpsf_fault_entry* in, uint64_t n, const Params& P,
                    uint8_t* sid, uint32_t* rid, DevSummary* sum, cudaStream_t st, const Marker& mk) {
  return staged_fits(W) ? classify_t<true>(W, S, in, n, P, sid, rid, sum, st, mk)
                        : classify_t<false>(W, S, in, n, P, sid, rid, sum, st, mk);
}

int launch_translate(const World& W, const Scratch& S, const mpsf_fault_entry* in, uint64_t n, const Params& P,
                     uint8_t* hit, mpsf_fault_entry* faults, uint32_t* fault_idx, uint32_t* pop_idx, DevSummary* sum,
                     cudaStream_t st, const Marker& mk) {
  if (launch_translate_prefetch(W, S, in, n, P, st, mk)) return -1;
  return launch_translate_finish(W, S, in, n, P, hit, faults, fault_idx, pop_idx, sum, st, mk);
}

int launch_hash_export(const Hash& h, uint64_t cap, unsigned long long* keys, uint32_t* vals, uint32_t* counter,
                       uint64_t out_cap, cudaStream_t st) {
  k_hash_export<<<2 * sm_count(), 256, 0, st>>>(h, cap, keys, vals, counter, out_cap);
  return ok_or_err();
}

int launch_hash_merge(const Hash& h, uint32_t* ctrl, const unsigned long long* keys, const uint32_t* vals,
                      uint64_t count, cudaStream_t st) {
  if (count == 0) return 0;
  k_hash_merge<<<2 * sm_count(), 256, 0, st>>>(h, ctrl, keys, vals, count);
  return ok_or_err();
}


}  // namespace mpsf
