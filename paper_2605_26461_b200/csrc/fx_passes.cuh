// Streaming passes for worlds within the fixed shared-memory layout (the common case: every
// BASELINE config).  Included by fault_kernels.cu after its helpers.
//
// Same computation as scan_fast / finalize_phase (rules C0-C9 of SURVEY.md Appendix C; the
// reference semantics they restate are cited there), laid out for instruction count -- both
// passes are issue-bound -- rather than generality:
//  * the world tables are rows read with one shared load per step: channel row (client word,
//    skip-table span / shift / offset) replicated 8x so a quarter-warp's 16-byte loads never
//    share a bank group; skip slot {range at the slot start, base of the next range inside the
//    slot}; range row {base, end, page-state slot, attributes}.  Attribution
//    (MemoryModel.range_at, memory.py:233-237) is three dependent loads, no loop, no compare
//    against a second row;
//  * one classification LUT indexed by (min(engine, 3), min(access, 3), range class, page state)
//    also rejects bad engine / access values;
//  * the pass-1 record carries exactly what pass 2 indexes with (scenario, dedup group,
//    mechanism class, location, channel engine, client, range index | page high bits, page slot |
//    page low bits) plus one "known duplicate" bit: pass 1 already saw a smaller index on the
//    entry's dedup slot, so pass 2 needs no dedup lookup for it unless its cancel flag depends on
//    the representative's index.
namespace fx {

constexpr uint32_t NCH = FX_CH + 1;            // channel rows (the last: invalid channel)
constexpr uint32_t CH_COPIES = 8;              // replicas of a channel row (one per quarter-warp lane)
constexpr uint32_t LUT2_XK = 16 * 16 * 8;      // [min(eng,3) * 4 + min(acc,3)][range class][state]
constexpr uint32_t LUT2_N = LUT2_XK + 16;      // + the non-translation kinds
// (not replicated per lane: a batch hits few distinct LUT words, which a single copy serves as
// broadcasts; 8 replicas made k_scan 1.2 -> 2.1 ms at config 3 -- profiles/r02/ab_lut_replicas.txt)

__host__ __device__ constexpr uint32_t a16(uint32_t x) { return (x + 15u) & ~15u; }

// shared-memory layout (fixed offsets: every table access is an immediate-offset load)
constexpr uint32_t O_LUT = 0;
constexpr uint32_t O_SLUT = a16(O_LUT + 4 * LUT2_N);
constexpr uint32_t O_CHAN = a16(O_SLUT + 4 * 32);
constexpr uint32_t O_SKIP = O_CHAN + NCH * CH_COPIES * 16;
constexpr uint32_t O_ROWS = O_SKIP + FX_SKIP * 8;
constexpr uint32_t O_PASS = O_ROWS + FX_R * 16;
// pass 1
constexpr uint32_t O_QUEUE = O_PASS;
constexpr uint32_t O_C64 = O_QUEUE + WARPS * QCAP * 16;
constexpr uint32_t O_ISO = a16(O_C64 + 8 * (3 * FX_C + 2));
constexpr uint32_t O_R32 = O_ISO + 4 * 3 * FX_C * 32;
constexpr uint32_t O_CNT = O_R32 + 4 * 2 * FX_R;
constexpr uint32_t O_USED = O_CNT + 4 * NSCEN * FX_C;
constexpr uint32_t SCAN_BYTES = O_USED + 16;
// pass 2 (its own layout: it needs neither the classification LUT nor the channel / skip tables)
constexpr uint32_t RID_COPIES = 8;             // replicas of the rid table (one per quarter-warp lane)
constexpr uint32_t F_DLUT = 0;                                     // [3 epoch bands][1024 classes] uint2
constexpr uint32_t F_SLUT = F_DLUT + 3 * 1024 * 8;
constexpr uint32_t F_ROWS = F_SLUT + 128;
constexpr uint32_t F_CROW = F_ROWS + FX_R * 16;                    // [(client, engine)][8 copies] uint4
constexpr uint32_t F_TRAP = F_CROW + FX_C * 4 * CH_COPIES * 16;    // [client] applied trap
constexpr uint32_t F_RRID = F_TRAP + 4 * FX_C;                     // [range][8 copies]
constexpr uint32_t F_EXT = F_RRID + 4 * FX_R * RID_COPIES;
constexpr uint32_t F_NR0 = F_EXT + 4 * FX_R;
constexpr uint32_t F_SLOWQ = F_NR0 + 4 * FX_R;
constexpr uint32_t FIN_BYTES = F_SLOWQ + WARPS * 96 * 16;
static_assert(SCAN_BYTES <= 227 * 1024 && FIN_BYTES <= 227 * 1024, "fixed layout exceeds shared memory");

__device__ __forceinline__ uint32_t lut2_word(uint32_t idx, bool isolation) {
  if (idx >= LUT2_XK) return lut_word((int)(LUT_XK + (idx - LUT2_XK)), isolation);
  const uint32_t st = idx & 7, rcls = (idx >> 3) & 15, e = idx >> 9, a = (idx >> 7) & 3;
  if (e > 2 || a > 2) return LF_VALID | LF_BAD;
  return lut_word((int)(((e * 3 + a) * 16 + rcls) * 8 + st), isolation);
}

// predicated L2 load (no branch): dflt when p is false
__device__ __forceinline__ uint32_t ldcg_if(bool p, const uint32_t* a, uint32_t dflt) {
  uint32_t v;
  asm("{.reg .pred q; setp.ne.u32 q, %2, 0; mov.b32 %0, %3; @q ld.global.cg.u32 %0, [%1];}"
      : "=r"(v) : "l"(a), "r"((uint32_t)p), "r"(dflt));
  return v;
}

// World tables into shared memory (both passes).
__device__ __forceinline__ void stage_tables(uint8_t* sm, const World& W, bool isolation) {
  const uint32_t tid = threadIdx.x, nb = blockDim.x;
  uint32_t* lut = reinterpret_cast<uint32_t*>(sm + O_LUT);
  for (uint32_t i = tid; i < LUT2_N; i += nb) lut[i] = lut2_word(i, isolation);
  uint32_t* slut = reinterpret_cast<uint32_t*>(sm + O_SLUT);
  if (tid < 32) slut[tid] = scen_word((int)tid, isolation);
  uint4* ch = reinterpret_cast<uint4*>(sm + O_CHAN);
  const uint32_t nch1 = W.n_channels + 1;
  for (uint32_t i = tid; i < nch1 * CH_COPIES; i += nb) ch[i] = __ldg(W.chan4 + i / CH_COPIES);
  uint2* sk = reinterpret_cast<uint2*>(sm + O_SKIP);
  for (uint32_t i = tid; i <= W.n_skip; i += nb) sk[i] = __ldg(W.skip2 + i);
  uint4* rows = reinterpret_cast<uint4*>(sm + O_ROWS);
  for (uint32_t i = tid; i <= W.n_ranges; i += nb) rows[i] = __ldg(W.row4 + i);
}

// Decoded entry.  f = LUT word (0: skipped or malformed -- the error bits are raised here).
struct D {
  uint32_t f, cw, page, slot, k;
  bool inr, grd;
};

__device__ __forceinline__ D decode(const uint8_t* sm, const uint8_t* __restrict__ ps, uint32_t nch, uint32_t copy16,
                                    const Scratch& S, uint4 e, uint32_t gidx) {
  D d;
  const uint32_t w3 = e.w, ek = (w3 >> 16) & 0xFFu;
  const uint32_t ch = min(e.z, nch);
  const uint4 cr = *reinterpret_cast<const uint4*>(sm + O_CHAN + ch * (CH_COPIES * 16) + copy16);
  d.page = __funnelshift_r(e.x, e.y, 12);
  const uint32_t j = min((d.page - cr.y) >> cr.z, cr.w >> 16);
  const uint2 sk = reinterpret_cast<const uint2*>(sm + O_SKIP)[(cr.w & 0xFFFFu) + j];
  d.k = sk.x + (d.page >= sk.y ? 1u : 0u);
  const uint4 row = reinterpret_cast<const uint4*>(sm + O_ROWS)[d.k];
  // translation entries below 2^44 - 4 KiB look their range up (no range reaches higher)
  const bool look = (ek == 0) & (e.y < 0x1000u) & (d.page != 0xFFFFFFFFu);
  d.inr = look & (d.page >= row.x) & (d.page < row.y);
  d.grd = look & (d.page == row.y);
  d.slot = row.z + (d.page - row.x);
  const bool pp = d.inr & ((row.w & ROW_PERPAGE) != 0);
  const uint32_t pst = pp ? ps[d.slot] : row.w;                 // per-page state byte, else the uniform one
  // LUT index: [engine][access][range class][state] (engine / access 3 -> a BAD word, > 3 caught
  // below), or the kind
  const uint32_t eng = w3 & 0xFFu;
  const bool ea_bad = (w3 & 0xFCFCu) != 0;
  const uint32_t ea = ((w3 & 3u) << 9) | ((w3 & 0x300u) >> 1);
  const uint32_t t = d.inr ? ((row.w & 0x38u) | (pst & 7u)) : 64u;
  const uint32_t idx = ek == 0 ? ea + t : LUT2_XK + min(ek, 15u);
  const uint32_t f = reinterpret_cast<const uint32_t*>(sm + O_LUT)[idx];
  d.cw = cr.x;
  const uint32_t ceng = (cr.x >> 16) & 3u;
  const bool tbad = (ek == 0) & (ea_bad | (eng != ceng) | (e.y >= (1u << 21)));
  const bool bad = !(cr.x & CH_VALID) | ((f & LF_BAD) != 0) | tbad;
  const bool valid = (w3 >> 24) & MPSF_ENTRY_VALID;
  // malformed entry (never in a valid trace): a warp-uniform test keeps the common path free of
  // a divergent branch
  if (__any_sync(0xFFFFFFFFu, valid && bad) && valid && bad) {
    const uint32_t bit = !(cr.x & CH_VALID) ? EB_NO_CHANNEL
                         : (((f & LF_BAD) != 0) | ((ek == 0) & ea_bad)) ? EB_BAD_ENTRY
                         : (eng != ceng ? EB_MISMATCH : EB_VA);
    raise_err(S, bit, gidx);
  }
  d.f = (valid & !bad) ? f : 0u;
  return d;
}

// pass-1 record: lo = scenario [4:0] | location [7:5] (L_*) | known duplicate [8] | non-replayable
// [9] | dedup group [12:10] | channel engine [14:13] | client [20:15] | range index, or page bits
// 32.. of a wild page, [31:21];  hi = page-state slot (in range / guard) or page bits 0..31.
// lo[9:0] is the entry's class: pass 2 indexes its decision LUT with it directly.
constexpr uint32_t L_SKIP = 0, L_INM = 1, L_INX = 2, L_GRD = 3, L_NONE = 4;   // in a managed / external range
constexpr uint32_t R_KDUP = 1u << 8;
__device__ __forceinline__ uint32_t rec_client(uint32_t lo) { return (lo >> 15) & 63u; }
__device__ __forceinline__ uint32_t rec_ceng(uint32_t lo) { return (lo >> 13) & 3u; }
__device__ __forceinline__ uint32_t rec_group(uint32_t lo) { return (lo >> 10) & 7u; }
__device__ __forceinline__ uint32_t rec_loc(uint32_t lo) { return (lo >> 5) & 7u; }
__device__ __forceinline__ uint32_t rec_k(uint32_t lo) { return lo >> 21; }

// entries per lane per step of pass 1 (4 measured: k_scan 1.27 -> 1.87-2.24 ms at config 3 for
// 512-1024-thread CTAs -- register spills / fewer warps; profiles/r02/ab_entries_per_lane.txt)
constexpr int EPL = 2;

// Entry stream of pass 1: warp w of the grid owns steps w, w + W, ... of 32 * EPL entries; lane l
// reads its EPL adjacent entries (32-byte non-allocating loads), the next step's requested before
// the current one is processed.
template <int N, typename F>
__device__ __forceinline__ void stream_n(const mpsf_fault_entry* in, uint64_t n64, F&& fn) {
  constexpr uint32_t CH = 32 * N;
  const uint32_t n = (uint32_t)n64;   // < MAX_GIDX
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t gw = blockIdx.x * (blockDim.x >> 5) + warp, GW = gridDim.x * (blockDim.x >> 5);
  const uint32_t nch = (n + CH - 1) / CH;
  const bool a32 = ((uintptr_t)in & 31u) == 0;
  uint4 nx[N];
  auto load = [&](uint32_t c) {
#pragma unroll
    for (int u = 0; u < N; u += 2) ld_pair(in, n, c * CH + N * lane + u, a32, nx[u], nx[u + 1]);
  };
  if (gw < nch) load(gw);
  for (uint32_t c = gw; c < nch; c += GW) {
    uint4 e[N];
#pragma unroll
    for (int u = 0; u < N; ++u) e[u] = nx[u];
    if (c + GW < nch) load(c + GW);
    fn(e, c * CH + N * lane);
  }
}

// Pass 1 over [0, n) (global index P.base_index + i).  As pass 2, the common path has no
// data-dependent branch: the block-local minima and counts are predicated shared-memory
// reductions, the global pre-check loads and minima predicated accesses; the work a warp would
// otherwise serialise on -- wild-page hash inserts and claimed-slot CAS claims -- goes to the
// per-warp queue, drained 32 operations at a time.  Traps and fatal reports (rare) keep a branch.
__device__ __forceinline__ void q_exec(const Scratch& S, uint32_t* used, const QOp& x) {
  const uint32_t t = x.tab & 3u;
  if (t == 2) {                                  // claimed-slot dedup (sparse worlds)
    uint32_t* slot = S.dd + (x.tab >> 2);
    claim_resolve(S, used, slot, x.val, __ldcg(slot), x.key);
  } else if (!hash_min(t ? S.hnr : S.hdd, used + t, x.key, x.val)) {
    atomicOr(S.ctrl + C_OVF, 1u);
  }
}

template <bool kSparse>
__device__ __forceinline__ void scan_body(const World& W, const Scratch& S, uint8_t* sm,
                                          const mpsf_fault_entry* __restrict__ in, uint64_t n, const Params& P) {
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t copy16 = (lane & (CH_COPIES - 1)) * 16;
  const uint32_t C = W.n_clients, nch = W.n_channels;
  const uint32_t base = (uint32_t)P.base_index;
  // claimed page slots (one per page, no first-eligible table) or dense (page, group) slots
  constexpr uint32_t G = kSparse ? 1u : 5u, gmask = kSparse ? 0u : 7u;
  uint32_t* counts = reinterpret_cast<uint32_t*>(sm + O_CNT);
  // per-warp copies of the per-(mechanism class, client) minima, one row per warp: a warp's lanes
  // spread over the banks (a column-per-warp layout put every lane of a warp on one bank)
  uint32_t* iso = reinterpret_cast<uint32_t*>(sm + O_ISO) + warp * (3 * FX_C);
  uint32_t* r32 = reinterpret_cast<uint32_t*>(sm + O_R32);
  uint32_t* used = reinterpret_cast<uint32_t*>(sm + O_USED);
  unsigned long long* c64 = reinterpret_cast<unsigned long long*>(sm + O_C64);
  QOp* q = reinterpret_cast<QOp*>(sm + O_QUEUE) + warp * QCAP;
  unsigned long long* const drec = S.drec + (P.base_index - S.drec_base);
  const uint8_t* __restrict__ ps = W.page_state;
  uint32_t* const nrall = S.nrall;   // present iff !kSparse
  struct O {
    uint32_t* pd; uint32_t vd;     // dedup slot and its value
    uint32_t* pa;                  // first eligible record of the page (dense worlds)
    uint32_t ok;
    bool p_dd, p_a, qn, qd;        // predicates: dedup slot, nrall; wild NR / dedup hash ops
    uint32_t lo, hi;               // record
    uint64_t page;
  };
  // per entry, in two halves: (a) decode and the addresses of the global pre-check loads (both
  // entries' loads are issued before either entry's shared-memory work, which covers them);
  // (b) counts, block-local minima, the record
  auto first = [&](uint4 e, uint32_t gidx, O& o, D& d) {
    d = decode(sm, ps, nch, copy16, S, e, gidx);
    const uint32_t f = d.f;
    o.ok = ((f & LF_REPL) ? 0u : 0x80000000u) | gidx;
    const bool elig = (f & LF_ELIG) != 0;
    const bool inw = d.inr | d.grd;
    o.p_a = elig & d.inr & !kSparse;
    o.pa = nrall + d.slot;
    const bool dd = (f & LF_DD) != 0;
    const uint32_t group = (f >> LF_GROUP_SH) & 7u;
    o.p_dd = dd & inw;
    o.pd = S.dd + (d.slot * G + (group & gmask));
    o.vd = (gidx << 3) | group;
  };
  auto second = [&](uint4 e, uint32_t gidx, O& o, const D& d) {
    const uint32_t f = d.f, c = d.cw & 0xFFFFu, sid = f & LF_S;
    red_add_s(f != 0, counts + (f ? c * NSCEN + sid : 0u));
    if (__any_sync(0xFFFFFFFFu, f & (LF_TRAP | LF_FATAL)) && (f & (LF_TRAP | LF_FATAL))) {   // rare: traps, fatal reports
      const bool sa = (d.cw >> 18) & 1u;
      const uint32_t ceng = (d.cw >> 16) & 3u;
      if (f & LF_TRAP) {
        smin64(sa ? c64 + 2 * C + c : c64 + 3 * C + 1, ((unsigned long long)gidx << 8) | sid);
      } else {
        smin64(sa ? c64 + C + c : (ceng == 1 ? c64 + c : c64 + 3 * C), ((unsigned long long)o.ok << 8) | sid);
      }
    }
    const bool elig = (f & LF_ELIG) != 0;
    const uint32_t m = (f >> LF_M_SH) & 3u;
    const bool inw = d.inr | d.grd;
    min_s_if(elig, iso + (m * C + c), o.ok);
    min_s_if(elig & (d.grd | (d.inr & (m == 2))), r32 + (d.grd ? FX_R : 0u) + d.k, o.ok);
    const bool dd = (f & LF_DD) != 0;
    o.qn = elig & !inw;
    o.qd = dd & !inw;
    const uint32_t loc = f ? (d.inr ? m : (d.grd ? L_GRD : L_NONE)) : L_SKIP;   // in range: m is 1 or 2
    const uint32_t pagehi = (e.y >> 12) & 0x7FFu;
    o.lo = (f & 31u) | (loc << 5) | ((f & LF_REPL) ? 0u : 0x200u) | ((f & 0xE0u) << 5) | ((d.cw >> 3) & 0x6000u) |
           ((c & 63u) << 15) | ((inw ? d.k : pagehi) << 21);
    o.hi = inw ? d.slot : d.page;
    o.page = (uint64_t)d.page | ((uint64_t)pagehi << 32);
  };
  auto key_of = [&](const O& o) {     // the entry's dedup key
    return dedup_key(rec_client(o.lo), (int)rec_ceng(o.lo), (int)(o.lo & 31u), o.page);
  };
  // wild-page hash operations: appended to the warp's queue (ballot ranks; the warp-uniform count
  // lives in a register), executed 32 at a time by the whole warp.  The count stays below 32
  // before each append, so an append (<= 32 operations) never overflows QCAP = 64.
  const uint32_t lt = (1u << lane) - 1u;
  uint32_t qn = 0;
  auto push = [&](bool has, unsigned long long key, uint32_t val, uint32_t tab) {
    const uint32_t m = __ballot_sync(0xFFFFFFFFu, has);
    if (!m) return;
    if (qn >= 32) {
      __syncwarp();
      q_exec(S, used, q[qn - 32 + lane]);
      qn -= 32;
      __syncwarp();
    }
    if (has) {
      QOp x; x.key = key; x.val = val; x.tab = tab;
      q[qn + __popc(m & lt)] = x;
    }
    qn += __popc(m);
  };
  stream_n<EPL>(in, n, [&](const uint4* e, uint32_t i0) {
    O o[EPL];
    D d[EPL];
    uint32_t ra[EPL], rd[EPL];
    bool ok[EPL], kd[EPL];
#pragma unroll
    for (int u = 0; u < EPL; ++u) {
      ok[u] = i0 + u < (uint32_t)n;
      uint4 eu = e[u];
      if (!ok[u]) eu.w = 0;                            // past the end: decodes as a skipped entry
      first(eu, base + i0 + u, o[u], d[u]);
      ra[u] = ldcg_if(o[u].p_a, o[u].pa, 0u);
      rd[u] = ldcg_if(o[u].p_dd, o[u].pd, EMPTY32);
    }
#pragma unroll
    for (int u = 0; u < EPL; ++u) second(e[u], base + i0 + u, o[u], d[u]);
    unsigned long long r[EPL];
#pragma unroll
    for (int u = 0; u < EPL; ++u) {
      // a smaller index of the same key already in the slot: a duplicate whatever comes later
      kd[u] = (rd[u] != EMPTY32) & ((rd[u] & 7u) == (o[u].vd & 7u)) & (rd[u] < o[u].vd);
      r[u] = (unsigned long long)(o[u].lo | (kd[u] ? R_KDUP : 0u)) | ((unsigned long long)o[u].hi << 32);
    }
    unsigned long long* rp = drec + i0;
#pragma unroll
    for (int u = 0; u < EPL; u += 2) {
      if (ok[u + 1] && (((uintptr_t)(rp + u) & 15u) == 0)) __stcs(reinterpret_cast<ulonglong2*>(rp + u), make_ulonglong2(r[u], r[u + 1]));
      else {
        if (ok[u]) __stcs(rp + u, r[u]);
        if (ok[u + 1]) __stcs(rp + u + 1, r[u + 1]);
      }
    }
    bool any_q = false;
#pragma unroll
    for (int u = 0; u < EPL; ++u) {
      if (!kSparse) min_g_if(o[u].p_a, ra[u], o[u].pa, o[u].ok);
      // dense slots: a predicated atomic MIN; claimed slots: claim (CAS), or MIN, or the hash
      if (!kSparse) min_g_if(o[u].p_dd & !kd[u], rd[u], o[u].pd, o[u].vd);
      if (kSparse && (o[u].p_dd & !kd[u])) claim_resolve(S, used, o[u].pd, o[u].vd, rd[u], key_of(o[u]));
      any_q |= o[u].qn | o[u].qd;
    }
    if (__any_sync(0xFFFFFFFFu, any_q)) {
#pragma unroll
      for (int u = 0; u < EPL; ++u) {
        push(o[u].qn, nr_key(rec_client(o[u].lo), 0, o[u].page), o[u].ok, 1);
        push(o[u].qd, key_of(o[u]), o[u].vd >> 3, 0);
      }
    }
  });
  __syncwarp();
  if (qn >= 32) {
    q_exec(S, used, q[qn - 32 + lane]);
    qn -= 32;
  }
  __syncwarp();
  if (lane < qn) q_exec(S, used, q[lane]);
}

template <bool kSparse>
__global__ void __launch_bounds__(BLOCK, 1) k_scan_fx(World W, Scratch S, const mpsf_fault_entry* __restrict__ in,
                                                      uint64_t n, Params P, unsigned long long* __restrict__ counts) {
  extern __shared__ __align__(128) uint8_t sm[];
  pdl_trigger();
  const uint32_t tid = threadIdx.x, nb = blockDim.x, C = W.n_clients, R1 = W.n_ranges + 1;
  stage_tables(sm, W, P.flags & MPSF_PF_ISOLATION);
  unsigned long long* c64 = reinterpret_cast<unsigned long long*>(sm + O_C64);
  for (uint32_t i = tid; i < 3 * C + 2; i += nb) c64[i] = EMPTY64;
  uint32_t* iso = reinterpret_cast<uint32_t*>(sm + O_ISO);
  for (uint32_t i = tid; i < 3 * FX_C * 32; i += nb) iso[i] = EMPTY32;
  uint32_t* r32 = reinterpret_cast<uint32_t*>(sm + O_R32);
  for (uint32_t i = tid; i < R1; i += nb) { r32[i] = EMPTY32; r32[FX_R + i] = EMPTY32; }
  uint32_t* cnt = reinterpret_cast<uint32_t*>(sm + O_CNT);
  for (uint32_t i = tid; i < NSCEN * C; i += nb) cnt[i] = 0;
  uint32_t* used = reinterpret_cast<uint32_t*>(sm + O_USED);
  if (tid < 2) used[tid] = 0;
  __syncthreads();
  pdl_wait();
  scan_body<kSparse>(W, S, sm, in, n, P);
  __syncthreads();
  for (uint32_t i = tid; i < NSCEN * C; i += nb)
    if (cnt[i]) atomicAdd(counts + i, (unsigned long long)cnt[i]);
  // fold the block-local minima into the global ones (same slots as flush_minima)
  for (uint32_t i = tid; i < 3 * C; i += nb) {
    uint32_t m = EMPTY32;
#pragma unroll 8
    for (int k = 0; k < 32; ++k) m = min(m, iso[k * (3 * FX_C) + i]);
    uint32_t* g = (i < C ? S.iso1 : (i < 2 * C ? S.iso2 : S.iso3)) + (i % C);
    if (m != EMPTY32) atomicMin(g, m);
    const unsigned long long t = c64[i];
    if (t != EMPTY64) atomicMin(i < C ? S.ft_ce + i : (i < 2 * C ? S.ft_sa + (i - C) : S.trap_sa + (i - 2 * C)), t);
  }
  if (tid < 2) {
    const unsigned long long t = c64[3 * C + tid];
    if (t != EMPTY64) atomicMin(tid ? S.trap_mps : S.ft_gr, t);
  }
  for (uint32_t i = tid; i < W.n_ranges; i += nb) {
    if (r32[i] != EMPTY32) atomicMin(S.ext + i, r32[i]);
    if (r32[FX_R + i] != EMPTY32) atomicMin(S.nr0 + i, r32[FX_R + i]);
  }
  if (tid < 2 && used[tid]) atomicAdd(S.ctrl + C_HASH_DD + tid, used[tid]);
}

// ---- pass 2 ----------------------------------------------------------------------------------
// Per entry: the OutRecord from the record's class, its client row and at most two L2 loads (its
// dedup slot, its first-isolation word).  Every decision that depends only on the class (scenario,
// location, known-duplicate bit -- lo[9:0]) and the entry's epoch band is evaluated once per CTA
// into a decision LUT (dlut_word), so the per-entry path is two shared loads (client row, LUT
// word), the predicated L2 / shared loads the word asks for, and a handful of compares and ORs,
// with no data-dependent branch.  Entries that need a wild-page hash lookup (no range and no
// guard page, or a claimed page slot held by another dedup group) are queued per warp and
// resolved 32 at a time; their mask bits are OR-ed into the chunk masks afterwards.
constexpr uint32_t SQ_CAP = 96;   // per-warp slow queue: < 32 kept + 64 per chunk

// decision word per scenario id (slot 31: skipped entry)
constexpr uint32_t S2_DD = 1u << 8, S2_SERV = 1u << 9, S2_ELIG = 1u << 10, S2_FATAL = 1u << 11,
                   S2_TRAP = 1u << 12, S2_NONREPL = 1u << 31;   // [6:0] static verdict bits

__device__ __forceinline__ uint32_t slut2_word(uint32_t sid, bool isolation) {
  const uint32_t f = scen_word((int)sid, isolation);
  if (!f) return 0u;
  const bool trap = f & LF_TRAP, elig = f & LF_ELIG, serv = f & LF_SERV;
  const uint32_t outcome = trap ? 0u : (elig ? 2u : (serv ? 1u : 3u));
  return outcome | ((f & LF_REPL) ? 0x40u : 0u) | ((f & LF_DD) ? S2_DD : 0u) | (serv ? S2_SERV : 0u) |
         (elig ? S2_ELIG : 0u) | ((!trap && !elig && !serv) ? S2_FATAL : 0u) | (trap ? S2_TRAP : 0u) |
         ((f & LF_REPL) ? 0u : S2_NONREPL);
}

// Decision LUT of pass 2: [epoch band E][class X] -> {w0 flags, w1 = scenario | static verdict << 8
// (0xFFFF00FF for a skipped entry: scenario 0xFF, client 0xFFFF)}.  E = 0: the entry precedes its
// client's release (epoch 0); 1: epoch 1; 2: epoch 1 with pass 1's first-record keys (a client
// released before the drain in a world with per-page keys).  The bits restate rules C2-C7
// for one class:
//   LDD_A / LDD_B  load the dedup slot (B: only if the client's benign-cancel threshold is a tie)
//   LD_NR, NR1     load the first-isolation word of the page (nr1: epoch-1 keys, else nrall)
//   SM_EXT/SM_NR0  read the range's first external-isolation / guard-page key from shared memory
//   SLOW_A/SLOW_B  wild page: resolved by the slow path (B: only with a tie threshold)
//   MH / MM        mechanism when the loaded key is / is not the entry's own (0: not isolating)
//   CGE / CNE      cancel compare: representative >= threshold (benign), != applied record
constexpr uint32_t D_LDD_A = 1u, D_LDD_B = 2u, D_LD_NR = 4u, D_NR1 = 8u, D_SM_EXT = 16u, D_SM_NR0 = 32u,
                   D_SLOW_A = 64u, D_SLOW_B = 128u, D_DD = 256u, D_INR = 512u, D_MH_SH = 10, D_MM_SH = 12,
                   D_CGE = 1u << 14, D_CNE = 1u << 15, D_CTRAP = 1u << 16;
constexpr uint32_t NCLASS = 1024, DBAND = NCLASS * 8;   // bytes per epoch band

__device__ __forceinline__ uint2 dlut_word(uint32_t X, uint32_t E, bool isolation) {
  const uint32_t sid = X & 31u, loc = (X >> 5) & 7u;
  const bool kd = (X >> 8) & 1u;
  const uint32_t sw = (loc == L_SKIP || loc > L_NONE) ? 0u : slut2_word(sid, isolation);
  if (!sw) return make_uint2(0u, 0xFFFF00FFu);
  const bool inr = loc == L_INM || loc == L_INX, grd = loc == L_GRD, wild = loc == L_NONE, inw = inr || grd;
  const bool ep1 = E >= 1, e1 = E == 1;
  const bool dd = sw & S2_DD, elig = sw & S2_ELIG, serv = sw & S2_SERV, fatal = sw & S2_FATAL, trap = sw & S2_TRAP;
  // the representative is needed unless the entry is a known duplicate whose verdict ignores it
  const bool want_a = dd && !(kd && (elig || serv));
  const bool want_b = dd && kd && serv;
  const bool needs_nr = elig && !kd && (!inr || ep1);
  const bool pe = elig && !kd && inr && !ep1 && loc == L_INX;
  const bool ld_nr = needs_nr && (e1 ? inw : inr);
  const bool smv = pe || (needs_nr && grd && !e1);
  const uint32_t mh = elig ? (needs_nr ? 1u : (pe ? 3u : 2u)) : 0u, mm = elig ? 2u : 0u;
  const uint32_t w0 = (want_a && inw ? D_LDD_A : 0u) | (want_b && inw ? D_LDD_B : 0u) | (ld_nr ? D_LD_NR : 0u) |
                      (e1 ? D_NR1 : 0u) | (smv ? (pe ? D_SM_EXT : D_SM_NR0) : 0u) |
                      (wild && (want_a || needs_nr) ? D_SLOW_A : 0u) | (wild && want_b ? D_SLOW_B : 0u) |
                      (dd ? D_DD : 0u) | (inr ? D_INR : 0u) | (mh << D_MH_SH) | (mm << D_MM_SH) |
                      (serv ? D_CGE : 0u) | (trap || fatal ? D_CNE : 0u) | (trap ? D_CTRAP : 0u);
  return make_uint2(w0, sid | ((sw & 0x7Fu) << 8));
}

// Client row per (client, channel engine): {epoch-1 threshold, benign-cancel threshold, applied
// fatal report of the channel's TSG class, byte offset of the client's epoch-1 LUT band}.
//   epoch 1 iff ok32 >= thr (rel = REL_PRE -> 0, REL_NONE -> ~0; ok32 < 2^32 - 1)
//   a benign completion is cancelled iff its representative's ok32 >= T: T = 0 when the client's
//   benign completions are always cancelled on this channel class, ~0 when never (no tie), else
//   tie + 1 (rules C5/C6); a fatal report iff its representative's ok32 != the applied one (C4)
__device__ __forceinline__ uint4 client_row(const FinClient& f, uint32_t ceng) {
  const bool ce = ceng == 1;
  uint4 a;
  a.x = f.rel < 0 ? 0u : (f.rel >= (long long)0xFFFFFFFEll ? 0xFFFFFFFFu : (uint32_t)f.rel + 1u);
  const bool always = (f.bflags >> (ce ? 1 : 0)) & 1u;
  a.y = always ? 0u : (f.tie == EMPTY32 ? 0xFFFFFFFFu : f.tie + 1u);
  a.z = ce ? f.ft1 : f.ft0;
  a.w = (f.pre_nrall ? 2u : 1u) * DBAND;
  return a;
}

__device__ __forceinline__ uint4 lds128_if(bool p, const void* a) {   // predicated shared load (zeros if !p)
  uint4 v;
  asm("{.reg .pred q; setp.ne.u32 q, %5, 0; mov.b32 %0, 0; mov.b32 %1, 0; mov.b32 %2, 0; mov.b32 %3, 0;"
      " @q ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];}"
      : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"((uint32_t)__cvta_generic_to_shared(a)), "r"((uint32_t)p));
  return v;
}

__device__ __forceinline__ uint32_t lds32_if(bool p, const void* a, uint32_t dflt) {
  uint32_t v;
  asm("{.reg .pred q; setp.ne.u32 q, %2, 0; mov.b32 %0, %3; @q ld.shared.u32 %0, [%1];}"
      : "=r"(v) : "r"((uint32_t)__cvta_generic_to_shared(a)), "r"((uint32_t)p), "r"(dflt));
  return v;
}

template <bool kSparse>
__global__ void __launch_bounds__(BLOCK, 1) k_finalize_fx(World W, Scratch S, uint64_t n, Params P,
                                                          mpsf_out_record* __restrict__ out, uint64_t q_base) {
  extern __shared__ __align__(128) uint8_t sm[];
  pdl_trigger();
  const uint32_t tid = threadIdx.x, nb = blockDim.x;
  const bool isolation = P.flags & MPSF_PF_ISOLATION;
  uint2* dl = reinterpret_cast<uint2*>(sm + F_DLUT);
  for (uint32_t i = tid; i < 3 * NCLASS; i += nb) dl[i] = dlut_word(i % NCLASS, i / NCLASS, isolation);
  uint32_t* slut2 = reinterpret_cast<uint32_t*>(sm + F_SLUT);
  if (tid < 32) slut2[tid] = tid == 31 ? 0u : slut2_word(tid, isolation);
  uint4* rows_w = reinterpret_cast<uint4*>(sm + F_ROWS);
  for (uint32_t i = tid; i <= W.n_ranges; i += nb) rows_w[i] = __ldg(W.row4 + i);
  uint32_t* rrid = reinterpret_cast<uint32_t*>(sm + F_RRID);
  for (uint32_t i = tid; i < FX_R * RID_COPIES; i += nb) {
    const uint32_t r = i / RID_COPIES;
    rrid[i] = r <= W.n_ranges ? __ldg(W.rrid + r) : NO_RID;
  }
  pdl_wait();
  if (__ldcg(S.ctrl + C_ERR) != 0) return;
  const bool gpath = __ldcg(S.ctrl + C_PATH) != 0;
  uint4* crow = reinterpret_cast<uint4*>(sm + F_CROW);
  uint32_t* trp = reinterpret_cast<uint32_t*>(sm + F_TRAP);
  for (uint32_t k = tid; k < FX_C * 4 * CH_COPIES; k += nb) {
    const uint32_t ci = k / CH_COPIES, c = ci >> 2;
    uint4 a = make_uint4(0xFFFFFFFFu, 0xFFFFFFFFu, EMPTY32, DBAND);
    if (c < W.n_clients) {
      // the general path's exact minima (what k_resolve2 folds in; idempotent if it ran)
      CState cs = S.cstate[c];
      if (gpath) resolve2_client(S, P, c, cs);
      const FinClient f = fin_client(cs, *S.glob, S.nrall != nullptr);
      a = client_row(f, ci & 3u);
      // an applied trap, as the ok32 of a (non-replayable) trap record
      if (k % (4 * CH_COPIES) == 0) trp[c] = f.trap_ok == EMPTY32 ? EMPTY32 : (f.trap_ok | 0x80000000u);
    }
    crow[k] = a;
  }
  uint32_t* ext = reinterpret_cast<uint32_t*>(sm + F_EXT);
  uint32_t* nr0 = reinterpret_cast<uint32_t*>(sm + F_NR0);
  for (uint32_t i = tid; i < FX_R; i += nb) {
    ext[i] = i < W.n_ranges ? __ldcg(S.ext + i) : EMPTY32;
    nr0[i] = i < W.n_ranges ? __ldcg(S.nr0 + i) : EMPTY32;
  }
  __syncthreads();
  const uint4* rows = reinterpret_cast<const uint4*>(sm + F_ROWS);
  const uint32_t lane = tid & 31, warp = tid >> 5;
  const uint32_t copy16 = (lane & (CH_COPIES - 1)) * 16, copy4 = (lane & (RID_COPIES - 1)) * 4;
  const uint8_t* crow_l = sm + F_CROW + copy16;       // this lane's replica: + (client, engine) * 128
  const uint8_t* rrid_l = sm + F_RRID + copy4;        // + k * 32
  const uint32_t base = (uint32_t)P.base_index;
  uint4* sq = reinterpret_cast<uint4*>(sm + F_SLOWQ) + warp * SQ_CAP;   // {lo, hi, batch index, dd word}
  uint32_t sqn = 0;

  // the general resolution of one queued entry (hash lookups allowed), by one lane
  auto slow_one = [&](uint4 q) {
    const uint32_t lo = q.x, hi = q.y, i = q.z, wd = q.w, gidx = base + i;
    const uint32_t sid = lo & 31u, c = rec_client(lo), ceng = rec_ceng(lo), k = rec_k(lo), loc = rec_loc(lo);
    const bool inr = loc == L_INM || loc == L_INX, inw = inr || loc == L_GRD;
    const uint32_t sw = slut2[sid];
    const uint4 r = crow[((lo >> 13) & 0xFFu) * CH_COPIES];
    const uint32_t ok = gidx | (sw & S2_NONREPL);
    const bool ep1 = ok >= r.x, pre = r.w == 2 * DBAND;
    const bool elig = sw & S2_ELIG, dd = sw & S2_DD;
    const uint64_t page = inw ? (uint64_t)(rows[k].x + (hi - rows[k].z)) : ((uint64_t)hi | ((uint64_t)k << 32));
    unsigned long long key = dd ? dedup_key(c, (int)ceng, (int)sid, page) : 0ull;
    uint32_t ri = ok;
    if (dd) ri = (inw && wd != EMPTY32 && (wd & 7u) == rec_group(lo)) ? (wd >> 3) : hash_get(S.hdd, key);
    const bool dup = dd && ri != gidx;
    const uint32_t rep_ok = dd ? ri : ok;
    bool canc = false;
    if (sw & S2_TRAP) canc = ok != trp[c];
    else if (sw & S2_SERV) canc = rep_ok >= r.y;
    else if (sw & S2_FATAL) canc = rep_ok != r.z;
    uint32_t mech = 0;
    if (elig && !dup) {
      const bool e1 = ep1 && !pre;
      if (!inr || ep1) {
        uint32_t nr;
        if (!inw) nr = hash_get(S.hnr, nr_key(c, e1 ? 1 : 0, page));
        else if (e1) nr = __ldcg(S.nr1 + hi);
        else nr = inr ? __ldcg(S.nrall + hi) : nr0[k];
        mech = nr == ok ? 1u : 2u;
      } else {
        mech = (loc == L_INX && ext[k] == ok) ? 3u : 2u;
      }
    }
    const uint32_t verdict = (sw & 0x7Fu) | (mech << 2) | (canc ? 0x10u : 0u) | (dup ? 0x20u : 0u);
    const uint32_t rid = inr ? rrid[k * RID_COPIES] : NO_RID;
    __stcs(reinterpret_cast<unsigned long long*>(out) + i, (unsigned long long)rid | ((unsigned long long)sid << 32) |
           ((unsigned long long)verdict << 40) | ((unsigned long long)c << 48));
    const uint64_t qq = q_base + i / WCHUNK;
    const uint32_t w = i % WCHUNK, bit = 1u << (w >> 1);
    uint32_t* mw = reinterpret_cast<uint32_t*>(S.cmask + qq);
    const bool rep = dd && !dup;
    if (canc) atomicOr(mw + (w & 1u), bit);
    if (rep) {
      atomicOr(mw + 2 + (w & 1u), bit);
      st_keep(S.dstage + qq * KSTAGE + w, key);
    }
    if (canc || rep) atomicAdd(S.segcnt + qq / SEG_CHUNKS, (canc ? 1ull : 0ull) | (rep ? (1ull << 32) : 0ull));
  };
  auto slow_drain = [&](uint32_t k) {   // queue entries [sqn - k, sqn) by lanes 0..k-1
    __syncwarp();
    if (lane < k) slow_one(sq[sqn - k + lane]);
    sqn -= k;
    __syncwarp();
  };

  // one entry: the class word and the loads (a), the outcome after the loads (b)
  struct A {
    uint32_t lo, hi, w0, w1, ok, T, ft, wd, wn;
    bool pdd;
  };
  auto fin_a = [&](uint32_t lo, uint32_t hi, uint32_t gidx, A& a) {
    a.lo = lo; a.hi = hi;
    a.ok = gidx | ((lo << 22) & 0x80000000u);
    const uint4 r = *reinterpret_cast<const uint4*>(crow_l + ((lo >> 13) & 0xFFu) * (CH_COPIES * 16));
    const uint2 w = *reinterpret_cast<const uint2*>(sm + F_DLUT + (a.ok >= r.x ? r.w : 0u) + (lo & 0x3FFu) * 8);
    a.w0 = w.x; a.w1 = w.y; a.T = r.y; a.ft = r.z;
    const bool tie = (r.y - 1u) < 0xFFFFFFFEu;
    a.pdd = ((w.x & D_LDD_A) != 0) | (((w.x & D_LDD_B) != 0) & tie);
    const uint32_t* pd = S.dd + (kSparse ? hi : hi * 5u + rec_group(lo));
    const uint32_t* pn = ((w.x & D_NR1) ? S.nr1 : S.nrall) + hi;
    const uint32_t smv = lds32_if(w.x & (D_SM_EXT | D_SM_NR0), sm + ((w.x & D_SM_EXT) ? F_EXT : F_NR0) + 4 * rec_k(lo),
                                  EMPTY32);
    a.wd = ldcg_if(a.pdd, pd, 0u);
    a.wn = ldcg_if(w.x & D_LD_NR, pn, smv);
  };
  auto fin_b = [&](const A& a, uint32_t gidx, unsigned long long& o8, bool& canc, bool& rep, bool& slow,
                   unsigned long long& key) {
    const uint32_t lo = a.lo, w0 = a.w0;
    const bool tie = (a.T - 1u) < 0xFFFFFFFEu;
    slow = ((w0 & D_SLOW_A) != 0) | (((w0 & D_SLOW_B) != 0) & tie) |
           (kSparse & a.pdd & ((a.wd == EMPTY32) | (((a.wd ^ (lo >> 10)) & 7u) != 0)));
    const uint32_t ri = a.wd >> 3;
    const bool dup = ((w0 & D_DD) != 0) & (ri != gidx);   // an unloaded slot reads 0: a known duplicate (gidx > 0)
    const uint32_t rep_ok = a.pdd ? ri : a.ok;
    const uint32_t ref = lds32_if(w0 & D_CTRAP, trp + rec_client(lo), a.ft);
    canc = (((w0 & D_CGE) != 0) & (rep_ok >= a.T)) | (((w0 & D_CNE) != 0) & (rep_ok != ref));
    const uint32_t mech = dup ? 0u : (a.wn == a.ok ? (w0 & 0xC00u) : ((w0 >> 2) & 0xC00u));
    const uint32_t h32 = a.w1 | ((lo & 0x1F8000u) << 1) | mech | (canc ? 0x1000u : 0u) | (dup ? 0x2000u : 0u);
    const uint32_t rid = lds32_if(w0 & D_INR, rrid_l + rec_k(lo) * (RID_COPIES * 4), NO_RID);
    o8 = (unsigned long long)rid | ((unsigned long long)h32 << 32);
    rep = ((w0 & D_DD) != 0) & !dup & !slow;
    canc = canc & !slow;
    const uint4 row = lds128_if(rep, rows + rec_k(lo));                  // representatives only
    key = (unsigned long long)(row.x + (a.hi - row.z)) |
          ((unsigned long long)(((lo & 0x1FE000u) << 1) | ((lo & 31u) << 9)) << 32);
  };

  const unsigned long long* rec = S.drec + (P.base_index - S.drec_base);
  const uint32_t below = (1u << lane) - 1u;
  rec_stream(rec, n, [&](ulonglong2 r, uint32_t i0, bool ok0, bool ok1) {
    A a0, a1;
    fin_a(ok0 ? (uint32_t)r.x : 0u, (uint32_t)(r.x >> 32), base + i0, a0);
    fin_a(ok1 ? (uint32_t)r.y : 0u, (uint32_t)(r.y >> 32), base + i0 + 1, a1);
    unsigned long long o0, o1, k0, k1;
    bool c0, c1, p0, p1, s0, s1;
    fin_b(a0, base + i0, o0, c0, p0, s0, k0);
    fin_b(a1, base + i0 + 1, o1, c1, p1, s1, k1);
    unsigned long long* o = reinterpret_cast<unsigned long long*>(out) + i0;
    if (ok1 && (((uintptr_t)o & 15u) == 0)) __stcs(reinterpret_cast<ulonglong2*>(o), make_ulonglong2(o0, o1));
    else {
      if (ok0) __stcs(o, o0);
      if (ok1) __stcs(o + 1, o1);
    }
    const uint32_t bc0 = __ballot_sync(0xFFFFFFFFu, ok0 && c0), bc1 = __ballot_sync(0xFFFFFFFFu, ok1 && c1);
    const uint32_t bd0 = __ballot_sync(0xFFFFFFFFu, ok0 && p0), bd1 = __ballot_sync(0xFFFFFFFFu, ok1 && p1);
    const uint64_t qq = q_base + i0 / WCHUNK;
    if (ok0 && p0) st_keep(S.dstage + qq * KSTAGE + 2 * lane, k0);
    if (ok1 && p1) st_keep(S.dstage + qq * KSTAGE + 2 * lane + 1, k1);
    if (lane == 0) {
      S.cmask[qq] = make_uint4(bc0, bc1, bd0, bd1);
      const uint32_t nc = __popc(bc0) + __popc(bc1), nd = __popc(bd0) + __popc(bd1);
      if (nc | nd) atomicAdd(S.segcnt + qq / SEG_CHUNKS, (unsigned long long)nc | ((unsigned long long)nd << 32));
    }
    // entries needing a hash lookup: queued, resolved 32 at a time (after this chunk's mask store)
    s0 = ok0 && s0;
    s1 = ok1 && s1;
    const uint32_t b0 = __ballot_sync(0xFFFFFFFFu, s0), b1 = __ballot_sync(0xFFFFFFFFu, s1);
    if (b0 | b1) {
      if (s0) sq[sqn + __popc(b0 & below)] = make_uint4(a0.lo, a0.hi, i0, a0.pdd ? a0.wd : EMPTY32);
      sqn += __popc(b0);
      if (s1) sq[sqn + __popc(b1 & below)] = make_uint4(a1.lo, a1.hi, i0 + 1, a1.pdd ? a1.wd : EMPTY32);
      sqn += __popc(b1);
      while (sqn >= 32) slow_drain(32);
    }
  });
  if (sqn) slow_drain(sqn);
}

}  // namespace fx
