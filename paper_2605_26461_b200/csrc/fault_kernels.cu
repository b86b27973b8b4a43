// Batched MMU-fault-buffer processing for sm_100a.
//
// One batch = N packed 16-byte fault-buffer entries resident in HBM.  The reference
// (pkg/src/mpssim/) handles them one record at a time: raise_mmu_fault classifies each
// (pipeline.py:96-129), service_bottom_half drains replayable-then-non-replayable and
// acts per record on the evolving world (pipeline.py:160-183).  Here the same result is
// computed with the parallel recipe C9 of SURVEY.md Appendix C -- every cross-record
// dependency is a first-in-group minimum over the drain key, so the batch needs:
//
//   k_scan      pass 1 over the entries: decode, attribute (binary search in the smem
//               interval table), classify, per-(client,scenario) counts, and the group
//               minima (fatal TSG teardowns, traps, first isolation per external range /
//               per unmapped page / per client, first record per dedup key)
//   k_resolve   one block: per-client release keys, kill thresholds, fates, fast/general
//   k_general1  [general path only] release-aware first-isolation keys (rule C3 epochs)
//   k_general2  [general path, m2 <= benign] exact per-client M2 minima
//   k_resolve2  [general path] kill thresholds from the exact minima
//   k_finalize  pass 2: re-decode, resolve dup / mechanism / cancel per entry, write the
//               8-byte OutRecord, compact the cancel list and the dedup set in index order
//               with a decoupled look-back over tiles
//
// The fast path (isolation off, or no client with isolation-eligible records is released
// in the batch, and m2_us > benign_us) reads the entries exactly twice.
#include <cuda_runtime.h>
#include <stdint.h>

#include "mpsf_device.cuh"
#include "mpsf_kernels.h"

namespace mpsf {

constexpr int BLOCK = 512;
constexpr int WARPS = BLOCK / 32;
constexpr int EPT = 8;                  // entries per lane per tile
constexpr int TILE = BLOCK * EPT;       // 4096 entries per tile

// ---- shared-memory staging of the world tables ------------------------------------
struct Smem {
  mpsf_range_entry* ranges;   // staged interval table (or global pointer)
  mpsf_channel_entry* channels;
  uint32_t* client_off;
  uint8_t* client_mode;
  // pass-1 write-through caches
  unsigned long long* ft_ce;
  unsigned long long* ft_sa;
  unsigned long long* trap_sa;
  uint32_t* elig;
  uint32_t* iso1;
  uint32_t* iso2;
  uint32_t* iso3;
  uint32_t* ext;
  uint32_t* nr0;
  uint32_t* counts;
};

__host__ __device__ inline size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

__host__ __device__ inline size_t staged_smem_bytes(uint32_t nr, uint32_t nc, uint32_t nch) {
  size_t s = 0;
  s += align16(sizeof(mpsf_range_entry) * nr);
  s += align16(sizeof(mpsf_channel_entry) * nch);
  s += align16(sizeof(uint32_t) * (nc + 1));
  s += align16(nc);
  s += align16(sizeof(unsigned long long) * 3 * nc);
  s += align16(sizeof(uint32_t) * 4 * nc);
  s += align16(sizeof(uint32_t) * 2 * nr);
  s += align16(sizeof(uint32_t) * NSCEN * nc);
  return s;
}

__device__ inline Smem carve(uint8_t* base, const World& W) {
  Smem s;
  size_t o = 0;
  s.ranges = reinterpret_cast<mpsf_range_entry*>(base + o); o += align16(sizeof(mpsf_range_entry) * W.n_ranges);
  s.channels = reinterpret_cast<mpsf_channel_entry*>(base + o); o += align16(sizeof(mpsf_channel_entry) * W.n_channels);
  s.client_off = reinterpret_cast<uint32_t*>(base + o); o += align16(sizeof(uint32_t) * (W.n_clients + 1));
  s.client_mode = base + o; o += align16(W.n_clients);
  s.ft_ce = reinterpret_cast<unsigned long long*>(base + o);
  s.ft_sa = s.ft_ce + W.n_clients;
  s.trap_sa = s.ft_sa + W.n_clients;
  o += align16(sizeof(unsigned long long) * 3 * W.n_clients);
  s.elig = reinterpret_cast<uint32_t*>(base + o);
  s.iso1 = s.elig + W.n_clients; s.iso2 = s.iso1 + W.n_clients; s.iso3 = s.iso2 + W.n_clients;
  o += align16(sizeof(uint32_t) * 4 * W.n_clients);
  s.ext = reinterpret_cast<uint32_t*>(base + o); s.nr0 = s.ext + W.n_ranges;
  o += align16(sizeof(uint32_t) * 2 * W.n_ranges);
  s.counts = reinterpret_cast<uint32_t*>(base + o);
  return s;
}

// Copy world tables into smem and initialise the caches.  kStaged=false keeps
// everything in global memory (worlds too large for one CTA's smem).
template <bool kStaged>
__device__ inline Smem stage(uint8_t* sm, const World& W, bool with_caches) {
  Smem s;
  if (!kStaged) {
    s.ranges = const_cast<mpsf_range_entry*>(W.ranges);
    s.channels = const_cast<mpsf_channel_entry*>(W.channels);
    s.client_off = const_cast<uint32_t*>(W.client_off);
    s.client_mode = nullptr;
    return s;
  }
  s = carve(sm, W);
  const int tid = threadIdx.x;
  {
    const uint4* src = reinterpret_cast<const uint4*>(W.ranges);
    uint4* dst = reinterpret_cast<uint4*>(s.ranges);
    for (uint32_t i = tid; i < W.n_ranges * 2; i += blockDim.x) dst[i] = __ldg(src + i);
  }
  for (uint32_t i = tid; i < W.n_channels; i += blockDim.x) s.channels[i] = W.channels[i];
  for (uint32_t i = tid; i <= W.n_clients; i += blockDim.x) s.client_off[i] = __ldg(W.client_off + i);
  for (uint32_t i = tid; i < W.n_clients; i += blockDim.x) s.client_mode[i] = W.clients[i].mode;
  if (with_caches) {
    for (uint32_t i = tid; i < 3 * W.n_clients; i += blockDim.x) s.ft_ce[i] = EMPTY64;
    for (uint32_t i = tid; i < 4 * W.n_clients; i += blockDim.x) s.elig[i] = EMPTY32;
    for (uint32_t i = tid; i < 2 * W.n_ranges; i += blockDim.x) s.ext[i] = EMPTY32;
    for (uint32_t i = tid; i < NSCEN * W.n_clients; i += blockDim.x) s.counts[i] = 0;
  }
  return s;
}

__device__ __forceinline__ uint32_t client_mode(const Smem& s, const World& W, uint32_t c, bool staged) {
  return staged ? s.client_mode[c] : W.clients[c].mode;
}

__device__ __forceinline__ void raise_err(const Scratch& S, uint32_t bit, uint64_t gidx) {
  atomicOr(S.ctrl + C_ERR, bit);
  atomicMin(S.err_idx, (unsigned long long)gidx);
}

// Decoded + classified view of one entry, shared by every pass.
struct Rec {
  bool valid;
  uint32_t c;       // client
  int ceng;         // channel engine
  int eng, acc, kind;
  int s;            // scenario id
  uint64_t va;
  Attr at;
  bool repl;        // replayable buffer
  uint32_t group;   // dedup group (replayable translation)
};

// Entry decode, validation, attribution, classification.  Returns valid=false for
// invalid-flag entries and for malformed ones (after raising the error bit).
template <bool kStaged>
__device__ __forceinline__ Rec decode(const World& W, const Smem& sm, const Scratch& S,
                                      uint64_t va, uint64_t w1, uint64_t gidx) {
  Rec r;
  r.valid = false;
  r.va = va;
  const uint32_t flags = (uint32_t)(w1 >> 56);
  if (!(flags & MPSF_ENTRY_VALID)) return r;
  const uint32_t ch = (uint32_t)w1;
  r.eng = (int)((w1 >> 32) & 0xFF);
  r.acc = (int)((w1 >> 40) & 0xFF);
  r.kind = (int)((w1 >> 48) & 0xFF);
  if (ch >= W.n_channels) { raise_err(S, EB_NO_CHANNEL, gidx); return r; }
  const mpsf_channel_entry ce = kStaged ? sm.channels[ch] : W.channels[ch];
  if (ce.client >= W.n_clients) { raise_err(S, EB_NO_CHANNEL, gidx); return r; }
  r.c = ce.client;
  r.ceng = ce.engine;
  r.group = 0;
  if (r.kind == 0) {
    if (r.eng > 2 || r.acc > 2) { raise_err(S, EB_BAD_ENTRY, gidx); return r; }
    if (r.eng != r.ceng) { raise_err(S, EB_MISMATCH, gidx); return r; }
    if (va >= VA_LIMIT) { raise_err(S, EB_VA, gidx); return r; }
    const uint32_t lo = sm.client_off[r.c], hi = sm.client_off[r.c + 1];
    r.at = attribute(sm.ranges, W.page_state, lo, hi, va);
    const bool has = r.at.in_range;
    r.s = classify(r.eng, r.acc, has, r.at.kind, r.at.lifecycle, r.at.migratable, r.at.st);
    r.repl = s_replayable(r.s);
    if (r.repl && r.eng == 0 && r.acc != 2) {
      const int sr = classify(0, 0, has, r.at.kind, r.at.lifecycle, r.at.migratable, r.at.st);
      const int sw = classify(0, 1, has, r.at.kind, r.at.lifecycle, r.at.migratable, r.at.st);
      r.group = dedup_group(0, r.acc, sr, sw);
    } else {
      r.group = dedup_group(r.eng, r.acc, 0, 0);
    }
  } else if (r.kind >= 1 && r.kind <= 5) {
    r.s = 23 + r.kind - 1;
    r.repl = true;
    r.at.ridx = -1; r.at.in_range = false; r.at.guard = false; r.at.rid = NO_RID;
  } else if (r.kind >= 8 && r.kind <= 12) {
    r.s = 18 + r.kind - 8;
    r.repl = false;
    r.at.ridx = -1; r.at.in_range = false; r.at.guard = false; r.at.rid = NO_RID;
  } else {
    raise_err(S, EB_BAD_ENTRY, gidx);
    return r;
  }
  r.valid = true;
  return r;
}

__device__ __forceinline__ uint32_t ok32_of(bool repl, uint64_t gidx) {
  return (repl ? 0u : 0x80000000u) | (uint32_t)gidx;
}

// ---- pass 1 ---------------------------------------------------------------------------
template <bool kStaged>
__global__ void __launch_bounds__(BLOCK) k_scan(World W, Scratch S, const mpsf_fault_entry* __restrict__ in,
                                                uint64_t n, Params P, unsigned long long* __restrict__ counts) {
  extern __shared__ __align__(16) uint8_t smem[];
  const Smem sm = stage<kStaged>(smem, W, true);
  if (kStaged) __syncthreads();
  const bool iso = P.flags & MPSF_PF_ISOLATION;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t ntiles = (n + TILE - 1) / TILE;
  const ulonglong2* src = reinterpret_cast<const ulonglong2*>(in);
  for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const uint64_t base = t * TILE + (uint64_t)warp * (32 * EPT) + lane;
    ulonglong2 e[EPT];
#pragma unroll
    for (int k = 0; k < EPT; ++k) {
      const uint64_t i = base + (uint64_t)k * 32;
      e[k] = i < n ? __ldg(src + i) : make_ulonglong2(0ull, 0ull);
    }
#pragma unroll
    for (int k = 0; k < EPT; ++k) {
      const uint64_t i = base + (uint64_t)k * 32;
      const uint64_t gidx = P.base_index + i;
      const Rec r = decode<kStaged>(W, sm, S, e[k].x, e[k].y, gidx);
      if (!r.valid) continue;
      const uint32_t c = r.c;
      if (kStaged) atomicAdd(sm.counts + c * NSCEN + r.s, 1u);
      else atomicAdd(counts + (uint64_t)c * NSCEN + r.s, 1ull);
      const uint32_t mode = client_mode(sm, W, c, kStaged);
      if (s_trap(r.s)) {
        const unsigned long long v = (gidx << 8) | (unsigned long long)r.s;
        if (mode == 0) min64(&S.glob->trap_mps, v);
        else if (kStaged) min64c(S.trap_sa + c, sm.trap_sa + c, v);
        else min64(S.trap_sa + c, v);
        continue;
      }
      const uint32_t ok = ok32_of(r.repl, gidx);
      const bool parse = s_parse(r.s);
      const bool serv = s_serviceable(r.s);
      if (parse || (!serv && !iso)) {                       // fatal report (pipeline.py:168-182)
        const unsigned long long v = ((unsigned long long)ok << 8) | (unsigned long long)r.s;
        if (mode == 1) { if (kStaged) min64c(S.ft_sa + c, sm.ft_sa + c, v); else min64(S.ft_sa + c, v); }
        else if (r.ceng == 1) { if (kStaged) min64c(S.ft_ce + c, sm.ft_ce + c, v); else min64(S.ft_ce + c, v); }
        else min64(&S.glob->ft_gr, v);
      } else if (!serv) {                                   // isolation-eligible (pipeline.py:177-179)
        if (kStaged) min32c(S.elig + c, sm.elig + c, ok); else min32(S.elig + c, ok);
        if (!r.at.in_range) {
          if (kStaged) min32c(S.iso1 + c, sm.iso1 + c, ok); else min32(S.iso1 + c, ok);
          if (r.at.guard) {
            if (kStaged) min32c(S.nr0 + r.at.ridx, sm.nr0 + r.at.ridx, ok); else min32(S.nr0 + r.at.ridx, ok);
          } else if (!hash_min(S.hnr, S.ctrl, nr_key(c, 0, r.va >> 12), ok)) {
            atomicOr(S.ctrl + C_OVF, 1u);
          }
        } else if (r.at.kind == 0) {
          if (kStaged) min32c(S.iso2 + c, sm.iso2 + c, ok); else min32(S.iso2 + c, ok);
        } else {
          if (kStaged) {
            min32c(S.iso3 + c, sm.iso3 + c, ok);
            min32c(S.ext + r.at.ridx, sm.ext + r.at.ridx, ok);
          } else {
            min32(S.iso3 + c, ok);
            min32(S.ext + r.at.ridx, ok);
          }
        }
      }
      if (r.kind == 0 && r.repl) {                          // dedup insert (rule C2)
        const uint32_t v = ((uint32_t)gidx << 3) | r.group;
        bool to_hash = !(r.at.in_range || r.at.guard);
        if (!to_hash) {
          uint32_t* slot = S.dd + r.at.slot;
          uint32_t cur = __ldcg(slot);
          while (true) {
            if (cur == EMPTY32) {
              const uint32_t prev = atomicCAS(slot, EMPTY32, v);
              if (prev == EMPTY32) break;
              cur = prev;
              continue;
            }
            if ((cur & 7u) == r.group) { if (cur > v) atomicMin(slot, v); break; }
            to_hash = true;
            break;
          }
        }
        if (to_hash && !hash_min(S.hdd, S.ctrl, dedup_key(c, r.eng, r.s, r.va >> 12), (uint32_t)gidx))
          atomicOr(S.ctrl + C_OVF, 1u);
      }
    }
  }
  if (kStaged) {
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < NSCEN * W.n_clients; i += blockDim.x) {
      const uint32_t v = sm.counts[i];
      if (v) atomicAdd(counts + i, (unsigned long long)v);
    }
  }
}

// ---- per-client resolution ----------------------------------------------------------
// Rules C4-C7 of SURVEY.md Appendix C (C9 "ROUND 1" + fate).  One block.
__device__ inline void kill_thresholds(const Params& P, uint32_t m1, uint32_t m2, uint32_t m3,
                                       bool use_m2, bool& kill_all, uint32_t& tie) {
  kill_all = false;
  tie = EMPTY32;
  const uint32_t lat[3] = {P.m1_us, P.m2_us, P.m3_us};
  const uint32_t v[3] = {m1, m2, m3};
  for (int m = 0; m < 3; ++m) {
    if (m == 1 && !use_m2) continue;
    if (v[m] == EMPTY32) continue;
    if (lat[m] < P.benign_us) kill_all = true;
    else if (lat[m] == P.benign_us && v[m] < tie) tie = v[m];
  }
}

__global__ void k_resolve(World W, Scratch S, Params P, mpsf_client_verdict* __restrict__ verdict) {
  __shared__ int s_general;
  if (threadIdx.x == 0) s_general = 0;
  __syncthreads();
  if (__ldcg(S.ctrl + C_ERR) != 0) return;
  const bool iso = P.flags & MPSF_PF_ISOLATION;
  Globals* G = S.glob;
  const bool gr_alive0 = W.has_mps && !(W.world_flags & MPSF_WF_GR_DEAD);
  const unsigned long long trap_mps = G->trap_mps, ft_gr = G->ft_gr;
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
    const unsigned long long tsa = S.trap_sa[c], fsa = S.ft_sa[c], fce = S.ft_ce[c];
    const bool trapped = sa ? (alive0 && tsa != EMPTY64) : trapped_mps;
    const bool sa_applied = sa && alive0 && !trapped && fsa != EMPTY64;
    long long rel;
    if (!alive0) rel = REL_PRE;
    else if (sa) rel = trapped ? REL_PRE : (sa_applied ? (long long)(fsa >> 8) : REL_NONE);
    else rel = gr_rel;
    const bool ce_applied = ce_alive0 && fce != EMPTY64 && !(rel < (long long)(fce >> 8));
    const uint32_t elig = S.elig[c];
    CState cs;
    cs.rel = rel;
    cs.ft_ce_ok = fce == EMPTY64 ? EMPTY32 : (uint32_t)(fce >> 8);
    cs.ft_sa_ok = fsa == EMPTY64 ? EMPTY32 : (uint32_t)(fsa >> 8);
    cs.trap_sa_idx = tsa == EMPTY64 ? EMPTY32 : (uint32_t)(tsa >> 8);
    bool kill_all;
    uint32_t tie;
    kill_thresholds(P, S.iso1[c], S.iso2[c], S.iso3[c], false, kill_all, tie);
    cs.kill_tie = tie;
    cs.flags = (alive0 ? CS_ALIVE0 : 0u) | (sa ? CS_SA : 0u) | (ce_alive0 ? CS_CE_ALIVE0 : 0u) |
               ((!sa && (!ce_alive0 || ce_applied)) ? CS_CE_TORN : 0u) | (kill_all ? CS_KILL_ALL : 0u) |
               (trapped ? CS_TRAPPED : 0u) | (elig != EMPTY32 ? CS_ELIG : 0u);
    cs.pad = 0;
    S.cstate[c] = cs;
    mpsf_client_verdict v;
    v.flags = 0;
    if (alive0) {
      if (trapped) { v.state = 1; v.reason = 2; v.notifier = (uint8_t)((sa ? tsa : trap_mps) & 0xFF); }
      else if (!sa && gr_applied) { v.state = 1; v.reason = 2; v.notifier = (uint8_t)(ft_gr & 0xFF); }
      else if (sa_applied) { v.state = 1; v.reason = 2; v.notifier = (uint8_t)(fsa & 0xFF); }
      else if (elig != EMPTY32) { v.state = 1; v.reason = 1; v.notifier = ce_applied ? (uint8_t)(fce & 0xFF) : 0xFF; }
      else if (ce_applied) { v.state = 0; v.reason = 0; v.notifier = (uint8_t)(fce & 0xFF); }
      else { v.state = 0; v.reason = 0; v.notifier = 0xFF; }
    } else {
      v.state = 1; v.reason = 3;
      v.notifier = (!sa && trapped_mps) ? (uint8_t)(trap_mps & 0xFF)
                   : ((!sa && gr_applied) ? (uint8_t)(ft_gr & 0xFF) : 0xFE);
    }
    verdict[c] = v;
    if (iso && elig != EMPTY32 && (rel != REL_NONE || P.m2_us <= P.benign_us)) general = 1;
  }
  if (general) atomicOr(&s_general, 1);
  __syncthreads();
  if (threadIdx.x == 0) {
    G->ft_gr_ok = gr_applied ? (uint32_t)(ft_gr >> 8) : EMPTY32;
    G->trap_mps_idx = trapped_mps ? (uint32_t)(trap_mps >> 8) : EMPTY32;
    G->gr_alive0 = gr_alive0;
    S.ctrl[C_PATH] = s_general;
  }
}

// ---- general path (rule C3 epochs) ----------------------------------------------------
__device__ __forceinline__ uint32_t dedup_rep(const Scratch& S, const Rec& r) {
  // smallest global index among records of r's dedup key
  if (r.at.in_range || r.at.guard) {
    const uint32_t cur = __ldcg(S.dd + r.at.slot);
    if (cur != EMPTY32 && (cur & 7u) == r.group) return cur >> 3;
  }
  return hash_get(S.hdd, dedup_key(r.c, r.eng, r.s, r.va >> 12));
}

__device__ __forceinline__ uint32_t nr_lookup(const Scratch& S, const Rec& r, bool epoch1) {
  if (epoch1) {
    if (r.at.in_range || r.at.guard) return __ldcg(S.nr1 + r.at.slot);
    return hash_get(S.hnr, nr_key(r.c, 1, r.va >> 12));
  }
  if (r.at.guard) return __ldcg(S.nr0 + r.at.ridx);
  return hash_get(S.hnr, nr_key(r.c, 0, r.va >> 12));
}

__global__ void k_clear_nr1(Scratch S, uint64_t n_pages) {
  if (__ldcg(S.ctrl + C_PATH) == 0) return;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n_pages; i += (uint64_t)gridDim.x * blockDim.x)
    S.nr1[i] = EMPTY32;
}

// stage 1: epoch-1 NR keys, exact M1 / M3 / direct-M2 minima (giso[3*c + m-1])
// stage 2: noRange non-first records -> M2 minima (needs NR complete)
template <bool kStaged, int kStage>
__global__ void __launch_bounds__(BLOCK) k_general(World W, Scratch S, const mpsf_fault_entry* __restrict__ in,
                                                   uint64_t n, Params P) {
  if (__ldcg(S.ctrl + C_PATH) == 0) return;
  extern __shared__ __align__(16) uint8_t smem[];
  const Smem sm = stage<kStaged>(smem, W, false);
  if (kStaged) __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t ntiles = (n + TILE - 1) / TILE;
  const ulonglong2* src = reinterpret_cast<const ulonglong2*>(in);
  for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const uint64_t base = t * TILE + (uint64_t)warp * (32 * EPT) + lane;
    ulonglong2 e[EPT];
#pragma unroll
    for (int k = 0; k < EPT; ++k) {
      const uint64_t i = base + (uint64_t)k * 32;
      e[k] = i < n ? __ldg(src + i) : make_ulonglong2(0ull, 0ull);
    }
#pragma unroll
    for (int k = 0; k < EPT; ++k) {
      const uint64_t i = base + (uint64_t)k * 32;
      const uint64_t gidx = P.base_index + i;
      const Rec r = decode<kStaged>(W, sm, S, e[k].x, e[k].y, gidx);
      if (!r.valid || r.kind != 0 || s_serviceable(r.s)) continue;   // elig translation only
      if (r.repl && dedup_rep(S, r) != (uint32_t)gidx) continue;      // dups excluded (C2)
      const uint32_t ok = ok32_of(r.repl, gidx);
      const long long rel = S.cstate[r.c].rel;
      const bool epoch1 = rel < (long long)ok;
      const bool no_range = !r.at.in_range || epoch1;
      uint32_t* giso = S.giso + 3 * r.c;
      if (kStage == 1) {
        if (no_range) {
          min32(giso + 0, ok);
          if (epoch1) {
            if (r.at.in_range || r.at.guard) min32(S.nr1 + r.at.slot, ok);
            else if (!hash_min(S.hnr, S.ctrl, nr_key(r.c, 1, r.va >> 12), ok)) atomicOr(S.ctrl + C_OVF, 1u);
          }
        } else if (r.at.kind == 0) {
          min32(giso + 1, ok);
        } else {
          const uint32_t ext = __ldcg(S.ext + r.at.ridx);
          if (ok == ext && (long long)ext < rel) min32(giso + 2, ok);
          else min32(giso + 1, ok);
        }
      } else {
        if (no_range && nr_lookup(S, r, epoch1) != ok) min32(giso + 1, ok);
      }
    }
  }
}

__global__ void k_resolve2(World W, Scratch S, Params P) {
  if (__ldcg(S.ctrl + C_PATH) == 0) return;
  for (uint32_t c = threadIdx.x; c < W.n_clients; c += blockDim.x) {
    bool kill_all;
    uint32_t tie;
    kill_thresholds(P, S.giso[3 * c], S.giso[3 * c + 1], S.giso[3 * c + 2], true, kill_all, tie);
    CState cs = S.cstate[c];
    cs.kill_tie = tie;
    cs.flags = (cs.flags & ~CS_KILL_ALL) | (kill_all ? CS_KILL_ALL : 0u);
    S.cstate[c] = cs;
  }
}

// ---- pass 2 -----------------------------------------------------------------------------
// Decoupled look-back descriptor: [63:62] status (0 none, 1 aggregate, 2 prefix),
// [61:31] dedup count, [30:0] cancel count.
constexpr unsigned long long LB_AGG = 1ull << 62, LB_PRE = 2ull << 62, LB_VAL = (1ull << 62) - 1;

__device__ __forceinline__ unsigned long long lb_pack(uint32_t nc, uint32_t nd) {
  return ((unsigned long long)nd << 31) | nc;
}

template <bool kStaged>
__global__ void __launch_bounds__(BLOCK) k_finalize(World W, Scratch S, const mpsf_fault_entry* __restrict__ in,
                                                    uint64_t n, Params P, mpsf_out_record* __restrict__ out,
                                                    unsigned long long* __restrict__ dkeys,
                                                    uint32_t* __restrict__ didx, uint32_t* __restrict__ cancel) {
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ uint32_t s_tile;
  __shared__ uint32_t s_wc[WARPS], s_wd[WARPS];
  __shared__ uint32_t s_pc, s_pd;
  if (__ldcg(S.ctrl + C_ERR) != 0) return;
  const Smem sm = stage<kStaged>(smem, W, false);
  // per-client derived state: reuse the cache region (kStaged) or read from global
  CState* cst = S.cstate;
  if (kStaged) {
    CState* dst = reinterpret_cast<CState*>(sm.ft_ce);   // ft_ce..iso3 region >= 40 B/client
    for (uint32_t c = threadIdx.x; c < W.n_clients; c += blockDim.x) dst[c] = S.cstate[c];
    cst = dst;
    __syncthreads();
  }
  const bool iso = P.flags & MPSF_PF_ISOLATION;
  const Globals G = *S.glob;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t ntiles = (uint32_t)((n + TILE - 1) / TILE);
  const ulonglong2* src = reinterpret_cast<const ulonglong2*>(in);
  const unsigned lt_mask = (1u << lane) - 1u;
  while (true) {
    if (threadIdx.x == 0) s_tile = atomicAdd(S.ctrl + C_TILE_FIN, 1u);
    __syncthreads();
    const uint32_t t = s_tile;
    if (t >= ntiles) break;
    const uint64_t base = (uint64_t)t * TILE + (uint64_t)warp * (32 * EPT) + lane;
    ulonglong2 e[EPT];
#pragma unroll
    for (int k = 0; k < EPT; ++k) {
      const uint64_t i = base + (uint64_t)k * 32;
      e[k] = i < n ? __ldcs(src + i) : make_ulonglong2(0ull, 0ull);
    }
    uint32_t cflag = 0, dflag = 0;             // bit k: entry k cancelled / dedup representative
    unsigned long long key[EPT];
    uint32_t wc = 0, wd = 0;                   // warp totals
    uint32_t my_c_off[EPT], my_d_off[EPT];
#pragma unroll
    for (int k = 0; k < EPT; ++k) {
      const uint64_t i = base + (uint64_t)k * 32;
      const uint64_t gidx = P.base_index + i;
      key[k] = 0;
      const Rec r = decode<kStaged>(W, sm, S, e[k].x, e[k].y, gidx);
      mpsf_out_record o;
      o.rid = NO_RID; o.scenario = 0xFF; o.verdict = 0; o.client = 0xFFFF;
      bool canc = false, rep = false;
      if (r.valid) {
        const CState cs = cst[r.c];
        o.scenario = (uint8_t)r.s;
        o.client = (uint16_t)r.c;
        o.rid = r.at.in_range ? r.at.rid : NO_RID;
        if (s_trap(r.s)) {
          // raise_sm_trap at raise time (pipeline.py:151-155); a second trap on a destroyed
          // TSG is cancelled (the reference raises UnknownTsg)
          if (!(cs.flags & CS_SA)) canc = !(G.gr_alive0 && (uint32_t)gidx == G.trap_mps_idx);
          else canc = !((cs.flags & CS_ALIVE0) && (uint32_t)gidx == cs.trap_sa_idx);
          o.verdict = canc ? 0x10 : 0;
        } else {
          const bool parse = s_parse(r.s), serv = s_serviceable(r.s);
          const int outcome = parse ? 3 : (serv ? 1 : (iso ? 2 : 3));
          const uint32_t ok = ok32_of(r.repl, gidx);
          uint32_t rep_ok = ok;
          bool dup = false;
          if (r.kind == 0 && r.repl) {
            const uint32_t ri = dedup_rep(S, r);
            dup = ri != (uint32_t)gidx;
            rep_ok = ri;                          // replayable: ok32 == idx
            rep = !dup;
            if (rep) key[k] = dedup_key(r.c, r.eng, r.s, r.va >> 12);
          }
          int mech = 0;
          if (outcome == 3) {                     // fatal: applies iff its TSG still lives (C4)
            bool applied;
            if (cs.flags & CS_SA) applied = (cs.flags & CS_ALIVE0) && !(cs.flags & CS_TRAPPED) && rep_ok == cs.ft_sa_ok;
            else if (r.ceng == 1) applied = (cs.flags & CS_CE_ALIVE0) && rep_ok == cs.ft_ce_ok && !(cs.rel < (long long)rep_ok);
            else applied = rep_ok == G.ft_gr_ok;
            canc = !applied;
          } else if (outcome == 1) {              // benign completion dropped on a torn channel (C5)
            canc = cs.rel != REL_NONE || (r.ceng == 1 && (cs.flags & CS_CE_TORN)) ||
                   (cs.flags & CS_KILL_ALL) || rep_ok > cs.kill_tie;
          } else if (!dup) {                      // isolation mechanism (C3)
            const bool epoch1 = cs.rel < (long long)ok;
            if (!r.at.in_range || epoch1) mech = nr_lookup(S, r, epoch1) == ok ? 1 : 2;
            else if (r.at.kind == 0) mech = 2;
            else mech = __ldcg(S.ext + r.at.ridx) == ok ? 3 : 2;
          }
          o.verdict = (uint8_t)(outcome | (mech << 2) | (canc ? 0x10 : 0) | (dup ? 0x20 : 0) | (r.repl ? 0x40 : 0));
        }
      }
      if (base + (uint64_t)k * 32 < n) __stcs(reinterpret_cast<unsigned long long*>(out) + base + (uint64_t)k * 32,
                                             *reinterpret_cast<unsigned long long*>(&o));
      const unsigned bc = __ballot_sync(0xFFFFFFFFu, canc);
      const unsigned bd = __ballot_sync(0xFFFFFFFFu, rep);
      my_c_off[k] = wc + __popc(bc & lt_mask);
      my_d_off[k] = wd + __popc(bd & lt_mask);
      wc += __popc(bc);
      wd += __popc(bd);
      cflag |= (canc ? 1u : 0u) << k;
      dflag |= (rep ? 1u : 0u) << k;
    }
    if (lane == 0) { s_wc[warp] = wc; s_wd[warp] = wd; }
    __syncthreads();
    if (threadIdx.x == 0) {
      uint32_t tc = 0, td = 0;
      for (int w = 0; w < WARPS; ++w) {
        const uint32_t a = s_wc[w], b = s_wd[w];
        s_wc[w] = tc; s_wd[w] = td;
        tc += a; td += b;
      }
      // decoupled look-back
      volatile unsigned long long* desc = S.tiles;
      uint32_t pc = 0, pd = 0;
      if (t == 0) {
        desc[0] = LB_PRE | lb_pack(tc, td);
      } else {
        desc[t] = LB_AGG | lb_pack(tc, td);
        int64_t j = (int64_t)t - 1;
        while (j >= 0) {
          const unsigned long long d = desc[j];
          const unsigned long long st = d & ~LB_VAL;
          if (st == 0) continue;
          pc += (uint32_t)(d & 0x7FFFFFFFull);
          pd += (uint32_t)((d >> 31) & 0x7FFFFFFFull);
          if (st == LB_PRE) break;
          --j;
        }
        __threadfence();
        desc[t] = LB_PRE | lb_pack(pc + tc, pd + td);
      }
      s_pc = pc; s_pd = pd;
    }
    __syncthreads();
    const uint32_t bc0 = s_pc + s_wc[warp], bd0 = s_pd + s_wd[warp];
#pragma unroll
    for (int k = 0; k < EPT; ++k) {
      const uint64_t gidx = P.base_index + base + (uint64_t)k * 32;
      if (cflag & (1u << k)) cancel[bc0 + my_c_off[k]] = (uint32_t)gidx;
      if (dflag & (1u << k)) {
        dkeys[bd0 + my_d_off[k]] = key[k];
        didx[bd0 + my_d_off[k]] = (uint32_t)gidx;
      }
    }
    __syncthreads();
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

bool staged_fits(const World& W) {
  return staged_smem_bytes(W.n_ranges, W.n_clients, W.n_channels) <= 96 * 1024;
}

template <bool kStaged>
static int launch_all(const World& W, const Scratch& S, const mpsf_fault_entry* in, uint64_t n,
                      const Params& P, mpsf_out_record* out, mpsf_client_verdict* verdict,
                      unsigned long long* counts, unsigned long long* dkeys, uint32_t* didx,
                      uint32_t* cancel, cudaStream_t st, int* launches, const Marker& mk) {
  const size_t smem = kStaged ? staged_smem_bytes(W.n_ranges, W.n_clients, W.n_channels) : 0;
  static bool attr_set = false;
  if (!attr_set) {
    const int mx = 200 * 1024;
    cudaFuncSetAttribute(k_scan<kStaged>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
    cudaFuncSetAttribute(k_general<kStaged, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
    cudaFuncSetAttribute(k_general<kStaged, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
    cudaFuncSetAttribute(k_finalize<kStaged>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
    attr_set = true;
  }
  const uint64_t ntiles = (n + TILE - 1) / TILE;
  int nl = 0;
  if (n > 0) {
    int g = grid_for(k_scan<kStaged>, smem);
    if ((uint64_t)g > ntiles) g = (int)ntiles;
    k_scan<kStaged><<<g, BLOCK, smem, st>>>(W, S, in, n, P, counts);
    mk.mark("k_scan");
    ++nl;
  }
  k_resolve<<<1, 1024, 0, st>>>(W, S, P, verdict);
  mk.mark("k_resolve");
  ++nl;
  if ((P.flags & MPSF_PF_ISOLATION) && n > 0) {
    k_clear_nr1<<<2 * sm_count(), 256, 0, st>>>(S, W.n_pages);
    mk.mark("k_clear_nr1");
    int g = grid_for(k_general<kStaged, 1>, smem);
    if ((uint64_t)g > ntiles) g = (int)ntiles;
    k_general<kStaged, 1><<<g, BLOCK, smem, st>>>(W, S, in, n, P);
    mk.mark("k_general1");
    nl += 2;
    if (P.m2_us <= P.benign_us) {
      k_general<kStaged, 2><<<g, BLOCK, smem, st>>>(W, S, in, n, P);
      mk.mark("k_general2");
      ++nl;
    }
    k_resolve2<<<1, 1024, 0, st>>>(W, S, P);
    mk.mark("k_resolve2");
    ++nl;
  }
  if (n > 0) {
    int g = grid_for(k_finalize<kStaged>, smem);
    if ((uint64_t)g > ntiles) g = (int)ntiles;
    k_finalize<kStaged><<<g, BLOCK, smem, st>>>(W, S, in, n, P, out, dkeys, didx, cancel);
    mk.mark("k_finalize");
    ++nl;
  }
  *launches = nl;
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

int launch_fault_path(const World& W, const Scratch& S, const mpsf_fault_entry* in, uint64_t n,
                      const Params& P, mpsf_out_record* out, mpsf_client_verdict* verdict,
                      unsigned long long* counts, unsigned long long* dkeys, uint32_t* didx,
                      uint32_t* cancel, cudaStream_t st, int* launches, const Marker& mk) {
  if (staged_fits(W))
    return launch_all<true>(W, S, in, n, P, out, verdict, counts, dkeys, didx, cancel, st, launches, mk);
  return launch_all<false>(W, S, in, n, P, out, verdict, counts, dkeys, didx, cancel, st, launches, mk);
}

uint64_t tiles_for(uint64_t n) { return (n + TILE - 1) / TILE; }

}  // namespace mpsf
