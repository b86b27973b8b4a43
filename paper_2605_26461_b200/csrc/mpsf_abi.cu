// C ABI of libmpsf.so (declared in include/mpsf.h): context, world upload, batch
// processing, summary, host-buffer end-to-end form, remap.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <stdio.h>

#include <algorithm>
#include <map>
#include <string>
#include <vector>

#include "mpsf.h"
#include "mpsf_device.cuh"
#include "mpsf_kernels.h"

using namespace mpsf;

namespace {

struct InitSegs {
  void* p[10];
  uint64_t words[10];
  uint32_t val[10];
  int n;
};

// Clears / fills the per-batch scratch: every thread of a 1-D grid strides over each segment
// in turn (16-byte stores), so the large segments (hash tables, dedup slots) get the whole
// grid rather than a slice of it.
__global__ void k_init(InitSegs segs) {
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x, stride = (uint64_t)gridDim.x * blockDim.x;
  for (int s = 0; s < segs.n; ++s) {
    uint32_t* p = reinterpret_cast<uint32_t*>(segs.p[s]);
    const uint64_t w = segs.words[s];
    const uint32_t v = segs.val[s];
    const uint64_t w4 = w / 4;
    uint4* p4 = reinterpret_cast<uint4*>(p);
    const uint4 v4 = make_uint4(v, v, v, v);
    for (uint64_t i = tid; i < w4; i += stride) p4[i] = v4;
    for (uint64_t i = w4 * 4 + tid; i < w; i += stride) p[i] = v;
  }
}

uint64_t next_pow2(uint64_t x) {
  uint64_t p = 1;
  while (p < x) p <<= 1;
  return p;
}

size_t a256(size_t x) { return (x + 255) & ~size_t(255); }

// mpsf_process_host splits a batch into at most this many tile-aligned chunks so the
// host->device copy of chunk k+1 overlaps pass 1 on chunk k, and the device->host copy
// of chunk k's records overlaps finalize on chunk k+1
constexpr int kMaxChunks = 8;

}  // namespace

constexpr int kSlots = MPSF_HOST_SLOTS;

// One in-flight batch of the asynchronous host-buffer form.
struct HostSlot {
  uint8_t* d_io = nullptr;
  size_t io_cap = 0;
  size_t o_in = 0, o_out = 0, o_v = 0, o_cnt = 0, o_dk = 0, o_di = 0, o_ca = 0;
  DevSummary* h_sum = nullptr;     // mapped pinned
  DevSummary* d_sum = nullptr;
  cudaEvent_t ev_done = nullptr;   // every output of the slot's batch is on the host
  bool busy = false, lists_copied = false;
  uint64_t n = 0;
  mpsf_params p{};
  const mpsf_fault_entry* h_in = nullptr;
  mpsf_out_record* h_out = nullptr;
  mpsf_client_verdict* h_verdict = nullptr;
  uint64_t* h_counts = nullptr;
  uint64_t* h_dkeys = nullptr;
  uint32_t* h_didx = nullptr;
  uint32_t* h_cancel = nullptr;
};

struct mpsf_ctx {
  int device = 0;
  cudaStream_t own_stream = nullptr;
  // world
  void* d_world = nullptr;
  World W{};
  bool has_world = false;
  // scratch
  uint32_t* d_dd = nullptr;
  uint32_t* d_nr1 = nullptr;
  uint32_t* d_pf = nullptr;     // first PREFETCH per page (batched translation)
  uint32_t* d_nrall = nullptr;
  uint64_t dd_cap = 0;
  int dedup_mode = 0;            // 1 dense slots, -1 claimed slots (large-world layout), 0 by size
  // exchange-group offsets inside d_small
  size_t x_u64 = 0, x_u32 = 0, x_giso = 0;
  uint64_t x_u64_n = 0, x_u32_n = 0, x_giso_n = 0;
  // state carried between phase calls
  uint64_t phase_n = 0;
  uint32_t* d_counter = nullptr;
  uint64_t pages_cap = 0;
  uint8_t* d_small = nullptr;
  size_t small_cap = 0;
  size_t small_empty_bytes = 0, small_zero_off = 0, small_zero_bytes = 0;
  uint8_t* d_masks = nullptr;   // per-chunk masks + segment counters (pass 2)
  unsigned long long* d_drec = nullptr;   // pass-1 records (8 B per entry)
  uint64_t drec_cap = 0;
  uint64_t tiles_cap = 0;
  unsigned long long* d_hdd = nullptr;  // keys then vals
  uint64_t hcap_dd = 0;
  unsigned long long* d_hnr = nullptr;
  uint64_t hcap_nr = 0;
  uint32_t hash_gen = 0;        // the batch generation of the hash tables (bumped by every batch)
  uint64_t want_dd = 0, want_nr = 0;
  Scratch S{};
  // summary (mapped pinned host memory)
  DevSummary* h_sum = nullptr;
  DevSummary* d_sum = nullptr;
  cudaEvent_t ev_done = nullptr;
  bool pending = false;
  bool pending_fault = true;      // the pending summary is a fault-path batch (not a translation)
  uint64_t last_n = 0;
  int last_launches = 0;
  // per-kernel profiling (events recorded after every launch)
  bool profiling = false;
  std::vector<cudaEvent_t> ev_pool;
  struct Pending {
    std::string name;
    cudaEvent_t a, b;
  };
  std::vector<Pending> pend;
  std::vector<cudaEvent_t> pend_events;
  cudaEvent_t last_mark = nullptr;
  cudaStream_t mark_stream = nullptr;
  std::map<std::string, std::pair<uint64_t, double>> acc;

  cudaEvent_t new_event() {
    if (!ev_pool.empty()) {
      cudaEvent_t e = ev_pool.back();
      ev_pool.pop_back();
      return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
  }
  void mark_begin(cudaStream_t st) {
    if (!profiling) return;
    mark_stream = st;
    last_mark = new_event();
    pend_events.push_back(last_mark);
    cudaEventRecord(last_mark, st);
  }
  static void mark_cb(void* p, const char* name) {
    mpsf_ctx* c = static_cast<mpsf_ctx*>(p);
    if (!c->profiling || !c->last_mark) return;
    cudaEvent_t e = c->new_event();
    c->pend_events.push_back(e);
    cudaEventRecord(e, c->mark_stream);
    c->pend.push_back({name, c->last_mark, e});
    c->last_mark = e;
  }
  mpsf::Marker marker() {
    mpsf::Marker m;
    if (profiling) {
      m.fn = &mpsf_ctx::mark_cb;
      m.ctx = this;
    }
    return m;
  }
  uint32_t* d_remap_err = nullptr;
  uint8_t* d_fold = nullptr;    // snapshot-fold scratch (grown on demand)
  uint4* d_trstage = nullptr;   // translation: staged miss entries, 64 per chunk (grown on demand)
  uint64_t trstage_cap = 0;     // chunks
  size_t fold_cap = 0;
  // host-path buffers and the copy streams of the chunked pipeline
  HostSlot slots[kSlots];
  cudaStream_t h2d_stream = nullptr, d2h_stream = nullptr;
  cudaEvent_t ev_in[kMaxChunks] = {}, ev_fin[kMaxChunks] = {}, ev_fork = nullptr, ev_d2h = nullptr;
};

#define CK(x)                                \
  do {                                       \
    if ((x) != cudaSuccess) return MPSF_E_CUDA; \
  } while (0)

// `fault`: a fault-path batch (translation summaries carry no hash counts and must not size
// the wild-page tables)
// Wild-page hash capacity: 8x the previous batch's keys (load <= 1/8 keeps the probe runs short;
// with generation-stamped slots a larger table costs no clearing)
constexpr uint64_t kHashSlack = 8;
static void fill_summary(mpsf_ctx* c, const DevSummary& d, mpsf_summary* out, bool fault) {
  memset(out, 0, sizeof(*out));
  const uint32_t err = d.ctrl[C_ERR];
  if (err & EB_NO_CHANNEL) out->status = MPSF_E_NO_CHANNEL;
  else if (err & EB_BAD_ENTRY) out->status = MPSF_E_BAD_ENTRY;
  else if (err & EB_MISMATCH) out->status = MPSF_E_ENGINE_MISMATCH;
  else if (err & EB_VA) out->status = MPSF_E_VA_RANGE;
  else if (d.ctrl[C_OVF]) out->status = MPSF_E_OVERFLOW;
  else out->status = MPSF_OK;
  out->path = d.ctrl[C_PATH];
  out->n_dedup = d.n_dedup;
  out->n_cancel = d.n_cancel;
  out->error_index = d.err_idx;
  out->hash_used = (uint64_t)d.ctrl[C_HASH_DD] + d.ctrl[C_HASH_NR];
  // adapt the wild-page hash tables for the next call
  if (!fault) return;
  if (out->status == MPSF_E_OVERFLOW) {
    if (d.ctrl[C_HASH_DD] * 2ull >= c->hcap_dd / 2) c->want_dd = c->hcap_dd * 4;
    if (d.ctrl[C_HASH_NR] * 2ull >= c->hcap_nr / 2) c->want_nr = c->hcap_nr * 4;
    if (c->want_dd == c->hcap_dd && c->want_nr == c->hcap_nr) { c->want_dd *= 4; c->want_nr *= 4; }
  } else if (out->status == MPSF_OK) {
    c->want_dd = next_pow2(std::max<uint64_t>(1ull << 16, kHashSlack * d.ctrl[C_HASH_DD]));
    c->want_nr = next_pow2(std::max<uint64_t>(1ull << 16, kHashSlack * d.ctrl[C_HASH_NR]));
  }
}

static int slot_buffers(mpsf_ctx* c, HostSlot& h, uint64_t n) {
  const uint32_t C = c->W.n_clients;
  h.o_in = 0;
  h.o_out = a256(16 * n);
  h.o_v = h.o_out + a256(8 * n);
  h.o_cnt = h.o_v + a256(4ull * C + 4);
  h.o_dk = h.o_cnt + a256(8ull * NSCEN * C + 8);
  h.o_di = h.o_dk + a256(8 * n);
  h.o_ca = h.o_di + a256(4 * n);
  const size_t total = h.o_ca + a256(4 * n + 4);
  if (total > h.io_cap) {
    if (h.ev_done) cudaEventSynchronize(h.ev_done);
    cudaFree(h.d_io);
    h.d_io = nullptr;
    h.io_cap = 0;
    CK(cudaMalloc(&h.d_io, total));
    h.io_cap = total;
  }
  if (!h.h_sum) {
    CK(cudaHostAlloc(reinterpret_cast<void**>(&h.h_sum), sizeof(DevSummary), cudaHostAllocMapped));
    CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&h.d_sum), h.h_sum, 0));
    CK(cudaEventCreateWithFlags(&h.ev_done, cudaEventDisableTiming));
  }
  return MPSF_OK;
}

template <typename T>
static T* device_view(T* host) {      // the device address of pinned host memory, or null
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, host) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return (at.type == cudaMemoryTypeHost && at.devicePointer) ? reinterpret_cast<T*>(at.devicePointer) : nullptr;
}

extern "C" {


int mpsf_version(void) { return MPSF_ABI_VERSION; }

const char* mpsf_strerror(int code) {
  switch (code) {
    case MPSF_OK: return "ok";
    case MPSF_E_CUDA: return "CUDA error (see cudaGetLastError)";
    case MPSF_E_ARG: return "invalid argument";
    case MPSF_E_NO_CHANNEL: return "fault entry channel has no client attribution";
    case MPSF_E_BAD_ENTRY: return "malformed fault entry (engine/access/kind)";
    case MPSF_E_ENGINE_MISMATCH: return "fault entry engine differs from its channel's engine";
    case MPSF_E_VA_RANGE: return "fault VA >= 2^53";
    case MPSF_E_WORLD: return "interval table not sorted/aligned/disjoint or inconsistent TSG state";
    case MPSF_E_OVERFLOW: return "wild-page hash table overflowed; call again (it has grown)";
    case MPSF_E_NO_WORLD: return "no world uploaded";
    case MPSF_E_TOO_LARGE: return "base_index + n exceeds 2^29 entries";
    default: return "unknown error";
  }
}

int mpsf_create(mpsf_ctx** out, int device) {
  if (!out) return MPSF_E_ARG;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) return MPSF_E_CUDA;
  CK(cudaSetDevice(device));
  mpsf_ctx* c = new mpsf_ctx();
  c->device = device;
  if (cudaStreamCreateWithFlags(&c->own_stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_done, cudaEventDisableTiming) != cudaSuccess ||
      cudaHostAlloc(reinterpret_cast<void**>(&c->h_sum), sizeof(DevSummary), cudaHostAllocMapped) != cudaSuccess ||
      cudaHostGetDevicePointer(reinterpret_cast<void**>(&c->d_sum), c->h_sum, 0) != cudaSuccess ||
      cudaMalloc(&c->d_remap_err, sizeof(uint32_t)) != cudaSuccess ||
      cudaStreamCreateWithFlags(&c->h2d_stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&c->d2h_stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_d2h, cudaEventDisableTiming) != cudaSuccess) {
    mpsf_destroy(c);
    return MPSF_E_CUDA;
  }
  for (int k = 0; k < kMaxChunks; ++k) {
    if (cudaEventCreateWithFlags(&c->ev_in[k], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_fin[k], cudaEventDisableTiming) != cudaSuccess) {
      mpsf_destroy(c);
      return MPSF_E_CUDA;
    }
  }
  memset(c->h_sum, 0, sizeof(DevSummary));
  *out = c;
  return MPSF_OK;
}

void mpsf_destroy(mpsf_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  cudaDeviceSynchronize();
  cudaFree(c->d_world);
  cudaFree(c->d_dd);
  cudaFree(c->d_nr1);
  cudaFree(c->d_nrall);
  cudaFree(c->d_counter);
  cudaFree(c->d_small);
  cudaFree(c->d_masks);
  cudaFree(c->d_pf);
  cudaFree(c->d_drec);
  cudaFree(c->d_hdd);
  cudaFree(c->d_hnr);
  for (int k = 0; k < kSlots; ++k) {
    cudaFree(c->slots[k].d_io);
    if (c->slots[k].h_sum) cudaFreeHost(c->slots[k].h_sum);
    if (c->slots[k].ev_done) cudaEventDestroy(c->slots[k].ev_done);
  }
  cudaFree(c->d_remap_err);
  cudaFree(c->d_fold);
  cudaFree(c->d_trstage);
  for (cudaEvent_t e : c->ev_pool) cudaEventDestroy(e);
  for (cudaEvent_t e : c->pend_events) cudaEventDestroy(e);
  if (c->h_sum) cudaFreeHost(c->h_sum);
  if (c->ev_done) cudaEventDestroy(c->ev_done);
  for (int k = 0; k < kMaxChunks; ++k) {
    if (c->ev_in[k]) cudaEventDestroy(c->ev_in[k]);
    if (c->ev_fin[k]) cudaEventDestroy(c->ev_fin[k]);
  }
  if (c->ev_fork) cudaEventDestroy(c->ev_fork);
  if (c->ev_d2h) cudaEventDestroy(c->ev_d2h);
  if (c->h2d_stream) cudaStreamDestroy(c->h2d_stream);
  if (c->d2h_stream) cudaStreamDestroy(c->d2h_stream);
  if (c->own_stream) cudaStreamDestroy(c->own_stream);
  delete c;
}

int mpsf_upload_world(mpsf_ctx* c, const mpsf_range_entry* ranges, uint32_t nr, const uint8_t* page_state,
                      uint64_t np, const mpsf_channel_entry* channels, uint32_t nch,
                      const mpsf_client_entry* clients, uint32_t ncl, uint32_t world_flags) {
  if (!c || (nr && !ranges) || (np && !page_state) || (nch && !channels) || (ncl && !clients)) return MPSF_E_ARG;
  if (ncl > 65535) return MPSF_E_ARG;
  CK(cudaSetDevice(c->device));
  // validation: sorted by (client, base), 4 KiB aligned, disjoint per client, slots in range
  std::vector<uint32_t> off(ncl + 1, 0);
  for (uint32_t i = 0; i < nr; ++i) {
    const mpsf_range_entry& r = ranges[i];
    if (r.client >= ncl || r.base >= r.end || (r.base & 0xFFF) || (r.end & 0xFFF)) return MPSF_E_WORLD;
    if (r.kind > 1 || r.lifecycle > 1 || r.migratable > 1) return MPSF_E_WORLD;   // RangeKind / Lifecycle / bool
    if (i > 0) {
      const mpsf_range_entry& p = ranges[i - 1];
      if (p.client > r.client) return MPSF_E_WORLD;
      if (p.client == r.client && p.end > r.base) return MPSF_E_WORLD;
    }
    const uint64_t npg = (r.end - r.base) >> 12;
    if ((uint64_t)r.page_off + npg + 1 > np) return MPSF_E_WORLD;
    off[r.client + 1]++;
  }
  for (uint32_t i = 0; i < ncl; ++i) off[i + 1] += off[i];
  uint32_t has_mps = 0;
  for (uint32_t i = 0; i < ncl; ++i) {
    if (clients[i].mode > 1) return MPSF_E_WORLD;
    if (clients[i].mode == 0) {
      has_mps = 1;
      if ((world_flags & MPSF_WF_GR_DEAD) && (clients[i].flags & 1)) return MPSF_E_WORLD;
    }
  }
  for (uint32_t i = 0; i < nch; ++i)
    if (channels[i].engine > 2) return MPSF_E_WORLD;
  if (nr > 65535) return MPSF_E_WORLD;
  // page-granular SoA interval table (padded with one sentinel row) + per-client skip tables
  std::vector<uint32_t> pg_base(nr + 1), pg_end(nr + 1), poff(nr + 1), rattr(nr + 1), rrid(nr + 1);
  for (uint32_t i = 0; i < nr; ++i) {
    const mpsf_range_entry& r = ranges[i];
    if (r.end > VA_TABLE_LIMIT) return MPSF_E_WORLD;
    pg_base[i] = (uint32_t)(r.base >> 12);
    pg_end[i] = (uint32_t)(r.end >> 12);
    poff[i] = r.page_off;
    rattr[i] = (uint32_t)r.kind | ((uint32_t)r.lifecycle << 8) | ((uint32_t)r.migratable << 16) |
               ((uint32_t)r.state << 24);
    rrid[i] = r.rid;
  }
  pg_base[nr] = 0xFFFFFFFFu; pg_end[nr] = 0; poff[nr] = 0; rattr[nr] = 0; rrid[nr] = NO_RID;
  // skip tables: slot size 2^sh <= the smallest gap between two consecutive bases, so a slot
  // holds at most one base and attribution is one table read plus at most one step
  std::vector<uint16_t> skip;
  std::vector<uint32_t> cinfo(4ull * std::max<uint32_t>(ncl, 1), 0);
  uint32_t exact1 = 1;
  for (uint32_t cl = 0; cl < ncl; ++cl) {
    const uint32_t lo = off[cl], hi = off[cl + 1];
    uint32_t* ci = &cinfo[4ull * cl];
    ci[0] = lo | (hi << 16);
    ci[3] = (uint32_t)skip.size();
    if (lo == hi) continue;
    const uint64_t span_lo = pg_base[lo], span_hi = (uint64_t)pg_end[hi - 1] + 1;
    uint64_t gap = span_hi - span_lo;
    for (uint32_t i = lo + 1; i < hi; ++i) gap = std::min<uint64_t>(gap, (uint64_t)pg_base[i] - pg_base[i - 1]);
    uint32_t sh = 0;
    while ((2ull << sh) <= gap) ++sh;
    auto slots_for = [&](uint32_t s_) { return (span_hi - span_lo + (1ull << s_) - 1) >> s_; };
    while (slots_for(sh) > SKIP_MAX) { ++sh; exact1 = 0; }
    const uint64_t slots = slots_for(sh);
    ci[1] = (uint32_t)span_lo;
    ci[2] = sh | ((uint32_t)(slots - 1) << 8);
    uint32_t k = lo;
    for (uint64_t j = 0; j < slots; ++j) {
      const uint64_t st = span_lo + (j << sh);
      while (k + 1 < hi && pg_base[k + 1] <= st) ++k;
      skip.push_back((uint16_t)k);
    }
  }
  const uint32_t n_skip = (uint32_t)skip.size();
  skip.push_back(0);
  std::vector<uint32_t> chan(nch + 1, 0);
  for (uint32_t i = 0; i < nch; ++i) {
    const uint32_t cl = channels[i].client;
    chan[i] = cl < ncl ? ((cl & 0xFFFFu) | ((uint32_t)channels[i].engine << 16) |
                          ((uint32_t)(clients[cl].mode & 1) << 18) | CH_VALID)
                       : 0u;
  }
  // row form for the streaming passes (mpsf_device.cuh World::chan4 / skip2 / row4)
  std::vector<uint32_t> chan4(4ull * (nch + 1), 0), skip2(2ull * (skip.size()), 0), row4(4ull * (nr + 1), 0);
  for (uint32_t i = 0; i <= nch; ++i) {
    uint32_t* o = &chan4[4ull * i];
    o[0] = chan[i];
    o[3] = n_skip;                                    // no ranges: the sentinel slot, jmax 0
    if (i < nch && (chan[i] & CH_VALID)) {
      const uint32_t* ci = &cinfo[4ull * (chan[i] & 0xFFFFu)];
      if ((ci[0] & 0xFFFFu) != (ci[0] >> 16)) {
        o[1] = ci[1];
        o[2] = ci[2] & 31u;
        o[3] = ci[3] | ((ci[2] >> 8) << 16);
      }
    }
  }
  for (uint32_t cl = 0; cl < ncl; ++cl) {
    const uint32_t* ci = &cinfo[4ull * cl];
    const uint32_t lo = ci[0] & 0xFFFFu, hi = ci[0] >> 16;
    if (lo == hi) continue;
    const uint32_t sh = ci[2] & 31u, slots = (ci[2] >> 8) + 1;
    for (uint32_t j = 0; j < slots; ++j) {
      const uint32_t k = skip[ci[3] + j];
      const uint64_t end_slot = (uint64_t)ci[1] + ((uint64_t)(j + 1) << sh);
      skip2[2ull * (ci[3] + j)] = k;
      skip2[2ull * (ci[3] + j) + 1] = (k + 1 < hi && pg_base[k + 1] < end_slot) ? pg_base[k + 1] : 0xFFFFFFFFu;
    }
  }
  skip2[2ull * n_skip] = nr;                          // sentinel slot -> sentinel row
  skip2[2ull * n_skip + 1] = 0xFFFFFFFFu;
  for (uint32_t i = 0; i < nr; ++i) {
    const mpsf_range_entry& r = ranges[i];
    row4[4ull * i] = pg_base[i];
    row4[4ull * i + 1] = pg_end[i];
    row4[4ull * i + 2] = r.page_off;
    row4[4ull * i + 3] = (r.state == 0xFF ? ROW_PERPAGE : (uint32_t)(r.state & 7u)) |
                         (((uint32_t)r.kind | ((uint32_t)r.lifecycle << 1) | ((uint32_t)r.migratable << 2)) << 3);
  }
  row4[4ull * nr] = 0xFFFFFFFFu;                      // sentinel: no page is in it or its guard
  row4[4ull * nr + 1] = 0xFFFFFFFFu;
  const size_t o_r = 0, o_off = a256(o_r + sizeof(mpsf_range_entry) * nr);
  const size_t o_ps = a256(o_off + sizeof(uint32_t) * (ncl + 1));
  const size_t o_ch = a256(o_ps + np);
  const size_t o_cl = a256(o_ch + sizeof(mpsf_channel_entry) * nch);
  const size_t o_soa = a256(o_cl + sizeof(mpsf_client_entry) * ncl);
  const size_t o_skip = a256(o_soa + 5ull * 4 * (nr + 1));
  const size_t o_cinfo4 = a256(o_skip + 2ull * skip.size());
  const size_t o_chan = a256(o_cinfo4 + 4ull * cinfo.size());
  const size_t o_chan4 = a256(o_chan + 4ull * chan.size());
  const size_t o_skip2 = a256(o_chan4 + 4ull * chan4.size());
  const size_t o_row4 = a256(o_skip2 + 4ull * skip2.size());
  const size_t total = a256(o_row4 + 4ull * row4.size()) + 256;
  cudaFree(c->d_world);
  c->d_world = nullptr;
  c->has_world = false;
  CK(cudaMalloc(&c->d_world, total));
  uint8_t* b = reinterpret_cast<uint8_t*>(c->d_world);
  if (nr) CK(cudaMemcpy(b + o_r, ranges, sizeof(mpsf_range_entry) * nr, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(b + o_off, off.data(), sizeof(uint32_t) * (ncl + 1), cudaMemcpyHostToDevice));
  if (np) CK(cudaMemcpy(b + o_ps, page_state, np, cudaMemcpyHostToDevice));
  if (nch) CK(cudaMemcpy(b + o_ch, channels, sizeof(mpsf_channel_entry) * nch, cudaMemcpyHostToDevice));
  if (ncl) CK(cudaMemcpy(b + o_cl, clients, sizeof(mpsf_client_entry) * ncl, cudaMemcpyHostToDevice));
  uint32_t* soa = reinterpret_cast<uint32_t*>(b + o_soa);
  const size_t R1 = nr + 1;
  CK(cudaMemcpy(soa, pg_base.data(), 4 * R1, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(soa + R1, pg_end.data(), 4 * R1, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(soa + 2 * R1, poff.data(), 4 * R1, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(soa + 3 * R1, rattr.data(), 4 * R1, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(soa + 4 * R1, rrid.data(), 4 * R1, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(b + o_skip, skip.data(), 2ull * skip.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(b + o_cinfo4, cinfo.data(), 4ull * cinfo.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(b + o_chan, chan.data(), 4ull * chan.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(b + o_chan4, chan4.data(), 4ull * chan4.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(b + o_skip2, skip2.data(), 4ull * skip2.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(b + o_row4, row4.data(), 4ull * row4.size(), cudaMemcpyHostToDevice));
  World& W = c->W;
  W.ranges = reinterpret_cast<const mpsf_range_entry*>(b + o_r);
  W.client_off = reinterpret_cast<const uint32_t*>(b + o_off);
  W.page_state = b + o_ps;
  W.channels = reinterpret_cast<const mpsf_channel_entry*>(b + o_ch);
  W.clients = reinterpret_cast<const mpsf_client_entry*>(b + o_cl);
  W.pg_base = soa;
  W.pg_end = soa + R1;
  W.poff = soa + 2 * R1;
  W.rattr = soa + 3 * R1;
  W.rrid = soa + 4 * R1;
  W.skip = reinterpret_cast<const uint16_t*>(b + o_skip);
  W.cinfo4 = reinterpret_cast<const uint4*>(b + o_cinfo4);
  W.chan = reinterpret_cast<const uint32_t*>(b + o_chan);
  W.chan4 = reinterpret_cast<const uint4*>(b + o_chan4);
  W.skip2 = reinterpret_cast<const uint2*>(b + o_skip2);
  W.row4 = reinterpret_cast<const uint4*>(b + o_row4);
  W.n_skip = n_skip;
  W.exact1 = exact1;
  W.n_ranges = nr;
  W.n_clients = ncl;
  W.n_channels = nch;
  W.world_flags = world_flags;
  W.n_pages = np;
  W.has_mps = has_mps;
  // dedup slots: one per (page, group) while that stays small (L2-resident), else one
  // claimed slot per page with overflow to the hash table
  // (mpsf_set_dense_dedup forces either layout: dense for sharded runs, claimed slots to test the
  // large-world path on small worlds)
  W.dd_groups = c->dedup_mode > 0 ? 5 : c->dedup_mode < 0 ? 1 : (np * 5 * 4 <= (64ull << 20)) ? 5 : 1;
  // page-sized scratch
  const uint64_t dd_words = np * W.dd_groups;
  if (!c->d_dd || dd_words > c->dd_cap || np > c->pages_cap) {
    cudaFree(c->d_dd);
    cudaFree(c->d_nr1);
    cudaFree(c->d_nrall);
    c->d_dd = c->d_nr1 = c->d_nrall = nullptr;
    c->pages_cap = c->dd_cap = 0;
    CK(cudaMalloc(&c->d_dd, sizeof(uint32_t) * std::max<uint64_t>(dd_words, 1)));
    CK(cudaMalloc(&c->d_nr1, sizeof(uint32_t) * std::max<uint64_t>(np, 1)));
    cudaFree(c->d_pf);
    c->d_pf = nullptr;
    CK(cudaMalloc(&c->d_pf, sizeof(uint32_t) * std::max<uint64_t>(np, 1)));
    CK(cudaMalloc(&c->d_nrall, sizeof(uint32_t) * std::max<uint64_t>(np, 1)));
    c->pages_cap = np;
    c->dd_cap = dd_words;
  }
  // small scratch: [EMPTY-init][ZERO-init][uninit]
  const uint32_t C = ncl, R = nr;
  size_t o = 0;
  auto take = [&](size_t bytes) { size_t r = o; o = (o + bytes + 15) & ~size_t(15); return r; };
  // exchange groups are contiguous: u64 minima [ft_ce | ft_sa | trap_sa | ft_gr | trap_mps],
  // u32 minima [nr0 | ext | iso1 | iso2 | iso3], general-path u32 minima [giso]
  const size_t s_u64 = take(8ull * (3ull * C + 2));
  const size_t s_u32 = take(4ull * (2ull * R + 3ull * C));
  const size_t s_giso = take(12ull * C), s_glob = take(sizeof(Globals)), s_err = take(8);
  c->x_u64 = s_u64; c->x_u64_n = 3ull * C + 2;
  c->x_u32 = s_u32; c->x_u32_n = 2ull * R + 3ull * C;
  c->x_giso = s_giso; c->x_giso_n = 3ull * C;
  const size_t empty_bytes = o;
  const size_t s_ctrl = take(4 * C_NCTRL);
  const size_t zero_bytes = o - empty_bytes;
  const size_t s_cst = take(sizeof(CState) * std::max<uint32_t>(C, 1));
  const size_t s_fcl = take(sizeof(FinClient) * std::max<uint32_t>(C, 1));
  if (o > c->small_cap) {
    cudaFree(c->d_small);
    c->d_small = nullptr;
    c->small_cap = 0;
    CK(cudaMalloc(&c->d_small, o));
    c->small_cap = o;
  }
  c->small_empty_bytes = empty_bytes;
  c->small_zero_off = empty_bytes;
  c->small_zero_bytes = zero_bytes;
  uint8_t* s = c->d_small;
  Scratch& S = c->S;
  S.dd = c->d_dd;
  S.nr1 = c->d_nr1;
  S.pf = c->d_pf;
  // per-page first-eligible keys only for dense (small) worlds; large worlds take the
  // release-aware pass instead when a client is released before the drain
  S.nrall = W.dd_groups == 5 ? c->d_nrall : nullptr;
  unsigned long long* u64 = reinterpret_cast<unsigned long long*>(s + s_u64);
  S.ft_ce = u64;
  S.ft_sa = u64 + C;
  S.trap_sa = u64 + 2ull * C;
  S.ft_gr = u64 + 3ull * C;
  S.trap_mps = u64 + 3ull * C + 1;
  uint32_t* u32 = reinterpret_cast<uint32_t*>(s + s_u32);
  S.nr0 = u32;
  S.ext = u32 + R;
  S.iso1 = u32 + 2ull * R;
  S.iso2 = u32 + 2ull * R + C;
  S.iso3 = u32 + 2ull * R + 2ull * C;
  S.giso = reinterpret_cast<uint32_t*>(s + s_giso);
  S.glob = reinterpret_cast<Globals*>(s + s_glob);
  S.err_idx = reinterpret_cast<unsigned long long*>(s + s_err);
  S.ctrl = reinterpret_cast<uint32_t*>(s + s_ctrl);
  S.cstate = reinterpret_cast<CState*>(s + s_cst);
  S.fclient = reinterpret_cast<FinClient*>(s + s_fcl);
  c->has_world = true;
  return MPSF_OK;
}

static int ensure_call_scratch(mpsf_ctx* c, uint64_t n) {
  const uint64_t nq = chunks_for(n), nseg = segments_for(n);
  const uint64_t mbytes = (16 + 8 * 64) * std::max<uint64_t>(nq, 1) + 16 * std::max<uint64_t>(nseg, 1);
  if (mbytes > c->tiles_cap) {
    cudaFree(c->d_masks);
    c->d_masks = nullptr;
    c->tiles_cap = 0;
    CK(cudaMalloc(&c->d_masks, mbytes));
    c->tiles_cap = mbytes;
  }
  if (n > c->drec_cap) {
    cudaFree(c->d_drec);
    c->d_drec = nullptr;
    c->drec_cap = 0;
    CK(cudaMalloc(&c->d_drec, 8 * std::max<uint64_t>(n, 2)));
    c->drec_cap = n;
  }
  c->S.drec = c->d_drec;
  c->S.cmask = reinterpret_cast<uint4*>(c->d_masks);
  c->S.dstage = reinterpret_cast<unsigned long long*>(c->d_masks + 16 * std::max<uint64_t>(nq, 1));
  c->S.segcnt = c->S.dstage + 64 * std::max<uint64_t>(nq, 1);
  c->S.segbase = c->S.segcnt + std::max<uint64_t>(nseg, 1);
  const uint64_t floor_cap = 1ull << 16;
  if (c->want_dd == 0 || c->last_n != n) {
    const uint64_t guess = next_pow2(std::max<uint64_t>(floor_cap, std::min<uint64_t>(n / 32, 1ull << 24)));
    c->want_dd = std::max(c->want_dd, guess);
    c->want_nr = std::max(c->want_nr, guess);
  }
  if (c->want_dd != c->hcap_dd) {
    cudaFree(c->d_hdd);
    c->d_hdd = nullptr;
    c->hcap_dd = 0;
    CK(cudaMalloc(&c->d_hdd, 16 * c->want_dd));
    CK(cudaMemset(c->d_hdd, 0, 16 * c->want_dd));   // generation 0: free in every batch
    c->hcap_dd = c->want_dd;
  }
  if (c->want_nr != c->hcap_nr) {
    cudaFree(c->d_hnr);
    c->d_hnr = nullptr;
    c->hcap_nr = 0;
    CK(cudaMalloc(&c->d_hnr, 16 * c->want_nr));
    CK(cudaMemset(c->d_hnr, 0, 16 * c->want_nr));
    c->hcap_nr = c->want_nr;
  }
  Scratch& S = c->S;
  S.hdd.keys = c->d_hdd;
  S.hdd.mask = (uint32_t)(c->hcap_dd - 1);
  S.hdd.used_slot = C_HASH_DD;
  S.hnr.keys = c->d_hnr;
  S.hnr.mask = (uint32_t)(c->hcap_nr - 1);
  S.hnr.used_slot = C_HASH_NR;
  return MPSF_OK;
}

static Params to_params(const mpsf_params* p) {
  Params P;
  P.flags = p->flags;
  P.benign_us = p->benign_us;
  P.m1_us = p->m1_us;
  P.m2_us = p->m2_us;
  P.m3_us = p->m3_us;
  P.base_index = p->base_index;
  return P;
}

int mpsf_set_dense_dedup(mpsf_ctx* c, int on) {
  if (!c) return MPSF_E_ARG;
  c->dedup_mode = on > 0 ? 1 : on < 0 ? -1 : 0;
  return MPSF_OK;
}

// phase 1: clear scratch + k_scan
static int batch_init(mpsf_ctx* c, uint64_t n, const mpsf_params* p, uint64_t* d_counts, cudaStream_t st);
static int scan_chunk(mpsf_ctx* c, const mpsf_fault_entry* d_chunk, uint64_t n_chunk, uint64_t chunk_off,
                      const mpsf_params* p, uint64_t* d_counts, cudaStream_t st);

int mpsf_scan(mpsf_ctx* c, const mpsf_fault_entry* d_in, uint64_t n, const mpsf_params* p, uint64_t* d_counts,
              void* stream) {
  if (!c || !p) return MPSF_E_ARG;
  if (!c->has_world) return MPSF_E_NO_WORLD;
  if (n && !d_in) return MPSF_E_ARG;
  if (c->W.n_clients && !d_counts) return MPSF_E_ARG;
  if (p->base_index + n > MAX_GIDX) return MPSF_E_TOO_LARGE;
  CK(cudaSetDevice(c->device));
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  int rc = batch_init(c, n, p, d_counts, st);
  if (!rc) rc = scan_chunk(c, d_in, n, 0, p, d_counts, st);
  c->last_launches = n ? 2 : 1;
  return rc;
}

// clear the per-batch scratch (k_init) and size it for n entries
static int batch_init(mpsf_ctx* c, uint64_t n, const mpsf_params* p, uint64_t* d_counts, cudaStream_t st) {
  int rc = ensure_call_scratch(c, n);
  if (rc) return rc;
  c->S.drec_base = p->base_index;
  InitSegs segs{};
  int k = 0;
  // (pass 1 probes the dedup slots and first-eligible keys at random: they are cleared last, so
  // they are the freshest lines in L2 when it starts; nr1 is only read by the release-aware pass)
  if (p->flags & MPSF_PF_ISOLATION) { segs.p[k] = c->d_nr1; segs.words[k] = c->W.n_pages; segs.val[k++] = EMPTY32; }
  segs.p[k] = c->d_small; segs.words[k] = c->small_empty_bytes / 4; segs.val[k++] = EMPTY32;
  segs.p[k] = c->d_small + c->small_zero_off; segs.words[k] = c->small_zero_bytes / 4; segs.val[k++] = 0;
  segs.p[k] = c->S.segcnt; segs.words[k] = 2 * segments_for(n); segs.val[k++] = 0;
  // (the wild-page hash tables need no clearing: a new generation frees every slot)
  if (++c->hash_gen == 0) c->hash_gen = 1;
  c->S.hdd.gen = c->S.hnr.gen = c->hash_gen;
  if (c->W.n_clients) { segs.p[k] = d_counts; segs.words[k] = 2ull * NSCEN * c->W.n_clients; segs.val[k++] = 0; }
  if ((p->flags & MPSF_PF_ISOLATION) && c->S.nrall) {
    segs.p[k] = c->S.nrall; segs.words[k] = c->W.n_pages; segs.val[k++] = EMPTY32;
  }
  segs.p[k] = c->d_dd; segs.words[k] = c->W.n_pages * c->W.dd_groups; segs.val[k++] = EMPTY32;
  segs.n = k;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device);
  c->mark_begin(st);
  k_init<<<dim3(8 * sms), 256, 0, st>>>(segs);
  c->marker().mark("k_init");
  c->phase_n = n;
  CK(cudaGetLastError());
  return MPSF_OK;
}

// pass 1 over entries [chunk_off, chunk_off + n_chunk) of the batch (d_chunk points at them)
static int scan_chunk(mpsf_ctx* c, const mpsf_fault_entry* d_chunk, uint64_t n_chunk, uint64_t chunk_off,
                      const mpsf_params* p, uint64_t* d_counts, cudaStream_t st) {
  Params P = to_params(p);
  P.base_index += chunk_off;
  if (launch_scan(c->W, c->S, d_chunk, n_chunk, P, reinterpret_cast<unsigned long long*>(d_counts),
                  st, c->marker()))
    return MPSF_E_CUDA;
  return MPSF_OK;
}

int mpsf_resolve(mpsf_ctx* c, const mpsf_params* p, mpsf_client_verdict* d_verdict, uint64_t* d_counts,
                 void* stream) {
  if (!c || !p) return MPSF_E_ARG;
  if (c->W.n_clients && (!d_verdict || !d_counts)) return MPSF_E_ARG;
  CK(cudaSetDevice(c->device));
  if (launch_resolve(c->W, c->S, to_params(p), d_verdict, reinterpret_cast<cudaStream_t>(stream), c->marker()))
    return MPSF_E_CUDA;
  c->last_launches += 1;
  return MPSF_OK;
}

int mpsf_general(mpsf_ctx* c, const mpsf_fault_entry* d_in, uint64_t n, const mpsf_params* p, int stage,
                 void* stream) {
  if (!c || !p || (stage != 1 && stage != 2)) return MPSF_E_ARG;
  if (!(p->flags & MPSF_PF_ISOLATION) || n == 0) return MPSF_OK;
  CK(cudaSetDevice(c->device));
  if (launch_general(c->W, c->S, d_in, n, to_params(p), stage, reinterpret_cast<cudaStream_t>(stream), c->marker()))
    return MPSF_E_CUDA;
  c->last_launches += 1;
  return MPSF_OK;
}

int mpsf_resolve2(mpsf_ctx* c, const mpsf_params* p, void* stream) {
  if (!c || !p) return MPSF_E_ARG;
  if (!(p->flags & MPSF_PF_ISOLATION)) return MPSF_OK;
  CK(cudaSetDevice(c->device));
  if (launch_resolve2(c->W, c->S, to_params(p), reinterpret_cast<cudaStream_t>(stream), c->marker()))
    return MPSF_E_CUDA;
  c->last_launches += 1;
  return MPSF_OK;
}

int mpsf_finalize(mpsf_ctx* c, const mpsf_fault_entry* d_in, uint64_t n, const mpsf_params* p,
                  mpsf_out_record* d_out, uint64_t* d_dkeys, uint32_t* d_didx, uint32_t* d_cancel, void* stream) {
  if (!c || !p) return MPSF_E_ARG;
  if (n && (!d_in || !d_out || !d_dkeys || !d_didx || !d_cancel)) return MPSF_E_ARG;
  if (n != c->phase_n) return MPSF_E_ARG;
  CK(cudaSetDevice(c->device));
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const Marker mk = c->marker();
  if (launch_finalize(c->W, c->S, d_in, n, to_params(p), d_out, 0, st, mk)) return MPSF_E_CUDA;
  if (launch_lists(c->S, d_in, d_out, n, p->base_index, reinterpret_cast<unsigned long long*>(d_dkeys), d_didx,
                   d_cancel, c->d_sum, st, mk))
    return MPSF_E_CUDA;
  CK(cudaEventRecord(c->ev_done, st));
  c->pending = true;
  c->pending_fault = true;
  c->last_n = n;
  c->last_launches += n ? 2 : 1;
  return MPSF_OK;
}

// Between the passes of a single-GPU batch: the client resolution and, when a client needs it,
// the release-aware pass.  On the fixed layout with isolation on, k_resolve + k_general stage 1 are
// one launch and pass 2 folds in k_resolve2; otherwise the separate kernels of the phase API.
static int mid_phases(mpsf_ctx* c, const mpsf_fault_entry* d_in, uint64_t n, const mpsf_params* p,
                      mpsf_client_verdict* d_verdict, cudaStream_t st, int& launches) {
  const Marker mk = c->marker();
  const Params P = to_params(p);
  const bool iso = (p->flags & MPSF_PF_ISOLATION) && n;
  if (iso && resolve_fused_fits(c->W)) {
    if (launch_resolve_general(c->W, c->S, d_in, n, P, d_verdict, st, mk)) return MPSF_E_CUDA;
    ++launches;
    if (p->m2_us <= p->benign_us) {
      if (launch_general(c->W, c->S, d_in, n, P, 2, st, mk)) return MPSF_E_CUDA;
      ++launches;
    }
    return MPSF_OK;
  }
  if (launch_resolve(c->W, c->S, P, d_verdict, st, mk)) return MPSF_E_CUDA;
  ++launches;
  if (iso) {
    if (launch_general(c->W, c->S, d_in, n, P, 1, st, mk)) return MPSF_E_CUDA;
    ++launches;
    if (p->m2_us <= p->benign_us) {
      if (launch_general(c->W, c->S, d_in, n, P, 2, st, mk)) return MPSF_E_CUDA;
      ++launches;
    }
    if (launch_resolve2(c->W, c->S, P, st, mk)) return MPSF_E_CUDA;
    ++launches;
  }
  return MPSF_OK;
}

int mpsf_process(mpsf_ctx* c, const mpsf_fault_entry* d_in, uint64_t n, const mpsf_params* p,
                 mpsf_out_record* d_out, mpsf_client_verdict* d_verdict, uint64_t* d_counts,
                 uint64_t* d_dkeys, uint32_t* d_didx, uint32_t* d_cancel, void* stream) {
  if (!c || !p) return MPSF_E_ARG;
  if (n && (!d_in || !d_out || !d_dkeys || !d_didx || !d_cancel)) return MPSF_E_ARG;
  if (c->W.n_clients && (!d_verdict || !d_counts)) return MPSF_E_ARG;
  int rc = mpsf_scan(c, d_in, n, p, d_counts, stream);
  if (!rc) {
    int launches = 0;
    rc = mid_phases(c, d_in, n, p, d_verdict, reinterpret_cast<cudaStream_t>(stream), launches);
    c->last_launches += launches;
  }
  if (!rc) rc = mpsf_finalize(c, d_in, n, p, d_out, d_dkeys, d_didx, d_cancel, stream);
  return rc;
}

int mpsf_classify(mpsf_ctx* c, const mpsf_fault_entry* d_in, uint64_t n, uint64_t base_index, uint8_t* d_scenario,
                  uint32_t* d_rid, void* stream) {
  if (!c) return MPSF_E_ARG;
  if (!c->has_world) return MPSF_E_NO_WORLD;
  if (n && (!d_in || !d_scenario || !d_rid)) return MPSF_E_ARG;
  if (base_index + n > MAX_GIDX) return MPSF_E_TOO_LARGE;
  CK(cudaSetDevice(c->device));
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  InitSegs segs{};
  int k = 0;
  segs.p[k] = c->d_small; segs.words[k] = c->small_empty_bytes / 4; segs.val[k++] = EMPTY32;
  segs.p[k] = c->d_small + c->small_zero_off; segs.words[k] = c->small_zero_bytes / 4; segs.val[k++] = 0;
  segs.n = k;
  c->mark_begin(st);
  k_init<<<dim3(16), 256, 0, st>>>(segs);
  CK(cudaGetLastError());
  mpsf_params p{};
  p.base_index = base_index;
  if (launch_classify(c->W, c->S, d_in, n, to_params(&p), d_scenario, d_rid, c->d_sum, st, c->marker()))
    return MPSF_E_CUDA;
  CK(cudaEventRecord(c->ev_done, st));
  c->pending = true;
  c->pending_fault = false;
  c->last_launches = n ? 3 : 2;
  return MPSF_OK;
}

int mpsf_translate_prefetch(mpsf_ctx* c, const mpsf_fault_entry* d_acc, uint64_t n, uint64_t base_index,
                            void* stream) {
  if (!c) return MPSF_E_ARG;
  if (!c->has_world) return MPSF_E_NO_WORLD;
  if (n && !d_acc) return MPSF_E_ARG;
  if (base_index + n > MAX_GIDX) return MPSF_E_TOO_LARGE;
  CK(cudaSetDevice(c->device));
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  int rc = ensure_call_scratch(c, n);
  if (rc) return rc;
  const uint64_t nq = std::max<uint64_t>(chunks_for(n), 1);
  if (nq > c->trstage_cap) {
    CK(cudaStreamSynchronize(st));
    cudaFree(c->d_trstage);
    c->d_trstage = nullptr;
    c->trstage_cap = 0;
    CK(cudaMalloc(&c->d_trstage, 16ull * 64 * nq));
    c->trstage_cap = nq;
  }
  c->S.trstage = c->d_trstage;
  InitSegs segs{};
  int k = 0;
  segs.p[k] = c->d_pf; segs.words[k] = c->W.n_pages; segs.val[k++] = EMPTY32;
  segs.p[k] = c->d_small; segs.words[k] = c->small_empty_bytes / 4; segs.val[k++] = EMPTY32;
  segs.p[k] = c->d_small + c->small_zero_off; segs.words[k] = c->small_zero_bytes / 4; segs.val[k++] = 0;
  segs.p[k] = c->S.segcnt; segs.words[k] = 2 * segments_for(n); segs.val[k++] = 0;
  segs.n = k;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device);
  c->mark_begin(st);
  k_init<<<dim3(8 * sms), 256, 0, st>>>(segs);
  c->marker().mark("k_init");
  mpsf_params p{};
  p.base_index = base_index;
  if (launch_translate_prefetch(c->W, c->S, d_acc, n, to_params(&p), st, c->marker())) return MPSF_E_CUDA;
  c->phase_n = n;
  c->last_launches = n ? 2 : 1;
  return MPSF_OK;
}

int mpsf_translate_finish(mpsf_ctx* c, const mpsf_fault_entry* d_acc, uint64_t n, uint64_t base_index,
                          uint8_t* d_hit, mpsf_fault_entry* d_faults, uint32_t* d_fault_idx, uint32_t* d_pop_idx,
                          void* stream) {
  if (!c) return MPSF_E_ARG;
  if (!c->has_world) return MPSF_E_NO_WORLD;
  if (n && (!d_acc || !d_hit || !d_faults || !d_fault_idx || !d_pop_idx)) return MPSF_E_ARG;
  if (base_index + n > MAX_GIDX) return MPSF_E_TOO_LARGE;
  if (n != c->phase_n) return MPSF_E_ARG;        // the batch mpsf_translate_prefetch started
  CK(cudaSetDevice(c->device));
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  mpsf_params p{};
  p.base_index = base_index;
  if (launch_translate_finish(c->W, c->S, d_acc, n, to_params(&p), d_hit, d_faults, d_fault_idx, d_pop_idx,
                              c->d_sum, st, c->marker()))
    return MPSF_E_CUDA;
  CK(cudaEventRecord(c->ev_done, st));
  c->pending = true;
  c->pending_fault = false;
  c->last_n = n;
  c->last_launches += n ? 2 : 1;
  return MPSF_OK;
}

int mpsf_translate(mpsf_ctx* c, const mpsf_fault_entry* d_acc, uint64_t n, uint64_t base_index, uint8_t* d_hit,
                   mpsf_fault_entry* d_faults, uint32_t* d_fault_idx, uint32_t* d_pop_idx, void* stream) {
  if (!c) return MPSF_E_ARG;
  if (n && (!d_acc || !d_hit || !d_faults || !d_fault_idx || !d_pop_idx)) return MPSF_E_ARG;
  int rc = mpsf_translate_prefetch(c, d_acc, n, base_index, stream);
  if (rc) return rc;
  return mpsf_translate_finish(c, d_acc, n, base_index, d_hit, d_faults, d_fault_idx, d_pop_idx, stream);
}

int mpsf_get_translate_summary(mpsf_ctx* c, mpsf_translate_summary* out) {
  if (!c || !out) return MPSF_E_ARG;
  mpsf_summary s;
  const int rc = mpsf_get_summary(c, &s);
  if (rc) return rc;
  memset(out, 0, sizeof(*out));
  out->status = s.status;
  out->n_miss = s.n_cancel;
  out->n_populated = s.n_dedup;
  out->error_index = s.error_index;
  return MPSF_OK;
}

int mpsf_exchange_buffers(mpsf_ctx* c, int stage, mpsf_xbuf* out, int cap) {
  if (!c || (cap && !out)) return MPSF_E_ARG;
  if (!c->has_world) return MPSF_E_NO_WORLD;
  mpsf_xbuf b[4];
  int k = 0;
  uint8_t* s = c->d_small;
  if (stage == 1) {
    b[k++] = {s + c->x_u64, c->x_u64_n, 8, MPSF_XOP_MIN};
    b[k++] = {s + c->x_u32, c->x_u32_n, 4, MPSF_XOP_MIN};
    if (c->W.dd_groups != 5) return MPSF_E_ARG;   // claimed slots are not combinable: set dense dedup
    b[k++] = {c->d_dd, c->W.n_pages * 5, 4, MPSF_XOP_MIN};
    if (c->S.nrall) b[k++] = {c->S.nrall, c->W.n_pages, 4, MPSF_XOP_MIN};
  } else if (stage == 2) {
    b[k++] = {s + c->x_giso, c->x_giso_n, 4, MPSF_XOP_MIN};
    b[k++] = {c->d_nr1, c->W.n_pages, 4, MPSF_XOP_MIN};
  } else if (stage == 3) {
    b[k++] = {s + c->x_giso, c->x_giso_n, 4, MPSF_XOP_MIN};
  } else if (stage == 4) {                        // translation: first PREFETCH per page
    b[k++] = {c->d_pf, c->W.n_pages, 4, MPSF_XOP_MIN};
  } else {
    return MPSF_E_ARG;
  }
  for (int i = 0; i < k && i < cap; ++i) out[i] = b[i];
  return k;
}

int64_t mpsf_hash_export(mpsf_ctx* c, int which, uint64_t* d_keys, uint32_t* d_vals, uint64_t cap, void* stream) {
  if (!c || (which != 0 && which != 1) || (cap && (!d_keys || !d_vals))) return MPSF_E_ARG;
  CK(cudaSetDevice(c->device));
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (!c->d_counter) CK(cudaMalloc(&c->d_counter, 4));
  CK(cudaMemsetAsync(c->d_counter, 0, 4, st));
  const Hash& h = which == 0 ? c->S.hdd : c->S.hnr;
  const uint64_t hcap = which == 0 ? c->hcap_dd : c->hcap_nr;
  if (launch_hash_export(h, hcap, reinterpret_cast<unsigned long long*>(d_keys), d_vals, c->d_counter, cap, st))
    return MPSF_E_CUDA;
  uint32_t cnt = 0;
  CK(cudaMemcpyAsync(&cnt, c->d_counter, 4, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return cnt > cap ? MPSF_E_OVERFLOW : (int64_t)cnt;
}

int mpsf_hash_merge(mpsf_ctx* c, int which, const uint64_t* d_keys, const uint32_t* d_vals, uint64_t count,
                    void* stream) {
  if (!c || (which != 0 && which != 1) || (count && (!d_keys || !d_vals))) return MPSF_E_ARG;
  CK(cudaSetDevice(c->device));
  const Hash& h = which == 0 ? c->S.hdd : c->S.hnr;
  if (launch_hash_merge(h, c->S.ctrl, reinterpret_cast<const unsigned long long*>(d_keys), d_vals, count,
                        reinterpret_cast<cudaStream_t>(stream)))
    return MPSF_E_CUDA;
  return MPSF_OK;
}

int64_t mpsf_sparse_export(mpsf_ctx* c, const uint32_t* d_buf, uint64_t count, uint32_t* d_idx, uint32_t* d_val,
                           uint64_t cap, void* stream) {
  if (!c || (count && !d_buf) || (cap && (!d_idx || !d_val)) || count > 0xFFFFFFFFull) return MPSF_E_ARG;
  CK(cudaSetDevice(c->device));
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (!c->d_counter) CK(cudaMalloc(&c->d_counter, 4));
  CK(cudaMemsetAsync(c->d_counter, 0, 4, st));
  if (launch_sparse_export(d_buf, count, d_idx, d_val, c->d_counter, cap, st)) return MPSF_E_CUDA;
  uint32_t cnt = 0;
  CK(cudaMemcpyAsync(&cnt, c->d_counter, 4, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return cnt > cap ? MPSF_E_OVERFLOW : (int64_t)cnt;
}

int mpsf_sparse_merge(mpsf_ctx* c, uint32_t* d_buf, uint64_t count, const uint32_t* d_idx, const uint32_t* d_val,
                      uint64_t n, void* stream) {
  if (!c || (count && !d_buf) || (n && (!d_idx || !d_val))) return MPSF_E_ARG;
  CK(cudaSetDevice(c->device));
  if (launch_sparse_merge(d_buf, count, d_idx, d_val, n, reinterpret_cast<cudaStream_t>(stream))) return MPSF_E_CUDA;
  return MPSF_OK;
}

int mpsf_get_summary(mpsf_ctx* c, mpsf_summary* out) {
  if (!c || !out) return MPSF_E_ARG;
  CK(cudaSetDevice(c->device));
  if (c->pending) {
    CK(cudaEventSynchronize(c->ev_done));
    c->pending = false;
  }
  fill_summary(c, *c->h_sum, out, c->pending_fault);
  return MPSF_OK;
}


int mpsf_last_launches(mpsf_ctx* c) { return c ? c->last_launches : 0; }

int mpsf_set_profiling(mpsf_ctx* c, int on) {
  if (!c) return MPSF_E_ARG;
  CK(cudaSetDevice(c->device));
  mpsf_kernel_time dummy;
  mpsf_get_profile(c, &dummy, 0);  // drain anything pending
  c->acc.clear();
  c->profiling = on != 0;
  return MPSF_OK;
}

int mpsf_get_profile(mpsf_ctx* c, mpsf_kernel_time* out, int cap) {
  if (!c || cap < 0 || (cap && !out)) return MPSF_E_ARG;
  CK(cudaSetDevice(c->device));
  for (auto& p : c->pend) {
    CK(cudaEventSynchronize(p.b));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, p.a, p.b));
    auto& slot = c->acc[p.name];
    slot.first += 1;
    slot.second += ms;
  }
  c->pend.clear();
  for (cudaEvent_t e : c->pend_events) c->ev_pool.push_back(e);
  c->pend_events.clear();
  c->last_mark = nullptr;
  int i = 0;
  for (auto& kv : c->acc) {
    if (i >= cap) break;
    memset(out[i].name, 0, sizeof(out[i].name));
    strncpy(out[i].name, kv.first.c_str(), sizeof(out[i].name) - 1);
    out[i].launches = kv.second.first;
    out[i].total_ms = kv.second.second;
    ++i;
  }
  return cap ? i : (int)c->acc.size();
}

// ---- host-buffer form: asynchronous two-slot pipeline -----------------------------------------
// A slot owns the device copies of one batch's input and outputs and its mapped summary.
// mpsf_submit_host enqueues: H2D of the entries in chunks (h2d stream) overlapping pass 1, the
// resolution, pass 2 in chunks with the D2H of each chunk's records (d2h stream) behind it, the
// lists, and the D2H of verdicts / counts / lists -- the lists copied by a kernel straight into
// the caller's host buffers when they are device-accessible (pinned), so nothing waits for the
// list lengths.  Batches run in submission order on the compute stream (the scratch is shared);
// with two slots the H2D of batch k+1 overlaps the passes and the D2H of batch k.
int mpsf_submit_host(mpsf_ctx* c, int slot, const mpsf_fault_entry* h_in, uint64_t n, const mpsf_params* p,
                     mpsf_out_record* h_out, mpsf_client_verdict* h_verdict, uint64_t* h_counts,
                     uint64_t* h_dkeys, uint32_t* h_didx, uint32_t* h_cancel) {
  if (!c || !p || slot < 0 || slot >= kSlots) return MPSF_E_ARG;
  if (!c->has_world) return MPSF_E_NO_WORLD;
  if (n && (!h_in || !h_out || !h_dkeys || !h_didx || !h_cancel)) return MPSF_E_ARG;
  if (c->W.n_clients && (!h_verdict || !h_counts)) return MPSF_E_ARG;
  if (p->base_index + n > MAX_GIDX) return MPSF_E_TOO_LARGE;
  HostSlot& h = c->slots[slot];
  if (h.busy) return MPSF_E_ARG;                   // collect it first
  CK(cudaSetDevice(c->device));
  int rc = slot_buffers(c, h, n);
  if (rc) return rc;
  h.n = n; h.p = *p; h.h_in = h_in; h.h_out = h_out; h.h_verdict = h_verdict; h.h_counts = h_counts;
  h.h_dkeys = h_dkeys; h.h_didx = h_didx; h.h_cancel = h_cancel;
  const uint32_t C = c->W.n_clients;
  uint8_t* b = h.d_io;
  cudaStream_t st = c->own_stream;
  const mpsf_fault_entry* d_in = reinterpret_cast<const mpsf_fault_entry*>(b + h.o_in);
  mpsf_out_record* d_out = reinterpret_cast<mpsf_out_record*>(b + h.o_out);
  mpsf_client_verdict* d_v = reinterpret_cast<mpsf_client_verdict*>(b + h.o_v);
  uint64_t* d_cnt = reinterpret_cast<uint64_t*>(b + h.o_cnt);
  unsigned long long* d_dk = reinterpret_cast<unsigned long long*>(b + h.o_dk);
  uint32_t* d_di = reinterpret_cast<uint32_t*>(b + h.o_di);
  uint32_t* d_ca = reinterpret_cast<uint32_t*>(b + h.o_ca);
  // chunk boundaries on 64-entry chunk multiples: host chunk k = entries [e_lo[k], e_lo[k+1])
  const uint64_t ce = chunk_entries(), nq = chunks_for(n);
  const int nch = n >= (1ull << 20) ? kMaxChunks : n >= (1ull << 18) ? 4 : 1;
  const uint64_t qpc = std::max<uint64_t>(1, (nq + nch - 1) / nch);
  uint64_t q_lo[kMaxChunks + 1];
  int chunks = 0;
  for (uint64_t q = 0; q < nq; q += qpc) q_lo[chunks++] = q;
  q_lo[chunks] = nq;
  auto ent = [&](int k) { return std::min<uint64_t>(q_lo[k] * ce, n); };
  // the slot's previous batch must have landed before its device buffers are overwritten
  CK(cudaStreamWaitEvent(c->h2d_stream, h.ev_done, 0));
  CK(cudaStreamWaitEvent(c->d2h_stream, h.ev_done, 0));
  rc = batch_init(c, n, p, d_cnt, st);
  if (rc) return rc;
  int launches = 1;
  for (int k = 0; k < chunks; ++k) {
    const uint64_t lo = ent(k), cnt = ent(k + 1) - lo;
    CK(cudaMemcpyAsync(b + h.o_in + 16 * lo, h_in + lo, 16 * cnt, cudaMemcpyHostToDevice, c->h2d_stream));
    CK(cudaEventRecord(c->ev_in[k], c->h2d_stream));
    CK(cudaStreamWaitEvent(st, c->ev_in[k], 0));
    if ((rc = scan_chunk(c, d_in + lo, cnt, lo, p, d_cnt, st))) return rc;
    ++launches;
  }
  const Marker mk = c->marker();
  const Params P = to_params(p);
  if ((rc = mid_phases(c, d_in, n, p, d_v, st, launches))) return rc;
  for (int k = 0; k < chunks; ++k) {
    const uint64_t lo = ent(k), cnt = ent(k + 1) - lo;
    Params Pk = P;
    Pk.base_index += lo;
    if (launch_finalize(c->W, c->S, d_in + lo, cnt, Pk, d_out + lo, q_lo[k], st, mk)) return MPSF_E_CUDA;
    ++launches;
    CK(cudaEventRecord(c->ev_fin[k], st));
    CK(cudaStreamWaitEvent(c->d2h_stream, c->ev_fin[k], 0));
    CK(cudaMemcpyAsync(h_out + lo, d_out + lo, 8 * cnt, cudaMemcpyDeviceToHost, c->d2h_stream));
  }
  if (launch_lists(c->S, d_in, d_out, n, p->base_index, d_dk, d_di, d_ca, h.d_sum, st, mk)) return MPSF_E_CUDA;
  ++launches;
  if (C) {
    CK(cudaMemcpyAsync(h_verdict, d_v, 4ull * C, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(h_counts, d_cnt, 8ull * NSCEN * C, cudaMemcpyDeviceToHost, st));
  }
  // the lists: straight into pinned host buffers by a copy kernel (lengths stay on the device)
  unsigned long long* hv_dk = device_view(reinterpret_cast<unsigned long long*>(h_dkeys));
  uint32_t* hv_di = device_view(h_didx);
  uint32_t* hv_ca = device_view(h_cancel);
  h.lists_copied = n && hv_dk && hv_di && hv_ca;
  if (h.lists_copied) {
    if (launch_copyout(c->S, n, d_dk, d_di, d_ca, hv_dk, hv_di, hv_ca, st)) return MPSF_E_CUDA;
    ++launches;
  }
  CK(cudaEventRecord(c->ev_fork, st));
  CK(cudaStreamWaitEvent(c->d2h_stream, c->ev_fork, 0));
  CK(cudaEventRecord(h.ev_done, c->d2h_stream));
  // No compute-stream wait on this batch's D2H: the copies read only this slot's buffers, and
  // the slot's next batch overwrites them only after its H2D, which waits for h.ev_done.
  h.busy = true;
  c->last_n = n;
  c->last_launches = launches + 1;
  return MPSF_OK;
}

int mpsf_collect_host(mpsf_ctx* c, int slot, mpsf_summary* summary) {
  if (!c || !summary || slot < 0 || slot >= kSlots) return MPSF_E_ARG;
  HostSlot& h = c->slots[slot];
  if (!h.busy) return MPSF_E_ARG;
  CK(cudaSetDevice(c->device));
  CK(cudaEventSynchronize(h.ev_done));
  h.busy = false;
  fill_summary(c, *h.h_sum, summary, true);
  const uint64_t n = h.n;
  uint8_t* b = h.d_io;
  cudaStream_t st = c->own_stream;
  if (summary->status == MPSF_OK) {
    if (!h.lists_copied) {
      if (summary->n_dedup) {
        CK(cudaMemcpyAsync(h.h_dkeys, b + h.o_dk, 8 * summary->n_dedup, cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(h.h_didx, b + h.o_di, 4 * summary->n_dedup, cudaMemcpyDeviceToHost, st));
      }
      if (summary->n_cancel)
        CK(cudaMemcpyAsync(h.h_cancel, b + h.o_ca, 4 * summary->n_cancel, cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
    }
    return MPSF_OK;
  }
  if (summary->status != MPSF_E_OVERFLOW) return MPSF_OK;
  // the wild-page hash overflowed (its capacity has grown): re-run on the resident entries
  const uint32_t C = c->W.n_clients;
  const mpsf_fault_entry* d_in = reinterpret_cast<const mpsf_fault_entry*>(b + h.o_in);
  for (int attempt = 1; attempt < 4; ++attempt) {
    int rc = mpsf_process(c, d_in, n, &h.p, reinterpret_cast<mpsf_out_record*>(b + h.o_out),
                          reinterpret_cast<mpsf_client_verdict*>(b + h.o_v), reinterpret_cast<uint64_t*>(b + h.o_cnt),
                          reinterpret_cast<uint64_t*>(b + h.o_dk), reinterpret_cast<uint32_t*>(b + h.o_di),
                          reinterpret_cast<uint32_t*>(b + h.o_ca), st);
    if (rc) return rc;
    CK(cudaMemcpyAsync(h.h_out, b + h.o_out, 8 * n, cudaMemcpyDeviceToHost, st));
    if (C) {
      CK(cudaMemcpyAsync(h.h_verdict, b + h.o_v, 4ull * C, cudaMemcpyDeviceToHost, st));
      CK(cudaMemcpyAsync(h.h_counts, b + h.o_cnt, 8ull * NSCEN * C, cudaMemcpyDeviceToHost, st));
    }
    rc = mpsf_get_summary(c, summary);
    if (rc) return rc;
    if (summary->status == MPSF_E_OVERFLOW) continue;
    if (summary->status != MPSF_OK) return MPSF_OK;
    if (summary->n_dedup) {
      CK(cudaMemcpyAsync(h.h_dkeys, b + h.o_dk, 8 * summary->n_dedup, cudaMemcpyDeviceToHost, st));
      CK(cudaMemcpyAsync(h.h_didx, b + h.o_di, 4 * summary->n_dedup, cudaMemcpyDeviceToHost, st));
    }
    if (summary->n_cancel) CK(cudaMemcpyAsync(h.h_cancel, b + h.o_ca, 4 * summary->n_cancel, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return MPSF_OK;
  }
  return MPSF_OK;
}

int mpsf_process_host(mpsf_ctx* c, const mpsf_fault_entry* h_in, uint64_t n, const mpsf_params* p,
                      mpsf_out_record* h_out, mpsf_client_verdict* h_verdict, uint64_t* h_counts,
                      uint64_t* h_dkeys, uint32_t* h_didx, uint32_t* h_cancel, mpsf_summary* summary) {
  if (!c || !summary) return MPSF_E_ARG;
  for (int s = 0; s < kSlots; ++s)
    if (c->slots[s].busy) return MPSF_E_ARG;      // not while batches are in flight
  int rc = mpsf_submit_host(c, 0, h_in, n, p, h_out, h_verdict, h_counts, h_dkeys, h_didx, h_cancel);
  if (rc) return rc;
  return mpsf_collect_host(c, 0, summary);
}

int mpsf_remap(mpsf_ctx* c, uint64_t va_base, const uint64_t* d_phys, uint64_t npages4k, uint32_t gran_log2,
               mpsf_remap_entry* d_out, void* stream) {
  if (!c || gran_log2 < 12 || gran_log2 > 30 || (npages4k && (!d_phys || !d_out))) return MPSF_E_ARG;
  CK(cudaSetDevice(c->device));
  c->mark_begin(reinterpret_cast<cudaStream_t>(stream));
  if (launch_remap(va_base, d_phys, npages4k, gran_log2, d_out, reinterpret_cast<cudaStream_t>(stream)))
    return MPSF_E_CUDA;
  c->marker().mark("k_remap");
  c->last_launches = npages4k ? 1 : 0;
  return MPSF_OK;
}

int mpsf_remap_blocks(mpsf_ctx* c, uint64_t va_base, const uint64_t* d_phys, uint64_t npages4k,
                      const uint32_t* d_blocks, uint64_t nblocks, mpsf_remap_entry* d_out, void* stream) {
  if (!c || (nblocks && (!d_phys || !d_blocks || !d_out))) return MPSF_E_ARG;
  CK(cudaSetDevice(c->device));
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  CK(cudaMemsetAsync(c->d_remap_err, 0, 4, st));
  if (launch_remap_blocks(va_base, d_phys, npages4k, d_blocks, nblocks, d_out, c->d_remap_err, st))
    return MPSF_E_CUDA;
  uint32_t err = 0;
  CK(cudaMemcpyAsync(&err, c->d_remap_err, 4, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  c->last_launches = nblocks ? 1 : 0;
  return err ? MPSF_E_ARG : MPSF_OK;
}

int mpsf_fold(mpsf_ctx* c, uint64_t n_snap, uint32_t n_req_ids, const uint32_t* d_req, const uint32_t* d_nblk,
              const uint32_t* d_ntok, const uint32_t* d_progress, const uint8_t* d_done, const uint32_t* d_blocks,
              uint64_t n_blocks, const uint32_t* d_tokens, uint64_t n_tokens, uint32_t* d_order, uint64_t* d_blk_off, uint32_t* d_blocks_out,
              uint64_t* d_tok_off, uint32_t* d_tokens_out, uint32_t* d_progress_out, uint8_t* d_done_out,
              mpsf_fold_summary* summary, void* stream) {
  if (!c || !summary) return MPSF_E_ARG;
  if (n_snap >= (1ull << 31) - 1 || n_blocks >= (1ull << 32) || n_tokens >= (1ull << 32) || n_req_ids > (1u << 30))
    return MPSF_E_TOO_LARGE;   // (the id space sizes four u32 tables of scratch)
  if ((n_blocks && (!d_blocks || !d_blocks_out)) || (n_tokens && (!d_tokens || !d_tokens_out))) return MPSF_E_ARG;
  if (n_snap && (!d_req || !d_nblk || !d_ntok || !d_progress || !d_done || !d_order || !d_blk_off ||
                 !d_tok_off || !d_progress_out || !d_done_out))
    return MPSF_E_ARG;
  *summary = mpsf_fold_summary{};
  summary->error_index = ~0ull;
  CK(cudaSetDevice(c->device));
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (!n_snap) {   // nothing folded: the CSR is the single zero offset
    if (d_blk_off) CK(cudaMemsetAsync(d_blk_off, 0, 8, st));
    if (d_tok_off) CK(cudaMemsetAsync(d_tok_off, 0, 8, st));
    return MPSF_OK;
  }
  const size_t need = fold_scratch_bytes(n_snap, n_req_ids ? n_req_ids : 1);
  if (need > c->fold_cap) {
    CK(cudaStreamSynchronize(st));
    cudaFree(c->d_fold);
    c->d_fold = nullptr;
    c->fold_cap = 0;
    CK(cudaMalloc(&c->d_fold, need));
    c->fold_cap = need;
  }
  FoldTotals tot{};
  c->mark_begin(st);
  if (launch_fold(c->d_fold, c->fold_cap, (uint32_t)n_snap, n_req_ids ? n_req_ids : 1, d_req, d_nblk, d_ntok,
                  d_progress, d_done, d_blocks, n_blocks, d_tokens, n_tokens, d_order, d_blk_off, d_blocks_out, d_tok_off, d_tokens_out,
                  d_progress_out, d_done_out, &tot, st, c->marker()))
    return MPSF_E_CUDA;
  c->last_launches = (int)tot.launches;
  summary->n_requests = tot.n_requests;
  summary->n_blocks = tot.n_blocks;
  summary->n_tokens = tot.n_tokens;
  summary->error_index = tot.error_index;
  summary->status = tot.error_index != ~0ull ? MPSF_E_BAD_ENTRY : tot.overrun ? MPSF_E_ARG : MPSF_OK;
  return summary->status;
}

int mpsf_kv_reserve(mpsf_ctx* c, uint32_t total_blocks, const uint32_t* d_block_ids, uint64_t n,
                    uint8_t* d_reserved, uint32_t* d_free, uint64_t* n_free, void* stream) {
  if (!c || !n_free || (n && !d_block_ids) || (total_blocks && (!d_reserved || !d_free))) return MPSF_E_ARG;
  *n_free = 0;
  if (!total_blocks) return MPSF_OK;
  CK(cudaSetDevice(c->device));
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const size_t need = kv_reserve_scratch_bytes(total_blocks);
  if (need > c->fold_cap) {
    CK(cudaStreamSynchronize(st));
    cudaFree(c->d_fold);
    c->d_fold = nullptr;
    c->fold_cap = 0;
    CK(cudaMalloc(&c->d_fold, need));
    c->fold_cap = need;
  }
  c->mark_begin(st);
  if (launch_kv_reserve(c->d_fold, c->fold_cap, total_blocks, d_block_ids, n, d_reserved, d_free, n_free, st))
    return MPSF_E_CUDA;
  c->marker().mark("k_kv_reserve");
  c->last_launches = n ? 4 : 3;
  return MPSF_OK;
}

}  // extern "C"
