// Trace-line rendering of a processed fault batch, host code.
//
// Reference: Trace.render_record (pkg/src/mpssim/kernel.py:127-132) -- one line per record,
// "t=<t> who=<who> kind=<kind> k=v ..." in emit order.  This renders, for a batch of fault
// entries and the OutRecords the device produced for it, the lines the reference emits:
//   top half (MPSF_RENDER_TOP), per entry in raise (= index) order:
//     raise_mmu_fault (pipeline.py:113-125): fault_raised scenario va access engine, and for
//       a non-replayable record rmgsp shadow_copy scenario channel;
//     raise_parse_time_fault (pipeline.py:142-143): fault_raised scenario=<category> va=0
//       access=n/a engine=sm;
//   drain (MPSF_RENDER_DRAIN), per record in drain order (replayable buffer first,
//     pipeline.py:164), as the batch bottom half applies the verdicts (shim.py):
//     bh_service scenario channel (pipeline.py:166-167);
//     parse-time: parse_fatal scenario (170-171), then unless cancelled _report_fatal's
//       tlb_invalidate channel + fatal_report scenario channel (pipeline.py:224-230);
//     isolated: isolate_begin mechanism scenario pid latency_us (pipeline.py:296-298);
//     fatal: unless cancelled, _report_fatal's lines;
//     serviced: nothing at drain time (benign_done is scheduled);
//     duplicates (rule C2): bh_service only.
// SM-trap entries have no buffer record (raise_sm_trap reports immediately) and render
// nothing; the DES follow-ups (rc_recovery teardown lines, benign_done, isolate_done) come
// from the simulator's own handlers.  Skipped entries (valid flag clear) render nothing.
//
// Rendering is split over host threads by entry ranges; each thread formats its range into a
// private buffer and the pieces are concatenated in order.
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <string>
#include <thread>
#include <vector>

#include "mpsf.h"

namespace {

const char* const kScen[28] = {
    "mmu.oob.sm", "mmu.am_cpu.sm", "mmu.am_gpu.sm", "mmu.am_vmm.sm", "mmu.zombie.sm", "mmu.nonmigratable.sm",
    "mmu.oob.ce", "mmu.am.ce", "mmu.zombie.ce", "mmu.nonmigratable.ce", "mmu.oob.pbdma", "mmu.am.pbdma",
    "mmu.zombie.pbdma", "mmu.nonmigratable.pbdma", "benign.demand_paging.sm", "benign.invalid_prefetch.sm",
    "benign.page_fault.ce", "benign.page_fault.pbdma", "sm.exc2.lane_user_stack_overflow",
    "sm.exc4.illegal_instruction", "sm.exc5.shared_local_oob", "sm.exc6.misaligned_address",
    "sm.exc7.invalid_address_space", "parse.mmu_structural", "parse.channel_state", "parse.privilege",
    "parse.aperture", "parse.ecc_poison"};
const char* const kEng[3] = {"sm", "ce", "pbdma"};
const char* const kAcc[3] = {"read", "write", "prefetch"};
constexpr uint8_t V_CANCELLED = 0x10, V_DUP = 0x20, V_REPL = 0x40;

struct Name {
  const char* p;
  uint32_t n;
};

// Line writer: each line reserves its worst case once (need), then writes unchecked.
struct Out {
  std::string s;
  size_t n = 0;
  void need(size_t k) {
    if (n + k > s.size()) s.resize(std::max(2 * s.size(), n + k + 65536));
  }
  template <size_t L>
  void lit(const char (&a)[L]) {
    memcpy(&s[n], a, L - 1);
    n += L - 1;
  }
  void name(const Name& x) {
    memcpy(&s[n], x.p, x.n);
    n += x.n;
  }
  void num(uint64_t v) {
    char b[24];
    int k = 0;
    do {
      b[k++] = (char)('0' + v % 10);
      v /= 10;
    } while (v);
    while (k) s[n++] = b[--k];
  }
  template <size_t L>
  void head(uint64_t t, const Name& who, const char (&kind)[L]) {
    lit("t=");
    num(t);
    lit(" who=");
    name(who);
    lit(" kind=");
    lit(kind);
  }
};

struct Job {
  const mpsf_fault_entry* e;
  const mpsf_out_record* o;
  const mpsf_render_params* p;
  std::vector<Name> chan, client;
  Name scen[28], eng[3], acc[3], mech[4], uvm, rmgsp, unknown;
  size_t line_max;   // worst-case line bytes
};

Name nm(const char* p) { return Name{p ? p : "?", (uint32_t)strlen(p ? p : "?")}; }

bool drained(const mpsf_fault_entry& e, const mpsf_out_record& o) {
  return (e.flags & 1u) && o.scenario < 28 && e.kind < 8;   // traps / skipped: no buffer record
}

const Name& chan_name(const Job& j, uint32_t ch) { return ch < j.chan.size() ? j.chan[ch] : j.unknown; }

void render_top(const Job& j, uint64_t lo, uint64_t hi, Out& w) {
  for (uint64_t i = lo; i < hi; ++i) {
    const mpsf_fault_entry& e = j.e[i];
    const mpsf_out_record& o = j.o[i];
    if (!drained(e, o)) continue;
    const uint64_t t = j.p->t_raise ? j.p->t_raise[i] : j.p->t_drain;
    const Name& ch = chan_name(j, e.channel);
    w.need(2 * j.line_max);
    w.head(t, ch, "fault_raised");
    w.lit(" scenario=");
    w.name(j.scen[o.scenario]);
    if (e.kind != 0) {
      w.lit(" va=0 access=n/a engine=sm\n");
      continue;
    }
    w.lit(" va=");
    w.num(e.va);
    w.lit(" access=");
    w.name(j.acc[e.access < 3 ? e.access : 0]);
    w.lit(" engine=");
    w.name(j.eng[e.engine < 3 ? e.engine : 0]);
    w.lit("\n");
    if (!(o.verdict & V_REPL)) {
      w.head(t, j.rmgsp, "shadow_copy");
      w.lit(" scenario=");
      w.name(j.scen[o.scenario]);
      w.lit(" channel=");
      w.name(ch);
      w.lit("\n");
    }
  }
}

void report_fatal(const Job& j, uint64_t t, const Name& scen, const Name& ch, bool repl, Out& w) {
  if (repl) {
    w.head(t, j.uvm, "tlb_invalidate");
    w.lit(" channel=");
    w.name(ch);
    w.lit("\n");
  }
  w.head(t, j.uvm, "fatal_report");
  w.lit(" scenario=");
  w.name(scen);
  w.lit(" channel=");
  w.name(ch);
  w.lit("\n");
}

// drain lines of the records i in [lo, hi) whose replayable flag equals `repl`
void render_drain(const Job& j, uint64_t lo, uint64_t hi, bool repl, Out& w) {
  const uint64_t t = j.p->t_drain;
  for (uint64_t i = lo; i < hi; ++i) {
    const mpsf_fault_entry& e = j.e[i];
    const mpsf_out_record& o = j.o[i];
    if (!drained(e, o) || ((o.verdict & V_REPL) != 0) != repl) continue;
    const Name& scen = j.scen[o.scenario];
    const Name& ch = chan_name(j, e.channel);
    w.need(4 * j.line_max);
    w.head(t, j.uvm, "bh_service");
    w.lit(" scenario=");
    w.name(scen);
    w.lit(" channel=");
    w.name(ch);
    w.lit("\n");
    if (o.verdict & V_DUP) continue;
    const uint32_t outcome = o.verdict & 3u, mech = (o.verdict >> 2) & 3u;
    const bool canc = o.verdict & V_CANCELLED;
    if (e.kind != 0) {   // parse-time
      w.head(t, j.uvm, "parse_fatal");
      w.lit(" scenario=");
      w.name(scen);
      w.lit("\n");
      if (!canc) report_fatal(j, t, scen, ch, true, w);
    } else if (outcome == 2) {
      w.head(t, j.uvm, "isolate_begin");
      w.lit(" mechanism=");
      w.name(j.mech[mech]);
      w.lit(" scenario=");
      w.name(scen);
      w.lit(" pid=");
      w.name(o.client < j.client.size() ? j.client[o.client] : j.unknown);
      w.lit(" latency_us=");
      w.num(mech == 1 ? j.p->m1_us : (mech == 3 ? j.p->m3_us : j.p->m2_us));
      w.lit("\n");
    } else if (outcome == 3 && !canc) {
      report_fatal(j, t, scen, ch, repl, w);
    }
  }
}

}  // namespace

extern "C" int64_t mpsf_render_trace(const mpsf_fault_entry* entries, const mpsf_out_record* out, uint64_t n,
                                     const mpsf_render_params* p, char* buf, uint64_t cap) {
  if (!p || (n && (!entries || !out)) || (p->n_channels && !p->channel_names) ||
      (p->n_clients && !p->client_names))
    return MPSF_E_ARG;
  Job j;
  j.e = entries;
  j.o = out;
  j.p = p;
  size_t longest = 32;
  for (uint32_t k = 0; k < p->n_channels; ++k) j.chan.push_back(nm(p->channel_names[k]));
  for (uint32_t k = 0; k < p->n_clients; ++k) j.client.push_back(nm(p->client_names[k]));
  for (const Name& x : j.chan) longest = std::max<size_t>(longest, x.n);
  for (const Name& x : j.client) longest = std::max<size_t>(longest, x.n);
  for (int k = 0; k < 28; ++k) j.scen[k] = nm(kScen[k]);
  for (int k = 0; k < 3; ++k) j.eng[k] = nm(kEng[k]), j.acc[k] = nm(kAcc[k]);
  static const char* const mn[4] = {"M?", "M1", "M2", "M3"};
  for (int k = 0; k < 4; ++k) j.mech[k] = nm(mn[k]);
  j.uvm = nm("uvm");
  j.rmgsp = nm("rmgsp");
  j.unknown = nm("?");
  j.line_max = 160 + 3 * longest;   // fixed text + numbers + the longest scenario + 3 names
  unsigned nt = p->threads ? p->threads : std::max(1u, std::thread::hardware_concurrency());
  nt = (unsigned)std::min<uint64_t>(nt, std::max<uint64_t>(1, n / 4096));
  // pieces in output order: top (per thread range), drain replayable, drain non-replayable
  const bool any = (p->parts & (MPSF_RENDER_TOP | MPSF_RENDER_DRAIN)) != 0;
  std::vector<Out> piece((size_t)nt * 3);
  auto work = [&](unsigned k) {
    const uint64_t lo = n * k / nt, hi = n * (k + 1) / nt;
    if (p->parts & MPSF_RENDER_TOP) render_top(j, lo, hi, piece[k]);
    if (p->parts & MPSF_RENDER_DRAIN) {
      render_drain(j, lo, hi, true, piece[nt + k]);
      render_drain(j, lo, hi, false, piece[2 * nt + k]);
    }
  };
  if (any) {
    std::vector<std::thread> th;
    for (unsigned k = 1; k < nt; ++k) th.emplace_back(work, k);
    work(0);
    for (auto& t : th) t.join();
  }
  uint64_t total = 0;
  for (const Out& o : piece) total += o.n;
  if (total > cap || !buf) return (int64_t)total;
  char* d = buf;
  for (const Out& o : piece) {
    memcpy(d, o.s.data(), o.n);
    d += o.n;
  }
  return (int64_t)total;
}
