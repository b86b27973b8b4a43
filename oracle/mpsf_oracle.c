/*
 * mpsf_oracle.c -- TEST INFRASTRUCTURE ONLY: the sequential CPU checker / CPU baseline.
 *
 * Plain-C restatement of oracle/seq_oracle.py (which is pinned against the reference
 * package by tests/test_oracle_vs_reference.py and tests/test_golden_oracle.py).  Only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
 * load it; the product path (libmpsf.so) never does.
 *
 * Algorithm, as the reference runs it (paths relative to pkg/src/mpssim/):
 *   A. top half per entry: channel -> client (pipeline.py:103), faults.classify
 *      (faults.py:134-171) with MemoryModel.range_at (memory.py:233-237: scan of the
 *      client's ranges), buffer by classified replayable flag (pipeline.py:116-123).
 *      Entries are independent here, so this phase runs on `threads` pthreads.
 *   B. sequential: SM traps at raise time (pipeline.py:151-155), then the drain
 *      replayable-then-non-replayable (pipeline.py:164) with rc_recovery / teardown
 *      (pipeline.py:235-265, execmodel.py:345-374, pipeline.py:329-365), isolation on the
 *      evolving range state (pipeline.py:270-304), then the (time, seq) event order of
 *      benign_done / isolation_done (kernel.py:206-265, pipeline.py:193-208, 307-324).
 *   Batch rules where the reference is undefined: SURVEY.md Appendix C (C2 dedup,
 *   C4 cancel of fatal records on destroyed TSGs, C5/C6 dropped benign completions).
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "mpsf.h"

#define EMPTY64 0xFFFFFFFFFFFFFFFFull

typedef struct {
  const mpsf_range_entry* R;
  const uint32_t* off;
  const uint8_t* ps;
  const mpsf_channel_entry* ch;
  uint32_t nch, ncl;
} world_t;

/* per-entry decoded record */
typedef struct {
  uint32_t c;
  int32_t ridx;
  uint8_t s, ceng, eng, kind, valid, repl, err;
} rec_t;

static int classify(int eng, int acc, int has, const mpsf_range_entry* r, uint32_t st) {
  if (acc == 2) return 15;
  int oob = eng == 0 ? 0 : 2 + 4 * eng;
  if (!has) return oob;
  if (r->lifecycle == 1) return 4 + 4 * eng;
  int res = st & 3, ro = (st & 4) != 0;
  if (!r->migratable && res == 1) return 5 + 4 * eng;
  if (acc == 1 && ro) {
    if (eng == 0) return r->kind == 1 ? 3 : (res == 2 ? 2 : 1);
    return 3 + 4 * eng;
  }
  if (r->kind == 0 && res <= 1) return eng == 0 ? 14 : 15 + eng;
  return oob;
}

static int replayable(int s) { return s <= 5 || s == 14 || s == 15 || s >= 23; }
static int serviceable(int s) { return s >= 14 && s <= 17; }

typedef struct {
  const world_t* w;
  const mpsf_fault_entry* in;
  rec_t* rec;
  uint64_t lo, hi;
} job_t;

static void* decode_range(void* arg) {
  job_t* j = (job_t*)arg;
  const world_t* w = j->w;
  for (uint64_t i = j->lo; i < j->hi; ++i) {
    const mpsf_fault_entry* e = &j->in[i];
    rec_t* r = &j->rec[i];
    memset(r, 0, sizeof(*r));
    r->ridx = -1;
    if (!(e->flags & 1)) continue;
    if (e->channel >= w->nch || w->ch[e->channel].client >= w->ncl) { r->err = 1; continue; }
    r->c = w->ch[e->channel].client;
    r->ceng = w->ch[e->channel].engine;
    r->eng = e->engine;
    r->kind = e->kind;
    if (e->kind == 0) {
      if (e->engine > 2 || e->access > 2) { r->err = 2; continue; }
      if (e->engine != r->ceng) { r->err = 3; continue; }
      if (e->va >= (1ull << 53)) { r->err = 4; continue; }
      int32_t found = -1;
      for (uint32_t k = w->off[r->c]; k < w->off[r->c + 1]; ++k)
        if (w->R[k].base <= e->va && e->va < w->R[k].end) { found = (int32_t)k; break; }
      uint32_t st = 0;
      if (found >= 0) {
        const mpsf_range_entry* rg = &w->R[found];
        st = rg->state != 0xFF ? rg->state : w->ps[rg->page_off + ((e->va - rg->base) >> 12)];
      }
      r->ridx = found;
      r->s = (uint8_t)classify(e->engine, e->access, found >= 0, found >= 0 ? &w->R[found] : NULL, st);
      r->repl = (uint8_t)replayable(r->s);
    } else if (e->kind >= 1 && e->kind <= 5) {
      r->s = (uint8_t)(23 + e->kind - 1);
      r->repl = 1;
    } else if (e->kind >= 8 && e->kind <= 12) {
      r->s = (uint8_t)(18 + e->kind - 8);
      r->repl = 0;
    } else {
      r->err = 2;
      continue;
    }
    r->valid = 1;
  }
  return NULL;
}

/* ---- open-addressing u64 -> u64 map ---- */
typedef struct { uint64_t* k; uint64_t* v; uint64_t mask; } map_t;

static uint64_t mix64(uint64_t x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull; x ^= x >> 33;
  return x;
}
static int map_init(map_t* m, uint64_t n) {
  uint64_t cap = 1024;
  while (cap < 2 * n + 16) cap <<= 1;
  m->k = (uint64_t*)malloc(cap * 8);
  m->v = (uint64_t*)malloc(cap * 8);
  if (!m->k || !m->v) return -1;
  memset(m->k, 0xFF, cap * 8);
  m->mask = cap - 1;
  return 0;
}
static void map_free(map_t* m) { free(m->k); free(m->v); }
/* returns pointer to value; *inserted set if new (value initialised to init) */
static uint64_t* map_get(map_t* m, uint64_t key, uint64_t init, int* inserted) {
  uint64_t s = mix64(key) & m->mask;
  for (;;) {
    if (m->k[s] == key) { *inserted = 0; return &m->v[s]; }
    if (m->k[s] == EMPTY64) { m->k[s] = key; m->v[s] = init; *inserted = 1; return &m->v[s]; }
    s = (s + 1) & m->mask;
  }
}
static uint64_t* map_find(map_t* m, uint64_t key) {
  uint64_t s = mix64(key) & m->mask;
  for (;;) {
    if (m->k[s] == key) return &m->v[s];
    if (m->k[s] == EMPTY64) return NULL;
    s = (s + 1) & m->mask;
  }
}

typedef struct { uint32_t t; uint64_t seq; uint64_t i; uint8_t benign; } event_t;
static int ev_cmp(const void* a, const void* b) {
  const event_t* x = (const event_t*)a;
  const event_t* y = (const event_t*)b;
  if (x->t != y->t) return x->t < y->t ? -1 : 1;
  return x->seq < y->seq ? -1 : (x->seq > y->seq);
}

/* per-client state of the drain */
typedef struct {
  uint8_t mode, state, reason, notifier, ce_alive, sa_alive, torn[3];
  uint32_t epoch;  /* incremented on release; 1 at start for dead clients */
} cl_t;

static void terminate(cl_t* c, uint8_t reason) {
  c->state = 1;
  c->reason = reason;
  c->torn[0] = c->torn[1] = c->torn[2] = 1;
  if (c->mode == 0) c->ce_alive = 0; else c->sa_alive = 0;
  c->epoch++;
}

int oracle_process(const mpsf_range_entry* R, uint32_t nr, const uint8_t* page_state, uint64_t np,
                   const mpsf_channel_entry* ch, uint32_t nch, const mpsf_client_entry* cl, uint32_t ncl,
                   uint32_t world_flags, const mpsf_fault_entry* in, uint64_t n, const mpsf_params* p,
                   int threads, mpsf_out_record* out, mpsf_client_verdict* verdict, uint64_t* counts,
                   uint64_t* dkeys, uint32_t* didx, uint64_t* n_dedup, uint32_t* cancel,
                   uint64_t* n_cancel, uint64_t* err_index) {
  (void)np;
  uint32_t* off = (uint32_t*)calloc(ncl + 1, 4);
  for (uint32_t i = 0; i < nr; ++i) off[R[i].client + 1]++;
  for (uint32_t i = 0; i < ncl; ++i) off[i + 1] += off[i];
  for (uint32_t c = 0; c < ncl; ++c)
    if (cl[c].mode == 0 && (cl[c].flags & 1) && (world_flags & 1)) { free(off); return MPSF_E_WORLD; }
  world_t w = {R, off, page_state, ch, nch, ncl};
  rec_t* rec = (rec_t*)malloc(sizeof(rec_t) * (n ? n : 1));
  if (threads < 1) threads = 1;
  if ((uint64_t)threads > n / 4096 + 1) threads = (int)(n / 4096 + 1);
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * threads);
  job_t* jobs = (job_t*)malloc(sizeof(job_t) * threads);
  for (int t = 0; t < threads; ++t) {
    jobs[t].w = &w; jobs[t].in = in; jobs[t].rec = rec;
    jobs[t].lo = n * t / threads; jobs[t].hi = n * (t + 1) / threads;
    if (t) pthread_create(&th[t], NULL, decode_range, &jobs[t]);
  }
  decode_range(&jobs[0]);
  for (int t = 1; t < threads; ++t) pthread_join(th[t], NULL);
  free(th); free(jobs);

  const uint64_t base = p->base_index;
  int rc = 0;
  for (uint64_t i = 0; i < n; ++i)
    if (rec[i].err) {
      *err_index = base + i;
      rc = rec[i].err == 1 ? MPSF_E_NO_CHANNEL : rec[i].err == 2 ? MPSF_E_BAD_ENTRY
         : rec[i].err == 3 ? MPSF_E_ENGINE_MISMATCH : MPSF_E_VA_RANGE;
      break;
    }
  if (rc) { free(rec); free(off); return rc; }

  uint8_t* vb = (uint8_t*)calloc(n ? n : 1, 1);
  uint8_t* canc = (uint8_t*)calloc(n ? n : 1, 1);
  uint64_t* rep = (uint64_t*)malloc(8 * (n ? n : 1));
  memset(counts, 0, 8ull * 28 * ncl);
  for (uint64_t i = 0; i < n; ++i) {
    const rec_t* r = &rec[i];
    mpsf_out_record o = {0xFFFFFFFFu, 0xFF, 0, 0xFFFF};
    rep[i] = EMPTY64;
    if (r->valid) {
      o.scenario = r->s;
      o.client = (uint16_t)r->c;
      if (r->ridx >= 0) o.rid = R[r->ridx].rid;
      counts[28ull * r->c + r->s]++;
      if (r->repl) vb[i] |= 0x40;
    }
    out[i] = o;
  }
  /* C2 dedup */
  map_t dm;
  map_init(&dm, n);
  uint64_t nd = 0;
  for (uint64_t i = 0; i < n; ++i) {
    const rec_t* r = &rec[i];
    if (!r->valid || r->kind != 0 || !r->repl) continue;
    uint64_t key = ((uint64_t)r->c << 48) | ((uint64_t)r->eng << 46) | ((uint64_t)r->s << 41) | (in[i].va >> 12);
    int ins;
    uint64_t* v = map_get(&dm, key, i, &ins);
    if (ins) { dkeys[nd] = key; didx[nd] = (uint32_t)(base + i); nd++; }
    else { rep[i] = *v; vb[i] |= 0x20; }
  }
  map_free(&dm);
  *n_dedup = nd;

  /* state */
  cl_t* C = (cl_t*)calloc(ncl ? ncl : 1, sizeof(cl_t));
  int has_mps = 0;
  for (uint32_t c = 0; c < ncl; ++c) {
    int alive = cl[c].flags & 1;
    C[c].mode = cl[c].mode;
    C[c].state = alive ? 0 : 1;
    C[c].reason = alive ? 0 : 3;
    C[c].notifier = alive ? 0xFF : 0xFE;
    C[c].ce_alive = cl[c].mode == 0 && alive && !(cl[c].flags & 2);
    C[c].sa_alive = cl[c].mode == 1 && alive;
    C[c].torn[0] = C[c].torn[1] = C[c].torn[2] = !alive;
    C[c].epoch = alive ? 0 : 1;
    if (cl[c].mode == 0) has_mps = 1;
  }
  int gr_alive = has_mps && !(world_flags & 1);
  for (uint32_t c = 0; c < ncl; ++c)
    if (C[c].mode == 0 && C[c].state == 0) {
      if (!C[c].ce_alive) C[c].torn[1] = 1;
      if (!gr_alive) C[c].torn[0] = C[c].torn[2] = 1;
    }
  /* rc_recovery on a live TSG: kind 0 GR, 1 CE_c, 2 SA_c */
#define RC(kind, cc, err)                                                          \
  do {                                                                             \
    if ((kind) == 0) {                                                             \
      for (uint32_t q = 0; q < ncl; ++q) if (C[q].mode == 0) C[q].notifier = (err);  \
      for (uint32_t q = 0; q < ncl; ++q) if (C[q].mode == 0) C[q].torn[0] = C[q].torn[2] = 1; \
      gr_alive = 0;                                                                \
      for (uint32_t q = 0; q < ncl; ++q) if (C[q].mode == 0 && C[q].state == 0) terminate(&C[q], 2); \
    } else if ((kind) == 1) {                                                      \
      C[cc].notifier = (err); C[cc].torn[1] = 1; C[cc].ce_alive = 0;               \
    } else {                                                                       \
      C[cc].notifier = (err); C[cc].torn[0] = C[cc].torn[1] = C[cc].torn[2] = 1;   \
      C[cc].sa_alive = 0;                                                          \
      if (C[cc].state == 0) terminate(&C[cc], 2);                                  \
    }                                                                              \
  } while (0)
  /* traps at raise time */
  for (uint64_t i = 0; i < n; ++i) {
    const rec_t* r = &rec[i];
    if (!r->valid || r->kind < 8) continue;
    uint32_t c = r->c;
    int kind = C[c].mode == 0 ? 0 : 2;
    int alive = kind == 0 ? gr_alive : C[c].sa_alive;
    if (!alive) { canc[i] = 1; continue; }
    RC(kind, c, r->s);
  }
  /* drain */
  const int iso = p->flags & 1;
  map_t pages;      /* (client, page) -> epoch+1 of an M1-created managed page */
  map_t conv;       /* range index -> epoch+1 of its M3 conversion            */
  map_init(&pages, n);
  map_init(&conv, nr + 1);
  event_t* ev = (event_t*)malloc(sizeof(event_t) * (n ? n : 1));
  uint64_t nev = 0, seq = 0;
  for (int pass = 0; pass < 2; ++pass) {
    for (uint64_t i = 0; i < n; ++i) {
      const rec_t* r = &rec[i];
      if (!r->valid || r->kind >= 8 || (int)r->repl != (pass == 0)) continue;
      const int parse = r->s >= 23, serv = serviceable(r->s);
      const int label = parse ? 3 : serv ? 1 : iso ? 2 : 3;
      vb[i] |= (uint8_t)label;
      if (vb[i] & 0x20) continue;
      const uint32_t c = r->c;
      if (label == 3) {
        int kind = C[c].mode == 1 ? 2 : (r->ceng == 1 ? 1 : 0);
        int alive = kind == 0 ? gr_alive : kind == 1 ? C[c].ce_alive : C[c].sa_alive;
        if (!alive) { canc[i] = 1; continue; }
        RC(kind, c, r->s);
      } else if (label == 1) {
        ev[nev].t = p->benign_us; ev[nev].seq = seq++; ev[nev].i = i; ev[nev].benign = 1; nev++;
      } else {
        const uint64_t va = in[i].va, page = va >> 12;
        int mech;
        int32_t k = -1;
        if (C[c].epoch == 0 && r->ridx >= 0) k = r->ridx;   /* snapshot range still mapped */
        if (k >= 0) {
          uint64_t* cv = map_find(&conv, (uint64_t)k);
          int managed = R[k].kind == 0 || (cv && *cv == (uint64_t)C[c].epoch + 1);
          if (managed) mech = 2;
          else { int ins; *map_get(&conv, (uint64_t)k, 0, &ins) = (uint64_t)C[c].epoch + 1; mech = 3; }
        } else {
          int ins;
          uint64_t* pv = map_get(&pages, ((uint64_t)c << 44) | page, 0, &ins);
          if (!ins && *pv == (uint64_t)C[c].epoch + 1) mech = 2;
          else { *pv = (uint64_t)C[c].epoch + 1; mech = 1; }
        }
        vb[i] |= (uint8_t)(mech << 2);
        uint32_t lat = mech == 1 ? p->m1_us : mech == 2 ? p->m2_us : p->m3_us;
        ev[nev].t = lat; ev[nev].seq = seq++; ev[nev].i = i; ev[nev].benign = 0; nev++;
      }
    }
  }
  qsort(ev, nev, sizeof(event_t), ev_cmp);
  for (uint64_t e = 0; e < nev; ++e) {
    const rec_t* r = &rec[ev[e].i];
    if (ev[e].benign) canc[ev[e].i] = C[r->c].torn[r->ceng];
    else if (C[r->c].state == 0) terminate(&C[r->c], 1);
  }
  uint64_t nc = 0;
  for (uint64_t i = 0; i < n; ++i) {
    if (rep[i] != EMPTY64) canc[i] = canc[rep[i]];
    if (canc[i]) { vb[i] |= 0x10; cancel[nc++] = (uint32_t)(base + i); }
    out[i].verdict = vb[i];
  }
  *n_cancel = nc;
  for (uint32_t c = 0; c < ncl; ++c) {
    verdict[c].state = C[c].state;
    verdict[c].reason = C[c].reason;
    verdict[c].notifier = C[c].notifier;
    verdict[c].flags = 0;
  }
  map_free(&pages); map_free(&conv);
  free(ev); free(C); free(vb); free(canc); free(rep); free(rec); free(off);
  return 0;
}
