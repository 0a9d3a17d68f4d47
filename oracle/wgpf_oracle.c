/*
 * oracle/wgpf_oracle.c -- TEST INFRASTRUCTURE ONLY: the CPU checker the CUDA
 * path is compared against.  Never linked into or called by the product.
 *
 * A line-by-line *semantic* restatement of the reference post-processor in
 * C11 (single-threaded, no SIMD).  Each function cites the reference lines it
 * follows; paths are relative to /root/reference/proj/include/wgprof/.
 * Where the reference has undefined or unspecified behaviour the choice made
 * here is stated in a comment marked DEVIATION.
 */
#define _GNU_SOURCE
#include "wgpf_oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* Errors (error.hpp:8-55)                                                   */
/* ------------------------------------------------------------------------ */

enum { K_PARSE, K_VALIDATE, K_INSTRUMENT, K_LOWER, K_CAPACITY, K_DEADLOCK,
       K_TRACE, K_CONFIG, K_IO };

static const char* category_of(int kind) {
  static const char* names[] = {"parse-error",    "validate-error",
                                "instrument-error", "lower-error",
                                "capacity-error", "simulation-deadlock",
                                "trace-error",    "config-error",
                                "io-error"};
  return (kind >= 0 && kind <= K_IO) ? names[kind] : "error";
}

static int fail(wgpo_status* st, int kind, const char* fmt, ...) {
  if (st) {
    st->code = 1 + kind;
    snprintf(st->category, sizeof st->category, "%s", category_of(kind));
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(st->message, sizeof st->message, fmt, ap);
    va_end(ap);
  }
  return 1 + kind;
}

static void ok(wgpo_status* st) {
  if (st) {
    st->code = 0;
    st->category[0] = 0;
    st->message[0] = 0;
  }
}

static void* xmalloc(size_t n) {
  void* p = malloc(n ? n : 1);
  if (!p) {
    fprintf(stderr, "wgpf_oracle: out of memory (%zu bytes)\n", n);
    abort();
  }
  return p;
}

static void* xcalloc(size_t n, size_t sz) {
  void* p = calloc(n ? n : 1, sz ? sz : 1);
  if (!p) {
    fprintf(stderr, "wgpf_oracle: out of memory\n");
    abort();
  }
  return p;
}

/* ------------------------------------------------------------------------ */
/* Labels (trace.hpp:302-306, instrument.hpp:29, trace.hpp:377-382)          */
/* ------------------------------------------------------------------------ */

const char* wgpo_label_of(const wgpo_plan* plan, uint32_t id, char* buf) {
  if (id < plan->n_labels)
    return plan->labels[id];
  snprintf(buf, 32, "region#%u", id);
  return buf;
}

static int is_wait_marker(const char* label) {
  size_t n = strlen(label);
  return n > 5 && memcmp(label + n - 5, ".wait", 5) == 0;
}

/* label(marker) == label(base) + ".wait" */
static int is_wait_of(const char* marker, const char* base) {
  size_t nb = strlen(base), nm = strlen(marker);
  return nm == nb + 5 && memcmp(marker, base, nb) == 0 &&
         memcmp(marker + nb, ".wait", 5) == 0;
}

/* ------------------------------------------------------------------------ */
/* KPFT parsing (deserialize_image, trace.hpp:181-209)                       */
/* ------------------------------------------------------------------------ */

static uint32_t rd32(const uint8_t* p) {
  return (uint32_t)p[0] | ((uint32_t)p[1] << 8) | ((uint32_t)p[2] << 16) |
         ((uint32_t)p[3] << 24);
}

typedef struct stream_view {
  wgpf_stream_hdr h;
  const uint8_t* slots; /* h.slot_capacity * 8 bytes */
} stream_view;

/* Parses a KPFT image into stream views (no copy).  v1 exactly as the
 * reference; v2 (this framework's container) with a u64 stream count. */
static int parse_image(const uint8_t* b, uint64_t n, stream_view** out,
                       uint64_t* n_streams, wgpo_status* st) {
  uint64_t pos = 0;
  *out = NULL;
  *n_streams = 0;
  if (n < 4)
    return fail(st, K_TRACE, "truncated trace image");
  if (memcmp(b, "KPFT", 4) != 0)
    return fail(st, K_TRACE, "bad magic: not a trace image");
  pos = 4;
  if (pos + 2 > n)
    return fail(st, K_TRACE, "truncated trace image");
  uint16_t version = (uint16_t)(b[pos] | (b[pos + 1] << 8));
  pos += 2;
  uint64_t count;
  if (version == 1) {
    if (pos + 2 > n)
      return fail(st, K_TRACE, "truncated trace image");
    count = (uint16_t)(b[pos] | (b[pos + 1] << 8));
    pos += 2;
  } else if (version == 2) { /* extension: u16 reserved, u64 count */
    if (pos + 10 > n)
      return fail(st, K_TRACE, "truncated trace image");
    pos += 2;
    count = (uint64_t)rd32(b + pos) | ((uint64_t)rd32(b + pos + 4) << 32);
    pos += 8;
  } else {
    return fail(st, K_TRACE, "unsupported trace version %u",
                (unsigned)version);
  }
  /* Streams are parsed lazily with bounds checks; a huge bogus count fails
   * with "truncated" like the reference (which would first try to resize). */
  uint64_t cap_guess = count < (n / 16 + 1) ? count : (n / 16 + 1);
  stream_view* v = (stream_view*)xmalloc(sizeof(stream_view) * cap_guess);
  uint64_t k = 0;
  for (uint64_t s = 0; s < count; ++s) {
    if (pos + 16 > n) {
      free(v);
      return fail(st, K_TRACE, "truncated trace image");
    }
    if (k == cap_guess) { /* cannot happen: each stream needs >= 16 bytes */
      free(v);
      return fail(st, K_TRACE, "truncated trace image");
    }
    v[k].h.block_index = rd32(b + pos);
    v[k].h.warp_group = rd32(b + pos + 4);
    v[k].h.record_count = rd32(b + pos + 8);
    v[k].h.slot_capacity = rd32(b + pos + 12);
    pos += 16;
    uint64_t need = (uint64_t)v[k].h.slot_capacity * 8u;
    if (pos + need > n) {
      free(v);
      return fail(st, K_TRACE, "truncated trace image");
    }
    v[k].slots = b + pos;
    pos += need;
    ++k;
  }
  if (pos != n) {
    free(v);
    return fail(st, K_TRACE, "trailing bytes after trace image");
  }
  *out = v;
  *n_streams = k;
  return 0;
}

static int parse_body(const uint8_t* b, uint64_t n, uint64_t count,
                      stream_view** out, uint64_t* n_streams,
                      wgpo_status* st) {
  uint64_t pos = 0;
  stream_view* v = (stream_view*)xmalloc(sizeof(stream_view) * (count + 1));
  for (uint64_t s = 0; s < count; ++s) {
    if (pos + 16 > n) {
      free(v);
      return fail(st, K_TRACE, "truncated trace image");
    }
    v[s].h.block_index = rd32(b + pos);
    v[s].h.warp_group = rd32(b + pos + 4);
    v[s].h.record_count = rd32(b + pos + 8);
    v[s].h.slot_capacity = rd32(b + pos + 12);
    pos += 16;
    uint64_t need = (uint64_t)v[s].h.slot_capacity * 8u;
    if (pos + need > n) {
      free(v);
      return fail(st, K_TRACE, "truncated trace image");
    }
    v[s].slots = b + pos;
    pos += need;
  }
  if (pos != n) {
    free(v);
    return fail(st, K_TRACE, "trailing bytes after trace image");
  }
  *out = v;
  *n_streams = count;
  return 0;
}

/* ------------------------------------------------------------------------ */
/* decode_image (trace.hpp:222-251)                                          */
/* ------------------------------------------------------------------------ */

static int check_decode(const stream_view* v, uint64_t ns,
                        const wgpo_plan* plan, wgpo_status* st) {
  for (uint64_t s = 0; s < ns; ++s) {
    const wgpf_stream_hdr* h = &v[s].h;
    if ((uint64_t)h->slot_capacity != plan->slots_per_warp_group)
      return fail(st, K_TRACE,
                  "stream capacity %u does not match the buffer plan (%llu)",
                  h->slot_capacity,
                  (unsigned long long)plan->slots_per_warp_group);
    if (h->record_count > h->slot_capacity) {
      if (plan->strategy == WGPF_STRATEGY_FLUSH)
        return fail(st, K_TRACE,
                    "flush stream claims more records than slots");
      /* DEVIATION: the reference computes count % 0 (UB) for a circular
       * zero-capacity stream with writes; reported as a trace error. */
      if (h->slot_capacity == 0)
        return fail(st, K_TRACE, "circular stream has zero slot capacity");
    }
  }
  return 0;
}

/* Chronological records of one stream; returns count, sets *dropped. */
static uint64_t decode_stream(const stream_view* sv, wgpf_record* out,
                              uint32_t* dropped) {
  const wgpf_stream_hdr* h = &sv->h;
  if (h->record_count <= h->slot_capacity) {
    for (uint32_t i = 0; i < h->record_count; ++i) {
      out[i].tag = rd32(sv->slots + 8u * i);
      out[i].payload = rd32(sv->slots + 8u * i + 4);
    }
    *dropped = 0;
    return h->record_count;
  }
  *dropped = h->record_count - h->slot_capacity;
  const uint32_t start = h->record_count % h->slot_capacity;
  for (uint32_t i = 0; i < h->slot_capacity; ++i) {
    uint32_t slot = (uint32_t)(((uint64_t)start + i) % h->slot_capacity);
    out[i].tag = rd32(sv->slots + 8u * slot);
    out[i].payload = rd32(sv->slots + 8u * slot + 4);
  }
  return h->slot_capacity;
}

int wgpo_decode_kpft(const uint8_t* bytes, uint64_t n, const wgpo_plan* plan,
                     wgpo_decode_out* out, wgpo_status* st) {
  memset(out, 0, sizeof *out);
  ok(st);
  stream_view* v = NULL;
  uint64_t ns = 0;
  int rc = parse_image(bytes, n, &v, &ns, st);
  if (rc)
    return rc;
  rc = check_decode(v, ns, plan, st);
  if (rc) {
    free(v);
    return rc;
  }
  uint64_t total = 0;
  for (uint64_t s = 0; s < ns; ++s)
    total += v[s].h.record_count <= v[s].h.slot_capacity
                 ? v[s].h.record_count
                 : v[s].h.slot_capacity;
  out->n_streams = ns;
  out->block = (uint32_t*)xmalloc(4 * ns);
  out->wg = (uint32_t*)xmalloc(4 * ns);
  out->dropped = (uint32_t*)xmalloc(4 * ns);
  out->offset = (uint64_t*)xmalloc(8 * (ns + 1));
  out->records = (wgpf_record*)xmalloc(sizeof(wgpf_record) * total);
  uint64_t k = 0;
  for (uint64_t s = 0; s < ns; ++s) {
    out->block[s] = v[s].h.block_index;
    out->wg[s] = v[s].h.warp_group;
    out->offset[s] = k;
    k += decode_stream(&v[s], out->records + k, &out->dropped[s]);
  }
  out->offset[ns] = k;
  out->n_records = k;
  free(v);
  return 0;
}

void wgpo_free_decode(wgpo_decode_out* out) {
  free(out->block);
  free(out->wg);
  free(out->dropped);
  free(out->offset);
  free(out->records);
  memset(out, 0, sizeof *out);
}

/* ------------------------------------------------------------------------ */
/* unwrap_clock (trace.hpp:257-272)                                          */
/* ------------------------------------------------------------------------ */

void wgpo_unwrap_clock(const uint32_t* v, uint64_t n, uint64_t* out) {
  uint64_t cur = 0;
  for (uint64_t i = 0; i < n; ++i) {
    if (i == 0)
      cur = v[0];
    else
      cur += (uint32_t)(v[i] - v[i - 1]);
    out[i] = cur;
  }
}

/* ------------------------------------------------------------------------ */
/* pair_records (trace.hpp:294-346)                                          */
/*                                                                           */
/* std::map<region, vector<Open>> is restated as a small open-addressing     */
/* table keyed by region id whose values are singly linked stacks threaded   */
/* through a node array (one node per START).                                */
/* ------------------------------------------------------------------------ */

typedef struct region_slot {
  uint32_t id;
  uint32_t used;
  int64_t top;        /* node index of the stack top, -1 when empty */
  uint64_t depth;
  uint32_t completed; /* completed[id] (u32 like the reference) */
} region_slot;

typedef struct open_node {
  uint64_t clock;
  uint64_t pos;
  int64_t next;
} open_node;

typedef struct region_table {
  region_slot* slots;
  uint64_t cap;
} region_table;

static void rt_init(region_table* t, uint64_t n) {
  uint64_t cap = 16;
  while (cap < 2 * n + 16)
    cap <<= 1;
  t->cap = cap;
  t->slots = (region_slot*)xcalloc(cap, sizeof(region_slot));
}

static region_slot* rt_get(region_table* t, uint32_t id) {
  uint64_t h = ((uint64_t)id * 0x9E3779B97F4A7C15ull) >> 20;
  for (uint64_t i = 0;; ++i) {
    region_slot* s = &t->slots[(h + i) & (t->cap - 1)];
    if (!s->used) {
      s->used = 1;
      s->id = id;
      s->top = -1;
      s->depth = 0;
      s->completed = 0;
      return s;
    }
    if (s->id == id)
      return s;
  }
}

static int pair_stream(const wgpf_record* r, uint64_t n,
                       const wgpo_plan* plan, wgpo_pair_out* out,
                       wgpo_status* st) {
  uint64_t* u = (uint64_t*)xmalloc(8 * n);
  {
    uint64_t cur = 0;
    for (uint64_t i = 0; i < n; ++i) {
      cur = i == 0 ? r[0].payload : cur + (uint32_t)(r[i].payload - r[i - 1].payload);
      u[i] = cur;
    }
  }
  region_table rt;
  rt_init(&rt, n);
  open_node* nodes = (open_node*)xmalloc(sizeof(open_node) * (n ? n : 1));
  uint64_t n_nodes = 0;
  out->iv = (wgpo_interval*)xmalloc(sizeof(wgpo_interval) * (n / 2 + 1));
  out->n = 0;
  out->dropped_heads = 0;
  out->truncated_tails = 0;
  for (uint64_t pos = 0; pos < n; ++pos) {
    const uint32_t tag = r[pos].tag;
    const uint32_t id = (tag >> 12) & (WGPF_MAX_REGIONS - 1u);
    region_slot* rs = rt_get(&rt, id);
    if (tag & WGPF_START_FLAG) {
      nodes[n_nodes].clock = u[pos];
      nodes[n_nodes].pos = pos;
      nodes[n_nodes].next = rs->top;
      rs->top = (int64_t)n_nodes++;
      rs->depth++;
    } else {
      if (rs->top < 0) {
        out->dropped_heads++;
        continue;
      }
      const open_node* top = &nodes[rs->top];
      wgpo_interval* iv = &out->iv[out->n];
      iv->region_id = id;
      iv->start = top->clock;
      iv->start_pos = top->pos;
      iv->end = u[pos];
      iv->end_pos = pos;
      iv->iteration = rs->completed++;
      rs->top = top->next;
      rs->depth--;
      if (iv->end - iv->start >= (1ull << 32)) {
        char buf[32];
        const char* label = wgpo_label_of(plan, id, buf);
        free(u);
        free(nodes);
        free(rt.slots);
        free(out->iv);
        out->iv = NULL;
        out->n = 0;
        return fail(st, K_TRACE,
                    "interval \"%s\" exceeds 2^32 cycles; the 32-bit clock "
                    "cannot represent it",
                    label);
      }
      out->n++;
    }
  }
  for (uint64_t i = 0; i < rt.cap; ++i)
    if (rt.slots[i].used)
      out->truncated_tails += (uint32_t)rt.slots[i].depth;
  free(u);
  free(nodes);
  free(rt.slots);
  return 0;
}

int wgpo_pair_records(const wgpf_record* recs, uint64_t n,
                      const wgpo_plan* plan, wgpo_pair_out* out,
                      wgpo_status* st) {
  memset(out, 0, sizeof *out);
  ok(st);
  return pair_stream(recs, n, plan, out, st);
}

void wgpo_free_pair(wgpo_pair_out* out) {
  free(out->iv);
  memset(out, 0, sizeof *out);
}

/* ------------------------------------------------------------------------ */
/* replay (trace.hpp:398-487)                                                */
/* ------------------------------------------------------------------------ */

typedef struct event_vec {
  wgpf_event* v;
  uint64_t n, cap;
} event_vec;

static void ev_push(event_vec* e, const wgpf_event* x) {
  if (e->n == e->cap) {
    e->cap = e->cap ? 2 * e->cap : 64;
    wgpf_event* nv = (wgpf_event*)realloc(e->v, sizeof(wgpf_event) * e->cap);
    if (!nv) {
      fprintf(stderr, "wgpf_oracle: out of memory\n");
      abort();
    }
    e->v = nv;
  }
  e->v[e->n++] = *x;
}

typedef struct pos_idx {
  uint64_t pos, idx;
} pos_idx;

static int cmp_pos_idx(const void* a, const void* b) {
  const pos_idx* x = (const pos_idx*)a;
  const pos_idx* y = (const pos_idx*)b;
  if (x->pos != y->pos) return x->pos < y->pos ? -1 : 1;
  return x->idx < y->idx ? -1 : (x->idx > y->idx);
}

typedef struct warn4 {
  uint32_t flagged, malformed;
} warn4;

static void replay_stream(const wgpo_interval* iv, uint64_t n,
                          const wgpo_plan* plan, uint32_t block, uint32_t wg,
                          uint64_t cost, event_vec* out, warn4* w) {
  /* marker_at: std::map<start_pos, index> (:405-410).  Later markers with
   * the same start_pos overwrite earlier ones, as map operator[] does. */
  uint64_t max_pos = 0;
  for (uint64_t i = 0; i < n; ++i) {
    if (iv[i].start_pos > max_pos) max_pos = iv[i].start_pos;
    if (iv[i].end_pos > max_pos) max_pos = iv[i].end_pos;
  }
  int64_t* marker_at = NULL;
  unsigned char* consumed = (unsigned char*)xcalloc(n, 1);
  char** labels = (char**)xmalloc(sizeof(char*) * (n ? n : 1));
  char* lbuf = (char*)xmalloc(32 * (n ? n : 1));
  unsigned char* marker = (unsigned char*)xcalloc(n, 1);
  for (uint64_t i = 0; i < n; ++i) {
    labels[i] = (char*)wgpo_label_of(plan, iv[i].region_id, lbuf + 32 * i);
    marker[i] = (unsigned char)is_wait_marker(labels[i]);
  }
  /* positions can be arbitrary u64 for caller-built intervals: index the
   * markers with a sorted (pos, idx) array; for equal positions the largest
   * index wins, as repeated map assignment does. */
  uint64_t n_mk = 0;
  for (uint64_t i = 0; i < n; ++i)
    n_mk += marker[i];
  pos_idx* mk = (pos_idx*)xmalloc(sizeof(pos_idx) * (n_mk + 1));
  {
    uint64_t k = 0;
    for (uint64_t i = 0; i < n; ++i)
      if (marker[i]) {
        mk[k].pos = iv[i].start_pos;
        mk[k].idx = i;
        ++k;
      }
    qsort(mk, n_mk, sizeof(pos_idx), cmp_pos_idx);
  }
  (void)marker_at;
  (void)max_pos;

  for (uint64_t i = 0; i < n; ++i) {
    if (consumed[i] || marker[i])
      continue;
    const wgpo_interval* a = &iv[i];
    wgpf_event ev;
    const uint64_t inside = a->end_pos - a->start_pos;
    const uint64_t overhead = cost * inside;
    const uint64_t measured = a->end - a->start;
    ev.start = a->start;
    ev.end = a->start + (measured >= overhead ? measured - overhead : 0);
    ev.region = a->region_id | WGPF_EV_CORRECTED;
    ev.iteration = a->iteration;
    ev.block_index = block;
    ev.warp_group = wg;
    ev_push(out, &ev);
    consumed[i] = 1;

    /* marker_at.find(end_pos + 1) */
    const uint64_t key = a->end_pos + 1;
    uint64_t lo = 0, hi = n_mk;
    while (lo < hi) { /* first entry with pos > key */
      uint64_t mid = (lo + hi) / 2;
      if (mk[mid].pos <= key) lo = mid + 1; else hi = mid;
    }
    if (lo == 0 || mk[lo - 1].pos != key)
      continue;
    const uint64_t m = mk[lo - 1].idx;
    if (!is_wait_of(labels[m], labels[i]))
      continue;
    consumed[m] = 1;
    wgpf_event wt;
    wt.start = a->end;
    wt.end = iv[m].start;
    wt.iteration = a->iteration;
    wt.block_index = block;
    wt.warp_group = wg;
    if (wt.end < wt.start) {
      w->malformed++;
      continue;
    }
    if (wt.end - wt.start <= cost) {
      wt.region = iv[m].region_id | WGPF_EV_WAIT;
      w->flagged++;
    } else {
      wt.region = iv[m].region_id | WGPF_EV_WAIT | WGPF_EV_CORRECTED;
    }
    ev_push(out, &wt);
  }
  /* Orphan markers (:469-485). */
  for (uint64_t i = 0; i < n; ++i) {
    if (consumed[i] || !marker[i])
      continue;
    wgpf_event ev;
    ev.start = iv[i].start;
    ev.end = iv[i].end;
    ev.region = iv[i].region_id;
    ev.iteration = iv[i].iteration;
    ev.block_index = block;
    ev.warp_group = wg;
    ev_push(out, &ev);
    w->malformed++;
  }
  free(consumed);
  free(labels);
  free(lbuf);
  free(marker);
  free(mk);
}

int wgpo_replay_pairs(const wgpo_interval* iv, uint64_t n,
                      const wgpo_plan* plan, uint32_t block, uint32_t wg,
                      uint64_t record_cost, wgpo_replay_out* out,
                      wgpo_status* st) {
  memset(out, 0, sizeof *out);
  ok(st);
  event_vec ev = {0};
  warn4 w = {0, 0};
  replay_stream(iv, n, plan, block, wg, record_cost, &ev, &w);
  out->events = ev.v;
  out->n_events = ev.n;
  out->flagged_preconditions = w.flagged;
  out->malformed_groups = w.malformed;
  return 0;
}

/* ------------------------------------------------------------------------ */
/* replay_image (pipeline.hpp:66-81)                                         */
/* ------------------------------------------------------------------------ */

static int replay_views(const stream_view* v, uint64_t ns,
                        const wgpo_plan* plan, uint64_t cost,
                        wgpo_replay_out* out, wgpo_status* st) {
  int rc = check_decode(v, ns, plan, st); /* decode_image runs first */
  if (rc)
    return rc;
  uint64_t maxn = 0;
  for (uint64_t s = 0; s < ns; ++s)
    if (v[s].h.slot_capacity > maxn)
      maxn = v[s].h.slot_capacity;
  wgpf_record* recs = (wgpf_record*)xmalloc(sizeof(wgpf_record) * (maxn + 1));
  event_vec ev = {0};
  uint32_t dh = 0, tt = 0;
  warn4 w = {0, 0};
  uint64_t total = 0;
  for (uint64_t s = 0; s < ns; ++s) {
    uint32_t dropped;
    uint64_t n = decode_stream(&v[s], recs, &dropped);
    total += n;
    wgpo_pair_out pr;
    rc = pair_stream(recs, n, plan, &pr, st);
    if (rc) {
      free(recs);
      free(ev.v);
      return rc;
    }
    dh += pr.dropped_heads;
    tt += pr.truncated_tails;
    replay_stream(pr.iv, pr.n, plan, v[s].h.block_index, v[s].h.warp_group,
                  cost, &ev, &w);
    free(pr.iv);
  }
  free(recs);
  out->events = ev.v;
  out->n_events = ev.n;
  out->dropped_heads = dh;
  out->truncated_tails = tt;
  out->flagged_preconditions = w.flagged;
  out->malformed_groups = w.malformed;
  out->n_streams = ns;
  out->records = total;
  return 0;
}

int wgpo_replay_kpft(const uint8_t* bytes, uint64_t n, const wgpo_plan* plan,
                     uint64_t record_cost, wgpo_replay_out* out,
                     wgpo_status* st) {
  memset(out, 0, sizeof *out);
  ok(st);
  stream_view* v = NULL;
  uint64_t ns = 0;
  int rc = parse_image(bytes, n, &v, &ns, st);
  if (rc)
    return rc;
  rc = replay_views(v, ns, plan, record_cost, out, st);
  free(v);
  return rc;
}

int wgpo_replay_body(const uint8_t* body, uint64_t body_bytes,
                     uint64_t n_streams, const wgpo_plan* plan,
                     uint64_t record_cost, wgpo_replay_out* out,
                     wgpo_status* st) {
  memset(out, 0, sizeof *out);
  ok(st);
  stream_view* v = NULL;
  uint64_t ns = 0;
  int rc = parse_body(body, body_bytes, n_streams, &v, &ns, st);
  if (rc)
    return rc;
  rc = replay_views(v, ns, plan, record_cost, out, st);
  free(v);
  return rc;
}

void wgpo_free_replay(wgpo_replay_out* out) {
  free(out->events);
  memset(out, 0, sizeof *out);
}

/* ------------------------------------------------------------------------ */
/* region_stats (pipeline.hpp:114-133) + extensions                          */
/* ------------------------------------------------------------------------ */

typedef struct label_key {
  const char* label;
  uint64_t idx; /* index into the stats array */
} label_key;

static int cmp_label(const void* a, const void* b) {
  return strcmp(((const wgpo_stat*)a)->label, ((const wgpo_stat*)b)->label);
}

int wgpo_region_stats(const wgpf_event* ev, uint64_t n, const wgpo_plan* plan,
                      wgpo_stats_out* out) {
  memset(out, 0, sizeof *out);
  /* Distinct region ids -> label; distinct labels -> stats slot.  Region ids
   * are hashed; labels compared with strcmp (std::string order). */
  region_table rt;
  rt_init(&rt, 64);
  uint64_t n_ids = 0;
  /* first pass: collect distinct ids */
  uint32_t* ids = (uint32_t*)xmalloc(4 * (n + 1));
  for (uint64_t i = 0; i < n; ++i) {
    uint32_t id = ev[i].region & WGPF_EV_REGION_MASK;
    if (n_ids * 2 + 16 > rt.cap) { /* grow: rebuild */
      region_table nt;
      rt_init(&nt, n_ids * 2 + 16);
      for (uint64_t k = 0; k < n_ids; ++k) {
        region_slot* s = rt_get(&nt, ids[k]);
        s->depth = 1;
        s->completed = (uint32_t)k;
      }
      free(rt.slots);
      rt = nt;
    }
    region_slot* s = rt_get(&rt, id);
    if (s->depth == 0) { /* new */
      s->depth = 1;
      s->completed = (uint32_t)n_ids;
      ids[n_ids++] = id;
    }
  }
  /* labels for each distinct id, merge equal labels */
  out->names = (char*)xmalloc(32 * (n_ids + 1));
  const char** lab = (const char**)xmalloc(sizeof(char*) * (n_ids + 1));
  for (uint64_t k = 0; k < n_ids; ++k)
    lab[k] = wgpo_label_of(plan, ids[k], out->names + 32 * k);
  /* slot of each distinct id: first id with an equal label */
  uint64_t* slot_of = (uint64_t*)xmalloc(8 * (n_ids + 1));
  uint64_t n_slots = 0;
  const char** slot_label = (const char**)xmalloc(sizeof(char*) * (n_ids + 1));
  for (uint64_t k = 0; k < n_ids; ++k) {
    uint64_t j;
    for (j = 0; j < n_slots; ++j)
      if (strcmp(slot_label[j], lab[k]) == 0)
        break;
    if (j == n_slots)
      slot_label[n_slots++] = lab[k];
    slot_of[k] = j;
  }
  wgpo_stat* s = (wgpo_stat*)xcalloc(n_slots, sizeof(wgpo_stat));
  for (uint64_t j = 0; j < n_slots; ++j)
    s[j].label = slot_label[j];
  uint32_t* cnt32 = (uint32_t*)xcalloc(n_slots, 4);
  for (uint64_t i = 0; i < n; ++i) {
    uint32_t id = ev[i].region & WGPF_EV_REGION_MASK;
    wgpo_stat* rs = &s[slot_of[rt_get(&rt, id)->completed]];
    uint32_t* c = &cnt32[rs - s];
    const uint64_t d = ev[i].end - ev[i].start;
    if (rs->count == 0) {
      rs->warp_group = ev[i].warp_group;
      rs->kind = (ev[i].region & WGPF_EV_WAIT) ? 1u : 0u;
      rs->min = d;
      rs->max = d;
      rs->first_event = i;
    } else {
      if (d < rs->min) rs->min = d;
      if (d > rs->max) rs->max = d;
    }
    /* rs.mean = (rs.mean * rs.count + double(d)) / (rs.count + 1) with the
     * reference's u32 count (:129-130).  Compiled with -ffp-contract=off. */
    {
      volatile double prod = rs->mean * (double)(*c);
      volatile double num = prod + (double)d;
      rs->mean = num / (double)(uint32_t)(*c + 1u);
    }
    *c += 1u;
    rs->count++;
    rs->sum += d;
    rs->hist[wgpf_hist_bin(d)]++;
  }
  for (uint64_t j = 0; j < n_slots; ++j)
    s[j].mean_exact = s[j].count ? (double)s[j].sum / (double)s[j].count : 0.0;
  qsort(s, n_slots, sizeof(wgpo_stat), cmp_label);
  out->n = (uint32_t)n_slots;
  out->s = s;
  free(cnt32);
  free(ids);
  free(lab);
  free(slot_of);
  free(slot_label);
  free(rt.slots);
  return 0;
}

void wgpo_free_stats(wgpo_stats_out* out) {
  free(out->s);
  free(out->names);
  memset(out, 0, sizeof *out);
}

/* ------------------------------------------------------------------------ */
/* analyze_critical_path (perfmodel.hpp:317-501)                             */
/* ------------------------------------------------------------------------ */

typedef struct ev_ref {
  const wgpf_event* e;
  uint64_t order; /* event index, for the stable tie order */
  uint32_t stage;
} ev_ref;

static int cmp_iter(const void* a, const void* b) {
  const ev_ref* x = (const ev_ref*)a;
  const ev_ref* y = (const ev_ref*)b;
  if (x->e->iteration != y->e->iteration)
    return x->e->iteration < y->e->iteration ? -1 : 1;
  /* DEVIATION: std::sort is unstable (:332-335); ties (same label in several
   * warp groups / blocks) are ordered by event index here. */
  return x->order < y->order ? -1 : (x->order > y->order);
}

static int close_to(uint64_t pred_end, uint64_t succ_start, uint64_t theta) {
  const uint64_t lo = pred_end > theta ? pred_end - theta : 0;
  return succ_start >= lo && succ_start <= pred_end + theta;
}

typedef struct sort_str {
  const char* s;
  uint32_t idx;
} sort_str;

static int cmp_sort_str(const void* a, const void* b) {
  return strcmp(((const sort_str*)a)->s, ((const sort_str*)b)->s);
}

int wgpo_critical_path(const wgpf_event* ev, uint64_t n, const wgpo_plan* plan,
                       const char* const* barrier_src,
                       const char* const* barrier_dst, uint32_t n_barrier,
                       uint64_t slack, int exclude_warmup, int gate_by_block,
                       wgpo_cp_out* out, wgpo_status* st) {
  memset(out, 0, sizeof *out);
  ok(st);
  /* by_region: labels of the kept events */
  out->names = (char*)xmalloc(32 * (n + 1));
  const char** lab = (const char**)xmalloc(sizeof(char*) * (n + 1));
  unsigned char* keep = (unsigned char*)xcalloc(n, 1);
  for (uint64_t i = 0; i < n; ++i) {
    lab[i] = wgpo_label_of(plan, ev[i].region & WGPF_EV_REGION_MASK,
                           out->names + 32 * i);
    keep[i] = !(!(ev[i].region & WGPF_EV_WAIT) && is_wait_marker(lab[i]));
  }
  /* distinct labels sorted */
  sort_str* ss = (sort_str*)xmalloc(sizeof(sort_str) * (n + 1));
  uint64_t m = 0;
  for (uint64_t i = 0; i < n; ++i)
    if (keep[i]) {
      ss[m].s = lab[i];
      ss[m].idx = (uint32_t)i;
      ++m;
    }
  qsort(ss, m, sizeof(sort_str), cmp_sort_str);
  uint32_t n_lab = 0;
  const char** labels = (const char**)xmalloc(sizeof(char*) * (m + 1));
  uint32_t* stage_of_ev = (uint32_t*)xmalloc(4 * (n + 1));
  for (uint64_t k = 0; k < m; ++k) {
    if (n_lab == 0 || strcmp(labels[n_lab - 1], ss[k].s) != 0)
      labels[n_lab++] = ss[k].s;
    stage_of_ev[ss[k].idx] = n_lab - 1;
  }
  /* per-label event lists (in event order), then sorted by iteration */
  uint64_t* lab_cnt = (uint64_t*)xcalloc(n_lab + 1, 8);
  for (uint64_t i = 0; i < n; ++i)
    if (keep[i]) lab_cnt[stage_of_ev[i]]++;
  uint64_t* lab_off = (uint64_t*)xcalloc(n_lab + 1, 8);
  for (uint32_t l = 0; l < n_lab; ++l)
    lab_off[l + 1] = lab_off[l] + lab_cnt[l];
  ev_ref* er = (ev_ref*)xmalloc(sizeof(ev_ref) * (m + 1));
  uint64_t* fill = (uint64_t*)xcalloc(n_lab + 1, 8);
  for (uint64_t i = 0; i < n; ++i)
    if (keep[i]) {
      uint32_t l = stage_of_ev[i];
      ev_ref* r = &er[lab_off[l] + fill[l]++];
      r->e = &ev[i];
      r->order = i;
      r->stage = l;
    }
  /* stages: steady window + mean (:330-353); labels with an empty window
   * are dropped from `stages` */
  uint32_t* stage_idx = (uint32_t*)xmalloc(4 * (n_lab + 1)); /* label->stage */
  out->stage_label = (const char**)xmalloc(sizeof(char*) * (n_lab + 1));
  out->stage_mean = (uint64_t*)xmalloc(8 * (n_lab + 1));
  out->stage_n = (uint64_t*)xmalloc(8 * (n_lab + 1));
  out->stage_wg = (uint32_t*)xmalloc(4 * (n_lab + 1));
  uint64_t* win_lo = (uint64_t*)xmalloc(8 * (n_lab + 1));
  uint64_t* win_hi = (uint64_t*)xmalloc(8 * (n_lab + 1));
  uint32_t ns = 0;
  for (uint32_t l = 0; l < n_lab; ++l) {
    ev_ref* base = er + lab_off[l];
    uint64_t cnt = lab_cnt[l];
    qsort(base, cnt, sizeof(ev_ref), cmp_iter);
    uint64_t lo = 0, hi = cnt;
    if (exclude_warmup && cnt >= 3) {
      lo = 1;
      hi = cnt - 1;
    }
    stage_idx[l] = UINT32_MAX;
    if (hi <= lo)
      continue;
    uint64_t sum = 0;
    for (uint64_t k = lo; k < hi; ++k)
      sum += base[k].e->end - base[k].e->start;
    double q = (double)sum / (double)(hi - lo);
    out->stage_label[ns] = labels[l];
    out->stage_mean[ns] = (uint64_t)llround(q);
    out->stage_n[ns] = hi - lo;
    out->stage_wg[ns] = base[0].e->warp_group;
    win_lo[ns] = lab_off[l] + lo;
    win_hi[ns] = lab_off[l] + hi;
    stage_idx[l] = ns++;
  }
  out->n_stages = ns;
  /* all steady events, in stage (label) order */
  uint64_t n_all = 0;
  for (uint32_t s = 0; s < ns; ++s)
    n_all += win_hi[s] - win_lo[s];
  ev_ref** all = (ev_ref**)xmalloc(sizeof(ev_ref*) * (n_all + 1));
  uint32_t* all_stage = (uint32_t*)xmalloc(4 * (n_all + 1));
  {
    uint64_t k = 0;
    for (uint32_t s = 0; s < ns; ++s)
      for (uint64_t j = win_lo[s]; j < win_hi[s]; ++j) {
        all[k] = &er[j];
        all_stage[k] = s;
        ++k;
      }
  }
  uint64_t* bind = (uint64_t*)xcalloc((uint64_t)ns * ns + 1, 8);
  /* program-order gating (:364-385), O(n^2) like the reference */
  for (uint64_t fi = 0; fi < n_all; ++fi) {
    const wgpf_event* f = all[fi]->e;
    int64_t gate = -1;
    for (uint64_t ei = 0; ei < n_all; ++ei) {
      const wgpf_event* e = all[ei]->e;
      if (ei == fi || e->warp_group != f->warp_group)
        continue;
      if (gate_by_block && e->block_index != f->block_index)
        continue;
      if (e->start > f->start)
        continue;
      if (!close_to(e->end, f->start, slack))
        continue;
      if (gate < 0 || e->end > all[gate]->e->end ||
          (e->end == all[gate]->e->end &&
           strcmp(out->stage_label[all_stage[ei]],
                  out->stage_label[all_stage[gate]]) < 0))
        gate = (int64_t)ei;
    }
    if (gate >= 0)
      bind[(uint64_t)all_stage[gate] * ns + all_stage[fi]]++;
  }
  /* barrier edges (:387-406) */
  for (uint32_t b = 0; b < n_barrier; ++b) {
    int64_t si = -1, di = -1;
    for (uint32_t s = 0; s < ns; ++s) {
      if (strcmp(out->stage_label[s], barrier_src[b]) == 0) si = s;
      if (strcmp(out->stage_label[s], barrier_dst[b]) == 0) di = s;
    }
    if (si < 0 || di < 0) {
      int rc = fail(st, K_TRACE,
                    "critical path: no events for stage \"%s\" referenced by "
                    "a barrier edge",
                    si < 0 ? barrier_src[b] : barrier_dst[b]);
      free(lab); free(keep); free(ss); free(labels); free(stage_of_ev);
      free(lab_cnt); free(lab_off); free(er); free(fill); free(stage_idx);
      free(win_lo); free(win_hi); free(all); free(all_stage); free(bind);
      return rc;
    }
    if (out->stage_wg[si] == out->stage_wg[di])
      continue;
    for (uint64_t fj = win_lo[di]; fj < win_hi[di]; ++fj)
      for (uint64_t ej = win_lo[si]; ej < win_hi[si]; ++ej)
        if (close_to(er[ej].e->end, er[fj].e->start, slack)) {
          bind[(uint64_t)si * ns + di]++;
          break;
        }
  }
  /* binding table + majority fold (:408-427) */
  uint32_t nb = 0;
  for (uint64_t k = 0; k < (uint64_t)ns * ns; ++k)
    nb += bind[k] != 0;
  out->n_bind = nb;
  out->bind_src = (uint32_t*)xmalloc(4 * (nb + 1));
  out->bind_dst = (uint32_t*)xmalloc(4 * (nb + 1));
  out->bind_count = (uint64_t*)xmalloc(8 * (nb + 1));
  unsigned char* adj = (unsigned char*)xcalloc((uint64_t)ns * ns + 1, 1);
  {
    uint32_t k = 0;
    for (uint32_t a = 0; a < ns; ++a)
      for (uint32_t b = 0; b < ns; ++b) {
        uint64_t c = bind[(uint64_t)a * ns + b];
        if (!c) continue;
        out->bind_src[k] = a;
        out->bind_dst[k] = b;
        out->bind_count[k] = c;
        ++k;
        if ((uint32_t)c * 2u < out->stage_n[b])
          continue;
        adj[(uint64_t)a * ns + b] = 1;
      }
  }
  /* max-weight simple cycle (:429-469): iterative DFS over succ in
   * ascending order, nodes > root only. */
  uint32_t* path = (uint32_t*)xmalloc(4 * (ns + 1));
  uint32_t* it = (uint32_t*)xmalloc(4 * (ns + 1));
  unsigned char* on = (unsigned char*)xcalloc(ns + 1, 1);
  uint32_t* best = (uint32_t*)xmalloc(4 * (ns + 1));
  uint32_t best_n = 0;
  uint64_t best_w = 0;
  for (uint32_t root = 0; root < ns; ++root) {
    memset(on, 0, ns);
    uint32_t depth = 1;
    path[0] = root;
    it[0] = 0;
    on[root] = 1;
    while (depth > 0) {
      uint32_t v = path[depth - 1];
      uint32_t s = it[depth - 1];
      while (s < ns && !adj[(uint64_t)v * ns + s])
        ++s;
      if (s >= ns) { /* pop */
        on[v] = (depth == 1);
        --depth;
        if (depth > 0) it[depth - 1]++;
        continue;
      }
      it[depth - 1] = s;
      if (s == root) {
        uint64_t w = 0;
        for (uint32_t k = 0; k < depth; ++k)
          w += out->stage_mean[path[k]];
        if (w > best_w ||
            (w == best_w && depth > 0 && (best_n == 0 || depth < best_n))) {
          best_w = w;
          best_n = depth;
          memcpy(best, path, 4 * depth);
        }
        it[depth - 1]++;
      } else if (s > root && !on[s]) {
        on[s] = 1;
        path[depth] = s;
        it[depth] = 0;
        ++depth;
      } else {
        it[depth - 1]++;
      }
    }
  }
  if (best_n) {
    uint32_t pivot = 0;
    for (uint32_t i = 1; i < best_n; ++i)
      if (strcmp(out->stage_label[best[i]], out->stage_label[best[pivot]]) < 0)
        pivot = i;
    out->cycle = (uint32_t*)xmalloc(4 * best_n);
    for (uint32_t i = 0; i < best_n; ++i)
      out->cycle[i] = best[(pivot + i) % best_n];
    out->n_cycle = best_n;
    out->period = best_w;
  }
  free(path); free(it); free(on); free(best); free(adj);
  free(lab); free(keep); free(ss); free(labels); free(stage_of_ev);
  free(lab_cnt); free(lab_off); free(er); free(fill); free(stage_idx);
  free(win_lo); free(win_hi); free(all); free(all_stage); free(bind);
  return 0;
}

void wgpo_free_cp(wgpo_cp_out* o) {
  free(o->stage_label);
  free(o->stage_mean);
  free(o->stage_n);
  free(o->stage_wg);
  free(o->bind_src);
  free(o->bind_dst);
  free(o->bind_count);
  free(o->cycle);
  free(o->names);
  memset(o, 0, sizeof *o);
}

/* ------------------------------------------------------------------------ */
/* Role overlap counters (framework definition, see header)                  */
/* ------------------------------------------------------------------------ */

typedef struct iv64 {
  uint64_t a, b;
} iv64;

static int cmp_iv(const void* x, const void* y) {
  const iv64* p = (const iv64*)x;
  const iv64* q = (const iv64*)y;
  if (p->a != q->a) return p->a < q->a ? -1 : 1;
  return p->b < q->b ? -1 : (p->b > q->b);
}

/* merges sorted intervals in place, returns count */
static uint64_t merge_iv(iv64* v, uint64_t n) {
  if (!n) return 0;
  uint64_t k = 0;
  for (uint64_t i = 1; i < n; ++i) {
    if (v[i].a <= v[k].b) {
      if (v[i].b > v[k].b) v[k].b = v[i].b;
    } else {
      v[++k] = v[i];
    }
  }
  return k + 1;
}

typedef struct blk_ev {
  uint32_t block;
  uint64_t idx;
} blk_ev;

static int cmp_blk(const void* x, const void* y) {
  const blk_ev* p = (const blk_ev*)x;
  const blk_ev* q = (const blk_ev*)y;
  if (p->block != q->block) return p->block < q->block ? -1 : 1;
  return p->idx < q->idx ? -1 : (p->idx > q->idx);
}

void wgpo_overlap(const wgpf_event* ev, uint64_t n, const uint8_t* role_of_wg,
                  uint32_t n_roles, wgpo_overlap_out* out) {
  memset(out, 0, sizeof *out);
  blk_ev* be = (blk_ev*)xmalloc(sizeof(blk_ev) * (n + 1));
  for (uint64_t i = 0; i < n; ++i) {
    be[i].block = ev[i].block_index;
    be[i].idx = i;
  }
  qsort(be, n, sizeof(blk_ev), cmp_blk);
  iv64* r0 = (iv64*)xmalloc(sizeof(iv64) * (n + 1));
  iv64* r1 = (iv64*)xmalloc(sizeof(iv64) * (n + 1));
  for (uint64_t i = 0; i < n;) {
    uint64_t j = i;
    uint64_t lo = UINT64_MAX, hi = 0;
    uint64_t n0 = 0, n1 = 0;
    while (j < n && be[j].block == be[i].block) {
      const wgpf_event* e = &ev[be[j].idx];
      if (e->start < lo) lo = e->start;
      if (e->end > hi) hi = e->end;
      if (!(e->region & WGPF_EV_WAIT) && e->warp_group < n_roles &&
          e->end > e->start) {
        uint8_t r = role_of_wg[e->warp_group];
        if (r == 0) { r0[n0].a = e->start; r0[n0].b = e->end; ++n0; }
        if (r == 1) { r1[n1].a = e->start; r1[n1].b = e->end; ++n1; }
      }
      ++j;
    }
    qsort(r0, n0, sizeof(iv64), cmp_iv);
    qsort(r1, n1, sizeof(iv64), cmp_iv);
    n0 = merge_iv(r0, n0);
    n1 = merge_iv(r1, n1);
    uint64_t b0 = 0, b1 = 0, both = 0;
    for (uint64_t k = 0; k < n0; ++k) b0 += r0[k].b - r0[k].a;
    for (uint64_t k = 0; k < n1; ++k) b1 += r1[k].b - r1[k].a;
    for (uint64_t p = 0, q = 0; p < n0 && q < n1;) {
      uint64_t a = r0[p].a > r1[q].a ? r0[p].a : r1[q].a;
      uint64_t b = r0[p].b < r1[q].b ? r0[p].b : r1[q].b;
      if (b > a) both += b - a;
      if (r0[p].b < r1[q].b) ++p; else ++q;
    }
    const uint64_t span = hi > lo ? hi - lo : 0;
    out->blocks++;
    out->span += span;
    out->busy[0] += b0;
    out->busy[1] += b1;
    out->both += both;
    out->bubble[0] += span - b0;
    out->bubble[1] += span - b1;
    i = j;
  }
  free(be);
  free(r0);
  free(r1);
}
