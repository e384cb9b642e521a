/* TEST INFRASTRUCTURE — CPU oracle for the broadcast hot path; see
 * bcast_oracle.h for the usage rule. Plain C restatement of the reference
 * bcastlab (paths relative to /root/reference/proj). Pinned against the
 * reference's own outputs by tests/test_oracle_golden.py (fixtures generated
 * by tests/golden/make_golden.py through oracle/_ref/ref_harness). */
#include "bcast_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ core */

/* make_chunks: src/core.cpp:67-85. */
int64_t orc_make_chunks(uint64_t m, uint64_t c, orc_chunk* out, uint64_t cap) {
  if (c == 0) return -1;
  if (m == 0) {
    if (cap >= 1) { out[0].chunk_id = 0; out[0].offset = 0; out[0].length = 0; }
    return 1;
  }
  uint64_t count = (m + c - 1) / c;
  uint64_t off = 0;
  for (uint64_t i = 0; i < count && i < cap; ++i) {
    uint64_t len = c < m - off ? c : m - off;
    out[i].chunk_id = (uint32_t)i;
    out[i].offset = off;
    out[i].length = len;
    off += len;
  }
  return (int64_t)count;
}

/* ceil_log: src/core.cpp:244-258. */
static int ceil_log(int base, int64_t n) {
  int steps = 0;
  int64_t reach = 1;
  while (reach < n) { reach *= base; ++steps; }
  return steps;
}

/* ------------------------------------------------------------- schedules */

typedef struct { orc_event* v; uint64_t n, cap; } evlist;

static void push(evlist* l, int kind, int peer, uint32_t chunk, uint32_t group) {
  if (l->n == l->cap) {
    l->cap = l->cap ? l->cap * 2 : 8;
    l->v = (orc_event*)realloc(l->v, l->cap * sizeof(orc_event));
  }
  orc_event e = {kind, peer, chunk, group};
  l->v[l->n++] = e;
}

/* rotate_to_root: src/schedules.cpp:24-44 (logical l -> (l + root) mod n). */
static void finish(orc_schedule* s, int n, int root, uint64_t m, int prologue,
                   orc_chunk* chunks, uint32_t n_chunks, evlist* logical) {
  s->n = n; s->root = root; s->message_bytes = m; s->prologue = prologue;
  s->chunks = chunks; s->n_chunks = n_chunks;
  s->ev_off = (uint64_t*)calloc((size_t)n + 1, sizeof(uint64_t));
  evlist* actual = (evlist*)calloc((size_t)n, sizeof(evlist));
  for (int l = 0; l < n; ++l) {
    int a = (l + root) % n;
    for (uint64_t i = 0; i < logical[l].n; ++i) logical[l].v[i].peer = (logical[l].v[i].peer + root) % n;
    actual[a] = logical[l];
  }
  uint64_t total = 0;
  for (int r = 0; r < n; ++r) { s->ev_off[r] = total; total += actual[r].n; }
  s->ev_off[n] = total;
  s->events = (orc_event*)malloc((total ? total : 1) * sizeof(orc_event));
  for (int r = 0; r < n; ++r) {
    if (actual[r].n) memcpy(s->events + s->ev_off[r], actual[r].v, actual[r].n * sizeof(orc_event));
    free(actual[r].v);
  }
  free(actual);
  free(logical);
}

static orc_chunk* chunks_for(uint64_t m, uint64_t c, uint32_t* count) {
  int64_t k = orc_make_chunks(m, c, NULL, 0);
  orc_chunk* v = (orc_chunk*)malloc((size_t)k * sizeof(orc_chunk));
  orc_make_chunks(m, c, v, (uint64_t)k);
  *count = (uint32_t)k;
  return v;
}

/* whole_message_chunk: src/schedules.cpp:46-49. */
static orc_chunk* whole(uint64_t m, uint32_t* count) { return chunks_for(m, m > 0 ? m : 1, count); }

/* knomial_logical_ops: src/schedules.cpp:73-111. */
static void knomial_ops(int n, int k, evlist* ops) {
  int rounds = ceil_log(k, n);
  uint32_t* next_group = (uint32_t*)malloc((size_t)n * sizeof(uint32_t));
  for (int r = 0; r < n; ++r) next_group[r] = 1;
  for (int rank = 0; rank < n; ++rank) {
    int top = rounds;
    if (rank != 0) {
      int64_t power = 1;
      int position = 0;
      while (rank % (power * k) == 0) { power *= k; ++position; }
      int digit = (int)((rank / power) % k);
      int parent = rank - digit * (int)power;
      push(&ops[rank], ORC_RECV, parent, 0, 0);
      top = position;
    }
    for (int position = top - 1; position >= 0; --position) {
      int64_t power = 1;
      for (int i = 0; i < position; ++i) power *= k;
      int children[64];
      int nc = 0;
      for (int digit = 1; digit < k; ++digit) {
        int64_t child = rank + digit * power;
        if (child < n && nc < 64) children[nc++] = (int)child;
      }
      if (nc == 0) continue;
      uint32_t group = nc > 1 ? next_group[rank]++ : 0;
      for (int i = 0; i < nc; ++i) push(&ops[rank], ORC_SEND, children[i], 0, group);
    }
  }
  free(next_group);
}

/* partition_chunks: src/schedules.cpp:53-66. */
static orc_chunk* partitions(int n, uint64_t m) {
  uint64_t base = m / (uint64_t)n, rem = m % (uint64_t)n, off = 0;
  orc_chunk* v = (orc_chunk*)malloc((size_t)n * sizeof(orc_chunk));
  for (uint64_t i = 0; i < (uint64_t)n; ++i) {
    uint64_t len = base + (i < rem ? 1 : 0);
    v[i].chunk_id = (uint32_t)i; v[i].offset = off; v[i].length = len;
    off += len;
  }
  return v;
}

/* schedule_scatter_ring_allgather: src/schedules.cpp:189-242. */
static void sra_ops(int n, evlist* ops) {
  uint32_t* next_group = (uint32_t*)malloc((size_t)n * sizeof(uint32_t));
  for (int r = 0; r < n; ++r) next_group[r] = 1;
  unsigned char* has = (unsigned char*)calloc((size_t)n * (size_t)n, 1);
  for (int c = 0; c < n; ++c) has[c] = 1; /* rank 0 holds everything */
  int* qlo = (int*)malloc((size_t)(2 * n + 2) * sizeof(int));
  int* qhi = (int*)malloc((size_t)(2 * n + 2) * sizeof(int));
  int head = 0, tail = 0;
  qlo[tail] = 0; qhi[tail] = n; ++tail;
  while (head < tail) {
    int lo = qlo[head], hi = qhi[head];
    ++head;
    while (hi - lo > 1) {
      int mid = lo + (hi - lo + 1) / 2;
      uint32_t group = hi - mid > 1 ? next_group[lo]++ : 0;
      for (int c = mid; c < hi; ++c) {
        push(&ops[lo], ORC_SEND, mid, (uint32_t)c, group);
        push(&ops[mid], ORC_RECV, lo, (uint32_t)c, 0);
        has[(size_t)mid * n + c] = 1;
      }
      qlo[tail] = mid; qhi[tail] = hi; ++tail;
      hi = mid;
    }
  }
  for (int step = 1; step < n; ++step) {
    for (int rank = 0; rank < n; ++rank) {
      int dst = (rank + 1) % n;
      int part = ((rank - step + 1) % n + n) % n;
      if (dst == 0 || has[(size_t)dst * n + part]) continue;
      push(&ops[rank], ORC_SEND, dst, (uint32_t)part, 0);
      push(&ops[dst], ORC_RECV, rank, (uint32_t)part, 0);
    }
  }
  free(qlo); free(qhi); free(has); free(next_group);
}

/* make_schedule dispatch: src/schedules.cpp:244-263, with the generators at
 * :115-187 and require_root :14-21, AlgorithmConfig::validate core.cpp:56-65. */
int orc_make_schedule(int algo, int radix, uint64_t chunk_bytes, int n,
                      int root, uint64_t m, orc_schedule* s) {
  memset(s, 0, sizeof *s);
  if (algo < 0 || algo >= ORC_ALGO_COUNT) return -1;
  if ((algo == ORC_KNOMIAL || algo == ORC_KNOMIAL_STAGED) && radix < 2) return -1;
  if (algo == ORC_CHAIN_PIPELINED && chunk_bytes == 0) return -1;
  if (n < 1 || root < 0 || root >= n) return -1;
  if (algo == ORC_CHAIN_PIPELINED && n < 2) return -1;
  evlist* ops = (evlist*)calloc((size_t)n, sizeof(evlist));
  uint32_t nch = 0;
  orc_chunk* ch = NULL;
  int prologue = 0;
  switch (algo) {
    case ORC_DIRECT:
      for (int r = 1; r < n; ++r) { push(&ops[0], ORC_SEND, r, 0, 0); push(&ops[r], ORC_RECV, 0, 0, 0); }
      ch = whole(m, &nch); prologue = 1;
      break;
    case ORC_CHAIN:
      for (int r = 0; r + 1 < n; ++r) { push(&ops[r], ORC_SEND, r + 1, 0, 0); push(&ops[r + 1], ORC_RECV, r, 0, 0); }
      ch = whole(m, &nch);
      break;
    case ORC_KNOMIAL:
    case ORC_KNOMIAL_STAGED:
      knomial_ops(n, radix, ops);
      ch = whole(m, &nch);
      prologue = algo == ORC_KNOMIAL_STAGED ? 2 : 0;
      break;
    case ORC_SRA:
      ch = partitions(n, m); nch = (uint32_t)n;
      sra_ops(n, ops);
      break;
    case ORC_CHAIN_PIPELINED:
      ch = chunks_for(m, chunk_bytes, &nch);
      for (uint32_t c = 0; c < nch; ++c) push(&ops[0], ORC_SEND, 1, c, 0);
      for (int r = 1; r + 1 < n; ++r)
        for (uint32_t c = 0; c < nch; ++c) { push(&ops[r], ORC_RECV, r - 1, c, 0); push(&ops[r], ORC_SEND, r + 1, c, 0); }
      for (uint32_t c = 0; c < nch; ++c) push(&ops[n - 1], ORC_RECV, n - 2, c, 0);
      break;
  }
  finish(s, n, root, m, prologue, ch, nch, ops);
  return 0;
}

void orc_free_schedule(orc_schedule* s) {
  free(s->chunks); free(s->ev_off); free(s->events);
  memset(s, 0, sizeof *s);
}

/* -------------------------------------------------------------- executor */

typedef struct { uint32_t chunk; uint64_t len; uint8_t* data; } msg;
typedef struct { msg* v; uint64_t head, n, cap; } fifo;

/* execute_rank (src/runtime.cpp:32-64) for every rank, interleaved on one
 * thread over per-pair FIFOs with the in-process transport's rules: send
 * copies eagerly (transport_inproc.cpp:79-88), recv takes the pair's head and
 * rejects an out-of-order chunk id (:90-105), the length must match
 * (runtime.cpp:51-57). Returns -2 on a stall (a schedule that would block). */
int orc_execute(const orc_schedule* s, uint8_t* const* bufs) {
  int n = s->n;
  fifo* q = (fifo*)calloc((size_t)n * (size_t)n, sizeof(fifo));
  uint64_t* pc = (uint64_t*)calloc((size_t)n, sizeof(uint64_t));
  int rc = 0;
  for (;;) {
    int progress = 0, done = 1;
    for (int r = 0; r < n && rc == 0; ++r) {
      uint64_t end = s->ev_off[r + 1] - s->ev_off[r];
      while (pc[r] < end) {
        const orc_event* e = &s->events[s->ev_off[r] + pc[r]];
        const orc_chunk* c = &s->chunks[e->chunk];
        if (e->kind == ORC_SEND) {
          fifo* f = &q[(size_t)r * n + e->peer];
          if (f->n == f->cap) { f->cap = f->cap ? 2 * f->cap : 8; f->v = (msg*)realloc(f->v, f->cap * sizeof(msg)); }
          msg mm = {e->chunk, c->length, (uint8_t*)malloc(c->length ? c->length : 1)};
          if (c->length) memcpy(mm.data, bufs[r] + c->offset, c->length);
          f->v[f->n++] = mm;
        } else {
          fifo* f = &q[(size_t)e->peer * n + r];
          if (f->head == f->n) break;
          msg mm = f->v[f->head++];
          if (mm.chunk != e->chunk || mm.len != c->length) { free(mm.data); rc = -3; break; }
          if (mm.len) memcpy(bufs[r] + c->offset, mm.data, mm.len);
          free(mm.data);
        }
        ++pc[r];
        progress = 1;
      }
      if (pc[r] < end) done = 0;
    }
    if (rc != 0 || done) break;
    if (!progress) { rc = -2; break; }
  }
  for (size_t i = 0; i < (size_t)n * n; ++i) {
    for (uint64_t j = q[i].head; j < q[i].n; ++j) free(q[i].v[j].data);
    free(q[i].v);
  }
  free(q); free(pc);
  return rc;
}

int orc_bcast(int algo, int radix, uint64_t chunk_bytes, int n, int root,
              uint64_t m, uint8_t* const* bufs) {
  orc_schedule s;
  int rc = orc_make_schedule(algo, radix, chunk_bytes, n, root, m, &s);
  if (rc) return rc;
  rc = orc_execute(&s, bufs);
  orc_free_schedule(&s);
  return rc;
}

/* mt19937_64 (the standard's parameters) for payload_for,
 * tools/bcastlab.cpp:140-145. */
void orc_payload(uint64_t seed, uint64_t size, uint8_t* out) {
  enum { NN = 312, MM = 156 };
  static const uint64_t MATRIX_A = 0xB5026F5AA96619E9ULL;
  uint64_t mt[NN];
  mt[0] = seed * 0x9e3779b97f4a7c15ULL + size + 1;
  for (int i = 1; i < NN; ++i) mt[i] = 6364136223846793005ULL * (mt[i - 1] ^ (mt[i - 1] >> 62)) + (uint64_t)i;
  int idx = NN;
  for (uint64_t k = 0; k < size; ++k) {
    if (idx >= NN) {
      for (int i = 0; i < NN; ++i) {
        uint64_t x = (mt[i] & 0xFFFFFFFF80000000ULL) | (mt[(i + 1) % NN] & 0x7FFFFFFFULL);
        uint64_t xa = x >> 1;
        if (x & 1) xa ^= MATRIX_A;
        mt[i] = mt[(i + MM) % NN] ^ xa;
      }
      idx = 0;
    }
    uint64_t y = mt[idx++];
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= y >> 43;
    out[k] = (uint8_t)y;
  }
}

uint64_t orc_fnv1a(const uint8_t* p, uint64_t n) {
  uint64_t h = 1469598103934665603ULL;
  for (uint64_t i = 0; i < n; ++i) { h ^= p[i]; h *= 1099511628211ULL; }
  return h;
}

/* ------------------------------------------------------------------ tuner */

static const char* kNames[ORC_ALGO_COUNT] = {"direct", "chain", "knomial",
    "scatter_ring_allgather", "chain_pipelined", "knomial_staged"};

/* cost_for and Eqs. 1-6: src/models.cpp:20-124 (make_cost sums the three
 * terms in order, :24-32). Returns NaN on a contract error. */
double orc_cost(const orc_config* c, int n, uint64_t m, double ts, double bw,
                double st) {
  if (ts < 0.0 || !(bw > 0.0) || !(st > 0.0)) return NAN;
  if ((c->algorithm == ORC_KNOMIAL || c->algorithm == ORC_KNOMIAL_STAGED) && c->radix_k < 2) return NAN;
  if (c->algorithm == ORC_CHAIN_PIPELINED && c->chunk_bytes == 0) return NAN;
  double bytes = (double)m / bw;
  double a, b, g = 0.0;
  switch (c->algorithm) {
    case ORC_DIRECT: { if (n < 1) return NAN; double k = (double)n; a = k * ts; b = k * bytes; break; }
    case ORC_CHAIN: { if (n < 1) return NAN; double k = (double)(n - 1); a = k * ts; b = k * bytes; break; }
    case ORC_KNOMIAL: { if (n < 1) return NAN; double k = (double)ceil_log(c->radix_k, n); a = k * ts; b = k * bytes; break; }
    case ORC_SRA: {
      if (n < 1) return NAN;
      double k = (double)(ceil_log(2, n) + n - 1);
      double frac = (double)(n - 1) / (double)n;
      a = k * ts; b = 2.0 * frac * bytes; break;
    }
    case ORC_CHAIN_PIPELINED: {
      if (n < 2) return NAN;
      uint64_t count = m == 0 ? 1 : (m + c->chunk_bytes - 1) / c->chunk_bytes;
      uint64_t first = m == 0 ? 0 : (c->chunk_bytes < m ? c->chunk_bytes : m);
      double k = (double)(count + (uint64_t)n - 2);
      a = k * ts; b = k * ((double)first / bw); break;
    }
    case ORC_KNOMIAL_STAGED: {
      if (n < 1) return NAN;
      double k = (double)ceil_log(c->radix_k, n);
      a = k * ts; b = k * bytes; g = (double)m / st; break;
    }
    default: return NAN;
  }
  return a + b + g;
}

/* beats: src/tuner.cpp:84-92. */
static int beats(double lc, const orc_config* l, double rc, const orc_config* r) {
  if (lc != rc) return lc < rc;
  if (l->algorithm != r->algorithm) return l->algorithm < r->algorithm;
  if (l->chunk_bytes != r->chunk_bytes) return l->chunk_bytes < r->chunk_bytes;
  return l->radix_k < r->radix_k;
}

static int cfg_eq(const orc_config* a, const orc_config* b) {
  return a->algorithm == b->algorithm && a->radix_k == b->radix_k && a->chunk_bytes == b->chunk_bytes;
}

/* geometric_mean: src/tuner.cpp:27-31. */
static uint64_t gmean(uint64_t lo, uint64_t hi) {
  return (uint64_t)llround(sqrt((double)lo * (double)hi));
}

/* tune: src/tuner.cpp:118-176 with expand_candidates :94-116 and
 * pick_winner :38-54, analytical oracle. */
int64_t orc_tune(const int* n_list, int n_count, const uint64_t* sizes,
                 int n_sizes, const orc_config* cands, int n_cands,
                 const uint64_t* chunks, int n_chunks, double ts, double bw,
                 double st, orc_entry* out) {
  if (ts < 0.0 || !(bw > 0.0) || !(st > 0.0)) return -1;
  if (n_count == 0 || n_sizes == 0 || n_cands == 0) return -1;
  for (int i = 0; i + 1 < n_sizes; ++i) if (sizes[i] >= sizes[i + 1]) return -1;
  if (sizes[0] == 0) return -1;
  uint64_t* bounds = (uint64_t*)malloc((size_t)(n_sizes + 1) * sizeof(uint64_t));
  bounds[0] = sizes[0];
  for (int i = 0; i + 1 < n_sizes; ++i) bounds[i + 1] = gmean(sizes[i], sizes[i + 1]);
  bounds[n_sizes] = sizes[n_sizes - 1] * 2;
  orc_config* exp = (orc_config*)malloc((size_t)(n_cands * (n_chunks + 1) + 1) * sizeof(orc_config));
  int64_t count = 0;
  for (int ni = 0; ni < n_count; ++ni) {
    int n = n_list[ni];
    int64_t row_start = count;
    for (int i = 0; i < n_sizes; ++i) {
      uint64_t m = sizes[i];
      int ne = 0;
      for (int c = 0; c < n_cands; ++c) {
        if (cands[c].algorithm != ORC_CHAIN_PIPELINED) { exp[ne++] = cands[c]; continue; }
        for (int k = 0; k < n_chunks; ++k) {
          orc_config p = cands[c];
          uint64_t mm = m > 1 ? m : 1;
          uint64_t v = chunks[k] < mm ? chunks[k] : mm;
          p.chunk_bytes = v > 1 ? v : 1;
          int dup = 0;
          for (int j = 0; j < ne; ++j) if (cfg_eq(&exp[j], &p)) { dup = 1; break; }
          if (!dup) exp[ne++] = p;
        }
      }
      if (ne == 0) { free(bounds); free(exp); return -1; }
      orc_config best = exp[0];
      double best_cost = 0.0;
      int have = 0;
      for (int j = 0; j < ne; ++j) {
        double cost = orc_cost(&exp[j], n, m, ts, bw, st);
        if (isnan(cost)) { free(bounds); free(exp); return -1; }
        if (!have || beats(cost, &exp[j], best_cost, &best)) { best = exp[j]; best_cost = cost; have = 1; }
      }
      if (count > row_start && cfg_eq(&out[count - 1].config, &best)) {
        out[count - 1].msg_max = bounds[i + 1];
        continue;
      }
      orc_entry e = {n, bounds[i], bounds[i + 1], best, 0.0};
      out[count++] = e;
    }
    for (int64_t j = row_start; j < count; ++j) {
      uint64_t mid = gmean(out[j].msg_min, out[j].msg_max);
      out[j].cost = orc_cost(&out[j].config, n, mid, ts, bw, st);
    }
  }
  /* stable sort by (n, msg_min): insertion sort keeps equal keys in order */
  for (int64_t i = 1; i < count; ++i) {
    orc_entry key = out[i];
    int64_t j = i - 1;
    while (j >= 0 && (out[j].n > key.n || (out[j].n == key.n && out[j].msg_min > key.msg_min))) { out[j + 1] = out[j]; --j; }
    out[j + 1] = key;
  }
  free(bounds); free(exp);
  return count;
}

/* select: src/tuner.cpp:178-197. */
int orc_select(const orc_entry* e, int64_t count, int n, uint64_t m, orc_config* out) {
  if (count <= 0) return -1;
  int chosen = -1;
  for (int64_t i = 0; i < count; ++i) if (e[i].n <= n && e[i].n > chosen) chosen = e[i].n;
  if (chosen < 0) return -2;
  const orc_entry* match = NULL;
  for (int64_t i = 0; i < count; ++i) {
    if (e[i].n != chosen) continue;
    match = &e[i];
    if (m < e[i].msg_max) break;
  }
  *out = match->config;
  return 0;
}

/* std::to_chars(double) plain overload: shortest round-trip digits, fixed
 * or scientific whichever is shorter, fixed on a tie (used by save_table,
 * src/tuner.cpp:56-60). */
int orc_format_double(double v, char* out, int cap) {
  char buf[64], digits[32], fixed[400], sci[64];
  if (v == 0.0) return snprintf(out, (size_t)cap, signbit(v) ? "-0" : "0");
  if (isnan(v)) return snprintf(out, (size_t)cap, signbit(v) ? "-nan" : "nan");
  if (isinf(v)) return snprintf(out, (size_t)cap, v < 0 ? "-inf" : "inf");
  int p;
  for (p = 1; p <= 17; ++p) {
    snprintf(buf, sizeof buf, "%.*e", p - 1, v);
    if (strtod(buf, NULL) == v) break;
  }
  const char* s = buf;
  int neg = 0;
  if (*s == '-') { neg = 1; ++s; }
  int nd = 0;
  for (; *s && *s != 'e'; ++s) if (*s != '.') digits[nd++] = *s;
  digits[nd] = 0;
  int ex = atoi(s + 1);
  /* scientific */
  int k = 0;
  if (neg) sci[k++] = '-';
  sci[k++] = digits[0];
  if (nd > 1) { sci[k++] = '.'; memcpy(sci + k, digits + 1, (size_t)nd - 1); k += nd - 1; }
  k += snprintf(sci + k, sizeof sci - (size_t)k, "e%c%02d", ex < 0 ? '-' : '+', ex < 0 ? -ex : ex);
  /* fixed */
  int f = 0;
  if (neg) fixed[f++] = '-';
  if (ex >= 0) {
    for (int i = 0; i <= ex; ++i) fixed[f++] = i < nd ? digits[i] : '0';
    if (nd > ex + 1) { fixed[f++] = '.'; for (int i = ex + 1; i < nd; ++i) fixed[f++] = digits[i]; }
  } else {
    fixed[f++] = '0'; fixed[f++] = '.';
    for (int i = 0; i < -ex - 1; ++i) fixed[f++] = '0';
    for (int i = 0; i < nd; ++i) fixed[f++] = digits[i];
  }
  fixed[f] = 0;
  const char* pick = f <= k ? fixed : sci;
  return snprintf(out, (size_t)cap, "%s", pick);
}

static const char* kHeader =
    "n,msg_min_bytes,msg_max_bytes,algorithm,radix,chunk_bytes,predicted_cost_s";

/* save_table: src/tuner.cpp:203-229 (unused parameters written as 0). */
int64_t orc_save_table(const orc_entry* e, int64_t count, int oracle, char* out, int64_t cap) {
  size_t sz = 4096 + (size_t)count * 160;
  char* text = (char*)malloc(sz);
  size_t k = 0;
  k += (size_t)snprintf(text + k, sz - k, "# oracle: %s\n%s\n", oracle ? "simulated" : "analytical", kHeader);
  for (int64_t i = 0; i < count; ++i) {
    const orc_config* c = &e[i].config;
    int uses_radix = c->algorithm == ORC_KNOMIAL || c->algorithm == ORC_KNOMIAL_STAGED;
    int uses_chunk = c->algorithm == ORC_CHAIN_PIPELINED;
    char num[64];
    orc_format_double(e[i].cost, num, sizeof num);
    k += (size_t)snprintf(text + k, sz - k, "%d,%llu,%llu,%s,%d,%llu,%s\n", e[i].n,
                          (unsigned long long)e[i].msg_min, (unsigned long long)e[i].msg_max,
                          kNames[c->algorithm], uses_radix ? c->radix_k : 0,
                          (unsigned long long)(uses_chunk ? c->chunk_bytes : 0), num);
  }
  if ((int64_t)k + 1 > cap) { free(text); return (int64_t)k + 1; }
  memcpy(out, text, k + 1);
  free(text);
  return (int64_t)k;
}

/* std::from_chars-strict integer parse (no sign for unsigned, no spaces). */
static int parse_u64(const char* s, size_t n, uint64_t* v) {
  if (n == 0) return -1;
  uint64_t x = 0;
  for (size_t i = 0; i < n; ++i) {
    if (s[i] < '0' || s[i] > '9') return -1;
    uint64_t d = (uint64_t)(s[i] - '0');
    if (x > (UINT64_MAX - d) / 10) return -1;
    x = x * 10 + d;
  }
  *v = x;
  return 0;
}

static int parse_int(const char* s, size_t n, int* v) {
  int neg = n > 0 && s[0] == '-';
  uint64_t x;
  if (parse_u64(s + neg, n - (size_t)neg, &x)) return -1;
  if (x > (uint64_t)2147483647 + (uint64_t)neg) return -1;
  *v = neg ? (int)(-(int64_t)x) : (int)x;
  return 0;
}

static int parse_double(const char* s, size_t n, double* v) {
  char buf[128];
  if (n == 0 || n >= sizeof buf) return -1;
  if (s[0] == ' ' || s[0] == '+' || s[0] == '\t') return -1;
  memcpy(buf, s, n); buf[n] = 0;
  const char* t = buf + (buf[0] == '-');
  if (t[0] == '0' && (t[1] == 'x' || t[1] == 'X')) return -1;
  char* end;
  *v = strtod(buf, &end);
  return end == buf + n ? 0 : -1;
}

/* load_table: src/tuner.cpp:267-345 (line-numbered TableParseError). */
int64_t orc_load_table(const char* text, orc_entry* out, int64_t cap, int* oracle_out) {
  int64_t count = 0, line_no = 0;
  int saw_header = 0;
  *oracle_out = 0;
  const char* p = text;
  while (*p) {
    const char* nl = strchr(p, '\n');
    size_t len = nl ? (size_t)(nl - p) : strlen(p);
    ++line_no;
    const char* line = p;
    p = nl ? nl + 1 : p + len;
    if (len > 0 && line[len - 1] == '\r') --len;
    if (len == 0) continue;
    if (len >= 9 && strncmp(line, "# oracle:", 9) == 0) {
      const char* nm = line + 9;
      size_t nl2 = len - 9;
      size_t skip = 0;
      while (skip < nl2 && nm[skip] == ' ') ++skip;
      if (skip == nl2) return -line_no;
      nm += skip; nl2 -= skip;
      if (nl2 == 10 && strncmp(nm, "analytical", 10) == 0) *oracle_out = 0;
      else if (nl2 == 9 && strncmp(nm, "simulated", 9) == 0) *oracle_out = 1;
      else return -line_no;
      continue;
    }
    if (line[0] == '#') continue;
    if (!saw_header) {
      if (len != strlen(kHeader) || strncmp(line, kHeader, len) != 0) return -line_no;
      saw_header = 1;
      continue;
    }
    const char* f[16];
    size_t fl[16];
    int nf = 0;
    size_t start = 0;
    for (size_t i = 0; i <= len; ++i) {
      if (i == len || line[i] == ',') {
        if (i == len && start == len && len > 0 && line[len - 1] != ',') break;
        if (nf < 16) { f[nf] = line + start; fl[nf] = i - start; }
        ++nf;
        start = i + 1;
      }
    }
    if (nf != 7) return -line_no;
    orc_entry e;
    memset(&e, 0, sizeof e);
    if (parse_int(f[0], fl[0], &e.n)) return -line_no;
    if (parse_u64(f[1], fl[1], &e.msg_min)) return -line_no;
    if (parse_u64(f[2], fl[2], &e.msg_max)) return -line_no;
    int algo = -1;
    for (int a = 0; a < ORC_ALGO_COUNT; ++a)
      if (strlen(kNames[a]) == fl[3] && strncmp(kNames[a], f[3], fl[3]) == 0) algo = a;
    if (algo < 0) return -line_no;
    e.config.algorithm = algo;
    if (parse_int(f[4], fl[4], &e.config.radix_k)) return -line_no;
    if (parse_u64(f[5], fl[5], &e.config.chunk_bytes)) return -line_no;
    if (parse_double(f[6], fl[6], &e.cost)) return -line_no;
    if (e.n < 1) return -line_no;
    if (e.msg_min >= e.msg_max) return -line_no;
    if (count < cap) out[count] = e;
    ++count;
  }
  if (!saw_header) return line_no ? -line_no : -1000000;
  if (count == 0) return line_no ? -line_no : -1000000;
  /* per-n ranges sorted and disjoint; the reported line is the last one read */
  for (int64_t i = 0; i < count && i < cap; ++i) {
    for (int64_t j = i - 1; j >= 0; --j) {
      if (out[j].n == out[i].n) {
        if (out[i].msg_min < out[j].msg_max) return -line_no;
        break;
      }
    }
  }
  return count;
}
