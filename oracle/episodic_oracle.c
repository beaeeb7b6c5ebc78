/* TEST INFRASTRUCTURE ONLY — CPU restatement of the reference counting path.
 * See episodic_oracle.h. Plain C11 + POSIX threads; compiled by oracle/Makefile
 * into oracle/_build/libepisodic_oracle.so. The product never links this.
 *
 * Reference anchors (paths relative to /root/reference/proj/include/episodic):
 *   validate / from_events   types.hpp:82-92, types.hpp:102-119
 *   run_fsm / count_fsm      fsm.hpp:45-106
 *   enumerate_all / extend   oracle.hpp:21-60
 *   max_nonoverlap           oracle.hpp:65-79
 *   episode-parallel batch   miner.hpp:146-150
 */
#include "episodic_oracle.h"

#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* E/types.hpp:102-119: checks in this order per event; first failure wins. */
int orc_validate_stream(const uint32_t* types, const int64_t* times, uint64_t n,
                        uint32_t alphabet, char* msg, size_t msg_len) {
  int64_t prev = 0;
  for (uint64_t i = 0; i < n; ++i) {
    const char* err = NULL;
    if (times[i] < 0) err = "negative event time";
    else if (i > 0 && times[i] < prev) err = "event times must be non-decreasing";
    else if (types[i] >= alphabet) err = "event type id out of range";
    if (err) {
      if (msg && msg_len) snprintf(msg, msg_len, "%s", err);
      return 2;
    }
    prev = times[i];
  }
  return 0;
}

/* E/types.hpp:82-92 */
static int episode_valid(const int64_t* lo, const int64_t* hi, uint32_t n_nodes) {
  if (n_nodes == 0) return 0;
  for (uint32_t k = 0; k + 1 < n_nodes; ++k)
    if (lo[k] < 0 || lo[k] >= hi[k]) return 0;
  return 1;
}

typedef struct {
  int64_t* t;
  uint64_t len, cap, head;
} tlist;

static void tl_push(tlist* l, int64_t t) {
  if (l->len == l->cap) {
    l->cap = l->cap ? l->cap * 2 : 16;
    l->t = (int64_t*)realloc(l->t, sizeof(int64_t) * l->cap);
  }
  l->t[l->len++] = t;
}

/* run_fsm (E/fsm.hpp:45-98) with count_fsm's arguments (E/fsm.hpp:101-106):
 * begin = 0, prev_end = -inf, count_start_limit = n (never binding), no scan
 * limit. One list of accepted event times per position (the min_start field
 * of E/fsm.hpp:26-29 only feeds count_start_limit, which count_fsm never
 * binds, so it is not carried). Positions are visited in increasing order per
 * event (E/fsm.hpp:61); the head pointer drops entries older than t-high
 * (E/fsm.hpp:73) and admission needs an entry older than t-low
 * (E/fsm.hpp:75-79); completing the last position counts, sets pe = t and
 * clears every list (E/fsm.hpp:83-91). */
uint64_t orc_count_fsm(const uint32_t* types, const int64_t* times, uint64_t n,
                       const uint32_t* ep_types, const int64_t* lo, const int64_t* hi,
                       uint32_t n_nodes) {
  if (!episode_valid(lo, hi, n_nodes)) return UINT64_MAX;
  tlist* lists = (tlist*)calloc(n_nodes, sizeof(tlist));
  uint64_t count = 0;
  int have_pe = 0;
  int64_t pe = 0;
  for (uint64_t i = 0; i < n; ++i) {
    const int64_t t = times[i];
    const uint32_t ty = types[i];
    for (uint32_t k = 0; k < n_nodes; ++k) {
      if (ep_types[k] != ty) continue;
      int admitted;
      if (k == 0) {
        admitted = !have_pe || t > pe;
      } else {
        tlist* p = &lists[k - 1];
        while (p->head < p->len && p->t[p->head] < t - hi[k - 1]) ++p->head;
        admitted = p->head < p->len && p->t[p->head] < t - lo[k - 1];
      }
      if (!admitted) continue;
      if (k + 1 == n_nodes) {
        ++count;
        pe = t;
        have_pe = 1;
        for (uint32_t j = 0; j < n_nodes; ++j) lists[j].len = lists[j].head = 0;
      } else {
        tl_push(&lists[k], t);
      }
    }
  }
  for (uint32_t j = 0; j < n_nodes; ++j) free(lists[j].t);
  free(lists);
  return count;
}

typedef struct {
  int64_t s, e;
} interval;

typedef struct {
  interval* v;
  uint64_t len, cap;
} ivec;

static void iv_push(ivec* a, int64_t s, int64_t e) {
  if (a->len == a->cap) {
    a->cap = a->cap ? a->cap * 2 : 64;
    a->v = (interval*)realloc(a->v, sizeof(interval) * a->cap);
  }
  a->v[a->len].s = s;
  a->v[a->len].e = e;
  ++a->len;
}

/* oracle_detail::extend (E/oracle.hpp:21-36) */
static void extend(const uint32_t* types, const int64_t* times, uint64_t n,
                   const uint32_t* ep_types, const int64_t* lo, const int64_t* hi,
                   uint32_t n_nodes, uint32_t k, uint64_t prev_index, int64_t start, ivec* out) {
  if (k == n_nodes) return;
  const int64_t prev_time = times[prev_index];
  for (uint64_t j = prev_index + 1; j < n; ++j) {
    const int64_t t = times[j];
    if (t > prev_time + hi[k - 1]) break;
    if (types[j] != ep_types[k]) continue;
    const int64_t gap = t - prev_time;
    if (!(gap > lo[k - 1] && gap <= hi[k - 1])) continue;
    if (k + 1 == n_nodes)
      iv_push(out, start, t);
    else
      extend(types, times, n, ep_types, lo, hi, n_nodes, k + 1, j, start, out);
  }
}

static int by_end_then_start(const void* a, const void* b) {
  const interval* x = (const interval*)a;
  const interval* y = (const interval*)b;
  if (x->e != y->e) return x->e < y->e ? -1 : 1;
  if (x->s != y->s) return x->s < y->s ? -1 : 1;
  return 0;
}

/* max_nonoverlap (E/oracle.hpp:65-79): greedy by (end, start); a later
 * occurrence must start strictly after the last selected end. */
static uint64_t greedy_sorted(const interval* v, uint64_t n) {
  uint64_t count = 0;
  int have = 0;
  int64_t prev_end = 0;
  for (uint64_t i = 0; i < n; ++i) {
    if (!have || prev_end < v[i].s) {
      prev_end = v[i].e;
      have = 1;
      ++count;
    }
  }
  return count;
}

uint64_t orc_max_nonoverlap(const int64_t* starts, const int64_t* ends, uint64_t n) {
  interval* v = (interval*)malloc(sizeof(interval) * (n ? n : 1));
  for (uint64_t i = 0; i < n; ++i) {
    v[i].s = starts[i];
    v[i].e = ends[i];
  }
  qsort(v, n, sizeof(interval), by_end_then_start);
  uint64_t c = greedy_sorted(v, n);
  free(v);
  return c;
}

/* enumerate_all + max_nonoverlap = oracle_count (E/oracle.hpp:42-85).
 * Duplicate intervals collapse (std::set in the reference); duplicates never
 * change the greedy count, but they are removed anyway for fidelity. */
uint64_t orc_oracle_count(const uint32_t* types, const int64_t* times, uint64_t n,
                          const uint32_t* ep_types, const int64_t* lo, const int64_t* hi,
                          uint32_t n_nodes) {
  if (!episode_valid(lo, hi, n_nodes)) return UINT64_MAX;
  if (n > 500 || n_nodes > 6) return UINT64_MAX; /* OracleLimits, E/oracle.hpp:14-17 */
  ivec found = {0, 0, 0};
  for (uint64_t i = 0; i < n; ++i) {
    if (types[i] != ep_types[0]) continue;
    if (n_nodes == 1)
      iv_push(&found, times[i], times[i]);
    else
      extend(types, times, n, ep_types, lo, hi, n_nodes, 1, i, times[i], &found);
  }
  qsort(found.v, found.len, sizeof(interval), by_end_then_start);
  uint64_t u = 0;
  for (uint64_t i = 0; i < found.len; ++i)
    if (u == 0 || found.v[i].s != found.v[u - 1].s || found.v[i].e != found.v[u - 1].e)
      found.v[u++] = found.v[i];
  uint64_t c = greedy_sorted(found.v, u);
  free(found.v);
  return c;
}

typedef struct {
  const uint32_t* types;
  const int64_t* times;
  uint64_t n;
  const uint32_t* off;
  const uint32_t* ep_types;
  const int64_t* lo;
  const int64_t* hi;
  uint64_t begin, end;
  uint64_t* out;
  int bad;
} batch_job;

static void* batch_worker(void* arg) {
  batch_job* j = (batch_job*)arg;
  for (uint64_t e = j->begin; e < j->end; ++e) {
    uint32_t b = j->off[e], nn = j->off[e + 1] - b;
    uint64_t cb = (uint64_t)b - e;
    uint64_t c = orc_count_fsm(j->types, j->times, j->n, j->ep_types + b, j->lo + cb,
                               j->hi + cb, nn);
    if (c == UINT64_MAX) j->bad = 1;
    j->out[e] = c;
  }
  return NULL;
}

int orc_count_batch(const uint32_t* types, const int64_t* times, uint64_t n,
                    const uint32_t* off, const uint32_t* ep_types, const int64_t* lo,
                    const int64_t* hi, uint64_t n_eps, unsigned threads, uint64_t* out) {
  if (threads < 1) threads = 1;
  if (threads > n_eps) threads = n_eps ? (unsigned)n_eps : 1;
  batch_job* jobs = (batch_job*)calloc(threads, sizeof(batch_job));
  pthread_t* tid = (pthread_t*)calloc(threads, sizeof(pthread_t));
  for (unsigned w = 0; w < threads; ++w) {
    batch_job* j = &jobs[w];
    j->types = types;
    j->times = times;
    j->n = n;
    j->off = off;
    j->ep_types = ep_types;
    j->lo = lo;
    j->hi = hi;
    j->begin = n_eps * w / threads;
    j->end = n_eps * (w + 1) / threads;
    j->out = out;
    if (w > 0) pthread_create(&tid[w], NULL, batch_worker, j);
  }
  batch_worker(&jobs[0]);
  int bad = jobs[0].bad;
  for (unsigned w = 1; w < threads; ++w) {
    pthread_join(tid[w], NULL);
    bad |= jobs[w].bad;
  }
  free(jobs);
  free(tid);
  return bad ? 1 : 0;
}

/* FNV-1a-64 over (n, alphabet, then type, time per event) as little-endian
 * u64 words: the stream digest recorded by oracle/make_golden.cpp. */
uint64_t orc_fnv_stream(const uint32_t* types, const int64_t* times, uint64_t n, uint32_t alphabet) {
  uint64_t h = 1469598103934665603ULL;
#define MIX(v)                                   \
  do {                                           \
    uint64_t x_ = (uint64_t)(v);                 \
    for (int b_ = 0; b_ < 8; ++b_) {             \
      h ^= (x_ >> (8 * b_)) & 0xff;              \
      h *= 1099511628211ULL;                     \
    }                                            \
  } while (0)
  MIX(n);
  MIX(alphabet);
  for (uint64_t i = 0; i < n; ++i) {
    MIX(types[i]);
    MIX(times[i]);
  }
#undef MIX
  return h;
}
