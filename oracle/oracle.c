/*
 * oracle.c -- CPU restatement of the reference's KV data path.  TEST INFRASTRUCTURE.
 *
 * Checker only (see oracle.h): tests/, __graft_entry__.smoke() and bench.py's CPU
 * baseline legs load it; the product path (paper_2604_12171_b200) never does.
 * Restates /root/reference/pkg/src/pipeshift/{events,kvstore,migrator}.py with
 * plain C data structures: a lazily invalidated min-heap of free block ids
 * (kvstore.py:104-134), per-block per-group cell maps, request tables, and a
 * sorted-set dirty bitmap.  Pinned against the JSON fixtures in tests/golden.
 */
#include "oracle.h"

#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

static __thread char g_err[256];
const char* or_last_error(void) { return g_err; }

/* ---------------------------------------------------------------- events.py:93-104 */
static uint32_t crc_table[256];
static int crc_ready = 0;
static void crc_init(void) {
  for (uint32_t i = 0; i < 256; ++i) {
    uint32_t c = i;
    for (int j = 0; j < 8; ++j) c = (c & 1) ? 0xEDB88320u ^ (c >> 1) : c >> 1;
    crc_table[i] = c;
  }
  crc_ready = 1;
}
uint32_t or_crc32(const uint8_t* data, int64_t n, uint32_t start) {
  if (!crc_ready) crc_init();
  uint32_t c = start ^ 0xFFFFFFFFu;
  for (int64_t i = 0; i < n; ++i) c = crc_table[(c ^ data[i]) & 0xFF] ^ (c >> 8);
  return c ^ 0xFFFFFFFFu;
}
uint64_t or_stable_hash(const uint8_t* text, int64_t n) {
  uint64_t hi = or_crc32(text, n, 0), lo = or_crc32(text, n, 0x9E3779B9u);
  return ((hi << 32) | lo) >> 1;
}
/* engine.py:259-261 */
uint64_t or_payload(uint64_t seed, int64_t pos) {
  return (seed * 0x9E3779B97F4A7C15ull + (uint64_t)pos * 0xBF58476D1CE4E5B9ull) &
         0x7FFFFFFFFFFFFFFFull;
}
uint64_t or_expand_word(uint64_t fp, uint32_t layer, uint32_t w) {
  uint64_t z = (fp ^ (((uint64_t)layer << 32) | w)) + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
void or_expand_cell(uint64_t fp, uint32_t layer, uint8_t* out, int64_t nbytes) {
  for (int64_t w = 0; w * 8 < nbytes; ++w) {
    uint64_t v = or_expand_word(fp, layer, (uint32_t)w);
    int64_t m = nbytes - w * 8 < 8 ? nbytes - w * 8 : 8;
    memcpy(out + w * 8, &v, (size_t)m);
  }
}

/* ---------------------------------------------------------------- kvstore.py */
typedef struct {
  int present;
  int64_t ins;
  int64_t* chain;
  int64_t nchain, capchain;
  int64_t* written;  /* per model group, 0 = absent */
  int32_t* order;    /* groups in insertion order */
  int norder;
} table_t;

struct or_store {
  int gpu_id, k, s, G, words;
  int64_t cell_bytes;
  int64_t serial, used, occupied, ins_counter;
  int64_t *list, nlist, caplist;  /* block list order (ids) */
  int64_t capid;                   /* id-indexed arrays sized capid */
  int32_t* owner;                  /* -1 free */
  uint8_t* exists;
  uint64_t* fp;                    /* [id][G][s] */
  uint64_t* occ;                   /* [id][G][words] */
  uint8_t* bytes;                  /* [id][G][k][s][cell_bytes] or NULL */
  int64_t *heap, nheap, capheap;   /* lazily invalidated min-heap of free ids */
  table_t* tables;
  int32_t ntab;
  uint8_t* resident;
};

#define GROW(ptr, cap, need, type)                                            \
  do {                                                                        \
    if ((need) > (cap)) {                                                     \
      int64_t nc__ = (cap) ? (cap) : 16;                                       \
      while (nc__ < (need)) nc__ *= 2;                                        \
      ptr = (type*)realloc(ptr, sizeof(type) * (size_t)nc__);                 \
      cap = nc__;                                                             \
    }                                                                         \
  } while (0)

static int64_t unit_cells(const or_store* st) { return (int64_t)st->G * st->s; }
static uint64_t* occ_of(or_store* st, int64_t id, int g) {
  return st->occ + ((size_t)id * st->G + g) * st->words;
}
static uint64_t* fp_of(or_store* st, int64_t id, int g) {
  return st->fp + ((size_t)id * st->G + g) * st->s;
}
static uint8_t* cell_bytes_of(or_store* st, int64_t id, int g, int layer, int off) {
  return st->bytes + ((((size_t)id * st->G + g) * st->k + layer) * st->s + off) * st->cell_bytes;
}
static int occ_test(or_store* st, int64_t id, int g, int off) {
  return (int)((occ_of(st, id, g)[off >> 6] >> (off & 63)) & 1);
}
static void occ_set(or_store* st, int64_t id, int g, int off) {
  occ_of(st, id, g)[off >> 6] |= 1ull << (off & 63);
}
static int64_t group_occ(or_store* st, int64_t id, int g) {
  int64_t c = 0;
  for (int w = 0; w < st->words; ++w) c += __builtin_popcountll(occ_of(st, id, g)[w]);
  return c;
}
int64_t or_block_occupied(or_store* st, int64_t id) {
  if (id < 0 || id >= st->serial || !st->exists[id]) return -1;
  int64_t c = 0;
  for (int g = 0; g < st->G; ++g) c += group_occ(st, id, g);
  return c;
}

static void heap_push(or_store* st, int64_t id) {
  GROW(st->heap, st->capheap, st->nheap + 1, int64_t);
  int64_t i = st->nheap++;
  st->heap[i] = id;
  while (i > 0) {
    int64_t p = (i - 1) / 2;
    if (st->heap[p] <= st->heap[i]) break;
    int64_t t = st->heap[p]; st->heap[p] = st->heap[i]; st->heap[i] = t;
    i = p;
  }
}
static int64_t heap_pop(or_store* st) {
  int64_t top = st->heap[0];
  st->heap[0] = st->heap[--st->nheap];
  int64_t i = 0;
  for (;;) {
    int64_t l = 2 * i + 1, r = l + 1, m = i;
    if (l < st->nheap && st->heap[l] < st->heap[m]) m = l;
    if (r < st->nheap && st->heap[r] < st->heap[m]) m = r;
    if (m == i) break;
    int64_t t = st->heap[m]; st->heap[m] = st->heap[i]; st->heap[i] = t;
    i = m;
  }
  return top;
}

/* kvstore.py:111-119 */
static int64_t new_block(or_store* st) {
  int64_t id = st->serial++;
  if (st->serial > st->capid) {
    int64_t old = st->capid, nc = old ? old : 16;
    while (nc < st->serial) nc *= 2;
    st->owner = (int32_t*)realloc(st->owner, sizeof(int32_t) * (size_t)nc);
    st->exists = (uint8_t*)realloc(st->exists, (size_t)nc);
    st->fp = (uint64_t*)realloc(st->fp, sizeof(uint64_t) * (size_t)(nc * unit_cells(st)));
    st->occ = (uint64_t*)realloc(st->occ, sizeof(uint64_t) * (size_t)(nc * st->G * st->words));
    if (st->cell_bytes)
      st->bytes = (uint8_t*)realloc(st->bytes, (size_t)(nc * unit_cells(st) * st->k * st->cell_bytes));
    st->capid = nc;
  }
  st->owner[id] = -1;
  st->exists[id] = 1;
  memset(fp_of(st, id, 0), 0, sizeof(uint64_t) * (size_t)unit_cells(st));
  memset(occ_of(st, id, 0), 0, sizeof(uint64_t) * (size_t)(st->G * st->words));
  heap_push(st, id);
  return id;
}
/* kvstore.py:121-128 */
static int64_t alloc_block(or_store* st, int32_t req) {
  while (st->nheap) {
    int64_t id = heap_pop(st);
    if (id < st->serial && st->exists[id] && st->owner[id] < 0) {
      st->owner[id] = req;
      st->used++;
      return id;
    }
  }
  return -1;
}
/* kvstore.py:130-134 */
static void release_block(or_store* st, int64_t id) {
  st->owner[id] = -1;
  memset(occ_of(st, id, 0), 0, sizeof(uint64_t) * (size_t)(st->G * st->words));
  st->used--;
  heap_push(st, id);
}

or_store* or_store_new(int gpu_id, int k, int s, int64_t capacity, const int32_t* groups,
                       int n_groups, int n_model_groups, int64_t cell_bytes) {
  if (s <= 0 || k <= 0 || capacity < 0 || n_model_groups <= 0) {
    snprintf(g_err, sizeof g_err, "tokens_per_block must be positive");
    return NULL;
  }
  or_store* st = (or_store*)calloc(1, sizeof(or_store));
  st->gpu_id = gpu_id;
  st->k = k;
  st->s = s;
  st->G = n_model_groups;
  st->words = (s + 63) / 64;
  st->cell_bytes = cell_bytes;
  st->resident = (uint8_t*)calloc((size_t)n_model_groups, 1);
  for (int i = 0; i < n_groups; ++i)
    if (groups[i] >= 0 && groups[i] < n_model_groups) st->resident[groups[i]] = 1;
  for (int64_t i = 0; i < capacity; ++i) {
    GROW(st->list, st->caplist, st->nlist + 1, int64_t);
    st->list[st->nlist++] = new_block(st);
  }
  return st;
}

void or_store_free(or_store* st) {
  if (!st) return;
  for (int32_t r = 0; r < st->ntab; ++r) {
    free(st->tables[r].chain);
    free(st->tables[r].written);
    free(st->tables[r].order);
  }
  free(st->tables);
  free(st->list); free(st->owner); free(st->exists); free(st->fp); free(st->occ);
  free(st->bytes); free(st->heap); free(st->resident);
  free(st);
}

int64_t or_capacity(or_store* st) { return st->nlist; }
int64_t or_used(or_store* st) { return st->used; }
int64_t or_occupied(or_store* st) { return st->occupied; }
int or_resident(or_store* st, int32_t* out, int cap) {
  int n = 0;
  for (int g = 0; g < st->G; ++g)
    if (st->resident[g]) {
      if (n < cap) out[n] = g;
      ++n;
    }
  return n;
}
int or_add_group(or_store* st, int g) {
  if (g < 0 || g >= st->G) return OR_E_INVALID;
  st->resident[g] = 1;
  return OR_OK;
}

static table_t* tab(or_store* st, int32_t req) {
  if (req < 0 || req >= st->ntab || !st->tables[req].present) return NULL;
  return &st->tables[req];
}
static table_t* tab_create(or_store* st, int32_t req) {
  if (req >= st->ntab) {
    int32_t nt = st->ntab ? st->ntab : 16;
    while (nt <= req) nt *= 2;
    st->tables = (table_t*)realloc(st->tables, sizeof(table_t) * (size_t)nt);
    memset(st->tables + st->ntab, 0, sizeof(table_t) * (size_t)(nt - st->ntab));
    st->ntab = nt;
  }
  table_t* t = &st->tables[req];
  if (!t->present) {
    t->present = 1;
    t->ins = st->ins_counter++;
    t->nchain = 0;
    if (!t->written) t->written = (int64_t*)calloc((size_t)st->G, sizeof(int64_t));
    else memset(t->written, 0, sizeof(int64_t) * (size_t)st->G);
    if (!t->order) t->order = (int32_t*)calloc((size_t)st->G, sizeof(int32_t));
    t->norder = 0;
  }
  return t;
}
static void tab_delete(or_store* st, int32_t req) {
  table_t* t = tab(st, req);
  if (t) t->present = 0;
}
static int64_t free_blocks(or_store* st) { return st->nlist - st->used; }
static int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

static void set_written(table_t* t, int g, int64_t v) {
  if (t->written[g] == 0) t->order[t->norder++] = g;
  t->written[g] = v;
}
static int extend(or_store* st, int32_t req, table_t* t, int64_t needed) {
  for (int64_t i = 0; i < needed; ++i) {
    int64_t id = alloc_block(st, req);
    GROW(t->chain, t->capchain, t->nchain + 1, int64_t);
    t->chain[t->nchain++] = id;
  }
  return OR_OK;
}
static void write_cell(or_store* st, int64_t id, int g, int off, uint64_t fp) {
  fp_of(st, id, g)[off] = fp;
  if (st->cell_bytes)
    for (int j = 0; j < st->k; ++j) or_expand_cell(fp, (uint32_t)j, cell_bytes_of(st, id, g, j, off), st->cell_bytes);
}

/* kvstore.py:163-199 */
int or_append(or_store* st, int32_t req, int g, int64_t n, const uint64_t* payloads) {
  if (n == 0) return OR_OK;
  if (g < 0 || g >= st->G || n < 0) return OR_E_INVALID;
  table_t* t = tab_create(st, req);
  int64_t start = t->written[g];
  int64_t needed = ceil_div(start + n, st->s) - t->nchain;
  if (needed > 0) {
    if (needed > free_blocks(st)) {
      snprintf(g_err, sizeof g_err, "gpu %d: need %lld blocks, %lld free", st->gpu_id,
               (long long)needed, (long long)free_blocks(st));
      if (t->nchain == 0 && t->norder == 0) tab_delete(st, req);
      return OR_E_OVERFLOW;
    }
    extend(st, req, t, needed);
  }
  for (int64_t i = 0; i < n; ++i) {
    int64_t pos = start + i, id = t->chain[pos / st->s];
    occ_set(st, id, g, (int)(pos % st->s));
    write_cell(st, id, g, (int)(pos % st->s), payloads[i]);
  }
  set_written(t, g, start + n);
  st->occupied += n;
  return OR_OK;
}

/* kvstore.py:201-227 */
int or_write_slots(or_store* st, int32_t req, int g, int64_t n, const int64_t* pos,
                   const uint64_t* payloads) {
  if (n == 0) return OR_OK;
  if (g < 0 || g >= st->G) return OR_E_INVALID;
  table_t* t = tab_create(st, req);
  int64_t top = 0;
  for (int64_t i = 0; i < n; ++i)
    if (pos[i] + 1 > top) top = pos[i] + 1;
  int64_t needed = ceil_div(top, st->s) - t->nchain;
  if (needed < 0) needed = 0;
  if (needed > free_blocks(st)) {
    snprintf(g_err, sizeof g_err, "gpu %d: need %lld blocks, %lld free", st->gpu_id,
             (long long)needed, (long long)free_blocks(st));
    if (t->nchain == 0 && t->norder == 0) tab_delete(st, req);
    return OR_E_OVERFLOW;
  }
  extend(st, req, t, needed);
  for (int64_t i = 0; i < n; ++i) {
    int64_t id = t->chain[pos[i] / st->s];
    int off = (int)(pos[i] % st->s);
    if (!occ_test(st, id, g, off)) {
      st->occupied++;
      occ_set(st, id, g, off);
    }
    write_cell(st, id, g, off, payloads[i]);
  }
  set_written(t, g, t->written[g] > top ? t->written[g] : top);
  return OR_OK;
}

/* kvstore.py:239-245 */
int or_read_checksum(or_store* st, int32_t req, int g, int64_t tok, uint64_t* out) {
  table_t* t = tab(st, req);
  if (!t || g < 0 || g >= st->G || tok < 0 || tok >= t->written[g]) return OR_E_UNKNOWN_SLOT;
  int64_t id = t->chain[tok / st->s];
  if (!occ_test(st, id, g, (int)(tok % st->s))) return OR_E_UNKNOWN_SLOT;
  *out = fp_of(st, id, g)[tok % st->s];
  return OR_OK;
}
int or_read_cell(or_store* st, int32_t req, int g, int64_t tok, int layer, uint8_t* out) {
  uint64_t fp;
  int rc = or_read_checksum(st, req, g, tok, &fp);
  if (rc != OR_OK || !st->cell_bytes) return rc ? rc : OR_E_INVALID;
  table_t* t = tab(st, req);
  memcpy(out, cell_bytes_of(st, t->chain[tok / st->s], g, layer, (int)(tok % st->s)),
         (size_t)st->cell_bytes);
  return OR_OK;
}

/* kvstore.py:247-257 */
int64_t or_compact(or_store* st) {
  int64_t* out = (int64_t*)malloc(sizeof(int64_t) * (size_t)(st->nlist + 1));
  int64_t n = 0, nfree = 0;
  for (int64_t i = 0; i < st->nlist; ++i)
    if (st->owner[st->list[i]] >= 0) out[n++] = st->list[i];
  for (int64_t i = 0; i < st->nlist; ++i)
    if (st->owner[st->list[i]] < 0) { out[n++] = st->list[i]; ++nfree; }
  memcpy(st->list, out, sizeof(int64_t) * (size_t)st->nlist);
  free(out);
  return nfree;
}

/* kvstore.py:259-282 */
int or_resize(or_store* st, int64_t cap) {
  if (cap < 0) { snprintf(g_err, sizeof g_err, "capacity must be non-negative"); return OR_E_INVALID; }
  if (cap == st->nlist) return OR_OK;
  if (cap > st->nlist) {
    while (st->nlist < cap) {
      GROW(st->list, st->caplist, st->nlist + 1, int64_t);
      st->list[st->nlist++] = new_block(st);
    }
    return OR_OK;
  }
  if (st->used > cap) {
    snprintf(g_err, sizeof g_err, "gpu %d: %lld live blocks > target %lld", st->gpu_id,
             (long long)st->used, (long long)cap);
    return OR_E_BELOW_LIVE;
  }
  int live_tail = 0;
  for (int64_t i = cap; i < st->nlist; ++i) live_tail |= st->owner[st->list[i]] >= 0;
  if (live_tail) or_compact(st);
  for (int64_t i = cap; i < st->nlist; ++i) st->exists[st->list[i]] = 0;
  st->nlist = cap;
  return OR_OK;
}

/* kvstore.py:284-309 */
int or_drop_groups(or_store* st, const int32_t* groups, int n, int64_t* freed_out) {
  for (int i = 0; i < n; ++i)
    if (groups[i] < 0 || groups[i] >= st->G || !st->resident[groups[i]]) {
      snprintf(g_err, sizeof g_err, "gpu %d: group %d not resident", st->gpu_id, groups[i]);
      return OR_E_UNKNOWN_GROUP;
    }
  int64_t freed = 0;
  uint8_t* in = (uint8_t*)calloc((size_t)st->G, 1);
  for (int i = 0; i < n; ++i) in[groups[i]] = 1;
  for (int32_t r = 0; r < st->ntab; ++r) {
    table_t* t = tab(st, r);
    if (!t) continue;
    for (int g = 0; g < st->G; ++g) {
      if (!in[g] || !t->written[g]) continue;
      freed += t->written[g];
      t->written[g] = 0;
      int w = 0;
      for (int i = 0; i < t->norder; ++i)
        if (t->order[i] != g) t->order[w++] = t->order[i];
      t->norder = w;
    }
    for (int64_t c = 0; c < t->nchain; ++c)
      for (int g = 0; g < st->G; ++g)
        if (in[g]) {
          st->occupied -= group_occ(st, t->chain[c], g);
          memset(occ_of(st, t->chain[c], g), 0, sizeof(uint64_t) * (size_t)st->words);
        }
    while (t->nchain && or_block_occupied(st, t->chain[t->nchain - 1]) == 0)
      release_block(st, t->chain[--t->nchain]);
    if (t->nchain == 0 && t->norder == 0) tab_delete(st, r);
  }
  for (int g = 0; g < st->G; ++g)
    if (in[g]) st->resident[g] = 0;
  free(in);
  *freed_out = freed;
  return OR_OK;
}

/* kvstore.py:311-322 */
int or_free_request(or_store* st, int32_t req, int64_t* stats, int cap) {
  table_t* t = tab(st, req);
  if (!t) return 0;
  int n = 0;
  for (int i = 0; i < t->norder; ++i, ++n)
    if (n < cap) {
      int64_t w = t->written[t->order[i]];
      stats[3 * n] = t->order[i];
      stats[3 * n + 1] = w;
      stats[3 * n + 2] = ceil_div(w, st->s) * st->s;
    }
  for (int64_t c = 0; c < t->nchain; ++c) {
    st->occupied -= or_block_occupied(st, t->chain[c]);
    release_block(st, t->chain[c]);
  }
  t->nchain = 0;
  tab_delete(st, req);
  return n;
}

/* kvstore.py:324-329 */
double or_utilization(or_store* st) {
  if (st->used == 0) return 1.0;
  int nres = 0;
  for (int g = 0; g < st->G; ++g) nres += st->resident[g];
  return (double)st->occupied / ((double)st->used * st->s * (nres > 1 ? nres : 1));
}

int64_t or_blocks(or_store* st, int64_t* ids, int32_t* owner, int64_t cap) {
  for (int64_t i = 0; i < st->nlist && i < cap; ++i) {
    ids[i] = st->list[i];
    owner[i] = st->owner[st->list[i]];
  }
  return st->nlist;
}
int64_t or_tables(or_store* st, int32_t* reqs, int64_t cap) {
  /* insertion order */
  int64_t n = 0;
  int64_t next_ins = -1;
  for (;;) {
    int32_t best = -1;
    for (int32_t r = 0; r < st->ntab; ++r)
      if (st->tables[r].present && st->tables[r].ins > next_ins &&
          (best < 0 || st->tables[r].ins < st->tables[best].ins))
        best = r;
    if (best < 0) break;
    if (n < cap) reqs[n] = best;
    ++n;
    next_ins = st->tables[best].ins;
  }
  return n;
}
int64_t or_chain(or_store* st, int32_t req, int64_t* ids, int64_t cap) {
  table_t* t = tab(st, req);
  if (!t) return 0;
  for (int64_t i = 0; i < t->nchain && i < cap; ++i) ids[i] = t->chain[i];
  return t->nchain;
}
int or_written(or_store* st, int32_t req, int32_t* groups, int64_t* counts, int cap) {
  table_t* t = tab(st, req);
  if (!t) return 0;
  for (int i = 0; i < t->norder && i < cap; ++i) {
    groups[i] = t->order[i];
    counts[i] = t->written[t->order[i]];
  }
  return t->norder;
}
int or_block_cells(or_store* st, int64_t id, int g, int64_t* offs, uint64_t* fps, int cap) {
  if (id < 0 || id >= st->serial || !st->exists[id]) return -1;
  int n = 0;
  for (int o = 0; o < st->s; ++o)
    if (occ_test(st, id, g, o)) {
      if (n < cap) { offs[n] = o; fps[n] = fp_of(st, id, g)[o]; }
      ++n;
    }
  return n;
}

/* ---------------------------------------------------------------- migrator.py:24-48 */
typedef struct { int32_t req, g; int64_t pos; } key_t_;
struct or_dirty { key_t_* k; int64_t n, cap; };

or_dirty* or_dirty_new(void) { return (or_dirty*)calloc(1, sizeof(or_dirty)); }
void or_dirty_free(or_dirty* d) { if (d) { free(d->k); free(d); } }
void or_dirty_mark(or_dirty* d, int32_t req, int32_t g, int64_t start, int64_t n) {
  GROW(d->k, d->cap, d->n + n, key_t_);
  for (int64_t i = 0; i < n; ++i) d->k[d->n++] = (key_t_){req, g, start + i};
}
static const int32_t* g_rank;
static int64_t g_nrank;
static int64_t rank_of(int32_t r) { return r < g_nrank && g_rank ? g_rank[r] : r; }
static int key_cmp(const void* a, const void* b) {
  const key_t_ *x = (const key_t_*)a, *y = (const key_t_*)b;
  int64_t rx = rank_of(x->req), ry = rank_of(y->req);
  if (rx != ry) return rx < ry ? -1 : 1;
  if (x->g != y->g) return x->g < y->g ? -1 : 1;
  if (x->pos != y->pos) return x->pos < y->pos ? -1 : 1;
  return 0;
}
static void dedupe(or_dirty* d, const int32_t* rank, int64_t nrank) {
  g_rank = rank;
  g_nrank = nrank;
  qsort(d->k, (size_t)d->n, sizeof(key_t_), key_cmp);
  int64_t w = 0;
  for (int64_t i = 0; i < d->n; ++i)
    if (w == 0 || key_cmp(&d->k[w - 1], &d->k[i]) != 0) d->k[w++] = d->k[i];
  d->n = w;
}
int64_t or_dirty_count(or_dirty* d) {
  dedupe(d, NULL, 0);
  return d->n;
}
int64_t or_dirty_discard(or_dirty* d, int32_t req) {
  dedupe(d, NULL, 0);
  int64_t w = 0, dropped = 0;
  for (int64_t i = 0; i < d->n; ++i) {
    if (d->k[i].req == req) ++dropped;
    else d->k[w++] = d->k[i];
  }
  d->n = w;
  return dropped;
}
/* DirtyBitmap.drain: sorted snapshot + clear */
int64_t or_dirty_drain(or_dirty* d, const int32_t* rank, int64_t n_rank, int32_t* reqs,
                       int32_t* groups, int64_t* pos, int64_t cap) {
  dedupe(d, rank, n_rank);
  int64_t n = d->n;
  for (int64_t i = 0; i < n && i < cap; ++i) {
    reqs[i] = d->k[i].req;
    groups[i] = d->k[i].g;
    pos[i] = d->k[i].pos;
  }
  d->n = 0;
  return n;
}

typedef struct {
  or_dirty* d;
  or_store *src, *dst;
  const int64_t *src_id, *dst_id;
  int64_t lo, hi;
} copy_job;
static void* copy_worker(void* arg) {
  copy_job* j = (copy_job*)arg;
  for (int64_t i = j->lo; i < j->hi; ++i) {
    if (j->src_id[i] < 0) continue;
    const key_t_* key = &j->d->k[i];
    for (int l = 0; l < j->src->k; ++l)
      memcpy(cell_bytes_of(j->dst, j->dst_id[i], key->g, l, (int)(key->pos % j->dst->s)),
             cell_bytes_of(j->src, j->src_id[i], key->g, l, (int)(key->pos % j->src->s)),
             (size_t)j->src->cell_bytes);
  }
  return NULL;
}

/* _drain + receiver apply with real bytes: the CPU baseline of one patch round */
int or_patch_round(or_dirty* d, or_store* src, or_store* dst, const int32_t* rank, int64_t n_rank,
                   int layers_per_group, int threads, int64_t* keys_out, int64_t* cells_out) {
  dedupe(d, rank, n_rank);
  int64_t n = d->n;
  /* snapshot reads (migrator.py:231-235): source cell ids and fingerprints */
  int64_t* src_id = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n + 1));
  uint64_t* fps = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)(n + 1));
  for (int64_t i = 0; i < n; ++i) {
    table_t* t = tab(src, d->k[i].req);
    if (!t || d->k[i].pos >= t->written[d->k[i].g]) { src_id[i] = -1; continue; }
    src_id[i] = t->chain[d->k[i].pos / src->s];
    fps[i] = fp_of(src, src_id[i], d->k[i].g)[d->k[i].pos % src->s];
  }
  /* receiver bookkeeping per (req, group) in sorted order (migrator.py:124-128) */
  int64_t* dst_id = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n + 1));
  int rc = OR_OK;
  for (int64_t i = 0; i < n && rc == OR_OK;) {
    int64_t j = i;
    while (j < n && d->k[j].req == d->k[i].req && d->k[j].g == d->k[i].g) ++j;
    table_t* t = tab_create(dst, d->k[i].req);
    int g = d->k[i].g;
    int64_t top = d->k[j - 1].pos + 1;
    int64_t needed = ceil_div(top, dst->s) - t->nchain;
    if (needed > free_blocks(dst)) { rc = OR_E_OVERFLOW; break; }
    if (needed > 0) extend(dst, d->k[i].req, t, needed);
    for (int64_t q = i; q < j; ++q) {
      int64_t id = t->chain[d->k[q].pos / dst->s];
      int off = (int)(d->k[q].pos % dst->s);
      if (!occ_test(dst, id, g, off)) { dst->occupied++; occ_set(dst, id, g, off); }
      dst_id[q] = id;
      fp_of(dst, id, g)[off] = fps[q];
    }
    set_written(t, g, t->written[g] > top ? t->written[g] : top);
    i = j;
  }
  /* byte movement, the part that parallelises (pthreads, contiguous key ranges) */
  if (rc == OR_OK && src->cell_bytes && dst->cell_bytes && n > 0) {
    if (threads < 1) threads = 1;
    if (threads > 256) threads = 256;
    pthread_t tid[256];
    copy_job jobs[256];
    for (int w = 0; w < threads; ++w) {
      jobs[w] = (copy_job){d, src, dst, src_id, dst_id, n * w / threads, n * (w + 1) / threads};
      if (threads > 1) pthread_create(&tid[w], NULL, copy_worker, &jobs[w]);
      else copy_worker(&jobs[w]);
    }
    if (threads > 1)
      for (int w = 0; w < threads; ++w) pthread_join(tid[w], NULL);
  }
  free(src_id); free(fps); free(dst_id);
  *keys_out = n;
  *cells_out = n * layers_per_group;
  d->n = 0;
  return rc;
}
