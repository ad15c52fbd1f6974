/* TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference hot path (Norouzi/Punjani/Fleet multi-index hashing
 * as implemented in /root/reference/proj/include/mih). It is the checker for the CUDA product
 * path: only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it. The
 * product library (paper_1307_2982_b200/libmihg.so) never links or calls it.
 *
 * Parity pinning: tests/test_oracle.py checks every function here against golden vectors
 * produced by the reference itself (oracle/_ref/libmihref.so, built from the reference headers
 * by oracle/Makefile; fixtures in tests/golden/, generator tests/golden/make_golden.py).
 *
 * Each function cites the reference file:line it restates (paths relative to
 * /root/reference/proj).
 */
#include "mih_oracle.h"

#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static _Thread_local char g_err[256];

static int fail(int code, const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return code;
}

const char* or_last_error(void) { return g_err; }

/* ---- std::mt19937_64 (io.hpp:268 uses it; parameters fixed by the C++ standard) ---- */
#define MT_N 312
#define MT_M 156
typedef struct {
  uint64_t s[MT_N];
  int i;
} mt64;

static void mt64_seed(mt64* g, uint64_t seed) {
  g->s[0] = seed;
  for (int i = 1; i < MT_N; ++i)
    g->s[i] = 6364136223846793005ULL * (g->s[i - 1] ^ (g->s[i - 1] >> 62)) + (uint64_t)i;
  g->i = MT_N;
}

static uint64_t mt64_next(mt64* g) {
  if (g->i >= MT_N) {
    for (int k = 0; k < MT_N; ++k) {
      uint64_t y = (g->s[k] & 0xFFFFFFFF80000000ULL) | (g->s[(k + 1) % MT_N] & 0x7FFFFFFFULL);
      uint64_t v = g->s[(k + MT_M) % MT_N] ^ (y >> 1);
      if (y & 1) v ^= 0xB5026F5AA96619E9ULL;
      g->s[k] = v;
    }
    g->i = 0;
  }
  uint64_t z = g->s[g->i++];
  z ^= (z >> 29) & 0x5555555555555555ULL;
  z ^= (z << 17) & 0x71D67FFFEDA60000ULL;
  z ^= (z << 37) & 0xFFF7EEE000000000ULL;
  z ^= z >> 43;
  return z;
}

static uint32_t wpc_of(uint32_t bits) { return (bits + 63) / 64; } /* codes.hpp:18 */

static uint64_t last_word_mask(uint32_t bits) { /* codes.hpp:21-24 */
  uint32_t used = bits & 63;
  return used == 0 ? ~0ULL : ((1ULL << used) - 1);
}

/* gen_uniform, io.hpp:266-277 */
int or_gen_uniform(uint64_t n, uint32_t bits, uint64_t seed, uint64_t* out) {
  if (bits == 0 || bits > 4096) return fail(1, "gen_uniform: bad width");
  mt64* g = (mt64*)malloc(sizeof(mt64));
  if (!g) return fail(3, "bad_alloc");
  mt64_seed(g, seed);
  const uint32_t wpc = wpc_of(bits);
  const uint64_t mask = last_word_mask(bits);
  for (uint64_t i = 0; i < n; ++i) {
    uint64_t* w = out + i * wpc;
    for (uint32_t k = 0; k < wpc; ++k) w[k] = mt64_next(g);
    w[wpc - 1] &= mask;
  }
  free(g);
  return 0;
}

/* consecutive_partition, codes.hpp:198-211: the first bits % m substrings get the extra bit. */
int or_consecutive_partition(uint32_t bits, uint32_t m, uint32_t* lengths, uint32_t* positions) {
  if (m == 0 || m > bits) return fail(1, "consecutive_partition: need 1 <= m <= bits");
  const uint32_t base = bits / m, extra = bits % m;
  uint32_t pos = 0;
  for (uint32_t j = 0; j < m; ++j) {
    lengths[j] = base + (j < extra ? 1 : 0);
    for (uint32_t i = 0; i < lengths[j]; ++i) positions[pos] = pos, ++pos;
  }
  return 0;
}

/* detail::hamming_words, codes.hpp:38-42 */
uint32_t or_hamming(const uint64_t* a, const uint64_t* b, uint32_t nwords) {
  uint32_t d = 0;
  for (uint32_t w = 0; w < nwords; ++w) d += (uint32_t)__builtin_popcountll(a[w] ^ b[w]);
  return d;
}

/* extract_substring, codes.hpp:214-231 (slow path semantics; equal to the fast path):
 * bit i of the result = code bit at the i-th position owned by the substring. */
static uint64_t extract(const uint64_t* code, const uint32_t* pos, uint32_t len) {
  uint64_t v = 0;
  for (uint32_t i = 0; i < len; ++i) v |= ((code[pos[i] >> 6] >> (pos[i] & 63)) & 1ULL) << i;
  return v;
}

/* ---- index: one table per substring (index.hpp:101-121, table.hpp:91-159) ---- */
typedef struct {
  uint32_t s;
  uint64_t* keys; /* sorted ascending; ties keep insertion (= id) order */
  uint32_t* ids;
} or_table;

struct or_index {
  uint32_t bits, m, wpc;
  uint64_t n;
  uint64_t* codes;
  uint32_t* lengths;
  uint32_t* positions; /* concatenated */
  uint32_t* pos_off;   /* m+1 */
  or_table* tables;
};

typedef struct {
  uint64_t key;
  uint32_t id;
} kv;

static int kv_cmp(const void* a, const void* b) {
  const kv* x = (const kv*)a;
  const kv* y = (const kv*)b;
  if (x->key != y->key) return x->key < y->key ? -1 : 1;
  /* stable_sort (table.hpp:98-99) keeps insertion order; inputs arrive in id order */
  return x->id < y->id ? -1 : (x->id > y->id);
}

/* Partition::validate, codes.hpp:152-176 */
static int validate_partition(uint32_t bits, uint32_t m, const uint32_t* lengths,
                              const uint32_t* positions) {
  if (bits == 0 || bits > 4096) return fail(1, "Partition: bad width");
  if (m == 0 || m > bits) return fail(1, "Partition: substring count must be in [1, bits]");
  char* seen = (char*)calloc(bits, 1);
  if (!seen) return fail(3, "bad_alloc");
  uint64_t total = 0, at = 0;
  uint32_t lo = bits, hi = 0;
  for (uint32_t j = 0; j < m; ++j) {
    if (lengths[j] < lo) lo = lengths[j];
    if (lengths[j] > hi) hi = lengths[j];
    for (uint32_t i = 0; i < lengths[j]; ++i) {
      uint32_t p = positions[at++];
      if (p >= bits || seen[p]) {
        free(seen);
        return fail(1, "Partition: bit position out of range or assigned twice");
      }
      seen[p] = 1;
    }
    total += lengths[j];
  }
  free(seen);
  if (total != bits) return fail(1, "Partition: positions do not cover the code");
  if (hi - lo > 1) return fail(1, "Partition: substring sizes differ by more than 1");
  return 0;
}

void or_index_free(or_index* idx) {
  if (!idx) return;
  if (idx->tables)
    for (uint32_t j = 0; j < idx->m; ++j) {
      free(idx->tables[j].keys);
      free(idx->tables[j].ids);
    }
  free(idx->tables);
  free(idx->codes);
  free(idx->lengths);
  free(idx->positions);
  free(idx->pos_off);
  free(idx);
}

int or_index_build(const uint64_t* codes, uint64_t n, uint32_t bits, uint32_t m,
                   const uint32_t* lengths, const uint32_t* positions, or_index** out) {
  uint32_t* own_len = NULL;
  uint32_t* own_pos = NULL;
  if (!lengths) { /* consecutive_partition default */
    if (m == 0 || m > bits) return fail(1, "consecutive_partition: need 1 <= m <= bits");
    own_len = (uint32_t*)malloc(sizeof(uint32_t) * m);
    own_pos = (uint32_t*)malloc(sizeof(uint32_t) * bits);
    or_consecutive_partition(bits, m, own_len, own_pos);
    lengths = own_len;
    positions = own_pos;
  }
  int rc = validate_partition(bits, m, lengths, positions);
  if (rc) goto out_err;
  for (uint32_t j = 0; j < m; ++j)
    if (lengths[j] > 32) { /* index.hpp:108-112, kMaxTableBits table.hpp:31 */
      rc = fail(1, "MihIndex::build: substring wider than 32 bits");
      goto out_err;
    }
  if (n > (1ULL << 32)) {
    rc = fail(1, "CodeDatabase: at most 2^32 codes supported");
    goto out_err;
  }
  or_index* idx = (or_index*)calloc(1, sizeof(or_index));
  idx->bits = bits;
  idx->m = m;
  idx->n = n;
  idx->wpc = wpc_of(bits);
  idx->codes = (uint64_t*)malloc(sizeof(uint64_t) * (n * idx->wpc + 1));
  if (n) memcpy(idx->codes, codes, sizeof(uint64_t) * n * idx->wpc);
  idx->lengths = (uint32_t*)malloc(sizeof(uint32_t) * m);
  memcpy(idx->lengths, lengths, sizeof(uint32_t) * m);
  idx->positions = (uint32_t*)malloc(sizeof(uint32_t) * bits);
  memcpy(idx->positions, positions, sizeof(uint32_t) * bits);
  idx->pos_off = (uint32_t*)malloc(sizeof(uint32_t) * (m + 1));
  idx->pos_off[0] = 0;
  for (uint32_t j = 0; j < m; ++j) idx->pos_off[j + 1] = idx->pos_off[j] + lengths[j];
  idx->tables = (or_table*)calloc(m, sizeof(or_table));
  kv* pairs = (kv*)malloc(sizeof(kv) * (n + 1));
  for (uint32_t j = 0; j < m; ++j) {
    for (uint64_t i = 0; i < n; ++i) {
      pairs[i].key = extract(idx->codes + i * idx->wpc, idx->positions + idx->pos_off[j], lengths[j]);
      pairs[i].id = (uint32_t)i;
    }
    qsort(pairs, n, sizeof(kv), kv_cmp);
    or_table* t = &idx->tables[j];
    t->s = lengths[j];
    t->keys = (uint64_t*)malloc(sizeof(uint64_t) * (n + 1));
    t->ids = (uint32_t*)malloc(sizeof(uint32_t) * (n + 1));
    for (uint64_t i = 0; i < n; ++i) {
      t->keys[i] = pairs[i].key;
      t->ids[i] = pairs[i].id;
    }
  }
  free(pairs);
  free(own_len);
  free(own_pos);
  *out = idx;
  return 0;
out_err:
  free(own_len);
  free(own_pos);
  return rc;
}

/* SubstringTable::probe, table.hpp:178-188: the ids of bucket `value`, in insertion order. */
static void probe(const or_table* t, uint64_t n, uint64_t value, uint64_t* lo, uint64_t* hi) {
  uint64_t a = 0, b = n;
  while (a < b) {
    uint64_t mid = (a + b) / 2;
    if (t->keys[mid] < value) a = mid + 1; else b = mid;
  }
  *lo = a;
  b = n;
  while (a < b) {
    uint64_t mid = (a + b) / 2;
    if (t->keys[mid] <= value) a = mid + 1; else b = mid;
  }
  *hi = a;
}

int or_bucket(const or_index* idx, uint32_t j, uint64_t value, uint32_t* out, uint64_t cap,
              uint64_t* count) {
  if (j >= idx->m) return fail(1, "table index out of range");
  if (value >> idx->tables[j].s) return fail(1, "bucket_lookup: value does not fit");
  uint64_t lo, hi;
  probe(&idx->tables[j], idx->n, value, &lo, &hi);
  *count = hi - lo;
  for (uint64_t i = lo; i < hi && i - lo < cap; ++i) out[i - lo] = idx->tables[j].ids[i];
  return 0;
}

/* RingEnumerator, enumerate.hpp:31-90: values at exactly `z` flips from `center`, flip tuples
 * in lexicographic order. The callback order only affects trace accumulation order. */
typedef struct {
  uint32_t s, z, pos[64];
  uint64_t center, mask;
  int done;
} ring;

static void ring_init(ring* r, uint32_t s, uint64_t center, uint32_t z) {
  r->s = s;
  r->z = z;
  r->center = center;
  r->mask = 0;
  r->done = z > s;
  for (uint32_t i = 0; i < z && i < 64; ++i) {
    r->pos[i] = i;
    r->mask |= 1ULL << i;
  }
}

static int ring_next(ring* r, uint64_t* out) {
  if (r->done) return 0;
  *out = r->center ^ r->mask;
  if (r->z == 0) {
    r->done = 1;
    return 1;
  }
  uint32_t i = r->z;
  while (i > 0) {
    --i;
    if (r->pos[i] < r->s - r->z + i) {
      uint32_t p = r->pos[i];
      for (uint32_t j = i; j < r->z; ++j) r->pos[j] = ++p;
      r->mask = 0;
      for (uint32_t j = 0; j < r->z; ++j) r->mask |= 1ULL << r->pos[j];
      return 1;
    }
  }
  r->done = 1;
  return 1;
}

static int u32_cmp(const void* a, const void* b) {
  uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
  return x < y ? -1 : (x > y);
}

/* MihIndex::knn_search, index.hpp:185-253 (Alg. 3): progressive radius r = 0,1,..; step r
 * probes ring r/m of table r%m; new ids (n-bit mark vector, :66-70) are verified and binned by
 * full distance; stop once the bins at distance <= r-1 hold >= k ids (:209, :232). Output:
 * bins ascending, each sorted by id, first k (:239-248). traces: 5 u64 per query
 * {lookups, candidates, unique, distance_evaluations, final_radius} (SearchTrace :45-51). */
int or_knn(const or_index* idx, const uint64_t* queries, uint64_t nq, uint32_t k, uint32_t* ids,
           uint32_t* dists, uint64_t* traces) {
  if (k > idx->n) return fail(1, "knn_search: k exceeds database size");
  const uint32_t m = idx->m, b = idx->bits, wpc = idx->wpc;
  uint64_t* marks = (uint64_t*)calloc((idx->n + 63) / 64 + 1, sizeof(uint64_t));
  uint32_t** bins = (uint32_t**)calloc(b + 1, sizeof(uint32_t*));
  uint64_t* cnt = (uint64_t*)calloc(b + 1, sizeof(uint64_t));
  uint64_t* capb = (uint64_t*)calloc(b + 1, sizeof(uint64_t));
  uint32_t* touched = (uint32_t*)malloc(sizeof(uint32_t) * (idx->n + 1));
  uint64_t sub_q[4096];
  for (uint64_t qi = 0; qi < nq; ++qi) {
    const uint64_t* q = queries + qi * wpc;
    uint64_t tr_lookups = 0, tr_cand = 0, ntouched = 0;
    uint32_t r = 0;
    if (k > 0) {
      for (uint32_t j = 0; j < m; ++j)
        sub_q[j] = extract(q, idx->positions + idx->pos_off[j], idx->lengths[j]);
      uint64_t settled = 0;
      for (;;) {
        if (settled >= k) break;
        const uint32_t r_sub = r / m, a = r % m;
        const or_table* t = &idx->tables[a];
        ring rg;
        ring_init(&rg, t->s, sub_q[a], r_sub);
        uint64_t v;
        while (ring_next(&rg, &v)) {
          ++tr_lookups;
          uint64_t lo, hi;
          probe(t, idx->n, v, &lo, &hi);
          tr_cand += hi - lo;
          for (uint64_t p = lo; p < hi; ++p) {
            uint32_t id = t->ids[p];
            if ((marks[id >> 6] >> (id & 63)) & 1) continue;
            marks[id >> 6] |= 1ULL << (id & 63);
            touched[ntouched++] = id;
            uint32_t d = or_hamming(q, idx->codes + (uint64_t)id * wpc, wpc);
            if (cnt[d] == capb[d]) {
              capb[d] = capb[d] ? 2 * capb[d] : 16;
              bins[d] = (uint32_t*)realloc(bins[d], sizeof(uint32_t) * capb[d]);
            }
            bins[d][cnt[d]++] = id;
          }
        }
        settled += cnt[r];
        ++r;
      }
      uint64_t outn = 0;
      for (uint32_t d = 0; d <= b && outn < k; ++d) {
        if (!cnt[d]) continue;
        qsort(bins[d], cnt[d], sizeof(uint32_t), u32_cmp);
        for (uint64_t i = 0; i < cnt[d] && outn < k; ++i, ++outn) {
          ids[qi * k + outn] = bins[d][i];
          dists[qi * k + outn] = d;
        }
      }
      for (uint64_t i = 0; i < ntouched; ++i) marks[touched[i] >> 6] &= ~(1ULL << (touched[i] & 63));
      for (uint32_t d = 0; d <= b; ++d) cnt[d] = 0;
    }
    if (traces) {
      uint64_t* o = traces + qi * 5;
      o[0] = tr_lookups;
      o[1] = tr_cand;
      o[2] = ntouched;
      o[3] = ntouched;
      o[4] = k > 0 ? r - 1 : 0;
    }
  }
  for (uint32_t d = 0; d <= b; ++d) free(bins[d]);
  free(bins);
  free(cnt);
  free(capb);
  free(marks);
  free(touched);
  return 0;
}

typedef struct {
  uint32_t dist, id;
} nb;

static int nb_cmp(const void* a, const void* b) { /* neighbor_less, scan.hpp:24-26 */
  const nb* x = (const nb*)a;
  const nb* y = (const nb*)b;
  if (x->dist != y->dist) return x->dist < y->dist ? -1 : 1;
  return x->id < y->id ? -1 : (x->id > y->id);
}

/* MihIndex::range_search, index.hpp:149-176 (Alg. 2 + split_radius :28-43): probe ball(r')
 * in tables 0..a and ball(r'-1) in the rest, cull by full distance, sort by (dist, id). */
int or_range(const or_index* idx, const uint64_t* q, uint32_t r, uint32_t* ids, uint32_t* dists,
             uint64_t cap, uint64_t* count, uint64_t* trace) {
  if (r > idx->bits) return fail(1, "range_search: radius exceeds code width");
  const uint32_t m = idx->m, wpc = idx->wpc, r_sub = r / m, a = r % m;
  uint64_t* marks = (uint64_t*)calloc((idx->n + 63) / 64 + 1, sizeof(uint64_t));
  uint32_t* touched = (uint32_t*)malloc(sizeof(uint32_t) * (idx->n + 1));
  uint64_t ntouched = 0, lookups = 0, cand = 0;
  for (uint32_t j = 0; j < m; ++j) {
    int32_t rj = j <= a ? (int32_t)r_sub : (int32_t)r_sub - 1;
    if (rj < 0) continue;
    const or_table* t = &idx->tables[j];
    uint64_t sq = extract(q, idx->positions + idx->pos_off[j], idx->lengths[j]);
    for (uint32_t z = 0; z <= (uint32_t)rj; ++z) { /* BallEnumerator, enumerate.hpp:93-112 */
      ring rg;
      ring_init(&rg, t->s, sq, z);
      uint64_t v;
      while (ring_next(&rg, &v)) {
        ++lookups;
        uint64_t lo, hi;
        probe(t, idx->n, v, &lo, &hi);
        cand += hi - lo;
        for (uint64_t p = lo; p < hi; ++p) {
          uint32_t id = t->ids[p];
          if ((marks[id >> 6] >> (id & 63)) & 1) continue;
          marks[id >> 6] |= 1ULL << (id & 63);
          touched[ntouched++] = id;
        }
      }
    }
  }
  nb* out = (nb*)malloc(sizeof(nb) * (ntouched + 1));
  uint64_t no = 0;
  for (uint64_t i = 0; i < ntouched; ++i) { /* cull, index.hpp:271-280 */
    uint32_t d = or_hamming(q, idx->codes + (uint64_t)touched[i] * wpc, wpc);
    if (d <= r) out[no].dist = d, out[no].id = touched[i], ++no;
  }
  qsort(out, no, sizeof(nb), nb_cmp);
  *count = no;
  for (uint64_t i = 0; i < no && i < cap; ++i) ids[i] = out[i].id, dists[i] = out[i].dist;
  if (trace) {
    trace[0] = lookups;
    trace[1] = cand;
    trace[2] = ntouched;
    trace[3] = ntouched;
    trace[4] = 0;
  }
  free(out);
  free(marks);
  free(touched);
  return 0;
}

/* scan_knn, scan.hpp:43-68: the k smallest (dist, id); ties at the cut go to smaller ids.
 * Restated as a counting select (distances are <= bits): histogram, find the cut distance,
 * then emit ids in ascending order per distance — same output as the bounded heap. */
int or_scan_knn(const uint64_t* codes, uint64_t n, uint32_t bits, const uint64_t* queries,
                uint64_t nq, uint32_t k, uint32_t* ids, uint32_t* dists) {
  if (k > n) return fail(1, "scan_knn: k exceeds database size");
  const uint32_t wpc = wpc_of(bits);
  uint64_t* hist = (uint64_t*)calloc(bits + 2, sizeof(uint64_t));
  uint32_t* dd = (uint32_t*)malloc(sizeof(uint32_t) * (n + 1));
  uint64_t* fill = (uint64_t*)calloc(bits + 2, sizeof(uint64_t));
  for (uint64_t qi = 0; qi < nq; ++qi) {
    if (k == 0) continue;
    const uint64_t* q = queries + qi * wpc;
    memset(hist, 0, sizeof(uint64_t) * (bits + 2));
    for (uint64_t i = 0; i < n; ++i) {
      dd[i] = or_hamming(q, codes + i * wpc, wpc);
      ++hist[dd[i]];
    }
    uint64_t acc = 0;
    uint32_t cut = 0;
    for (cut = 0; cut <= bits; ++cut) {
      if (acc + hist[cut] >= k) break;
      acc += hist[cut];
    }
    /* slot start per distance */
    uint64_t at = 0;
    for (uint32_t d = 0; d <= cut; ++d) {
      fill[d] = at;
      at += hist[d];
    }
    for (uint64_t i = 0; i < n; ++i) {
      uint32_t d = dd[i];
      if (d > cut) continue;
      uint64_t slot = fill[d]++;
      if (slot < k) {
        ids[qi * k + slot] = (uint32_t)i;
        dists[qi * k + slot] = d;
      }
    }
  }
  free(hist);
  free(dd);
  free(fill);
  return 0;
}

/* ---- Gaussian-mixture sign-projection generator: C restatement of
 * paper_1307_2982_b200/csrc/gen.cu (exact integer arithmetic; see the definition there). Used to
 * pin the GPU generator and to give the CPU reference arm its inputs without the GPU. */
static uint64_t sm64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ULL;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
  return x ^ (x >> 31);
}
static int g5(uint64_t u) {
  return (int)(u & 31) + (int)((u >> 5) & 31) + (int)((u >> 10) & 31) + (int)((u >> 15) & 31) - 62;
}
static int g6(uint64_t u) {
  return (int)(u & 63) + (int)((u >> 6) & 63) + (int)((u >> 12) & 63) + (int)((u >> 18) & 63) - 126;
}

typedef struct {
  uint64_t first, lo, hi;
  uint32_t bits, dim, comps;
  const float* Wt; /* [dim][bits]: transposed so the inner loop runs over output bits */
  const int8_t* mu;
  uint64_t hC, hX;
  uint64_t* out;
} mix_job;

static void* mix_worker(void* arg) {
  const mix_job* j = (const mix_job*)arg;
  const uint32_t per = (j->dim + 2) / 3, wpc = (j->bits + 63) / 64, bits = j->bits;
  /* |partial sums| <= 128 * 126 * 124 < 2^24: float32 FMA is exact integer arithmetic here */
  float acc[256];
  for (uint64_t r = j->lo; r < j->hi; ++r) {
    const uint64_t i = j->first + r;
    const uint32_t c = (uint32_t)(sm64(j->hC ^ i) % j->comps);
    float x[258];
    const int8_t* mc = j->mu + (size_t)c * j->dim;
    for (uint32_t t = 0; t < per; ++t) { /* one hash per 3 dims: g5(u >> 0|20|40) */
      const uint64_t u = sm64(j->hX ^ (i * per + t));
      x[3 * t] = (float)(mc[3 * t] + g5(u));
      x[3 * t + 1] = (float)(3 * t + 1 < j->dim ? mc[3 * t + 1] + g5(u >> 20) : 0);
      x[3 * t + 2] = (float)(3 * t + 2 < j->dim ? mc[3 * t + 2] + g5(u >> 40) : 0);
    }
    for (uint32_t b = 0; b < bits; ++b) acc[b] = 0.0f;
    for (uint32_t d = 0; d < j->dim; ++d) {
      const float xd = x[d];
      const float* wc = j->Wt + (size_t)d * bits;
      for (uint32_t b = 0; b < bits; ++b) acc[b] += wc[b] * xd;
    }
    for (uint32_t w = 0; w < wpc; ++w) j->out[r * wpc + w] = 0;
    for (uint32_t b = 0; b < bits; ++b)
      if (acc[b] >= 0.0f) j->out[r * wpc + b / 64] |= 1ULL << (b % 64);
  }
  return NULL;
}

int or_gen_mixture(uint64_t first, uint64_t n, uint32_t bits, uint32_t dim, uint32_t comps,
                   uint64_t model_seed, uint64_t data_seed, uint64_t* out, int nthreads) {
  if (bits == 0 || bits > 256 || dim == 0 || dim % 4 || dim > 256 || comps == 0 || comps > 256)
    return fail(1, "gen_mixture: bad shape");
  float* W = (float*)malloc(sizeof(float) * bits * dim);
  int8_t* mu = (int8_t*)malloc((size_t)comps * dim);
  const uint64_t hW = sm64(model_seed ^ (1ULL * 0xD6E8FEB86659FD93ULL));
  const uint64_t hMu = sm64(model_seed ^ (2ULL * 0xD6E8FEB86659FD93ULL));
  /* W[j][d] = g6(h(model_seed, 1, j*dim + d)), stored transposed */
  for (uint64_t t = 0; t < (uint64_t)bits * dim; ++t) W[(t % dim) * bits + t / dim] = (float)g6(sm64(hW ^ t));
  for (uint64_t t = 0; t < (uint64_t)comps * dim; ++t) mu[t] = (int8_t)g5(sm64(hMu ^ t));
  if (nthreads < 1) nthreads = 1;
  if (nthreads > 256) nthreads = 256;
  pthread_t th[256];
  mix_job jobs[256];
  for (int t = 0; t < nthreads; ++t) {
    mix_job* j = &jobs[t];
    j->first = first;
    j->lo = n * (uint64_t)t / (uint64_t)nthreads;
    j->hi = n * (uint64_t)(t + 1) / (uint64_t)nthreads;
    j->bits = bits, j->dim = dim, j->comps = comps, j->Wt = W, j->mu = mu, j->out = out;
    j->hC = sm64(data_seed ^ (3ULL * 0xD6E8FEB86659FD93ULL));
    j->hX = sm64(data_seed ^ (4ULL * 0xD6E8FEB86659FD93ULL));
    pthread_create(&th[t], NULL, mix_worker, j);
  }
  for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
  free(W);
  free(mu);
  return 0;
}

/* ---- substring optimisation (optimize.hpp) ---- */

/* estimate_correlations (optimize.hpp:47-92): bit columns as packed bitsets, ones(i) and
 * ones(i AND j) by popcount, |Pearson| = |p_ij - p_i p_j| / sqrt(var_i var_j) clamped to 1;
 * bits with zero sample variance are flagged constant and stay 0 against every other bit.
 * `counts` (optional, b*b) receives the integer AND counts (diagonal = ones).
 * The reference as its CMake compiles it (-O3 -march=native; g++ contracts by default on an FMA
 * host) evaluates p_ij - p_i*p_j as fma(-p_i, p_j, p_ij): restated explicitly, pinned bitwise. */
int or_estimate_correlations(const uint64_t* codes, uint64_t n, uint32_t bits, double* corr,
                             uint8_t* constant, uint64_t* counts) {
  if (n < 2) return fail(1, "estimate_correlations: need at least 2 codes");
  const uint32_t wpc = wpc_of(bits);
  const uint64_t cw = (n + 63) / 64;
  uint64_t* cols = (uint64_t*)calloc((size_t)bits * cw, 8);
  uint64_t* ones = (uint64_t*)malloc((size_t)bits * 8);
  double* var = (double*)malloc((size_t)bits * sizeof(double));
  if (!cols || !ones || !var) {
    free(cols);
    free(ones);
    free(var);
    return fail(3, "bad_alloc");
  }
  for (uint64_t i = 0; i < n; ++i)
    for (uint32_t pos = 0; pos < bits; ++pos)
      if ((codes[i * wpc + pos / 64] >> (pos % 64)) & 1) cols[(uint64_t)pos * cw + (i >> 6)] |= 1ULL << (i & 63);
  for (uint32_t i = 0; i < bits; ++i) {
    uint64_t c = 0;
    for (uint64_t w = 0; w < cw; ++w) c += (uint64_t)__builtin_popcountll(cols[(uint64_t)i * cw + w]);
    ones[i] = c;
    const double p = (double)c / (double)n;
    var[i] = p * (1.0 - p);
    constant[i] = (c == 0 || c == n) ? 1 : 0;
  }
  for (uint32_t i = 0; i < bits; ++i)
    for (uint32_t j = 0; j < bits; ++j) corr[(uint64_t)i * bits + j] = i == j ? 1.0 : 0.0;
  for (uint32_t i = 0; i < bits; ++i) {
    if (counts) counts[(uint64_t)i * bits + i] = ones[i];
    for (uint32_t j = i + 1; j < bits; ++j) {
      uint64_t c = 0;
      for (uint64_t w = 0; w < cw; ++w)
        c += (uint64_t)__builtin_popcountll(cols[(uint64_t)i * cw + w] & cols[(uint64_t)j * cw + w]);
      if (counts) counts[(uint64_t)i * bits + j] = counts[(uint64_t)j * bits + i] = c;
      if (var[i] == 0.0 || var[j] == 0.0) continue;
      const double pi = (double)ones[i] / (double)n, pj = (double)ones[j] / (double)n;
      const double pij = (double)c / (double)n;
      double v = __builtin_fabs(__builtin_fma(-pi, pj, pij)) / __builtin_sqrt(var[i] * var[j]);
      if (v > 1.0) v = 1.0;
      corr[(uint64_t)i * bits + j] = corr[(uint64_t)j * bits + i] = v;
    }
  }
  free(cols);
  free(ones);
  free(var);
  return 0;
}

/* std::uniform_int_distribution<size_t>(0, range-1) over mt19937_64 as libstdc++ draws it:
 * the generator's range is exactly 2^64, so it downscales with Lemire's multiply-shift and
 * rejects low products below (2^64 - range) mod range. */
static uint64_t uniform_below(mt64* g, uint64_t range) {
  unsigned __int128 prod = (unsigned __int128)mt64_next(g) * range;
  uint64_t low = (uint64_t)prod;
  if (low < range) {
    const uint64_t threshold = (0 - range) % range;
    while (low < threshold) {
      prod = (unsigned __int128)mt64_next(g) * range;
      low = (uint64_t)prod;
    }
  }
  return (uint64_t)(prod >> 64);
}

static void take_value(uint32_t* v, uint32_t* len, uint32_t value) {
  uint32_t i = 0;
  while (v[i] != value) ++i;
  memmove(v + i, v + i + 1, (size_t)(*len - i - 1) * 4);
  --*len;
}

/* greedy_assign (optimize.hpp:101-172): chain initialisation from a seed-chosen opener, then
 * rounds giving each substring with spare capacity the unused bit of least worst-case
 * correlation with its current bits (ties to the lowest index), constant bits last
 * round-robin; each substring's positions sorted ascending. */
int or_greedy_assign(const double* corr, const uint8_t* constant, uint32_t bits, uint32_t m,
                     uint64_t seed, uint32_t* lengths, uint32_t* positions) {
  if (m == 0 || m > bits) return fail(1, "greedy_assign: need 1 <= m <= bits");
  uint32_t *cap = calloc(m, 4), *len = calloc(m, 4), *sub = calloc((size_t)m * bits, 4);
  uint32_t *pool = malloc((size_t)bits * 4), *consts = malloc((size_t)bits * 4);
  mt64* g = malloc(sizeof(mt64));
  if (!cap || !len || !sub || !pool || !consts || !g) {
    free(cap); free(len); free(sub); free(pool); free(consts); free(g);
    return fail(3, "bad_alloc");
  }
  uint32_t np = 0, nc = 0;
  for (uint32_t j = 0; j < m; ++j) cap[j] = bits / m + (j < bits % m ? 1 : 0);
  for (uint32_t i = 0; i < bits; ++i) {
    if (constant[i]) consts[nc++] = i;
    else pool[np++] = i;
  }
#define SUB(j, t) sub[(size_t)(j) * bits + (t)]
  if (np) {
    mt64_seed(g, seed);
    const uint32_t first = pool[uniform_below(g, np)];
    SUB(0, len[0]++) = first;
    take_value(pool, &np, first);
    for (uint32_t j = 1; j < m && np; ++j) {
      const uint32_t prev = len[j - 1] == 0 ? first : SUB(j - 1, 0);
      uint32_t best = pool[0];
      double best_c = -1.0;
      for (uint32_t t = 0; t < np; ++t) {
        const double c = corr[(uint64_t)pool[t] * bits + prev];
        if (c > best_c) {
          best_c = c;
          best = pool[t];
        }
      }
      SUB(j, len[j]++) = best;
      take_value(pool, &np, best);
    }
  }
  while (np) {
    int any = 0;
    for (uint32_t j = 0; j < m && np; ++j) {
      if (len[j] >= cap[j]) continue;
      any = 1;
      uint32_t best = pool[0];
      double best_worst = 2.0;
      for (uint32_t t = 0; t < np; ++t) {
        double worst = 0.0;
        for (uint32_t o = 0; o < len[j]; ++o) {
          const double c = corr[(uint64_t)pool[t] * bits + SUB(j, o)];
          if (c > worst) worst = c;
        }
        if (worst < best_worst) {
          best_worst = worst;
          best = pool[t];
        }
      }
      SUB(j, len[j]++) = best;
      take_value(pool, &np, best);
    }
    if (!any) break;
  }
  uint32_t j = 0;
  for (uint32_t t = 0; t < nc; ++t) {
    while (len[j] >= cap[j]) j = (j + 1) % m;
    SUB(j, len[j]++) = consts[t];
    j = (j + 1) % m;
  }
  uint32_t at = 0;
  for (uint32_t q = 0; q < m; ++q) {
    qsort(&SUB(q, 0), len[q], 4, u32_cmp);
    lengths[q] = len[q];
    for (uint32_t t = 0; t < len[q]; ++t) positions[at++] = SUB(q, t);
  }
#undef SUB
  free(cap); free(len); free(sub); free(pool); free(consts); free(g);
  return 0;
}
