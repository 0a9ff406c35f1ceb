/*
 * tess_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C, fp64 restatement of the reference's Tesseract hot path
 * (tesseract-sim, /root/reference/proj), used as the parity CHECKER for the
 * B200 library. Nothing in the product (paper_2105_14500_b200/) links,
 * loads or calls this file; only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg do.
 *
 * Parity of this restatement is PINNED two ways (tests/test_oracle.py):
 *   1. against the reference's own golden values (RNG
 *      stream words, FNV-1a fingerprints of A, B and of every TesseractA/B
 *      block, the NN [2,2,2] result fingerprint) and the SPEC.md KATs;
 *   2. against the reference itself, compiled from its sources into
 *      oracle/_ref/libtsim_ref.so (oracle/Makefile, oracle/ref_shim.cpp),
 *      on the same seeded inputs (tesseract_matmul NN/NT/TN, backward,
 *      layer_run for every LayerOp, CommStats).
 *
 * Every function cites the reference file:line it restates.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define TOR_EXPORT __attribute__((visibility("default")))

/* ------------------------------------------------------------------ RNG */
/* std::mt19937_64 as fully specified by the C++ standard, seeded through
 * one splitmix64 round per (seed, stream): proj/include/tsim/rng.hpp:20-47 */

typedef struct {
  uint64_t mt[312];
  int idx;
} tor_rng;

static void mt_seed(tor_rng* r, uint64_t seed) {
  r->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
  r->idx = 312;
}

static uint64_t mt_next(tor_rng* r) {
  const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
  if (r->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      uint64_t x = (r->mt[i] & UM) | (r->mt[(i + 1) % 312] & LM);
      uint64_t xa = x >> 1;
      if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
      r->mt[i] = r->mt[(i + 156) % 312] ^ xa;
    }
    r->idx = 0;
  }
  uint64_t x = r->mt[r->idx++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= (x >> 43);
  return x;
}

/* rng.hpp:39-44 */
static uint64_t splitmix(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

/* Rng::stream, rng.hpp:24-26 */
static void rng_stream(tor_rng* r, uint64_t seed, uint64_t stream) {
  mt_seed(r, splitmix(seed + 0x9e3779b97f4a7c15ULL * (stream + 1)));
}

/* Rng::uniform_signed, rng.hpp:31-36 */
static double uniform_signed(tor_rng* r) {
  double u = (double)(mt_next(r) >> 11) * 0x1.0p-53;
  return 2.0 * u - 1.0;
}

TOR_EXPORT void tor_stream_words(uint64_t seed, uint64_t stream, int64_t n,
                                 uint64_t* out) {
  tor_rng r;
  rng_stream(&r, seed, stream);
  for (int64_t i = 0; i < n; ++i) out[i] = mt_next(&r);
}

/* random_matrix, matrix.cpp:72-76 */
TOR_EXPORT void tor_random_matrix(uint64_t seed, uint64_t stream, int64_t rows,
                                  int64_t cols, double* out) {
  tor_rng r;
  rng_stream(&r, seed, stream);
  for (int64_t i = 0; i < rows * cols; ++i) out[i] = uniform_signed(&r);
}

/* random_block_params, layers.cpp:76-99: one stream consumed in the order
 * w_qkv [h,3h], w_proj [h,h], w_ff1 [h,4h], w_ff2 [4h,h] (x 1/sqrt(h)), then
 * ln1_gain (1 + 0.1u), ln1_bias (0.1u), ln2_gain, ln2_bias. */
TOR_EXPORT void tor_random_block_params(int64_t h, uint64_t seed, uint64_t stream,
                                        double* wqkv, double* wproj, double* wff1,
                                        double* wff2, double* ln1g, double* ln1b,
                                        double* ln2g, double* ln2b) {
  tor_rng r;
  rng_stream(&r, seed, stream);
  const double ws = 1.0 / sqrt((double)h);
  for (int64_t i = 0; i < h * 3 * h; ++i) wqkv[i] = ws * uniform_signed(&r);
  for (int64_t i = 0; i < h * h; ++i) wproj[i] = ws * uniform_signed(&r);
  for (int64_t i = 0; i < h * 4 * h; ++i) wff1[i] = ws * uniform_signed(&r);
  for (int64_t i = 0; i < 4 * h * h; ++i) wff2[i] = ws * uniform_signed(&r);
  for (int64_t i = 0; i < h; ++i) ln1g[i] = 1.0 + 0.1 * uniform_signed(&r);
  for (int64_t i = 0; i < h; ++i) ln1b[i] = 0.0 + 0.1 * uniform_signed(&r);
  for (int64_t i = 0; i < h; ++i) ln2g[i] = 1.0 + 0.1 * uniform_signed(&r);
  for (int64_t i = 0; i < h; ++i) ln2b[i] = 0.0 + 0.1 * uniform_signed(&r);
}

/* checksum, matrix.cpp:352-370: FNV-1a over rows, cols, then the
 * little-endian bit images of the doubles. */
TOR_EXPORT uint64_t tor_checksum(int64_t rows, int64_t cols, const double* v) {
  uint64_t h = 0xcbf29ce484222325ULL;
#define FEED(val)                                 \
  do {                                            \
    uint64_t w_ = (val);                          \
    for (int i_ = 0; i_ < 8; ++i_) {              \
      h ^= (w_ >> (8 * i_)) & 0xff;               \
      h *= 0x100000001b3ULL;                      \
    }                                             \
  } while (0)
  FEED((uint64_t)rows);
  FEED((uint64_t)cols);
  for (int64_t i = 0; i < rows * cols; ++i) {
    uint64_t bits;
    memcpy(&bits, &v[i], 8);
    FEED(bits);
  }
#undef FEED
  return h;
}

/* ----------------------------------------------------------------- grid */
/* grid.cpp:43-131. Group kinds: 0 = Row (fixed i,k; slot j), 1 = Column
 * (fixed j,k; slot i), 2 = Depth (fixed i,j; slot k). */

TOR_EXPORT int tor_rank_of(int q, int i, int j, int k) { return k * q * q + i * q + j; }

TOR_EXPORT void tor_coord_of(int q, int rank, int* i, int* j, int* k) {
  *k = rank / (q * q);
  *i = (rank / q) % q;
  *j = rank % q;
}

TOR_EXPORT int tor_block_row(int q, int i, int k) { return i + k * q; }

TOR_EXPORT int tor_group_index(int q, int i, int j, int k, int kind) {
  return kind == 0 ? k * q + i : kind == 1 ? k * q + j : i * q + j;
}

TOR_EXPORT int tor_slot_in_group(int i, int j, int k, int kind) {
  return kind == 0 ? j : kind == 1 ? i : k;
}

TOR_EXPORT void tor_member_at(int q, int kind, int gi, int slot, int* i, int* j,
                              int* k) {
  if (kind == 0) { *i = gi % q; *j = slot; *k = gi / q; }
  else if (kind == 1) { *i = slot; *j = gi % q; *k = gi / q; }
  else { *i = gi / q; *j = gi % q; *k = slot; }
}

/* ------------------------------------------------------------ partition */
/* shard.cpp:68-98 (TesseractA: block-row h = i + k*q of rows/(q*d),
 * block-col j of cols/q; TesseractB: block (i, j) of [rows/q, cols/q],
 * replicated over k). scheme 0 = TesseractA, 1 = TesseractB. Returns -1 on
 * a divisibility error (shard.cpp:14-21). */
TOR_EXPORT int tor_partition(const double* m, int64_t rows, int64_t cols, int q,
                             int d, int scheme, int rank, double* block) {
  int i, j, k;
  tor_coord_of(q, rank, &i, &j, &k);
  int64_t rb, cb, r0, c0;
  if (scheme == 0) {
    if (rows % ((int64_t)q * d) || cols % q) return -1;
    rb = rows / ((int64_t)q * d);
    cb = cols / q;
    r0 = (int64_t)tor_block_row(q, i, k) * rb;
  } else {
    if (rows % q || cols % q) return -1;
    rb = rows / q;
    cb = cols / q;
    r0 = (int64_t)i * rb;
  }
  c0 = (int64_t)j * cb;
  for (int64_t r = 0; r < rb; ++r)
    memcpy(block + r * cb, m + (r0 + r) * cols + c0, (size_t)cb * sizeof(double));
  return 0;
}

/* combine, shard.cpp:139-183: blocks indexed by linear rank. TesseractB
 * replicas (k > 0) must equal the k = 0 block bit for bit; returns -2 on
 * divergence. */
TOR_EXPORT int tor_combine(const double* const* blocks, int64_t rows, int64_t cols,
                           int q, int d, int scheme, double* out) {
  const int p = d * q * q;
  for (int rank = 0; rank < p; ++rank) {
    int i, j, k;
    tor_coord_of(q, rank, &i, &j, &k);
    int64_t rb, cb, r0;
    if (scheme == 0) {
      rb = rows / ((int64_t)q * d);
      cb = cols / q;
      r0 = (int64_t)tor_block_row(q, i, k) * rb;
    } else {
      rb = rows / q;
      cb = cols / q;
      r0 = (int64_t)i * rb;
      if (k > 0) {
        const double* ref = blocks[tor_rank_of(q, i, j, 0)];
        if (memcmp(ref, blocks[rank], (size_t)(rb * cb) * sizeof(double)) != 0) return -2;
        continue;
      }
    }
    const int64_t c0 = (int64_t)j * cb;
    for (int64_t r = 0; r < rb; ++r)
      memcpy(out + (r0 + r) * cols + c0, blocks[rank] + r * cb, (size_t)cb * sizeof(double));
  }
  return 0;
}

/* ---------------------------------------------------------- local GEMMs */
/* matmul_serial, matrix.cpp:168-183 (i-t-j order) */
TOR_EXPORT void tor_matmul(const double* a, int64_t m, int64_t k, const double* b,
                           int64_t n, double* c) {
  memset(c, 0, (size_t)(m * n) * sizeof(double));
  for (int64_t i = 0; i < m; ++i)
    for (int64_t t = 0; t < k; ++t) {
      const double av = a[i * k + t];
      const double* br = b + t * n;
      double* cr = c + i * n;
      for (int64_t j = 0; j < n; ++j) cr[j] += av * br[j];
    }
}

/* matmul_nt, matrix.cpp:185-199: c[m,n] = a[m,k] * b[n,k]^T */
TOR_EXPORT void tor_matmul_nt(const double* a, int64_t m, int64_t k, const double* b,
                              int64_t n, double* c) {
  for (int64_t i = 0; i < m; ++i)
    for (int64_t j = 0; j < n; ++j) {
      double acc = 0.0;
      for (int64_t t = 0; t < k; ++t) acc += a[i * k + t] * b[j * k + t];
      c[i * n + j] = acc;
    }
}

/* matmul_tn, matrix.cpp:201-216: c[m,n] = a[k,m]^T * b[k,n] */
TOR_EXPORT void tor_matmul_tn(const double* a, int64_t k, int64_t m, const double* b,
                              int64_t n, double* c) {
  memset(c, 0, (size_t)(m * n) * sizeof(double));
  for (int64_t t = 0; t < k; ++t)
    for (int64_t i = 0; i < m; ++i) {
      const double av = a[t * m + i];
      for (int64_t j = 0; j < n; ++j) c[i * n + j] += av * b[t * n + j];
    }
}

static double* dalloc(int64_t n) { return (double*)calloc((size_t)(n > 0 ? n : 1), sizeof(double)); }

static void vadd(double* acc, const double* v, int64_t n) {
  for (int64_t i = 0; i < n; ++i) acc[i] += v[i];
}

/* --------------------------------------------------------------- meter */
/* CommStats flat counting, runtime.hpp:24-69, runtime.cpp:287-344: a g-party
 * broadcast charges g-1 messages of numel to the root's send side and 1 to
 * each receiver; reduce charges 1 send per non-root and g-1 receives at the
 * root; all-reduce additionally charges the broadcast leg. Kinds: 0 bcast,
 * 1 reduce, 2 all-reduce. Counters per rank: [sent_msgs, sent_elems,
 * recv_msgs, recv_elems]; per kind: [msgs, elems]. */
typedef struct {
  int q, d, p;
  uint64_t* per_rank; /* p x 4 */
  uint64_t kind[5][2];
} tor_meter;

static void meter_collective(tor_meter* mt, int family, int kind, int root,
                             uint64_t numel) {
  const int q = mt->q, d = mt->d;
  const int gsize = family == 2 ? d : q;
  const int gcount = family == 2 ? q * q : q * d;
  if (gsize <= 1) return;
  for (int gi = 0; gi < gcount; ++gi) {
    for (int s = 0; s < gsize; ++s) {
      int i, j, k;
      tor_member_at(q, family, gi, s, &i, &j, &k);
      uint64_t* c = mt->per_rank + 4 * tor_rank_of(q, i, j, k);
      if (kind == 0) {
        if (s == root) {
          c[0] += gsize - 1;
          c[1] += (uint64_t)(gsize - 1) * numel;
          mt->kind[0][0] += gsize - 1;
          mt->kind[0][1] += (uint64_t)(gsize - 1) * numel;
        } else {
          c[2] += 1;
          c[3] += numel;
        }
      } else {
        const int all = kind == 2;
        const int rt = all ? 0 : root;
        if (s == rt) {
          c[2] += gsize - 1;
          c[3] += (uint64_t)(gsize - 1) * numel;
          if (all) {
            c[0] += gsize - 1;
            c[1] += (uint64_t)(gsize - 1) * numel;
            mt->kind[kind][0] += gsize - 1;
            mt->kind[kind][1] += (uint64_t)(gsize - 1) * numel;
          }
        } else {
          c[0] += 1;
          c[1] += numel;
          mt->kind[kind][0] += 1;
          mt->kind[kind][1] += numel;
          if (all) {
            c[2] += 1;
            c[3] += numel;
          }
        }
      }
    }
  }
}

/* ------------------------------------------------- Tesseract products */
/* Per-rank bodies restated over all ranks at once (algorithms.cpp:34-76).
 * The runtime's collectives are synchronous with slot-ascending sums
 * (runtime.cpp:308-344), so simulating rank by rank in slot order gives the
 * reference's values. Blocks are indexed by linear rank. */

/* nn_product_rank, algorithms.cpp:34-45: C(h,j) = sum_t A(h,t) B(t,j),
 * t ascending (row bcast of A from slot t, column bcast of B from slot t). */
static void nn_all(int q, int d, double* const* ab, int64_t ar, int64_t ak,
                   double* const* bb, int64_t bn, double** cb, tor_meter* mt) {
  const int p = d * q * q;
  double* prod = dalloc(ar * bn);
  for (int t = 0; t < q; ++t) {
    if (mt) {
      meter_collective(mt, 0, 0, t, (uint64_t)(ar * ak));
      meter_collective(mt, 1, 0, t, (uint64_t)(ak * bn));
    }
    for (int rank = 0; rank < p; ++rank) {
      int i, j, k;
      tor_coord_of(q, rank, &i, &j, &k);
      const double* at = ab[tor_rank_of(q, i, t, k)];
      const double* bt = bb[tor_rank_of(q, t, j, k)];
      tor_matmul(at, ar, ak, bt, bn, prod);
      if (t == 0) memcpy(cb[rank], prod, (size_t)(ar * bn) * sizeof(double));
      else vadd(cb[rank], prod, ar * bn);
    }
  }
  free(prod);
}

/* nt_product_rank, algorithms.cpp:47-59: C(h,t) = sum_j A(h,j) B(t,j)^T,
 * column bcast of B(t,j), row reduce (slot ascending) to slot j == t. */
static void nt_all(int q, int d, double* const* ab, int64_t ar, int64_t an,
                   double* const* bb, int64_t br, double** cb, tor_meter* mt) {
  const int p = d * q * q;
  double** partial = (double**)malloc(sizeof(double*) * p);
  for (int r = 0; r < p; ++r) partial[r] = dalloc(ar * br);
  for (int t = 0; t < q; ++t) {
    if (mt) {
      meter_collective(mt, 1, 0, t, (uint64_t)(br * an));
      meter_collective(mt, 0, 1, t, (uint64_t)(ar * br));
    }
    for (int rank = 0; rank < p; ++rank) {
      int i, j, k;
      tor_coord_of(q, rank, &i, &j, &k);
      tor_matmul_nt(ab[rank], ar, an, bb[tor_rank_of(q, t, j, k)], br, partial[rank]);
    }
    for (int rank = 0; rank < p; ++rank) {
      int i, j, k;
      tor_coord_of(q, rank, &i, &j, &k);
      if (j != t) continue;
      memcpy(cb[rank], partial[tor_rank_of(q, i, 0, k)], (size_t)(ar * br) * sizeof(double));
      for (int s = 1; s < q; ++s) vadd(cb[rank], partial[tor_rank_of(q, i, s, k)], ar * br);
    }
  }
  for (int r = 0; r < p; ++r) free(partial[r]);
  free(partial);
}

/* tn_product_rank, algorithms.cpp:61-76: C(t,j) = sum_{i} A(h,t)^T B(h,j)
 * reduced down the column to slot i == t, then (sum_over_depth) all-reduced
 * over the depth group (slot-ascending). */
static void tn_all(int q, int d, double* const* ab, int64_t ar, int64_t an,
                   double* const* bb, int64_t bn, int sum_over_depth, double** cb,
                   tor_meter* mt) {
  const int p = d * q * q;
  double** partial = (double**)malloc(sizeof(double*) * p);
  for (int r = 0; r < p; ++r) partial[r] = dalloc(an * bn);
  for (int t = 0; t < q; ++t) {
    if (mt) {
      meter_collective(mt, 0, 0, t, (uint64_t)(ar * an));
      meter_collective(mt, 1, 1, t, (uint64_t)(an * bn));
    }
    for (int rank = 0; rank < p; ++rank) {
      int i, j, k;
      tor_coord_of(q, rank, &i, &j, &k);
      tor_matmul_tn(ab[tor_rank_of(q, i, t, k)], ar, an, bb[rank], bn, partial[rank]);
    }
    for (int rank = 0; rank < p; ++rank) {
      int i, j, k;
      tor_coord_of(q, rank, &i, &j, &k);
      if (i != t) continue;
      memcpy(cb[rank], partial[tor_rank_of(q, 0, j, k)], (size_t)(an * bn) * sizeof(double));
      for (int s = 1; s < q; ++s) vadd(cb[rank], partial[tor_rank_of(q, s, j, k)], an * bn);
    }
  }
  if (sum_over_depth) {
    if (mt) meter_collective(mt, 2, 2, 0, (uint64_t)(an * bn));
    if (d > 1) {
      double* tmp = dalloc(an * bn);
      for (int i = 0; i < q; ++i)
        for (int j = 0; j < q; ++j) {
          memcpy(tmp, cb[tor_rank_of(q, i, j, 0)], (size_t)(an * bn) * sizeof(double));
          for (int k = 1; k < d; ++k) vadd(tmp, cb[tor_rank_of(q, i, j, k)], an * bn);
          for (int k = 0; k < d; ++k)
            memcpy(cb[tor_rank_of(q, i, j, k)], tmp, (size_t)(an * bn) * sizeof(double));
        }
      free(tmp);
    }
  }
  for (int r = 0; r < p; ++r) free(partial[r]);
  free(partial);
}

static double** blocks_new(int p, int64_t n) {
  double** b = (double**)malloc(sizeof(double*) * p);
  for (int r = 0; r < p; ++r) b[r] = dalloc(n);
  return b;
}

static void blocks_free(double** b, int p) {
  for (int r = 0; r < p; ++r) free(b[r]);
  free(b);
}

static tor_meter* meter_new(int q, int d, uint64_t* per_rank) {
  tor_meter* mt = (tor_meter*)calloc(1, sizeof(tor_meter));
  mt->q = q;
  mt->d = d;
  mt->p = d * q * q;
  mt->per_rank = per_rank;
  return mt;
}

static void meter_finish(tor_meter* mt, uint64_t* kind_out) {
  if (kind_out)
    for (int kk = 0; kk < 5; ++kk) {
      kind_out[2 * kk] = mt->kind[kk][0];
      kind_out[2 * kk + 1] = mt->kind[kk][1];
    }
  free(mt);
}

/* tesseract_matmul, algorithms.cpp:131-186. variant 0 = NN (C=[a,c] from
 * A [a,b], B [b,c]), 1 = NT (C=[m,r] from A [m,n], B [r,n]), 2 = TN
 * (C=[n,r] from A [m,n], B [m,r]). stats_rank: p x 4 counters (may be NULL),
 * stats_kind: 5 x 2 (may be NULL). Returns -1 on shape/divisibility error. */
TOR_EXPORT int tor_tesseract_matmul(int variant, int q, int d, const double* a,
                                    int64_t arows, int64_t acols, const double* b,
                                    int64_t brows, int64_t bcols, double* c,
                                    uint64_t* stats_rank, uint64_t* stats_kind) {
  const int p = d * q * q;
  int bscheme = variant == 2 ? 0 : 1;
  if (variant == 0 && acols != brows) return -1;
  if (variant == 1 && acols != bcols) return -1;
  if (variant == 2 && arows != brows) return -1;
  if (arows % ((int64_t)q * d) || acols % q) return -1;
  if (bscheme == 0 ? (brows % ((int64_t)q * d) || bcols % q) : (brows % q || bcols % q))
    return -1;
  const int64_t ar = arows / ((int64_t)q * d), ac = acols / q;
  const int64_t br = bscheme == 0 ? brows / ((int64_t)q * d) : brows / q, bc = bcols / q;
  double** ab = blocks_new(p, ar * ac);
  double** bb = blocks_new(p, br * bc);
  for (int r = 0; r < p; ++r) {
    tor_partition(a, arows, acols, q, d, 0, r, ab[r]);
    tor_partition(b, brows, bcols, q, d, bscheme, r, bb[r]);
  }
  if (stats_rank) memset(stats_rank, 0, sizeof(uint64_t) * 4 * p);
  uint64_t* scratch = stats_rank ? stats_rank : (uint64_t*)calloc(4 * p, sizeof(uint64_t));
  tor_meter* mt = meter_new(q, d, scratch);
  int rc = 0;
  if (variant == 0) {
    double** cb = blocks_new(p, ar * bc);
    nn_all(q, d, ab, ar, ac, bb, bc, cb, mt);
    rc = tor_combine((const double* const*)cb, arows, bcols, q, d, 0, c);
    blocks_free(cb, p);
  } else if (variant == 1) {
    double** cb = blocks_new(p, ar * br);
    nt_all(q, d, ab, ar, ac, bb, br, cb, mt);
    rc = tor_combine((const double* const*)cb, arows, brows, q, d, 0, c);
    blocks_free(cb, p);
  } else {
    double** cb = blocks_new(p, ac * bc);
    tn_all(q, d, ab, ar, ac, bb, bc, 1, cb, mt);
    rc = tor_combine((const double* const*)cb, acols, bcols, q, d, 1, c);
    blocks_free(cb, p);
  }
  meter_finish(mt, stats_kind);
  if (!stats_rank) free(scratch);
  blocks_free(ab, p);
  blocks_free(bb, p);
  return rc;
}

/* tesseract_backward_dense, algorithms.cpp:188-242: dA = NT(dC, B) and
 * dB = TN(A, dC) with the depth all-reduce. */
TOR_EXPORT int tor_tesseract_backward(int q, int d, const double* dc, const double* a,
                                      const double* b, int64_t m, int64_t k, int64_t n,
                                      double* da, double* db, uint64_t* stats_rank,
                                      uint64_t* stats_kind) {
  const int p = d * q * q;
  if (m % ((int64_t)q * d) || k % q || n % q) return -1;
  const int64_t mr = m / ((int64_t)q * d), kc = k / q, nc = n / q;
  double** dcb = blocks_new(p, mr * nc);
  double** ab = blocks_new(p, mr * kc);
  double** bb = blocks_new(p, kc * nc);
  for (int r = 0; r < p; ++r) {
    tor_partition(dc, m, n, q, d, 0, r, dcb[r]);
    tor_partition(a, m, k, q, d, 0, r, ab[r]);
    tor_partition(b, k, n, q, d, 1, r, bb[r]);
  }
  if (stats_rank) memset(stats_rank, 0, sizeof(uint64_t) * 4 * p);
  uint64_t* scratch = stats_rank ? stats_rank : (uint64_t*)calloc(4 * p, sizeof(uint64_t));
  tor_meter* mt = meter_new(q, d, scratch);
  double** dab = blocks_new(p, mr * kc);
  double** dbb = blocks_new(p, kc * nc);
  nt_all(q, d, dcb, mr, nc, bb, kc, dab, mt);
  tn_all(q, d, ab, mr, kc, dcb, nc, 1, dbb, mt);
  int rc = tor_combine((const double* const*)dab, m, k, q, d, 0, da);
  if (!rc) rc = tor_combine((const double* const*)dbb, k, n, q, d, 1, db);
  meter_finish(mt, stats_kind);
  if (!stats_rank) free(scratch);
  blocks_free(dcb, p);
  blocks_free(ab, p);
  blocks_free(bb, p);
  blocks_free(dab, p);
  blocks_free(dbb, p);
  return rc;
}

/* ------------------------------------------------------- serial layers */
/* The reference's own serial oracle ref::* (layers.cpp:696-905), which
 * layer_run's sharded results match to <= 1.1e-15 (SURVEY App. A probe5;
 * re-checked against oracle/_ref in tests/test_oracle.py). */

static const double kInvSqrt2 = 0.7071067811865475244;
static const double kInvSqrt2Pi = 0.3989422804014326779;

/* gelu / gelu_grad, layers.cpp:25-42 (exact erf form) */
static double gelu(double v) { return 0.5 * v * (1.0 + erf(v * kInvSqrt2)); }
static double gelu_grad(double v) {
  return 0.5 * (1.0 + erf(v * kInvSqrt2)) + v * kInvSqrt2Pi * exp(-0.5 * v * v);
}

static void transpose(const double* a, int64_t r, int64_t c, double* out) {
  for (int64_t i = 0; i < r; ++i)
    for (int64_t j = 0; j < c; ++j) out[j * r + i] = a[i * c + j];
}

/* ref::matmul_serial(a, transpose(b)) without forming b^T explicitly would
 * change nothing numerically (same i-t-j order on identical values), but we
 * keep the reference's explicit transposes for clarity. */
static void mm_bt(const double* a, int64_t m, int64_t k, const double* b, int64_t n,
                  double* c) {
  double* bt = dalloc(k * n);
  transpose(b, n, k, bt);
  tor_matmul(a, m, k, bt, n, c);
  free(bt);
}

static void mm_at(const double* a, int64_t k, int64_t m, const double* b, int64_t n,
                  double* c) {
  double* at = dalloc(m * k);
  transpose(a, k, m, at);
  tor_matmul(at, m, k, b, n, c);
  free(at);
}

/* ref::layernorm, layers.cpp:698-728 */
static void layernorm(const double* x, int64_t rows, int64_t w, const double* gain,
                      const double* bias, double eps, double* y, double* xhat,
                      double* isv_out) {
  const double n = (double)w;
  for (int64_t r = 0; r < rows; ++r) {
    double s = 0.0, s2 = 0.0;
    for (int64_t c = 0; c < w; ++c) {
      const double v = x[r * w + c];
      s += v;
      s2 += v * v;
    }
    const double mean = s / n;
    double var = s2 / n - mean * mean;
    if (var < 0.0) var = 0.0;
    const double isv = 1.0 / sqrt(var + eps);
    isv_out[r] = isv;
    for (int64_t c = 0; c < w; ++c) {
      const double xh = (x[r * w + c] - mean) * isv;
      xhat[r * w + c] = xh;
      y[r * w + c] = gain[c] * xh + bias[c];
    }
  }
}

/* ref::layernorm_backward, layers.cpp:730-770 */
static void layernorm_backward(const double* dy, int64_t rows, int64_t w,
                               const double* xhat, const double* isv,
                               const double* gain, double* dx, double* dgain,
                               double* dbias) {
  const double n = (double)w;
  for (int64_t r = 0; r < rows; ++r) {
    double s = 0.0, sx = 0.0;
    for (int64_t c = 0; c < w; ++c) {
      const double dxh = dy[r * w + c] * gain[c];
      s += dxh;
      sx += xhat[r * w + c] * dxh;
    }
    const double mean_d = s / n, mean_xd = sx / n;
    for (int64_t c = 0; c < w; ++c) {
      const double dxh = dy[r * w + c] * gain[c];
      dx[r * w + c] = isv[r] * (dxh - mean_d - xhat[r * w + c] * mean_xd);
    }
  }
  if (dgain)
    for (int64_t c = 0; c < w; ++c) {
      double dg = 0.0;
      for (int64_t r = 0; r < rows; ++r) dg += dy[r * w + c] * xhat[r * w + c];
      dgain[c] += dg;
    }
  if (dbias)
    for (int64_t c = 0; c < w; ++c) {
      double db = 0.0;
      for (int64_t r = 0; r < rows; ++r) db += dy[r * w + c];
      dbias[c] += db;
    }
}

/* softmax_rows / softmax_backward_rows, layers.cpp:44-74 */
static void softmax_rows(const double* s, int64_t rows, int64_t cols, double* p) {
  for (int64_t r = 0; r < rows; ++r) {
    double mx = s[r * cols];
    for (int64_t c = 1; c < cols; ++c) mx = fmax(mx, s[r * cols + c]);
    double sum = 0.0;
    for (int64_t c = 0; c < cols; ++c) {
      const double e = exp(s[r * cols + c] - mx);
      p[r * cols + c] = e;
      sum += e;
    }
    for (int64_t c = 0; c < cols; ++c) p[r * cols + c] /= sum;
  }
}

static void softmax_backward_rows(const double* p, const double* dp, int64_t rows,
                                  int64_t cols, double* ds) {
  for (int64_t r = 0; r < rows; ++r) {
    double dot = 0.0;
    for (int64_t c = 0; c < cols; ++c) dot += p[r * cols + c] * dp[r * cols + c];
    for (int64_t c = 0; c < cols; ++c) ds[r * cols + c] = p[r * cols + c] * (dp[r * cols + c] - dot);
  }
}

typedef struct {
  const double *wqkv, *wproj, *wff1, *wff2, *ln1g, *ln1b, *ln2g, *ln2b;
  double eps;
} params_t;

typedef struct {
  double *wqkv, *wproj, *wff1, *wff2, *ln1g, *ln1b, *ln2g, *ln2b;
} grads_t;

typedef struct {
  double *x, *z, *h;
} ffc_t;

typedef struct {
  double *x, *qkv, *o, *probs;
} attc_t;

/* ref::feedforward, layers.cpp:772-783 */
static void feedforward(const double* x, int64_t T, int64_t h, const params_t* p,
                        double* y, ffc_t* c) {
  c->x = dalloc(T * h);
  memcpy(c->x, x, (size_t)(T * h) * sizeof(double));
  c->z = dalloc(T * 4 * h);
  c->h = dalloc(T * 4 * h);
  tor_matmul(x, T, h, p->wff1, 4 * h, c->z);
  for (int64_t i = 0; i < T * 4 * h; ++i) c->h[i] = gelu(c->z[i]);
  tor_matmul(c->h, T, 4 * h, p->wff2, h, y);
}

/* ref::feedforward_backward, layers.cpp:785-796 */
static void feedforward_backward(const double* dy, int64_t T, int64_t h,
                                 const params_t* p, const ffc_t* c, double* dx,
                                 grads_t* g) {
  double* dh = dalloc(T * 4 * h);
  mm_bt(dy, T, h, p->wff2, 4 * h, dh);
  for (int64_t i = 0; i < T * 4 * h; ++i) dh[i] *= gelu_grad(c->z[i]);
  mm_bt(dh, T, 4 * h, p->wff1, h, dx);
  double* t2 = dalloc(4 * h * h);
  mm_at(c->h, T, 4 * h, dy, h, t2);
  vadd(g->wff2, t2, 4 * h * h);
  mm_at(c->x, T, h, dh, 4 * h, t2);
  vadd(g->wff1, t2, 4 * h * h);
  free(t2);
  free(dh);
}

static void get_block(const double* m, int64_t ld, int64_t r0, int64_t nr, int64_t c0,
                      int64_t nc, double* out) {
  for (int64_t r = 0; r < nr; ++r)
    memcpy(out + r * nc, m + (r0 + r) * ld + c0, (size_t)nc * sizeof(double));
}

static void put_block(double* m, int64_t ld, int64_t r0, int64_t nr, int64_t c0,
                      int64_t nc, const double* in) {
  for (int64_t r = 0; r < nr; ++r)
    memcpy(m + (r0 + r) * ld + c0, in + r * nc, (size_t)nc * sizeof(double));
}

/* ref::attention, layers.cpp:798-827 (no mask; per-head interleaved Q|K|V
 * column triples of width 3*hd, layers.hpp:38-41) */
static void attention(const double* x, int64_t batch, int64_t s, int64_t h,
                      int64_t heads, const params_t* p, double* y, attc_t* c) {
  const int64_t T = batch * s, hd = h / heads;
  const double inv = 1.0 / sqrt((double)hd);
  c->x = dalloc(T * h);
  memcpy(c->x, x, (size_t)(T * h) * sizeof(double));
  c->qkv = dalloc(T * 3 * h);
  c->o = dalloc(T * h);
  c->probs = dalloc(batch * heads * s * s);
  tor_matmul(x, T, h, p->wqkv, 3 * h, c->qkv);
  double *qm = dalloc(s * hd), *km = dalloc(s * hd), *vm = dalloc(s * hd);
  double *sc = dalloc(s * s), *oh = dalloc(s * hd);
  for (int64_t smp = 0; smp < batch; ++smp)
    for (int64_t hh = 0; hh < heads; ++hh) {
      const int64_t row0 = smp * s, base = hh * 3 * hd;
      get_block(c->qkv, 3 * h, row0, s, base, hd, qm);
      get_block(c->qkv, 3 * h, row0, s, base + hd, hd, km);
      get_block(c->qkv, 3 * h, row0, s, base + 2 * hd, hd, vm);
      mm_bt(qm, s, hd, km, s, sc);
      for (int64_t i = 0; i < s * s; ++i) sc[i] *= inv;
      double* prob = c->probs + (smp * heads + hh) * s * s;
      softmax_rows(sc, s, s, prob);
      tor_matmul(prob, s, s, vm, hd, oh);
      put_block(c->o, h, row0, s, hh * hd, hd, oh);
    }
  tor_matmul(c->o, T, h, p->wproj, h, y);
  free(qm); free(km); free(vm); free(sc); free(oh);
}

/* ref::attention_backward, layers.cpp:829-867 */
static void attention_backward(const double* dy, int64_t batch, int64_t s, int64_t h,
                               int64_t heads, const params_t* p, const attc_t* c,
                               double* dx, grads_t* g) {
  const int64_t T = batch * s, hd = h / heads;
  const double inv = 1.0 / sqrt((double)hd);
  double* dout = dalloc(T * h);
  mm_bt(dy, T, h, p->wproj, h, dout);
  double* t2 = dalloc(3 * h * h);
  mm_at(c->o, T, h, dy, h, t2);
  vadd(g->wproj, t2, h * h);
  double* dqkv = dalloc(T * 3 * h);
  double *qm = dalloc(s * hd), *km = dalloc(s * hd), *vm = dalloc(s * hd);
  double *doh = dalloc(s * hd), *dprob = dalloc(s * s), *ds = dalloc(s * s);
  double *dq = dalloc(s * hd), *dk = dalloc(s * hd), *dv = dalloc(s * hd);
  for (int64_t smp = 0; smp < batch; ++smp)
    for (int64_t hh = 0; hh < heads; ++hh) {
      const int64_t row0 = smp * s, base = hh * 3 * hd;
      get_block(c->qkv, 3 * h, row0, s, base, hd, qm);
      get_block(c->qkv, 3 * h, row0, s, base + hd, hd, km);
      get_block(c->qkv, 3 * h, row0, s, base + 2 * hd, hd, vm);
      const double* prob = c->probs + (smp * heads + hh) * s * s;
      get_block(dout, h, row0, s, hh * hd, hd, doh);
      mm_bt(doh, s, hd, vm, s, dprob);
      mm_at(prob, s, s, doh, hd, dv);
      softmax_backward_rows(prob, dprob, s, s, ds);
      for (int64_t i = 0; i < s * s; ++i) ds[i] *= inv;
      tor_matmul(ds, s, s, km, hd, dq);
      mm_at(ds, s, s, qm, hd, dk);
      put_block(dqkv, 3 * h, row0, s, base, hd, dq);
      put_block(dqkv, 3 * h, row0, s, base + hd, hd, dk);
      put_block(dqkv, 3 * h, row0, s, base + 2 * hd, hd, dv);
    }
  mm_bt(dqkv, T, 3 * h, p->wqkv, h, dx);
  mm_at(c->x, T, h, dqkv, 3 * h, t2);
  vadd(g->wqkv, t2, 3 * h * h);
  free(t2); free(dout); free(dqkv);
  free(qm); free(km); free(vm); free(doh); free(dprob); free(ds);
  free(dq); free(dk); free(dv);
}

/* layer_run (layers.cpp:604-692) computed with the serial ref::* path.
 * op: 0 Feedforward, 1 Attention, 2 Layernorm, 3 BiasAdd, 4 Block
 * (LayerOp, layers.hpp:187). params/grads: 8 arrays in BlockParams order
 * (w_qkv, w_proj, w_ff1, w_ff2, ln1_gain, ln1_bias, ln2_gain, ln2_bias);
 * grads are ACCUMULATED into (callers zero them). dbias (BiasAdd) [h]. */
TOR_EXPORT int tor_layer_run(int op, int64_t batch, int64_t seq, int64_t hidden,
                             int64_t heads, const double* x, const double* dy,
                             const double* const* prm, double eps, double* y,
                             double* dx, double* const* grd, double* dbias) {
  const int64_t T = batch * seq, h = hidden;
  if (heads <= 0 || h % heads) return -1;
  params_t p = {prm[0], prm[1], prm[2], prm[3], prm[4], prm[5], prm[6], prm[7], eps};
  grads_t g = {grd[0], grd[1], grd[2], grd[3], grd[4], grd[5], grd[6], grd[7]};
  switch (op) {
    case 0: {
      ffc_t c;
      feedforward(x, T, h, &p, y, &c);
      feedforward_backward(dy, T, h, &p, &c, dx, &g);
      free(c.x); free(c.z); free(c.h);
      break;
    }
    case 1: {
      attc_t c;
      attention(x, batch, seq, h, heads, &p, y, &c);
      attention_backward(dy, batch, seq, h, heads, &p, &c, dx, &g);
      free(c.x); free(c.qkv); free(c.o); free(c.probs);
      break;
    }
    case 2: {
      double* xhat = dalloc(T * h);
      double* isv = dalloc(T);
      layernorm(x, T, h, p.ln1g, p.ln1b, eps, y, xhat, isv);
      layernorm_backward(dy, T, h, xhat, isv, p.ln1g, dx, g.ln1g, g.ln1b);
      free(xhat); free(isv);
      break;
    }
    case 3: {
      /* bias_add_forward/backward (layers.cpp:491-517, 664-675): the bias
       * is params.ln1_bias; dx = dy; dbias = column sums of dy. */
      for (int64_t r = 0; r < T; ++r)
        for (int64_t c = 0; c < h; ++c) y[r * h + c] = x[r * h + c] + p.ln1b[c];
      memcpy(dx, dy, (size_t)(T * h) * sizeof(double));
      for (int64_t c = 0; c < h; ++c) {
        double sacc = 0.0;
        for (int64_t r = 0; r < T; ++r) sacc += dy[r * h + c];
        dbias[c] = sacc;
      }
      break;
    }
    case 4: {
      /* ref::transformer_block / _backward, layers.cpp:878-903 */
      double *xh1 = dalloc(T * h), *isv1 = dalloc(T), *ln1 = dalloc(T * h);
      double *xh2 = dalloc(T * h), *isv2 = dalloc(T), *ln2 = dalloc(T * h);
      double *att = dalloc(T * h), *r1 = dalloc(T * h), *ff = dalloc(T * h);
      attc_t ac;
      ffc_t fc;
      layernorm(x, T, h, p.ln1g, p.ln1b, eps, ln1, xh1, isv1);
      attention(ln1, batch, seq, h, heads, &p, att, &ac);
      for (int64_t i = 0; i < T * h; ++i) r1[i] = x[i] + att[i];
      layernorm(r1, T, h, p.ln2g, p.ln2b, eps, ln2, xh2, isv2);
      feedforward(ln2, T, h, &p, ff, &fc);
      for (int64_t i = 0; i < T * h; ++i) y[i] = r1[i] + ff[i];
      double *dff = dalloc(T * h), *dln2 = dalloc(T * h), *dr1 = dalloc(T * h);
      double *dat = dalloc(T * h), *dln1 = dalloc(T * h);
      feedforward_backward(dy, T, h, &p, &fc, dff, &g);
      layernorm_backward(dff, T, h, xh2, isv2, p.ln2g, dln2, g.ln2g, g.ln2b);
      for (int64_t i = 0; i < T * h; ++i) dr1[i] = dy[i] + dln2[i];
      attention_backward(dr1, batch, seq, h, heads, &p, &ac, dat, &g);
      layernorm_backward(dat, T, h, xh1, isv1, p.ln1g, dln1, g.ln1g, g.ln1b);
      for (int64_t i = 0; i < T * h; ++i) dx[i] = dr1[i] + dln1[i];
      free(xh1); free(isv1); free(ln1); free(xh2); free(isv2); free(ln2);
      free(att); free(r1); free(ff); free(dff); free(dln2); free(dr1);
      free(dat); free(dln1);
      free(ac.x); free(ac.qkv); free(ac.o); free(ac.probs);
      free(fc.x); free(fc.z); free(fc.h);
      break;
    }
    default:
      return -1;
  }
  return 0;
}

/* Metered collective schedule of layer_run (layers.cpp:604-692) on a
 * [q,q,d] grid without computing values: the per-rank programs issue the
 * same collectives in the same order for every rank, so the totals follow
 * from the op sequence (layers.cpp:242-517, algorithms.cpp:34-76). Shapes
 * are per-rank local extents. */
TOR_EXPORT void tor_layer_stats(int op, int q, int d, int64_t batch, int64_t seq,
                                int64_t hidden, uint64_t* stats_rank,
                                uint64_t* stats_kind) {
  const int p = d * q * q;
  memset(stats_rank, 0, sizeof(uint64_t) * 4 * p);
  tor_meter* mt = meter_new(q, d, stats_rank);
  const uint64_t rows = (uint64_t)(batch / (d * q) * seq), hq = (uint64_t)(hidden / q);
#define NN(ar, ak, bn) do { for (int t = 0; t < q; ++t) { \
    meter_collective(mt, 0, 0, t, (ar) * (ak)); meter_collective(mt, 1, 0, t, (ak) * (bn)); } } while (0)
#define NT(ar, an, br) do { for (int t = 0; t < q; ++t) { \
    meter_collective(mt, 1, 0, t, (br) * (an)); meter_collective(mt, 0, 1, t, (ar) * (br)); } } while (0)
#define TN(ar, an, bn) do { for (int t = 0; t < q; ++t) { \
    meter_collective(mt, 0, 0, t, (ar) * (an)); meter_collective(mt, 1, 1, t, (an) * (bn)); } \
    meter_collective(mt, 2, 2, 0, (an) * (bn)); } while (0)
#define LNF() meter_collective(mt, 0, 2, 0, rows * 2)
#define LNB() do { meter_collective(mt, 0, 2, 0, rows * 2); \
    meter_collective(mt, 1, 2, 0, 2 * hq); meter_collective(mt, 2, 2, 0, 2 * hq); } while (0)
#define FFF() do { NN(rows, hq, 4 * hq); NN(rows, 4 * hq, hq); } while (0)
#define FFB() do { NT(rows, hq, 4 * hq); NT(rows, 4 * hq, hq); TN(rows, 4 * hq, hq); TN(rows, hq, 4 * hq); } while (0)
#define ATF() do { NN(rows, hq, 3 * hq); NN(rows, hq, hq); } while (0)
#define ATB() do { NT(rows, hq, hq); TN(rows, hq, hq); NT(rows, 3 * hq, hq); TN(rows, hq, 3 * hq); } while (0)
  switch (op) {
    case 0: FFF(); FFB(); break;
    case 1: ATF(); ATB(); break;
    case 2: LNF(); LNB(); break;
    case 3:
      meter_collective(mt, 1, 0, 0, hq);
      meter_collective(mt, 1, 1, 0, hq);
      /* depth all-reduce only among the i == 0 ranks (layers.cpp:513-515) */
      if (d > 1) {
        for (int j = 0; j < q; ++j)
          for (int k = 0; k < d; ++k) {
            uint64_t* c = stats_rank + 4 * tor_rank_of(q, 0, j, k);
            if (k == 0) {
              c[2] += d - 1; c[3] += (d - 1) * hq; c[0] += d - 1; c[1] += (d - 1) * hq;
              mt->kind[2][0] += d - 1; mt->kind[2][1] += (d - 1) * hq;
            } else {
              c[0] += 1; c[1] += hq; c[2] += 1; c[3] += hq;
              mt->kind[2][0] += 1; mt->kind[2][1] += hq;
            }
          }
      }
      break;
    case 4:
      LNF(); ATF(); LNF(); FFF();
      FFB(); LNB(); ATB(); LNB();
      break;
  }
#undef NN
#undef NT
#undef TN
#undef LNF
#undef LNB
#undef FFF
#undef FFB
#undef ATF
#undef ATB
  meter_finish(mt, stats_kind);
}

/* ------------------------------------------------------------ toy training */
/* Serial half of train_toy (layers.cpp:947-1004): `layers` pre-norm blocks,
 * MSE loss sum(diff^2)/(rows*hidden) against a random target, dy =
 * 2*diff/denom, plain SGD on every parameter (including LayerNorm vectors),
 * seeds: x = stream(seed,0), target = stream(seed,1), block l params =
 * stream(seed,100+l). Writes the loss of every step (before its update). */
typedef struct {
  double *xh1, *isv1, *ln1, *r1, *xh2, *isv2, *ln2, *y;
  attc_t ac;
  ffc_t fc;
} blkc_t;

static void block_fwd(const double* x, int64_t b, int64_t s, int64_t h, int64_t nh,
                      const params_t* p, blkc_t* c) {
  const int64_t T = b * s;
  c->xh1 = dalloc(T * h); c->isv1 = dalloc(T); c->ln1 = dalloc(T * h);
  c->r1 = dalloc(T * h); c->xh2 = dalloc(T * h); c->isv2 = dalloc(T);
  c->ln2 = dalloc(T * h); c->y = dalloc(T * h);
  double* att = dalloc(T * h);
  double* ff = dalloc(T * h);
  layernorm(x, T, h, p->ln1g, p->ln1b, p->eps, c->ln1, c->xh1, c->isv1);
  attention(c->ln1, b, s, h, nh, p, att, &c->ac);
  for (int64_t i = 0; i < T * h; ++i) c->r1[i] = x[i] + att[i];
  layernorm(c->r1, T, h, p->ln2g, p->ln2b, p->eps, c->ln2, c->xh2, c->isv2);
  feedforward(c->ln2, T, h, p, ff, &c->fc);
  for (int64_t i = 0; i < T * h; ++i) c->y[i] = c->r1[i] + ff[i];
  free(att);
  free(ff);
}

static void block_bwd(const double* dy, int64_t b, int64_t s, int64_t h, int64_t nh,
                      const params_t* p, blkc_t* c, double* dx, grads_t* g) {
  const int64_t T = b * s;
  double *dff = dalloc(T * h), *dln2 = dalloc(T * h), *dr1 = dalloc(T * h);
  double *dat = dalloc(T * h), *dln1 = dalloc(T * h);
  feedforward_backward(dy, T, h, p, &c->fc, dff, g);
  layernorm_backward(dff, T, h, c->xh2, c->isv2, p->ln2g, dln2, g->ln2g, g->ln2b);
  for (int64_t i = 0; i < T * h; ++i) dr1[i] = dy[i] + dln2[i];
  attention_backward(dr1, b, s, h, nh, p, &c->ac, dat, g);
  layernorm_backward(dat, T, h, c->xh1, c->isv1, p->ln1g, dln1, g->ln1g, g->ln1b);
  for (int64_t i = 0; i < T * h; ++i) dx[i] = dr1[i] + dln1[i];
  free(dff); free(dln2); free(dr1); free(dat); free(dln1);
  free(c->xh1); free(c->isv1); free(c->ln1); free(c->r1); free(c->xh2); free(c->isv2);
  free(c->ln2); free(c->y);
  free(c->ac.x); free(c->ac.qkv); free(c->ac.o); free(c->ac.probs);
  free(c->fc.x); free(c->fc.z); free(c->fc.h);
}

TOR_EXPORT int tor_train_toy(int64_t batch, int64_t seq, int64_t hidden, int64_t heads,
                             int layers, int steps, double lr, uint64_t seed, double eps,
                             double* losses) {
  const int64_t T = batch * seq, h = hidden;
  if (heads <= 0 || h % heads || layers < 1) return -1;
  const double denom = (double)(T * h);
  double* x = dalloc(T * h);
  double* target = dalloc(T * h);
  tor_random_matrix(seed, 0, T, h, x);
  tor_random_matrix(seed, 1, T, h, target);
  const int64_t sz[8] = {h * 3 * h, h * h, h * 4 * h, 4 * h * h, h, h, h, h};
  double** W = (double**)calloc((size_t)layers * 8, sizeof(double*));
  double** G = (double**)calloc((size_t)layers * 8, sizeof(double*));
  for (int l = 0; l < layers; ++l) {
    for (int k = 0; k < 8; ++k) {
      W[l * 8 + k] = dalloc(sz[k]);
      G[l * 8 + k] = dalloc(sz[k]);
    }
    tor_random_block_params(h, seed, 100 + (uint64_t)l, W[l * 8 + 0], W[l * 8 + 1],
                            W[l * 8 + 2], W[l * 8 + 3], W[l * 8 + 4], W[l * 8 + 5],
                            W[l * 8 + 6], W[l * 8 + 7]);
  }
  blkc_t* cache = (blkc_t*)calloc((size_t)layers, sizeof(blkc_t));
  double* dy = dalloc(T * h);
  double* dxb = dalloc(T * h);
  for (int st = 0; st < steps; ++st) {
    const double* cur = x;
    for (int l = 0; l < layers; ++l) {
      params_t p = {W[l * 8 + 0], W[l * 8 + 1], W[l * 8 + 2], W[l * 8 + 3], W[l * 8 + 4],
                    W[l * 8 + 5], W[l * 8 + 6], W[l * 8 + 7], eps};
      block_fwd(cur, batch, seq, h, heads, &p, &cache[l]);
      cur = cache[l].y;
    }
    double loss = 0.0;
    for (int64_t i = 0; i < T * h; ++i) {
      const double dv = cur[i] - target[i];
      loss += dv * dv;
      dy[i] = 2.0 / denom * dv;
    }
    losses[st] = loss / denom;
    for (int l = layers - 1; l >= 0; --l) {
      params_t p = {W[l * 8 + 0], W[l * 8 + 1], W[l * 8 + 2], W[l * 8 + 3], W[l * 8 + 4],
                    W[l * 8 + 5], W[l * 8 + 6], W[l * 8 + 7], eps};
      for (int k = 0; k < 8; ++k) memset(G[l * 8 + k], 0, (size_t)sz[k] * sizeof(double));
      grads_t g = {G[l * 8 + 0], G[l * 8 + 1], G[l * 8 + 2], G[l * 8 + 3],
                   G[l * 8 + 4], G[l * 8 + 5], G[l * 8 + 6], G[l * 8 + 7]};
      block_bwd(dy, batch, seq, h, heads, &p, &cache[l], dxb, &g);
      memcpy(dy, dxb, (size_t)(T * h) * sizeof(double));
    }
    for (int l = 0; l < layers; ++l)
      for (int k = 0; k < 8; ++k)
        for (int64_t i = 0; i < sz[k]; ++i) W[l * 8 + k][i] -= lr * G[l * 8 + k][i];
  }
  for (int i = 0; i < layers * 8; ++i) {
    free(W[i]);
    free(G[i]);
  }
  free(W); free(G); free(cache); free(x); free(target); free(dy); free(dxb);
  return 0;
}

/* megatron_1d_linear, algorithms.cpp:244-265: line grid [1,1,p]; W1 split by
 * column blocks (Column1D, shard.cpp:110-118), W2 by row blocks (Row1D,
 * shard.cpp:119-127); out = sum_k (X W1_k) W2_k with the slot-ascending sum of
 * the depth all-reduce. Returns -1 on shape / divisibility errors. */
TOR_EXPORT int tor_megatron_1d_linear(int p, const double* x, int64_t xr, int64_t xc,
                                      const double* w1, int64_t w1c, const double* w2,
                                      int64_t w2c, double* out) {
  if (p < 1 || w1c % p) return -1;
  const int64_t kb = w1c / p;
  double* b1 = dalloc(xc * kb);
  double* h = dalloc(xr * kb);
  double* part = dalloc(xr * w2c);
  memset(out, 0, (size_t)(xr * w2c) * sizeof(double));
  for (int k = 0; k < p; ++k) {
    for (int64_t r = 0; r < xc; ++r)
      memcpy(b1 + r * kb, w1 + r * w1c + (int64_t)k * kb, (size_t)kb * sizeof(double));
    tor_matmul(x, xr, xc, b1, kb, h);
    tor_matmul(h, xr, kb, w2 + (int64_t)k * kb * w2c, w2c, part);
    if (k == 0) memcpy(out, part, (size_t)(xr * w2c) * sizeof(double));
    else vadd(out, part, xr * w2c);
  }
  free(b1);
  free(h);
  free(part);
  return 0;
}
