/*
 * oracle.c -- CPU oracle for the LiRank sparse-embedding hot path.
 * TEST INFRASTRUCTURE ONLY (see oracle.h).  Each function follows SURVEY.md §8(c)
 * step by step; the paper passages are cited at each definition in oracle.h.
 *
 * Build: gcc -O2 -std=c99 -ffp-contract=off -fno-fast-math -fPIC -shared oracle.c -lm
 * (liboracle.so, sequential), and the same source with -fopenmp (liboracle_omp.so): the
 * OpenMP pragmas only split loops whose iterations are independent -- bags (a2, a10),
 * segments (a6), unique rows (a8), table rows (a9), and the a5 sort into key ranges (the
 * concatenation of range-sorted buckets is the same total (key, occurrence) order) -- so
 * every arithmetic operation, and its order within an output, is the sequential one and
 * both builds give bit-identical results (tests/test_oracle_omp.py).  The global norm
 * (one running fp64 sum in (u, d) order) stays sequential.
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static int ora_nthreads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

int32_t ora_threads(void) { return (int32_t)ora_nthreads(); }

void ora_set_threads(int32_t n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
#else
  (void)n;
#endif
}

/* ------------------------------------------------------------------------- */
/* Row addressing                                    */
/* ------------------------------------------------------------------------- */

/* base[t] = sum of the rows of tables < t (caller frees). */
static int64_t* table_bases(const ora_cfg* c) {
  int64_t* base = (int64_t*)malloc(sizeof(int64_t) * (size_t)(c->num_tables + 1));
  base[0] = 0;
  for (int32_t t = 0; t < c->num_tables; ++t) base[t + 1] = base[t] + c->table_rows[t];
  return base;
}

/* Global key of id `id` read by feature f, or -1 if the id is out of range. */
static int64_t row_key(const ora_cfg* c, const int64_t* base, int32_t f, int32_t id) {
  int32_t t = c->feature_table[f];
  if (id < 0 || (int64_t)id >= c->table_rows[t]) return -1;
  return base[t] + id;
}

/* ------------------------------------------------------------------------- */
/* a2 forward pooled lookup                                                   */
/* ------------------------------------------------------------------------- */

int64_t ora_forward(const ora_cfg* c, const float* W, const int32_t* ids,
                    const int32_t* offsets, int32_t B, float* out) {
  const int32_t D = c->dim, F = c->num_features;
  const int64_t nbags = (int64_t)F * B;
  int64_t invalid = 0;
  int64_t* base = table_bases(c);
#pragma omp parallel reduction(+ : invalid)
  {
    float* acc = (float*)malloc(sizeof(float) * (size_t)D);
#pragma omp for schedule(dynamic, 512)
    for (int64_t bag = 0; bag < nbags; ++bag) {
      int32_t f = (int32_t)(bag / B), b = (int32_t)(bag % B);
      int32_t lo = offsets[bag], hi = offsets[bag + 1];
      for (int32_t d = 0; d < D; ++d) acc[d] = 0.0f;
      for (int32_t j = lo; j < hi; ++j) {
        int64_t key = row_key(c, base, f, ids[j]);
        if (key < 0) { ++invalid; continue; }
        const float* row = W + key * D;
        for (int32_t d = 0; d < D; ++d) acc[d] = acc[d] + row[d];
      }
      if (c->pooling == 1) {
        int32_t L = hi - lo;
        for (int32_t d = 0; d < D; ++d) acc[d] = (L > 0) ? acc[d] / (float)L : 0.0f;
      }
      float* o = out + ((int64_t)b * F + f) * D;
      for (int32_t d = 0; d < D; ++d) o[d] = acc[d];
    }
    free(acc);
  }
  free(base);
  return invalid;
}

/* ------------------------------------------------------------------------- */
/* a5 dedup: stable sort by key (ties by occurrence index), then run-length   */
/* ------------------------------------------------------------------------- */

typedef struct { int64_t key, occ, bag; } occ_t;

static int cmp_occ(const void* a, const void* b) {
  const occ_t* x = (const occ_t*)a;
  const occ_t* y = (const occ_t*)b;
  if (x->key != y->key) return x->key < y->key ? -1 : 1;
  if (x->occ != y->occ) return x->occ < y->occ ? -1 : 1; /* stability, explicitly */
  return 0;
}

/* Sort by (key, occurrence).  With several threads: P buckets of equal key ranges,
 * scattered in occurrence order and sorted each on its own thread; buckets hold disjoint,
 * increasing key ranges, so their concatenation is the one (key, occurrence) order. */
static void sort_occ(occ_t* v, int64_t n) {
  const int P = ora_nthreads();
  if (P <= 1 || n < 65536) {
    qsort(v, (size_t)n, sizeof(occ_t), cmp_occ);
    return;
  }
  int64_t kmax = 0;
  for (int64_t k = 0; k < n; ++k)
    if (v[k].key > kmax) kmax = v[k].key;
  const int64_t span = kmax / P + 1;
  int64_t* start = (int64_t*)calloc((size_t)P + 1, sizeof(int64_t));
  for (int64_t k = 0; k < n; ++k) ++start[v[k].key / span + 1];
  for (int p = 0; p < P; ++p) start[p + 1] += start[p];
  int64_t* at = (int64_t*)malloc(sizeof(int64_t) * (size_t)P);
  memcpy(at, start, sizeof(int64_t) * (size_t)P);
  occ_t* tmp = (occ_t*)malloc(sizeof(occ_t) * (size_t)n);
  for (int64_t k = 0; k < n; ++k) tmp[at[v[k].key / span]++] = v[k];
#pragma omp parallel for schedule(dynamic, 1)
  for (int p = 0; p < P; ++p)
    qsort(tmp + start[p], (size_t)(start[p + 1] - start[p]), sizeof(occ_t), cmp_occ);
  memcpy(v, tmp, sizeof(occ_t) * (size_t)n);
  free(tmp);
  free(at);
  free(start);
}

int64_t ora_dedup(const ora_cfg* c, const int32_t* ids, const int32_t* offsets, int32_t B,
                  int64_t* unique_keys, int64_t* seg_offsets, int64_t* sorted_bags,
                  int64_t* n_valid) {
  const int32_t F = c->num_features;
  int64_t nnz = offsets[(int64_t)F * B];
  int64_t* base = table_bases(c);
  occ_t* v = (occ_t*)malloc(sizeof(occ_t) * (size_t)(nnz > 0 ? nnz : 1));
  int64_t n = 0;
  for (int32_t f = 0; f < F; ++f)
    for (int32_t b = 0; b < B; ++b) {
      int64_t bag = (int64_t)f * B + b;
      for (int32_t j = offsets[bag]; j < offsets[bag + 1]; ++j) {
        int64_t key = row_key(c, base, f, ids[j]);
        if (key < 0) continue;
        v[n].key = key; v[n].occ = j; v[n].bag = bag; ++n;
      }
    }
  sort_occ(v, n);
  int64_t U = 0;
  for (int64_t k = 0; k < n; ++k) {
    if (k == 0 || v[k].key != v[k - 1].key) {
      unique_keys[U] = v[k].key;
      seg_offsets[U] = k;
      ++U;
    }
    sorted_bags[k] = v[k].bag;
  }
  seg_offsets[U] = n;
  *n_valid = n;
  free(v);
  free(base);
  return U;
}

/* ------------------------------------------------------------------------- */
/* a6 segment-reduce                                                          */
/* ------------------------------------------------------------------------- */

void ora_segment_reduce(const ora_cfg* c, const int32_t* offsets, int32_t B, int64_t U,
                        const int64_t* seg_offsets, const int64_t* sorted_bags,
                        const float* grad, float* G) {
  const int32_t D = c->dim, F = c->num_features;
#pragma omp parallel
  {
    double* acc = (double*)malloc(sizeof(double) * (size_t)D);
#pragma omp for schedule(dynamic, 256)
    for (int64_t u = 0; u < U; ++u) {
      for (int32_t d = 0; d < D; ++d) acc[d] = 0.0;
      for (int64_t k = seg_offsets[u]; k < seg_offsets[u + 1]; ++k) {
        int64_t bag = sorted_bags[k];
        int64_t f = bag / B, b = bag % B;
        const float* g = grad + (b * F + f) * D;
        if (c->pooling == 1) {
          int32_t L = offsets[bag + 1] - offsets[bag];
          double inv = 1.0 / (double)L;
          for (int32_t d = 0; d < D; ++d) acc[d] = acc[d] + (double)g[d] * inv;
        } else {
          for (int32_t d = 0; d < D; ++d) acc[d] = acc[d] + (double)g[d];
        }
      }
      for (int32_t d = 0; d < D; ++d) G[u * D + d] = (float)acc[d];
    }
    free(acc);
  }
}

/* ------------------------------------------------------------------------- */
/* a7 global norm and clip factor                                             */
/* ------------------------------------------------------------------------- */

double ora_sq_norm(const float* G, int64_t U, int32_t dim, double extra) {
  double S = 0.0;
  for (int64_t u = 0; u < U; ++u)
    for (int32_t d = 0; d < dim; ++d) {
      double x = (double)G[u * dim + d];
      S = S + x * x;
    }
  return S + extra;
}

float ora_clip_factor(double S, float max_norm, int* nonfinite) {
  *nonfinite = 0;
  if (!isfinite(S)) { *nonfinite = 1; return 0.0f; }
  double n = sqrt(S);
  return (n > (double)max_norm) ? (float)((double)max_norm / n) : 1.0f;
}

void ora_clip(const float* G, int64_t n, float c, float* g) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) g[i] = G[i] * c;
}

/* ------------------------------------------------------------------------- */
/* a8 sparse AdaGrad on touched rows                                          */
/* ------------------------------------------------------------------------- */

void ora_adagrad_rowwise(float* W, float* A, const int64_t* keys, int64_t U,
                         const float* g, int32_t dim, float lr, float eps) {
#pragma omp parallel for schedule(static)
  for (int64_t u = 0; u < U; ++u) {
    int64_t r = keys[u];
    const float* gu = g + u * dim;
    double ss = 0.0;
    for (int32_t d = 0; d < dim; ++d) ss = ss + (double)gu[d] * (double)gu[d];
    float s = (float)(ss / (double)dim);
    float a = A[r] + s;
    A[r] = a;
    float den = sqrtf(a) + eps;
    float mult = lr / den;
    float* w = W + r * dim;
    for (int32_t d = 0; d < dim; ++d) w[d] = w[d] - mult * gu[d];
  }
}

void ora_adagrad_elementwise(float* W, float* A, const int64_t* keys, int64_t U,
                             const float* g, int32_t dim, float lr, float eps) {
#pragma omp parallel for schedule(static)
  for (int64_t u = 0; u < U; ++u) {
    int64_t r = keys[u];
    const float* gu = g + u * dim;
    float* w = W + r * dim;
    float* a = A + r * dim;
    for (int32_t d = 0; d < dim; ++d) {
      float sq = gu[d] * gu[d];
      float an = a[d] + sq;
      a[d] = an;
      float den = sqrtf(an) + eps;
      float step = (-lr * gu[d]) / den;
      w[d] = w[d] + step;
    }
  }
}

/* ------------------------------------------------------------------------- */
/* a9 middle-max quantization                                                 */
/* ------------------------------------------------------------------------- */

int32_t ora_quantize_row(const float* x, int32_t dim, int8_t* codes, float* middle, float* scale) {
  for (int32_t d = 0; d < dim; ++d)
    if (!isfinite(x[d])) {
      for (int32_t e = 0; e < dim; ++e) codes[e] = 0;
      *middle = 0.0f; *scale = 0.0f;
      return 1;
    }
  float mn = x[0], mx = x[0];
  for (int32_t d = 1; d < dim; ++d) {
    if (x[d] < mn) mn = x[d];
    if (x[d] > mx) mx = x[d];
  }
  if (mx == mn) {
    *middle = mx; *scale = 0.0f;
    for (int32_t d = 0; d < dim; ++d) codes[d] = 0;
    return 0;
  }
  /* X^middle = (X^max * 2^(b-1) + X^min * (2^(b-1) - 1)) / (2^b - 1), b = 8 */
  float hi = mx * 128.0f;
  float lo = mn * 127.0f;
  float mid = (hi + lo) / 255.0f;
  /* X^scale = (X^max - X^min) / (2^b - 1) */
  float sc = (mx - mn) / 255.0f;
  *middle = mid; *scale = sc;
  for (int32_t d = 0; d < dim; ++d) {
    if (sc == 0.0f) { codes[d] = 0; continue; }
    /* X^int = round((X - X^middle) / X^scale), half away from zero, saturated */
    float q = (x[d] - mid) / sc;
    float r = roundf(q);
    if (r < -128.0f) r = -128.0f;
    if (r > 127.0f) r = 127.0f;
    codes[d] = (int8_t)r;
  }
  return 0;
}

int64_t ora_quantize_mm8(const float* X, int64_t rows, int32_t dim, int8_t* codes,
                         float* middle, float* scale) {
  int64_t bad = 0;
#pragma omp parallel for schedule(static) reduction(+ : bad)
  for (int64_t r = 0; r < rows; ++r)
    bad += ora_quantize_row(X + r * dim, dim, codes + r * dim, middle + r, scale + r);
  return bad;
}

/* ------------------------------------------------------------------------- */
/* a10 quantized-table pooled lookup                                          */
/* ------------------------------------------------------------------------- */

int64_t ora_forward_q8(const ora_cfg* c, const int8_t* codes, const float* middle,
                       const float* scale, const int32_t* ids, const int32_t* offsets,
                       int32_t B, float* out) {
  const int32_t D = c->dim, F = c->num_features;
  const int64_t nbags = (int64_t)F * B;
  int64_t invalid = 0;
  int64_t* base = table_bases(c);
#pragma omp parallel reduction(+ : invalid)
  {
    float* acc = (float*)malloc(sizeof(float) * (size_t)D);
#pragma omp for schedule(dynamic, 512)
    for (int64_t bag = 0; bag < nbags; ++bag) {
      int32_t f = (int32_t)(bag / B), b = (int32_t)(bag % B);
      int32_t lo = offsets[bag], hi = offsets[bag + 1];
      for (int32_t d = 0; d < D; ++d) acc[d] = 0.0f;
      for (int32_t j = lo; j < hi; ++j) {
        int64_t key = row_key(c, base, f, ids[j]);
        if (key < 0) { ++invalid; continue; }
        const int8_t* q = codes + key * D;
        for (int32_t d = 0; d < D; ++d) {
          float v = fmaf((float)q[d], scale[key], middle[key]); /* middle + int * scale */
          acc[d] = acc[d] + v;
        }
      }
      if (c->pooling == 1) {
        int32_t L = hi - lo;
        for (int32_t d = 0; d < D; ++d) acc[d] = (L > 0) ? acc[d] / (float)L : 0.0f;
      }
      float* o = out + ((int64_t)b * F + f) * D;
      for (int32_t d = 0; d < D; ++d) o[d] = acc[d];
    }
    free(acc);
  }
  free(base);
  return invalid;
}

/* ------------------------------------------------------------------------- */
/* one whole training step                                                    */
/* ------------------------------------------------------------------------- */

int32_t ora_train_step(const ora_cfg* c, float* W, float* A, int32_t adagrad_mode,
                       const int32_t* ids, const int32_t* offsets, int32_t B,
                       const float* grad, float lr, float eps, float max_norm,
                       double extra_sq_norm, float* out, double* S_out, float* c_out,
                       int64_t* U_out) {
  const int32_t D = c->dim;
  int64_t nnz = offsets[(int64_t)c->num_features * B];
  size_t n1 = (size_t)(nnz > 0 ? nnz : 1);
  if (out) ora_forward(c, W, ids, offsets, B, out);
  int64_t* keys = (int64_t*)malloc(sizeof(int64_t) * n1);
  int64_t* segs = (int64_t*)malloc(sizeof(int64_t) * (n1 + 1));
  int64_t* bags = (int64_t*)malloc(sizeof(int64_t) * n1);
  int64_t n_valid = 0;
  int64_t U = ora_dedup(c, ids, offsets, B, keys, segs, bags, &n_valid);
  float* G = (float*)malloc(sizeof(float) * (size_t)(U > 0 ? U : 1) * D);
  ora_segment_reduce(c, offsets, B, U, segs, bags, grad, G);
  double S = ora_sq_norm(G, U, D, extra_sq_norm);
  int nonfinite = 0;
  float cf = ora_clip_factor(S, max_norm, &nonfinite);
  if (S_out) *S_out = S;
  if (c_out) *c_out = cf;
  if (U_out) *U_out = U;
  if (!nonfinite) {
    ora_clip(G, U * D, cf, G);
    if (adagrad_mode == 0) ora_adagrad_rowwise(W, A, keys, U, G, D, lr, eps);
    else ora_adagrad_elementwise(W, A, keys, U, G, D, lr, eps);
  }
  free(keys); free(segs); free(bags); free(G);
  return nonfinite ? 1 : 0;
}

/* ------------------------------------------------------------------------------------ */
/* NEXT-1: MurmurHash3 x64-128 (Austin Appleby's public-domain algorithm, written out from
 * its definition: 16-byte blocks mixed into h1/h2 with constants c1, c2, a tail of 0..15
 * bytes, then the length and the 64-bit finalizer fmix64).                              */
static uint64_t rotl64(uint64_t x, int r) { return (x << r) | (x >> (64 - r)); }
static uint64_t fmix64(uint64_t k) {
  k ^= k >> 33;
  k *= 0xff51afd7ed558ccdULL;
  k ^= k >> 33;
  k *= 0xc4ceb9fe1a85ec53ULL;
  k ^= k >> 33;
  return k;
}
static uint64_t load_le64(const uint8_t* p) {
  uint64_t v = 0;
  for (int i = 7; i >= 0; --i) v = (v << 8) | p[i];
  return v;
}

void ora_murmur3_x64_128(const uint8_t* key, int64_t len, uint32_t seed, uint64_t out[2]) {
  const uint64_t c1 = 0x87c37b91114253d5ULL, c2 = 0x4cf5ad432745937fULL;
  uint64_t h1 = seed, h2 = seed;
  const int64_t nblocks = len / 16;
  for (int64_t i = 0; i < nblocks; ++i) {
    uint64_t k1 = load_le64(key + 16 * i), k2 = load_le64(key + 16 * i + 8);
    k1 *= c1; k1 = rotl64(k1, 31); k1 *= c2; h1 ^= k1;
    h1 = rotl64(h1, 27); h1 += h2; h1 = h1 * 5 + 0x52dce729;
    k2 *= c2; k2 = rotl64(k2, 33); k2 *= c1; h2 ^= k2;
    h2 = rotl64(h2, 31); h2 += h1; h2 = h2 * 5 + 0x38495ab5;
  }
  const uint8_t* tail = key + 16 * nblocks;
  const int rem = (int)(len & 15);
  uint64_t k1 = 0, k2 = 0;
  for (int i = rem - 1; i >= 8; --i) k2 = (k2 << 8) | tail[i];  /* bytes 8..14 */
  if (rem > 8) { k2 *= c2; k2 = rotl64(k2, 33); k2 *= c1; h2 ^= k2; }
  for (int i = (rem < 8 ? rem : 8) - 1; i >= 0; --i) k1 = (k1 << 8) | tail[i];  /* 0..7 */
  if (rem > 0) { k1 *= c1; k1 = rotl64(k1, 31); k1 *= c2; h1 ^= k1; }
  h1 ^= (uint64_t)len; h2 ^= (uint64_t)len;
  h1 += h2; h2 += h1;
  h1 = fmix64(h1); h2 = fmix64(h2);
  h1 += h2; h2 += h1;
  out[0] = h1;
  out[1] = h2;
}

void ora_hash_ids(const uint8_t* bytes, const int64_t* str_off, int64_t n, uint64_t* h) {
  for (int64_t i = 0; i < n; ++i) {
    uint64_t d[2];
    ora_murmur3_x64_128(bytes + str_off[i], str_off[i + 1] - str_off[i], 0u, d);
    h[i] = d[0];
  }
}

void ora_qr_expand(const uint64_t* h, const int32_t* offsets, int64_t nbags, int64_t nnz,
                   int32_t R, int64_t Q, int32_t dual, int32_t* ids_out, int32_t* offsets_out) {
  const int k = dual ? 4 : 2;
  for (int64_t b = 0; b <= nbags; ++b) offsets_out[b] = k * offsets[b];
  for (int64_t i = 0; i < nnz; ++i) {
    const uint32_t nB = (uint32_t)(h[i] & 0xffffffffULL);  /* bitcast: low half  = B */
    const uint32_t nC = (uint32_t)(h[i] >> 32);            /*          high half = C */
    ids_out[k * i + 0] = (int32_t)((int64_t)(nB / (uint32_t)R) % Q);
    ids_out[k * i + 1] = (int32_t)(Q + (int64_t)(nB % (uint32_t)R));
    if (dual) {
      ids_out[k * i + 2] = (int32_t)(Q + R + (int64_t)(nC / (uint32_t)R) % Q);
      ids_out[k * i + 3] = (int32_t)(2 * Q + R + (int64_t)(nC % (uint32_t)R));
    }
  }
}

/* ------------------------------------------------------------------------------------ */
/* NEXT-4: min-max row-wise 8-bit quantization (oracle.h)                                 */
int32_t ora_quantize_row_minmax(const float* x, int32_t dim, uint8_t* codes, float* mn_out,
                                float* scale) {
  for (int32_t d = 0; d < dim; ++d)
    if (!isfinite(x[d])) {
      for (int32_t e = 0; e < dim; ++e) codes[e] = 0;
      *mn_out = 0.0f; *scale = 0.0f;
      return 1;
    }
  float mn = x[0], mx = x[0];
  for (int32_t d = 1; d < dim; ++d) {
    if (x[d] < mn) mn = x[d];
    if (x[d] > mx) mx = x[d];
  }
  *mn_out = (mx == mn) ? mx : mn;
  if (mx == mn) {
    *scale = 0.0f;
    for (int32_t d = 0; d < dim; ++d) codes[d] = 0;
    return 0;
  }
  float sc = (mx - mn) / 255.0f; /* X^scale = (X^max - X^min) / (2^b - 1) */
  *scale = sc;
  for (int32_t d = 0; d < dim; ++d) {
    if (sc == 0.0f) { codes[d] = 0; continue; }
    float q = (x[d] - mn) / sc;   /* X^int = round((X - X^min) / X^scale) */
    float r = roundf(q);
    if (r < 0.0f) r = 0.0f;
    if (r > 255.0f) r = 255.0f;
    codes[d] = (uint8_t)r;
  }
  return 0;
}

int64_t ora_quantize_minmax(const float* X, int64_t rows, int32_t dim, uint8_t* codes,
                            float* mn, float* scale) {
  int64_t bad = 0;
  for (int64_t r = 0; r < rows; ++r)
    bad += ora_quantize_row_minmax(X + r * dim, dim, codes + r * dim, mn + r, scale + r);
  return bad;
}

int64_t ora_forward_q8_minmax(const ora_cfg* c, const uint8_t* codes, const float* mn,
                              const float* scale, const int32_t* ids, const int32_t* offsets,
                              int32_t B, float* out) {
  const int32_t D = c->dim, F = c->num_features;
  const int64_t nbags = (int64_t)F * B;
  int64_t invalid = 0;
  int64_t* base = table_bases(c);
#pragma omp parallel reduction(+ : invalid)
  {
    float* acc = (float*)malloc(sizeof(float) * (size_t)D);
#pragma omp for schedule(dynamic, 512)
    for (int64_t bag = 0; bag < nbags; ++bag) {
      int32_t f = (int32_t)(bag / B), b = (int32_t)(bag % B);
      int32_t lo = offsets[bag], hi = offsets[bag + 1];
      for (int32_t d = 0; d < D; ++d) acc[d] = 0.0f;
      for (int32_t j = lo; j < hi; ++j) {
        int64_t key = row_key(c, base, f, ids[j]);
        if (key < 0) { ++invalid; continue; }
        const uint8_t* q = codes + key * D;
        for (int32_t d = 0; d < D; ++d) acc[d] = acc[d] + fmaf((float)q[d], scale[key], mn[key]);
      }
      if (c->pooling == 1) {
        int32_t L = hi - lo;
        for (int32_t d = 0; d < D; ++d) acc[d] = (L > 0) ? acc[d] / (float)L : 0.0f;
      }
      float* o = out + ((int64_t)b * F + f) * D;
      for (int32_t d = 0; d < D; ++d) o[d] = acc[d];
    }
    free(acc);
  }
  free(base);
  return invalid;
}

/* ------------------------------------------------------------------------------------ */
/* NEXT-3: incremental training (oracle.h)                                                */
void ora_cold_weight_init(const float* w0, const float* w1, int64_t n, float alpha, float* w) {
  const float beta = 1.0f - alpha;
  for (int64_t i = 0; i < n; ++i) w[i] = alpha * w0[i] + beta * w1[i];
}

double ora_fim_penalty(const float* W, int64_t n, const float* w0, const float* H0,
                       const float* w1, const float* H1, float lambda, float alpha) {
  double s0 = 0.0, s1 = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    if (w0 && H0) { const double d = (double)W[i] - (double)w0[i]; s0 += (double)H0[i] * d * d; }
    if (w1 && H1) { const double d = (double)W[i] - (double)w1[i]; s1 += (double)H1[i] * d * d; }
  }
  return (double)lambda / 2.0 * ((double)alpha * s0 + (1.0 - (double)alpha) * s1);
}

void ora_fim_penalty_grad(const float* W, const int64_t* keys, int64_t U, int32_t dim,
                          const float* w0, const float* H0, const float* w1, const float* H1,
                          float lambda, float alpha, float* G) {
  const float beta = 1.0f - alpha;
  for (int64_t u = 0; u < U; ++u)
    for (int32_t d = 0; d < dim; ++d) {
      const int64_t i = keys[u] * dim + d;
      float t0 = 0.0f, t1 = 0.0f;
      if (w0 && H0) t0 = alpha * (H0[i] * (W[i] - w0[i]));
      if (w1 && H1) t1 = beta * (H1[i] * (W[i] - w1[i]));
      const float pen = lambda * (t0 + t1);
      G[u * dim + d] = G[u * dim + d] + pen;
    }
}

int32_t ora_train_step_fim(const ora_cfg* c, float* W, float* A, int32_t adagrad_mode,
                           const int32_t* ids, const int32_t* offsets, int32_t B,
                           const float* grad, float lr, float eps, float max_norm,
                           double extra_sq_norm, const float* w0, const float* H0,
                           const float* w1, const float* H1, float lambda, float alpha,
                           double* S_out, float* c_out) {
  const int32_t D = c->dim;
  int64_t nnz = offsets[(int64_t)c->num_features * B];
  size_t n1 = (size_t)(nnz > 0 ? nnz : 1);
  int64_t* keys = (int64_t*)malloc(sizeof(int64_t) * n1);
  int64_t* segs = (int64_t*)malloc(sizeof(int64_t) * (n1 + 1));
  int64_t* bags = (int64_t*)malloc(sizeof(int64_t) * n1);
  int64_t n_valid = 0;
  int64_t U = ora_dedup(c, ids, offsets, B, keys, segs, bags, &n_valid);
  float* G = (float*)malloc(sizeof(float) * (size_t)(U > 0 ? U : 1) * D);
  ora_segment_reduce(c, offsets, B, U, segs, bags, grad, G);
  ora_fim_penalty_grad(W, keys, U, D, w0, H0, w1, H1, lambda, alpha, G);
  double S = ora_sq_norm(G, U, D, extra_sq_norm);
  int nonfinite = 0;
  float cf = ora_clip_factor(S, max_norm, &nonfinite);
  if (S_out) *S_out = S;
  if (c_out) *c_out = cf;
  if (!nonfinite) {
    ora_clip(G, U * D, cf, G);
    if (adagrad_mode == 0) ora_adagrad_rowwise(W, A, keys, U, G, D, lr, eps);
    else ora_adagrad_elementwise(W, A, keys, U, G, D, lr, eps);
  }
  free(keys); free(segs); free(bags); free(G);
  return nonfinite ? 1 : 0;
}
