/*
 * rsot_oracle.c -- CPU restatement of the reference RSOT dual evaluator.
 * TEST INFRASTRUCTURE ONLY (see rsot_oracle.h).  Compile with
 * -ffp-contract=off so every product and sum rounds exactly as the x86
 * reference build does (the reference object has no FMA instructions).
 */
#define _GNU_SOURCE
#include "rsot_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

static _Thread_local const char* g_last_error = "";
const char* oracle_last_error(void) { return g_last_error; }

/* ---------------------------------------------------------------------- */
/* point.hpp:35-40: dx*dx + dy*dy + dz*dz, evaluated left to right. */
static inline double sqdist(const double* a, const double* b) {
  const double dx = a[0] - b[0];
  const double dy = a[1] - b[1];
  const double dz = a[2] - b[2];
  return dx * dx + dy * dy + dz * dz;
}

uint64_t oracle_candidate_hash_term(uint64_t j) {
  uint64_t z = j + 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

/* ---------------------------------------------------------------------- */
/* Exact uniform grid (stands in for the R*-tree of spatial_index.cpp).    */
struct oracle_grid {
  size_t n;
  double* pts;     /* n*3, copy of the input (spatial_index.cpp:40) */
  double lo[3];
  double h[3];     /* cell side per dim */
  int dims[3];     /* cells per dim */
  size_t* start;   /* ncells+1 */
  uint64_t* idx;   /* point indices, grouped by cell, ascending in a cell */
};

static int cell_coord(const oracle_grid* g, int d, double v) {
  double t = (v - g->lo[d]) / g->h[d];
  if (!(t >= 0.0)) return 0; /* also catches NaN */
  if (t >= (double)g->dims[d]) return g->dims[d] - 1;
  return (int)t;
}

oracle_grid* oracle_grid_create(const double* xyz, size_t n) {
  if (n == 0) {
    g_last_error = "spatial index: empty point set";
    return NULL;
  }
  oracle_grid* g = (oracle_grid*)calloc(1, sizeof(oracle_grid));
  if (!g) return NULL;
  g->n = n;
  g->pts = (double*)malloc(sizeof(double) * 3 * n);
  memcpy(g->pts, xyz, sizeof(double) * 3 * n);
  double hi[3];
  for (int d = 0; d < 3; ++d) g->lo[d] = hi[d] = xyz[d];
  for (size_t i = 1; i < n; ++i)
    for (int d = 0; d < 3; ++d) {
      const double v = xyz[3 * i + d];
      if (v < g->lo[d]) g->lo[d] = v;
      if (v > hi[d]) hi[d] = v;
    }
  /* Aim for about two points per cell over the active dimensions. */
  int active = 0;
  double vol = 1.0;
  for (int d = 0; d < 3; ++d)
    if (hi[d] > g->lo[d]) {
      ++active;
      vol *= hi[d] - g->lo[d];
    }
  double side = 1.0;
  if (active > 0) {
    const double cells = n > 2 ? (double)n / 2.0 : 1.0;
    side = pow(vol / cells, 1.0 / active);
  }
  for (int d = 0; d < 3; ++d) {
    const double ext = hi[d] - g->lo[d];
    if (ext > 0.0) {
      double nd = floor(ext / side) + 1.0;
      if (nd > 2048.0) nd = 2048.0;
      g->dims[d] = (int)nd;
      g->h[d] = ext / (double)g->dims[d] * (1.0 + 1e-12);
    } else {
      g->dims[d] = 1;
      g->h[d] = 1.0;
    }
  }
  const size_t ncell = (size_t)g->dims[0] * g->dims[1] * g->dims[2];
  g->start = (size_t*)calloc(ncell + 1, sizeof(size_t));
  g->idx = (uint64_t*)malloc(sizeof(uint64_t) * n);
  size_t* cell_of = (size_t*)malloc(sizeof(size_t) * n);
  for (size_t i = 0; i < n; ++i) {
    const int cx = cell_coord(g, 0, xyz[3 * i]);
    const int cy = cell_coord(g, 1, xyz[3 * i + 1]);
    const int cz = cell_coord(g, 2, xyz[3 * i + 2]);
    cell_of[i] = ((size_t)cz * g->dims[1] + cy) * g->dims[0] + cx;
    g->start[cell_of[i] + 1]++;
  }
  for (size_t c = 0; c < ncell; ++c) g->start[c + 1] += g->start[c];
  size_t* fill = (size_t*)malloc(sizeof(size_t) * ncell);
  memcpy(fill, g->start, sizeof(size_t) * ncell);
  for (size_t i = 0; i < n; ++i) g->idx[fill[cell_of[i]]++] = i; /* stable */
  free(fill);
  free(cell_of);
  return g;
}

void oracle_grid_destroy(oracle_grid* g) {
  if (!g) return;
  free(g->pts);
  free(g->start);
  free(g->idx);
  free(g);
}

size_t oracle_grid_size(const oracle_grid* g) { return g ? g->n : 0; }

static int cmp_u64(const void* a, const void* b) {
  const uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
  return (x > y) - (x < y);
}

/* spatial_index.cpp:47-61: strict d^2 < r*r, then sort ascending. */
static size_t ball_query_into(const oracle_grid* g, const double* c,
                              double radius, uint64_t** buf, size_t* cap) {
  if (!(radius > 0.0)) return 0;
  const double r2 = radius * radius;
  int lo[3], hi[3];
  for (int d = 0; d < 3; ++d) {
    lo[d] = cell_coord(g, d, c[d] - radius) - 1;
    hi[d] = cell_coord(g, d, c[d] + radius) + 1;
    if (lo[d] < 0) lo[d] = 0;
    if (hi[d] > g->dims[d] - 1) hi[d] = g->dims[d] - 1;
  }
  size_t count = 0;
  for (int z = lo[2]; z <= hi[2]; ++z)
    for (int y = lo[1]; y <= hi[1]; ++y) {
      const size_t row = ((size_t)z * g->dims[1] + y) * g->dims[0];
      const size_t b = g->start[row + lo[0]], e = g->start[row + hi[0] + 1];
      for (size_t k = b; k < e; ++k) {
        const uint64_t j = g->idx[k];
        if (sqdist(c, g->pts + 3 * j) < r2) {
          if (count == *cap) {
            *cap = *cap ? 2 * *cap : 256;
            *buf = (uint64_t*)realloc(*buf, sizeof(uint64_t) * *cap);
          }
          (*buf)[count++] = j;
        }
      }
    }
  qsort(*buf, count, sizeof(uint64_t), cmp_u64);
  return count;
}

size_t oracle_grid_ball_query(const oracle_grid* g, const double center[3],
                              double radius, uint64_t* out, size_t cap) {
  uint64_t* buf = NULL;
  size_t bcap = 0;
  const size_t n = ball_query_into(g, center, radius, &buf, &bcap);
  if (out)
    memcpy(out, buf, sizeof(uint64_t) * (n < cap ? n : cap));
  free(buf);
  return n;
}

/* spatial_index.cpp:70-84 semantics: argmin of (d^2, j) lexicographically.
 * Exact search by expanding rings of cells around the center's cell. */
uint64_t oracle_grid_nearest(const oracle_grid* g, const double c[3]) {
  int cc[3];
  for (int d = 0; d < 3; ++d) cc[d] = cell_coord(g, d, c[d]);
  double best_d2 = INFINITY;
  uint64_t best = g->n;
  const int maxk = g->dims[0] + g->dims[1] + g->dims[2];
  for (int k = 0; k <= maxk; ++k) {
    int lo[3], hi[3], full[3];
    for (int d = 0; d < 3; ++d) {
      lo[d] = cc[d] - k;
      hi[d] = cc[d] + k;
      full[d] = 0;
      if (lo[d] < 0) lo[d] = 0;
      if (hi[d] > g->dims[d] - 1) hi[d] = g->dims[d] - 1;
    }
    for (int z = lo[2]; z <= hi[2]; ++z)
      for (int y = lo[1]; y <= hi[1]; ++y)
        for (int x = lo[0]; x <= hi[0]; ++x) {
          /* only cells on the ring shell (Chebyshev distance == k) */
          const int dz = abs(z - cc[2]), dy = abs(y - cc[1]), dx = abs(x - cc[0]);
          int m = dx > dy ? dx : dy;
          m = m > dz ? m : dz;
          if (m != k) continue;
          const size_t cell = ((size_t)z * g->dims[1] + y) * g->dims[0] + x;
          for (size_t t = g->start[cell]; t < g->start[cell + 1]; ++t) {
            const uint64_t j = g->idx[t];
            const double d2 = sqdist(c, g->pts + 3 * j);
            if (d2 < best_d2 || (d2 == best_d2 && j < best)) {
              best_d2 = d2;
              best = j;
            }
          }
        }
    /* Distance from c to the outside of the scanned box, over the sides
     * that still have unscanned cells. */
    double margin = INFINITY;
    int any_left = 0;
    for (int d = 0; d < 3; ++d) {
      if (cc[d] - k > 0) {
        const double face = g->lo[d] + (double)(cc[d] - k) * g->h[d];
        const double m = c[d] - face;
        if (m < margin) margin = m;
        any_left = 1;
      }
      if (cc[d] + k < g->dims[d] - 1) {
        const double face = g->lo[d] + (double)(cc[d] + k + 1) * g->h[d];
        const double m = face - c[d];
        if (m < margin) margin = m;
        any_left = 1;
      }
      (void)full;
    }
    if (!any_left) break;
    if (best < g->n && margin > 0.0 && margin * margin > best_d2 * (1.0 + 1e-9) + 1e-300)
      break;
  }
  return best;
}

/* ---------------------------------------------------------------------- */
/* evaluate.cpp:86-174                                                    */

typedef struct {
  double J, D;
  double* g;
  uint64_t pairs, empty;
  int ran;
} partial_t;

typedef struct {
  size_t lo, hi;
  size_t n;
  const double *ax, *am, *ty, *psi, *log_nu;
  double eps, radius;
  int truncated;
  const oracle_grid* grid;
  partial_t* part;
  uint32_t* cnt;
  uint64_t* hash;
  double* log_s;
} job_t;

static void* eval_block(void* arg) {
  job_t* jb = (job_t*)arg;
  partial_t* part = jb->part;
  const size_t n = jb->n;
  part->g = (double*)calloc(n, sizeof(double)); /* evaluate.cpp:111 */
  part->ran = 1;
  uint64_t* cand = NULL;
  size_t ccap = 0;
  double* expo = NULL;
  size_t ecap = 0;
  if (!jb->truncated) {
    ccap = n;
    cand = (uint64_t*)malloc(sizeof(uint64_t) * n);
    for (size_t j = 0; j < n; ++j) cand[j] = j; /* :119-121 */
  }
  for (size_t q = jb->lo; q < jb->hi; ++q) {
    const double* x = jb->ax + 3 * q;
    const double mq = jb->am[q];
    size_t nc;
    if (!jb->truncated) {
      nc = n;
    } else {
      nc = ball_query_into(jb->grid, x, jb->radius, &cand, &ccap); /* :122-123 */
    }
    int was_empty = 0;
    if (nc == 0) { /* :129-132 */
      ++part->empty;
      was_empty = 1;
      if (ccap == 0) {
        ccap = 256;
        cand = (uint64_t*)malloc(sizeof(uint64_t) * ccap);
      }
      cand[0] = oracle_grid_nearest(jb->grid, x);
      nc = 1;
    }
    part->pairs += nc; /* :133 */
    if (nc > ecap) {
      ecap = nc;
      expo = (double*)realloc(expo, sizeof(double) * ecap);
    }
    double emax = -INFINITY; /* :136-142 */
    for (size_t i = 0; i < nc; ++i) {
      const uint64_t j = cand[i];
      const double c = 0.5 * sqdist(x, jb->ty + 3 * j); /* cost.hpp:26 */
      expo[i] = (jb->psi[j] - c) / jb->eps + jb->log_nu[j];
      emax = (emax < expo[i]) ? expo[i] : emax; /* std::max */
    }
    double sum = 0.0; /* :143-147 */
    for (size_t i = 0; i < nc; ++i) {
      expo[i] = exp(expo[i] - emax);
      sum += expo[i];
    }
    const double log_S = emax + log(sum); /* :148-150 */
    part->J += jb->eps * log_S * mq;
    part->D += mq * exp(-log_S);
    const double scale = mq / sum; /* :151-153 */
    for (size_t i = 0; i < nc; ++i) part->g[cand[i]] += expo[i] * scale;
    if (jb->cnt) jb->cnt[q] = (uint32_t)nc;
    if (jb->hash) {
      uint64_t h = 0;
      for (size_t i = 0; i < nc; ++i) h += oracle_candidate_hash_term(cand[i]);
      jb->hash[q] = h;
    }
    if (jb->log_s) jb->log_s[q] = log_S;
    (void)was_empty;
  }
  free(cand);
  free(expo);
  return NULL;
}

int oracle_evaluate_dual(size_t nq, const double* ax, const double* am,
                         size_t n, const double* ty, const double* nu,
                         const double* psi, double eps, double cutoff,
                         int workers, const oracle_grid* grid, double* g_out,
                         oracle_scalars* out, uint32_t* cnt, uint64_t* hash,
                         double* log_s) {
  /* :90-93 and potential.hpp:42-46 */
  for (size_t j = 0; j < n; ++j)
    if (!isfinite(psi[j])) {
      g_last_error = "potential has non-finite entries";
      return ORACLE_INVALID_ARGUMENT;
    }
  const int truncated = isfinite(cutoff); /* :95-99 */
  const double radius = oracle_ball_radius(cutoff);
  oracle_grid* own = NULL;
  if (!grid && nq > 0 && (truncated || 1)) {
    /* The reference always has an index (its ctor throws on empty). */
    own = oracle_grid_create(ty, n);
    if (!own) return ORACLE_INVALID_ARGUMENT;
    grid = own;
  }
  double* log_nu = (double*)malloc(sizeof(double) * (n ? n : 1));
  for (size_t j = 0; j < n; ++j) log_nu[j] = log(nu[j]); /* :101-103 */

  /* parallel.hpp:14-31 */
  int w = workers < 1 ? 1 : workers;
  size_t nthreads = 1, chunk = nq;
  if (!(w <= 1 || nq < 2)) {
    nthreads = (size_t)w < nq ? (size_t)w : nq;
    chunk = (nq + nthreads - 1) / nthreads;
  }
  partial_t* parts = (partial_t*)calloc(nthreads, sizeof(partial_t));
  job_t* jobs = (job_t*)calloc(nthreads, sizeof(job_t));
  pthread_t* th = (pthread_t*)calloc(nthreads, sizeof(pthread_t));
  size_t launched = 0;
  for (size_t t = 0; t < nthreads; ++t) {
    size_t lo = t * chunk, hi = lo + chunk;
    if (hi > nq) hi = nq;
    if (nthreads == 1) {
      lo = 0;
      hi = nq;
    } else if (lo >= hi) {
      break;
    }
    job_t* jb = &jobs[t];
    jb->lo = lo;
    jb->hi = hi;
    jb->n = n;
    jb->ax = ax;
    jb->am = am;
    jb->ty = ty;
    jb->psi = psi;
    jb->log_nu = log_nu;
    jb->eps = eps;
    jb->radius = radius;
    jb->truncated = truncated;
    jb->grid = grid;
    jb->part = &parts[t];
    jb->cnt = cnt;
    jb->hash = hash;
    jb->log_s = log_s;
    ++launched;
  }
  if (launched == 1) {
    eval_block(&jobs[0]);
  } else {
    for (size_t t = 0; t < launched; ++t)
      pthread_create(&th[t], NULL, eval_block, &jobs[t]);
    for (size_t t = 0; t < launched; ++t) pthread_join(th[t], NULL);
  }
  /* :157-172, merge in worker order */
  double J = 0.0, D = 0.0;
  uint64_t pairs = 0, empty = 0;
  for (size_t j = 0; j < n; ++j) g_out[j] = 0.0;
  for (size_t t = 0; t < launched; ++t) {
    const partial_t* p = &parts[t];
    if (!p->ran || n == 0) continue;
    J += p->J;
    D += p->D;
    pairs += p->pairs;
    empty += p->empty;
    for (size_t j = 0; j < n; ++j) g_out[j] += p->g[j];
  }
  for (size_t j = 0; j < n; ++j) {
    J -= psi[j] * nu[j];
    g_out[j] -= nu[j];
  }
  out->J = J;
  out->D = D;
  out->candidate_pairs = pairs;
  out->empty_candidate_atoms = empty;
  out->atoms_visited = nq;
  for (size_t t = 0; t < launched; ++t) free(parts[t].g);
  free(parts);
  free(jobs);
  free(th);
  free(log_nu);
  oracle_grid_destroy(own);
  return ORACLE_OK;
}

/* solve.cpp:62-142, SqEuclidean cost, one worker (parallel_blocks with
 * workers = 1 runs the same loops in order). */
int oracle_softmax_refine(size_t n_coarse, const double* cy, const double* cnu,
                          const double* cpsi, size_t n_fine, const double* fy,
                          size_t nq, const double* ax, const double* am,
                          double eps, double cutoff, double* psi_out) {
  for (size_t j = 0; j < n_coarse; ++j)
    if (!isfinite(cpsi[j])) {
      g_last_error = "potential has non-finite entries";
      return ORACLE_INVALID_ARGUMENT;
    }
  const int truncated = isfinite(cutoff);
  double* log_nu = (double*)malloc(sizeof(double) * (n_coarse ? n_coarse : 1));
  for (size_t j = 0; j < n_coarse; ++j) log_nu[j] = log(cnu[j]);
  double* log_S = (double*)malloc(sizeof(double) * (nq ? nq : 1));
  double* expo = (double*)malloc(sizeof(double) * (n_coarse ? n_coarse : 1));
  size_t* cand = (size_t*)malloc(sizeof(size_t) * (n_coarse ? n_coarse : 1));
  for (size_t q = 0; q < nq; ++q) { /* :79-118 */
    const double* x = ax + 3 * q;
    size_t nc = 0;
    if (truncated) {
      for (size_t j = 0; j < n_coarse; ++j)
        if (0.5 * sqdist(x, cy + 3 * j) < cutoff) cand[nc++] = j;
      if (nc == 0) {
        size_t best = 0;
        double best_c = 0.5 * sqdist(x, cy);
        for (size_t j = 1; j < n_coarse; ++j) {
          const double c = 0.5 * sqdist(x, cy + 3 * j);
          if (c < best_c) {
            best_c = c;
            best = j;
          }
        }
        cand[nc++] = best;
      }
    } else {
      for (size_t j = 0; j < n_coarse; ++j) cand[nc++] = j;
    }
    double emax = -INFINITY;
    for (size_t i = 0; i < nc; ++i) {
      const size_t j = cand[i];
      expo[i] = (cpsi[j] - 0.5 * sqdist(x, cy + 3 * j)) / eps + log_nu[j];
      emax = (emax < expo[i]) ? expo[i] : emax;
    }
    double sum = 0.0;
    for (size_t i = 0; i < nc; ++i) sum += exp(expo[i] - emax);
    log_S[q] = emax + log(sum);
  }
  int rc = ORACLE_OK;
  for (size_t k = 0; k < n_fine; ++k) { /* :120-139 */
    const double* y = fy + 3 * k;
    double emax = -INFINITY;
    for (size_t q = 0; q < nq; ++q) {
      const double t = -(0.5 * sqdist(ax + 3 * q, y)) / eps - log_S[q] + log(am[q]);
      emax = (emax < t) ? t : emax;
    }
    double sum = 0.0;
    for (size_t q = 0; q < nq; ++q) {
      const double t = -(0.5 * sqdist(ax + 3 * q, y)) / eps - log_S[q] + log(am[q]);
      sum += exp(t - emax);
    }
    psi_out[k] = -eps * (emax + log(sum));
    if (!isfinite(psi_out[k])) rc = ORACLE_INVALID_ARGUMENT;
  }
  if (rc) g_last_error = "potential has non-finite entries";
  free(log_nu);
  free(log_S);
  free(expo);
  free(cand);
  return rc;
}

/* spatial_index.cpp:101-121 (SqEuclidean branch) */
int oracle_covering_cost(size_t nq, const double* ax, size_t n,
                         const double* ty, double* out) {
  if (nq == 0 || n == 0) {
    g_last_error = "covering cost: empty input";
    return ORACLE_INVALID_ARGUMENT;
  }
  oracle_grid* g = oracle_grid_create(ty, n);
  double c0 = 0.0;
  for (size_t q = 0; q < nq; ++q) {
    const uint64_t j = oracle_grid_nearest(g, ax + 3 * q);
    const double c = 0.5 * sqdist(ax + 3 * q, ty + 3 * j);
    c0 = (c0 < c) ? c : c0; /* std::max */
  }
  oracle_grid_destroy(g);
  *out = c0;
  return ORACLE_OK;
}

/* cost.hpp:38-42 */
double oracle_ball_radius(double cutoff) {
  if (cutoff < 0.0) return 0.0;
  return sqrt(2.0 * cutoff);
}

/* evaluate.cpp:22-25 */
double oracle_cutoff_pointwise(double psi_max, double nu_max, double eps,
                               double delta_thr) {
  return psi_max + eps * log(nu_max / delta_thr);
}

static double dmax(double a, double b) { return (a < b) ? b : a; }

/* evaluate.cpp:27-34 */
int oracle_cutoff_integrated(double psi_max, double covering, double cached_D,
                             double cached_absJ, double eps, double tau,
                             double* out) {
  const double absJ = dmax(cached_absJ, 1e-30);
  if (absJ <= 1e-30) {
    g_last_error = "functional estimate degenerate";
    return ORACLE_RUNTIME_ERROR;
  }
  const double c = psi_max + eps * log(eps * cached_D / (tau * absJ));
  *out = dmax(c, covering);
  return ORACLE_OK;
}

/* evaluate.cpp:36-43 */
int oracle_cutoff_geometric(double covering, double psi_range, double nu_min,
                            double cached_absJ, double eps, double tau,
                            double* out) {
  const double absJ = dmax(cached_absJ, 1e-30);
  if (absJ <= 1e-30) {
    g_last_error = "functional estimate degenerate";
    return ORACLE_RUNTIME_ERROR;
  }
  const double c =
      covering + psi_range + eps * log(eps / (nu_min * tau * absJ));
  *out = dmax(c, covering);
  return ORACLE_OK;
}

/* evaluate.cpp:45-49 */
double oracle_cutoff_bootstrap(double covering, double psi_range,
                               double nu_min, double eps, double tau) {
  const double c = covering + psi_range + eps * log(eps / (nu_min * tau));
  return dmax(c, covering);
}

/* ---- PlanView (proj/src/plan.cpp) ---------------------------------------
 * ctor (:12-59): candidate sets (all targets, or the ball query with the
 * nearest-target fallback) and log_S_q; target_marginals (:85-91);
 * all_conditional_barycenters (:123-140, unnormalised first moments and
 * tilde returned, plus the normalised barycentres); barycentric_map
 * (:142-156); modal_map (:158-182).  SqEuclidean, single worker. */
int oracle_plan_view(size_t nq, const double* ax, const double* am, size_t n,
                     const double* ty, const double* nu, const double* psi,
                     double eps, double cutoff, double* log_s_out,
                     uint64_t* count_out, double* marginal_out,
                     double* moment_out, double* bary_out, double* map_out,
                     uint64_t* modal_out, int64_t* starved_out) {
  for (size_t j = 0; j < n; ++j)
    if (!isfinite(psi[j])) {
      g_last_error = "potential has non-finite entries";
      return ORACLE_INVALID_ARGUMENT;
    }
  const int truncated = isfinite(cutoff);
  const double radius = oracle_ball_radius(cutoff);
  oracle_grid* grid = oracle_grid_create(ty, n); /* plan.cpp:31 */
  if (!grid) return ORACLE_INVALID_ARGUMENT;
  double* log_nu = (double*)malloc(sizeof(double) * (n ? n : 1));
  for (size_t j = 0; j < n; ++j) log_nu[j] = log(nu[j]);
  uint64_t* cand = (uint64_t*)malloc(sizeof(uint64_t) * (n ? n : 1));
  size_t ccap = n ? n : 1;
  double* expo = (double*)malloc(sizeof(double) * (n ? n : 1));
  if (marginal_out)
    for (size_t j = 0; j < n; ++j) marginal_out[j] = 0.0;
  if (moment_out)
    for (size_t j = 0; j < 3 * n; ++j) moment_out[j] = 0.0;
  for (size_t q = 0; q < nq; ++q) {
    const double* x = ax + 3 * q;
    size_t nc;
    if (!truncated) {
      nc = n;
      for (size_t j = 0; j < n; ++j) cand[j] = j;
    } else {
      nc = ball_query_into(grid, x, radius, &cand, &ccap);
    }
    if (nc == 0) {
      cand[0] = oracle_grid_nearest(grid, x);
      nc = 1;
    }
    double emax = -INFINITY; /* :47-57 */
    for (size_t i = 0; i < nc; ++i) {
      const uint64_t j = cand[i];
      expo[i] = (psi[j] - 0.5 * sqdist(x, ty + 3 * j)) / eps + log_nu[j];
      emax = (emax < expo[i]) ? expo[i] : emax;
    }
    double sum = 0.0;
    for (size_t i = 0; i < nc; ++i) sum += exp(expo[i] - emax);
    const double lS = emax + log(sum);
    if (log_s_out) log_s_out[q] = lS;
    if (count_out) count_out[q] = nc;
    /* plan_density (:70-83) recomputes e with std::log(weights[j]) */
    double t0 = 0.0, t1 = 0.0, t2 = 0.0;
    uint64_t best = n;
    double best_score = -INFINITY;
    for (size_t i = 0; i < nc; ++i) {
      const uint64_t j = cand[i];
      const double c = 0.5 * sqdist(x, ty + 3 * j);
      const double e = (psi[j] - c) / eps + log(nu[j]);
      const double p = exp(e - lS);
      const double w = p * am[q];
      if (marginal_out) marginal_out[j] += w;
      if (moment_out) {
        moment_out[3 * j] += w * x[0];
        moment_out[3 * j + 1] += w * x[1];
        moment_out[3 * j + 2] += w * x[2];
      }
      t0 += p * ty[3 * j];
      t1 += p * ty[3 * j + 1];
      t2 += p * ty[3 * j + 2];
      const double score = psi[j] - c + eps * log(nu[j]); /* :172-175 */
      if (score > best_score) {
        best_score = score;
        best = j;
      }
    }
    if (map_out) {
      map_out[3 * q] = t0;
      map_out[3 * q + 1] = t1;
      map_out[3 * q + 2] = t2;
    }
    if (modal_out) modal_out[q] = best;
  }
  if (starved_out) *starved_out = -1;
  if (bary_out && marginal_out && moment_out)
    for (size_t j = 0; j < n; ++j) { /* :134-139 */
      if (marginal_out[j] < 1e-30) {
        if (starved_out && *starved_out < 0) *starved_out = (int64_t)j;
        bary_out[3 * j] = bary_out[3 * j + 1] = bary_out[3 * j + 2] = 0.0;
        continue;
      }
      const double inv = 1.0 / marginal_out[j];
      for (int d = 0; d < 3; ++d) bary_out[3 * j + d] = inv * moment_out[3 * j + d];
    }
  free(log_nu);
  free(cand);
  free(expo);
  oracle_grid_destroy(grid);
  return ORACLE_OK;
}

/* ---- evaluate_dual for CostKind::SqGeodesicSphere ------------------------
 * evaluate.cpp:86-174 with cost.hpp:19-33: c = acos(clamp(x.y, -1, 1))^2,
 * a finite cutoff selects {j : c < cutoff} by a full scan (:124-128; no ball
 * radius for this cost), an empty set takes index.nearest (Euclidean, lowest
 * index on ties, :129-132).  Single worker (the reference's workers = 1). */
static double geo_cost(const double* x, const double* y) {
  const double d = (x[0] * y[0] + x[1] * y[1]) + x[2] * y[2];
  const double t = d < -1.0 ? -1.0 : (1.0 < d ? 1.0 : d);
  const double g = acos(t);
  return g * g;
}

int oracle_evaluate_dual_geodesic(size_t nq, const double* ax, const double* am, size_t n,
                                  const double* ty, const double* nu, const double* psi,
                                  double eps, double cutoff, double* g_out,
                                  oracle_scalars* out, uint32_t* cnt, double* log_s) {
  for (size_t j = 0; j < n; ++j)
    if (!isfinite(psi[j])) {
      g_last_error = "potential has non-finite entries";
      return ORACLE_INVALID_ARGUMENT;
    }
  oracle_grid* grid = oracle_grid_create(ty, n);
  if (!grid) return ORACLE_INVALID_ARGUMENT;
  const int truncated = isfinite(cutoff);
  double* log_nu = (double*)malloc(sizeof(double) * (n ? n : 1));
  for (size_t j = 0; j < n; ++j) log_nu[j] = log(nu[j]);
  uint64_t* cand = (uint64_t*)malloc(sizeof(uint64_t) * (n ? n : 1));
  double* expo = (double*)malloc(sizeof(double) * (n ? n : 1));
  double J = 0.0, D = 0.0;
  uint64_t pairs = 0, empty = 0;
  for (size_t j = 0; j < n; ++j) g_out[j] = 0.0;
  for (size_t q = 0; q < nq; ++q) {
    const double* x = ax + 3 * q;
    size_t nc = 0;
    for (size_t j = 0; j < n; ++j)
      if (!truncated || geo_cost(x, ty + 3 * j) < cutoff) cand[nc++] = j;
    if (nc == 0) {
      ++empty;
      cand[nc++] = oracle_grid_nearest(grid, x);
    }
    pairs += nc;
    double emax = -INFINITY;
    for (size_t i = 0; i < nc; ++i) {
      const uint64_t j = cand[i];
      expo[i] = (psi[j] - geo_cost(x, ty + 3 * j)) / eps + log_nu[j];
      emax = (emax < expo[i]) ? expo[i] : emax;
    }
    double sum = 0.0;
    for (size_t i = 0; i < nc; ++i) {
      expo[i] = exp(expo[i] - emax);
      sum += expo[i];
    }
    const double lS = emax + log(sum);
    J += eps * lS * am[q];
    D += am[q] * exp(-lS);
    const double scale = am[q] / sum;
    for (size_t i = 0; i < nc; ++i) g_out[cand[i]] += expo[i] * scale;
    if (cnt) cnt[q] = (uint32_t)nc;
    if (log_s) log_s[q] = lS;
  }
  for (size_t j = 0; j < n; ++j) {
    J -= psi[j] * nu[j];
    g_out[j] -= nu[j];
  }
  out->J = J;
  out->D = D;
  out->candidate_pairs = pairs;
  out->empty_candidate_atoms = empty;
  out->atoms_visited = nq;
  free(log_nu);
  free(cand);
  free(expo);
  oracle_grid_destroy(grid);
  return ORACLE_OK;
}
