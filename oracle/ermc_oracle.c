/*
 * ermc_oracle.c — TEST INFRASTRUCTURE ONLY. Plain-C restatement of the
 * reference ERMC solve path (see ermc_oracle.h for the file:line map).
 * Compiled with -ffp-contract=off so every add/mul/div rounds like the
 * reference's x86-64 build; libm (glibc) is the same library the reference
 * links, so results are expected bitwise (pinned in tests/test_oracle.py).
 */
#define _GNU_SOURCE
#include "ermc_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static const double kPi = 3.14159265358979323846;
static const double kSigma = 5.670374419e-8;
static const double kInfD = 1.0 / 0.0;
#define ERMC_B200_MAX_LEVELS_ORACLE 16

/* ------------------------------------------------------------ tables */

typedef struct {
  int nb, nq, nt;
  const double *nu_lo, *nu_hi, *w, *temps, *k, *ib;
  int uniform;
  double t0, dt;
} tables_t;

static void tables_init(tables_t* v, const ermc_model_t* m) {
  /* SpectralModel constructor, uniform detection (spectral.cpp:119-129) */
  v->nb = m->n_bands;
  v->nq = m->n_quad;
  v->nt = m->n_temps;
  v->nu_lo = m->band_nu_lo;
  v->nu_hi = m->band_nu_hi;
  v->w = m->g_weights;
  v->temps = m->temp_grid;
  v->k = m->k_table;
  v->ib = m->ib_table;
  v->uniform = 0;
  v->t0 = 0.0;
  v->dt = 1.0;
  if (v->nt >= 2) {
    v->t0 = v->temps[0];
    v->dt = v->temps[1] - v->temps[0];
    v->uniform = 1;
    for (int t = 1; t < v->nt; ++t)
      if (fabs(v->temps[t] - (v->t0 + t * v->dt)) > 1e-9 * v->dt) {
        v->uniform = 0;
        break;
      }
  }
}

static double knode(const tables_t* v, int n, int g, int t) {
  return v->k[((size_t)n * v->nq + g) * v->nt + t];
}
static double ibnode(const tables_t* v, int n, int t) {
  return v->ib[(size_t)n * v->nt + t];
}

static void seterr(char* err, size_t len, const char* msg) {
  if (err && len) snprintf(err, len, "%s", msg);
}

/* SpectralModel::lookup (spectral.cpp:148-177). */
static int lookup(const tables_t* v, double T, int* idx, double* frac,
                  char* err, size_t len) {
  const double* tg = v->temps;
  if (!(T >= tg[0] && T <= tg[v->nt - 1])) {
    char buf[256];
    snprintf(buf, sizeof buf, "temperature %f K outside table range [%f, %f]",
             T, tg[0], tg[v->nt - 1]);
    seterr(err, len, buf);
    return 1;
  }
  if (v->nt < 2) {
    *idx = 0;
    *frac = 0.0;
    return 0;
  }
  if (v->uniform) {
    int lo = (int)((T - v->t0) / v->dt);
    if (lo < 0) lo = 0;
    if (lo > v->nt - 2) lo = v->nt - 2;
    double f = (T - tg[lo]) / (tg[lo + 1] - tg[lo]);
    if (f < 0.0 && lo > 0) {
      --lo;
      f = (T - tg[lo]) / (tg[lo + 1] - tg[lo]);
    } else if (f > 1.0 && lo < v->nt - 2) {
      ++lo;
      f = (T - tg[lo]) / (tg[lo + 1] - tg[lo]);
    }
    *idx = lo;
    *frac = f;
    return 0;
  }
  int first = 0, count = v->nt; /* upper_bound */
  while (count > 0) {
    int step = count / 2, it = first + step;
    if (!(T < tg[it])) {
      first = it + 1;
      count -= step + 1;
    } else {
      count = step;
    }
  }
  if (first == 0) {
    *idx = 0;
    *frac = 0.0;
  } else if (first == v->nt) {
    *idx = v->nt - 2;
    *frac = 1.0;
  } else {
    *idx = first - 1;
    *frac = (T - tg[first - 1]) / (tg[first] - tg[first - 1]);
  }
  return 0;
}

static double lerp_node(double a, double b, double f) {
  if (f == 0.0) return a;
  return a + f * (b - a);
}

static int interp_k(const tables_t* v, int n, int g, double T, double* out,
                    char* err, size_t len) {
  int lo;
  double f;
  if (lookup(v, T, &lo, &f, err, len)) return 1;
  *out = lerp_node(knode(v, n, g, lo), f == 0.0 ? 0.0 : knode(v, n, g, lo + 1), f);
  return 0;
}

static int interp_ib(const tables_t* v, int n, double T, double* out,
                     char* err, size_t len) {
  int lo;
  double f;
  if (lookup(v, T, &lo, &f, err, len)) return 1;
  *out = lerp_node(ibnode(v, n, lo), f == 0.0 ? 0.0 : ibnode(v, n, lo + 1), f);
  return 0;
}

static double sig4(double t) { return kSigma * t * t * t * t; }

int oracle_planck_mean(const ermc_model_t* m, double T, double* out, char* err,
                       size_t len) {
  /* spectral.cpp:207-218 */
  tables_t v;
  tables_init(&v, m);
  int lo;
  double f;
  if (lookup(&v, T, &lo, &f, err, len)) return 1;
  if (T <= 0.0) {
    *out = 0.0;
    return 0;
  }
  double sum = 0.0;
  for (int n = 0; n < v.nb; ++n) {
    double gk = 0.0, k, ib;
    for (int g = 0; g < v.nq; ++g) {
      interp_k(&v, n, g, T, &k, NULL, 0);
      gk += v.w[g] * k;
    }
    interp_ib(&v, n, T, &ib, NULL, 0);
    sum += kPi * (v.nu_hi[n] - v.nu_lo[n]) * ib * gk;
  }
  *out = sum / sig4(T);
  return 0;
}

int oracle_build_cdfs(const ermc_model_t* m, double t_max, double* band_cdf,
                      double* quad_cdf, char* err, size_t len) {
  /* spectral.cpp:306-354 */
  tables_t v;
  tables_init(&v, m);
  double* bw = (double*)malloc(sizeof(double) * (size_t)v.nb);
  double* w = (double*)malloc(sizeof(double) * (size_t)v.nq);
  double total = 0.0;
  int rc = 0;
  for (int n = 0; n < v.nb && !rc; ++n) {
    double gk = 0.0, k, ib;
    for (int g = 0; g < v.nq; ++g) {
      if ((rc = interp_k(&v, n, g, t_max, &k, err, len))) break;
      gk += v.w[g] * k;
    }
    if (rc || (rc = interp_ib(&v, n, t_max, &ib, err, len))) break;
    bw[n] = kPi * (v.nu_hi[n] - v.nu_lo[n]) * ib * gk;
    total += bw[n];
  }
  if (!rc && !(total > 0.0)) {
    seterr(err, len, "build_cdfs: medium is transparent at T_max (kappa_p = 0)");
    rc = 1;
  }
  if (!rc) {
    double cum = 0.0;
    for (int n = 0; n < v.nb; ++n) {
      cum += bw[n] / total;
      band_cdf[n] = cum;
    }
    band_cdf[v.nb - 1] = 1.0;
    for (int n = 0; n < v.nb; ++n) {
      double gsum = 0.0, k;
      for (int g = 0; g < v.nq; ++g) {
        interp_k(&v, n, g, t_max, &k, NULL, 0);
        w[g] = v.w[g] * k;
        gsum += w[g];
      }
      if (gsum <= 0.0) {
        for (int g = 0; g < v.nq; ++g) w[g] = v.w[g];
        gsum = 1.0;
      }
      double c = 0.0;
      for (int g = 0; g < v.nq; ++g) {
        c += w[g] / gsum;
        quad_cdf[(size_t)n * v.nq + g] = c;
      }
      quad_cdf[(size_t)n * v.nq + v.nq - 1] = 1.0;
    }
  }
  free(bw);
  free(w);
  return rc;
}

/* ------------------------------------------------------------ RNG */

static uint64_t mix64(uint64_t x) {
  /* sampling.cpp:13-20 */
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdULL;
  x ^= x >> 33;
  x *= 0xc4ceb9fe1a85ec53ULL;
  x ^= x >> 33;
  return x;
}

double oracle_uniform(uint64_t seed, uint64_t cell, uint32_t ray, uint32_t draw) {
  /* sampling.cpp:24-29 */
  uint64_t h = mix64(seed + 0x9e3779b97f4a7c15ULL);
  h = mix64(h ^ cell);
  h = mix64(h ^ (((uint64_t)ray << 32) | draw));
  return (double)(h >> 11) * 0x1.0p-53;
}

/* ------------------------------------------------------------ hierarchy */

typedef struct {
  int n[3];
  double d[3], origin[3];
  double* field; /* owned for l >= 1 */
  int cap;
} level_t;

typedef struct {
  int nl;
  level_t lv[ERMC_B200_MAX_LEVELS_ORACLE];
} hier_t;

static double extent(const level_t* L, int a) { return L->n[a] * L->d[a]; }
static double min3(double a, double b, double c) {
  double m = a < b ? a : b;
  return m < c ? m : c;
}
static double geps(const level_t* L) { return 1e-12 * min3(L->d[0], L->d[1], L->d[2]); }

static int build_hier(hier_t* h, const ermc_grid_t* g, const double* T, int nl,
                      int ratio, int spl, char* err, size_t len) {
  /* geometry.cpp:51-110 */
  if (nl > ERMC_B200_MAX_LEVELS_ORACLE) {
    seterr(err, len, "oracle: too many levels");
    return 1;
  }
  if (nl > 1 && ratio < 2) {
    seterr(err, len, "build_hierarchy: ratio must be >= 2");
    return 1;
  }
  h->nl = nl;
  level_t* L0 = &h->lv[0];
  L0->n[0] = g->nx;
  L0->n[1] = g->ny;
  L0->n[2] = g->nz;
  L0->d[0] = g->dx;
  L0->d[1] = g->dy;
  L0->d[2] = g->dz;
  for (int a = 0; a < 3; ++a) L0->origin[a] = g->origin[a];
  L0->field = (double*)T;
  for (int l = 1; l < nl; ++l) {
    const level_t* F = &h->lv[l - 1];
    level_t* Cl = &h->lv[l];
    if (F->n[0] == 1 && F->n[1] == 1 && F->n[2] == 1) {
      char buf[160];
      snprintf(buf, sizeof buf,
               "build_hierarchy: cannot coarsen below one cell; achievable depth is %d", l);
      seterr(err, len, buf);
      h->nl = l;
      return 1;
    }
    for (int a = 0; a < 3; ++a) {
      Cl->n[a] = (F->n[a] + ratio - 1) / ratio;
      Cl->d[a] = extent(F, a) / Cl->n[a];
      Cl->origin[a] = F->origin[a];
    }
    Cl->field = (double*)malloc(sizeof(double) * (size_t)Cl->n[0] * Cl->n[1] * Cl->n[2]);
    for (int ci = 0; ci < Cl->n[0]; ++ci)
      for (int cj = 0; cj < Cl->n[1]; ++cj)
        for (int ck = 0; ck < Cl->n[2]; ++ck) {
          double sum = 0.0;
          int cnt = 0;
          for (int i = ci * ratio; i < (ci + 1) * ratio && i < F->n[0]; ++i)
            for (int j = cj * ratio; j < (cj + 1) * ratio && j < F->n[1]; ++j)
              for (int k = ck * ratio; k < (ck + 1) * ratio && k < F->n[2]; ++k) {
                sum += F->field[((int64_t)i * F->n[1] + j) * F->n[2] + k];
                ++cnt;
              }
          Cl->field[((int64_t)ci * Cl->n[1] + cj) * Cl->n[2] + ck] = sum / cnt;
        }
  }
  for (int l = 0; l < nl; ++l) h->lv[l].cap = (l + 1 == nl) ? -1 : spl;
  return 0;
}

static void free_hier(hier_t* h) {
  for (int l = 1; l < h->nl; ++l) free(h->lv[l].field);
  h->nl = 0;
}

/* ------------------------------------------------------------ rays */

typedef struct {
  double pos[3], dir[3];
  int idx[3];
  int band, quad;
  double prefactor, ib_source;
  uint64_t seed, cell_id;
  uint32_t ray_id, next_draw;
} ray_t;

typedef struct {
  const tables_t* v;
  const double* band_cdf;
  const double* quad_cdf;
  double t_max;
  const hier_t* h;
  const ermc_boundary_t* b;
  double qe, tol;
  int64_t max_steps;
  int specular, volume;
} ctx_t;

static int upper_bound(const double* a, int n, double x) {
  int first = 0, count = n;
  while (count > 0) {
    int step = count / 2, it = first + step;
    if (!(x < a[it])) {
      first = it + 1;
      count -= step + 1;
    } else {
      count = step;
    }
  }
  return first;
}

static double draw(ray_t* r) {
  return oracle_uniform(r->seed, r->cell_id, r->ray_id, r->next_draw++);
}

static int init_ray(const ctx_t* X, int i, int j, int k, uint32_t ray_id,
                    uint64_t seed, ray_t* r, char* err, size_t len) {
  /* sampling.cpp:55-96 */
  const level_t* L = &X->h->lv[0];
  memset(r, 0, sizeof *r);
  r->seed = seed;
  r->cell_id = (uint64_t)(((int64_t)i * L->n[1] + j) * L->n[2] + k);
  r->ray_id = ray_id;
  double rt = draw(r), rp = draw(r), rn = draw(r), rg = draw(r);
  /* sample_direction (sampling.cpp:31-40) */
  double ct = 1.0 - 2.0 * rt;
  double phi = 2.0 * kPi * rp;
  double mx = 1.0 - ct * ct;
  double st = sqrt(mx > 0.0 ? mx : 0.0);
  r->dir[0] = st * cos(phi);
  r->dir[1] = st * sin(phi);
  r->dir[2] = ct;
  /* sample_band (sampling.cpp:42-53) */
  int n = upper_bound(X->band_cdf, X->v->nb, rn);
  if (n >= X->v->nb) n = X->v->nb - 1;
  int g = upper_bound(X->quad_cdf + (size_t)n * X->v->nq, X->v->nq, rg);
  if (g >= X->v->nq) g = X->v->nq - 1;
  r->band = n;
  r->quad = g;
  r->idx[0] = i;
  r->idx[1] = j;
  r->idx[2] = k;
  int ijk[3] = {i, j, k};
  for (int a = 0; a < 3; ++a) r->pos[a] = L->origin[a] + (ijk[a] + 0.5) * L->d[a];
  if (X->volume)
    for (int a = 0; a < 3; ++a) r->pos[a] += (draw(r) - 0.5) * L->d[a];
  double tc = L->field[r->cell_id];
  double kmax, ibmax, kc;
  if (interp_ib(X->v, n, tc, &r->ib_source, err, len)) return 1;
  if (interp_k(X->v, n, g, X->t_max, &kmax, err, len)) return 1;
  if (interp_ib(X->v, n, X->t_max, &ibmax, err, len)) return 1;
  if (kmax <= 0.0 || ibmax <= 0.0) {
    seterr(err, len,
           "init_ray: sampled a transparent point at T_max; spectral tables are "
           "inconsistent with the sampling CDFs");
    return 1;
  }
  if (interp_k(X->v, n, g, tc, &kc, err, len)) return 1;
  r->prefactor = kc * r->ib_source / (kmax * ibmax);
  return 0;
}

typedef struct {
  double tn[3], td[3];
  int step[3];
} dda_t;

static void dda_setup(dda_t* d, const level_t* L, const double* pos,
                      const double* dir, const int* idx) {
  /* tracer.cpp:17-38 */
  for (int a = 0; a < 3; ++a) {
    if (dir[a] == 0.0) {
      d->tn[a] = kInfD;
      d->td[a] = kInfD;
      d->step[a] = 0;
      continue;
    }
    d->step[a] = dir[a] > 0.0 ? 1 : -1;
    int fi = idx[a] + (dir[a] > 0.0 ? 1 : 0);
    double face = L->origin[a] + fi * L->d[a];
    d->tn[a] = (face - pos[a]) / dir[a];
    d->td[a] = L->d[a] / fabs(dir[a]);
  }
}

typedef struct {
  double q, w_abs, w_walls, w_res;
  int64_t steps;
  int64_t level_steps[ERMC_B200_MAX_LEVELS_ORACLE];
  int term, reflections;
} march_t;

static int locate_dir(const level_t* L, const double* p, const double* dir,
                      int* idx, char* err, size_t len) {
  /* geometry.cpp:112-138 */
  double e = geps(L);
  for (int a = 0; a < 3; ++a) {
    double q = p[a] + e * dir[a];
    double rel = (q - L->origin[a]) / L->d[a];
    int i = (int)floor(rel);
    if (i < 0 || i >= L->n[a]) {
      if (rel >= -1e-9 && i < 0)
        i = 0;
      else if (rel <= L->n[a] + 1e-9 && i >= L->n[a])
        i = L->n[a] - 1;
      else {
        char buf[96];
        snprintf(buf, sizeof buf, "locate: point outside domain on axis %d", a);
        seterr(err, len, buf);
        return 1;
      }
    }
    idx[a] = i;
  }
  return 0;
}

static int march(const ctx_t* X, ray_t ray, march_t* out, char* err, size_t len) {
  /* tracer.cpp:57-194 */
  memset(out, 0, sizeof *out);
  const tables_t* v = X->v;
  const double ib1 = ray.ib_source, pref = ray.prefactor, qe = X->qe;
  double q = 0.0, last = ib1, tau = 1.0;
  int level = 0, sal = 0;
  int idx[3] = {ray.idx[0], ray.idx[1], ray.idx[2]};
  double pos[3] = {ray.pos[0], ray.pos[1], ray.pos[2]};
  double dir[3] = {ray.dir[0], ray.dir[1], ray.dir[2]};
  const level_t* L = &X->h->lv[0];
  double eps = geps(L);
  dda_t d;
  dda_setup(&d, L, pos, dir, idx);
  int term = 0;
  for (;;) {
    if (tau <= X->tol) {
      term = 0;
      break;
    }
    if (out->steps >= X->max_steps) {
      term = 2;
      break;
    }
    int cap = X->h->lv[level].cap;
    if (cap >= 0 && sal >= cap && level + 1 < X->h->nl) {
      ++level;
      L = &X->h->lv[level];
      eps = geps(L);
      if (locate_dir(L, pos, dir, idx, err, len)) return 1;
      sal = 0;
      dda_setup(&d, L, pos, dir, idx);
    }
    int axis = 0;
    double ds = d.tn[0];
    if (d.tn[1] < ds) {
      ds = d.tn[1];
      axis = 1;
    }
    if (d.tn[2] < ds) {
      ds = d.tn[2];
      axis = 2;
    }
    if (ds < 0.0) ds = 0.0;
    double tc = L->field[((int64_t)idx[0] * L->n[1] + idx[1]) * L->n[2] + idx[2]];
    int lo;
    double f;
    if (lookup(v, tc, &lo, &f, err, len)) return 1;
    double kap = lerp_node(knode(v, ray.band, ray.quad, lo),
                           f == 0.0 ? 0.0 : knode(v, ray.band, ray.quad, lo + 1), f);
    double ib2 = lerp_node(ibnode(v, ray.band, lo),
                           f == 0.0 ? 0.0 : ibnode(v, ray.band, lo + 1), f);
    double alpha = -expm1(-kap * ds);
    last = ib2;
    q += qe * tau * alpha * ((ib2 - ib1) / ib1) * pref;
    out->w_abs += tau * alpha;
    tau *= 1.0 - alpha;
    double adv = ds + eps;
    for (int a = 0; a < 3; ++a) pos[a] += adv * dir[a];
    for (int a = 0; a < 3; ++a) d.tn[a] -= adv;
    d.tn[axis] += d.td[axis];
    ++out->steps;
    ++out->level_steps[level];
    ++sal;
    if (!isfinite(q) || !isfinite(tau)) {
      char buf[160];
      snprintf(buf, sizeof buf, "march: non-finite value at cell %llu ray %u step %lld",
               (unsigned long long)ray.cell_id, ray.ray_id, (long long)out->steps);
      seterr(err, len, buf);
      return 1;
    }
    idx[axis] += d.step[axis];
    if (idx[axis] >= 0 && idx[axis] < L->n[axis]) continue;
    if (X->b->kind[axis] == ERMC_AXIS_PERIODIC) {
      double ext = extent(L, axis);
      if (idx[axis] < 0) {
        idx[axis] = L->n[axis] - 1;
        pos[axis] += ext;
      } else {
        idx[axis] = 0;
        pos[axis] -= ext;
      }
      continue;
    }
    int at_hi = d.step[axis] > 0;
    double wt = at_hi ? X->b->hi_temperature[axis] : X->b->lo_temperature[axis];
    double we = at_hi ? X->b->hi_emissivity[axis] : X->b->lo_emissivity[axis];
    double ibw = 0.0;
    if (wt > 0.0 && interp_ib(v, ray.band, wt, &ibw, err, len)) return 1;
    q += qe * tau * we * ((ibw - ib1) / ib1) * pref;
    out->w_walls += tau * we;
    tau *= 1.0 - we;
    if (tau <= X->tol) {
      term = 1;
      break;
    }
    ++out->reflections;
    idx[axis] -= d.step[axis];
    pos[axis] = L->origin[axis] + (at_hi ? extent(L, axis) : 0.0);
    int inward = at_hi ? -1 : 1;
    if (X->specular) {
      dir[axis] = -dir[axis];
    } else {
      /* diffuse_reflection (tracer.cpp:42-53) */
      double r1 = draw(&ray), r2 = draw(&ray);
      double s = sqrt(r1), c = sqrt(1.0 - r1), ph = 2.0 * kPi * r2;
      int t1 = (axis + 1) % 3, t2 = (axis + 2) % 3;
      dir[axis] = inward * c;
      dir[t1] = s * cos(ph);
      dir[t2] = s * sin(ph);
    }
    for (int a = 0; a < 3; ++a) pos[a] += eps * dir[a];
    dda_setup(&d, L, pos, dir, idx);
  }
  q += qe * tau * ((last - ib1) / ib1) * pref;
  out->w_res = tau;
  out->q = q;
  out->term = term;
  return 0;
}

/* ------------------------------------------------------------ solve */

typedef struct {
  const ctx_t* X;
  const ermc_config_t* c;
  int64_t lo, hi;
  int stride, offset;
  double *q, *sd;
  int64_t steps[ERMC_B200_MAX_LEVELS_ORACLE];
  int64_t fail_cell;
  char err[512];
} job_t;

static void* worker(void* arg) {
  job_t* J = (job_t*)arg;
  const ctx_t* X = J->X;
  const level_t* L = &X->h->lv[0];
  int R = J->c->rays_per_cell;
  double* per = (double*)malloc(sizeof(double) * (size_t)R);
  J->fail_cell = -1;
  for (int64_t c = J->lo + J->offset; c < J->hi; c += J->stride) {
    int i = (int)(c / ((int64_t)L->n[1] * L->n[2]));
    int j = (int)((c / L->n[2]) % L->n[1]);
    int k = (int)(c % L->n[2]);
    for (int r = 0; r < R; ++r) {
      ray_t ray;
      march_t m;
      if (init_ray(X, i, j, k, (uint32_t)r, J->c->seed, &ray, J->err, sizeof J->err) ||
          march(X, ray, &m, J->err, sizeof J->err)) {
        J->fail_cell = c;
        free(per);
        return NULL;
      }
      per[r] = m.q;
      for (int l = 0; l < X->h->nl; ++l) J->steps[l] += m.level_steps[l];
    }
    /* per-cell tally in ray-id order (solver.cpp:142-155) */
    double sum = 0.0, mean = 0.0, m2 = 0.0;
    for (int r = 0; r < R; ++r) {
      double x = per[r];
      sum += x;
      double delta = x - mean;
      mean += delta / (r + 1);
      m2 += delta * (x - mean);
    }
    J->q[c - J->lo] = sum;
    J->sd[c - J->lo] = R > 1 ? sqrt(m2 * R / (R - 1.0)) : 0.0;
  }
  free(per);
  return NULL;
}

static int setup_ctx(ctx_t* X, tables_t* v, hier_t* h, double** cdf_mem,
                     const ermc_grid_t* g, const double* T, const ermc_boundary_t* b,
                     const ermc_model_t* m, const ermc_config_t* c, double t_max,
                     double qe, char* err, size_t len) {
  tables_init(v, m);
  double* mem = (double*)malloc(sizeof(double) * (size_t)m->n_bands * (1 + m->n_quad));
  *cdf_mem = mem;
  if (oracle_build_cdfs(m, t_max, mem, mem + m->n_bands, err, len)) return 1;
  if (build_hier(h, g, T, c->n_levels, c->coarsen_ratio, c->steps_per_level, err, len))
    return 1;
  X->v = v;
  X->band_cdf = mem;
  X->quad_cdf = mem + m->n_bands;
  X->t_max = t_max;
  X->h = h;
  X->b = b;
  X->qe = qe;
  X->tol = c->tolerance;
  X->max_steps = c->max_steps;
  X->specular = c->specular_walls;
  X->volume = c->volume_sampling;
  return 0;
}

int oracle_solve(const ermc_grid_t* g, const double* T, const ermc_boundary_t* b,
                 const ermc_model_t* m, const ermc_config_t* c, int64_t lo,
                 int64_t hi, double* q, double* sd, int64_t* steps, int nthreads,
                 char* err, size_t len) {
  /* solver.cpp:82-180 (inputs assumed validated; validation lives in the
   * product and is tested against the reference directly) */
  int64_t n = (int64_t)g->nx * g->ny * g->nz;
  double tmax = T[0];
  for (int64_t i = 1; i < n; ++i)
    if (T[i] > tmax) tmax = T[i];
  for (int a = 0; a < 3; ++a) {
    if (b->kind[a] == ERMC_AXIS_PERIODIC) continue;
    if (b->lo_temperature[a] > tmax) tmax = b->lo_temperature[a];
    if (b->hi_temperature[a] > tmax) tmax = b->hi_temperature[a];
  }
  tables_t v;
  hier_t h;
  memset(&h, 0, sizeof h);
  ctx_t X;
  double* mem = NULL;
  double kp;
  int rc = 0;
  /* solver.cpp:88-93; planck_mean cannot fail for an in-range T_max, so
   * evaluating it before build_cdfs keeps the reference's error order. */
  if (oracle_planck_mean(m, tmax, &kp, err, len)) return 1;
  double qe = 4.0 * kp * kSigma * tmax * tmax * tmax * tmax / c->rays_per_cell;
  if (setup_ctx(&X, &v, &h, &mem, g, T, b, m, c, tmax, qe, err, len)) {
    free(mem);
    free_hier(&h);
    return 1;
  }
  if (nthreads < 1) nthreads = 1;
  job_t* jobs = (job_t*)calloc((size_t)nthreads, sizeof(job_t));
  pthread_t* th = (pthread_t*)calloc((size_t)nthreads, sizeof(pthread_t));
  for (int w = 0; w < nthreads; ++w) {
    jobs[w].X = &X;
    jobs[w].c = c;
    jobs[w].lo = lo;
    jobs[w].hi = hi;
    jobs[w].stride = nthreads;
    jobs[w].offset = w;
    jobs[w].q = q;
    jobs[w].sd = sd;
    pthread_create(&th[w], NULL, worker, &jobs[w]);
  }
  int64_t first = -1;
  for (int w = 0; w < nthreads; ++w) {
    pthread_join(th[w], NULL);
    if (jobs[w].fail_cell >= 0 && (first < 0 || jobs[w].fail_cell < first)) {
      first = jobs[w].fail_cell;
      seterr(err, len, jobs[w].err);
      rc = 1;
    }
  }
  for (int l = 0; l < c->n_levels; ++l) {
    steps[l] = 0;
    for (int w = 0; w < nthreads; ++w) steps[l] += jobs[w].steps[l];
  }
  free(jobs);
  free(th);
  free(mem);
  free_hier(&h);
  return rc;
}

int oracle_trace_rays(const ermc_grid_t* g, const double* T, const ermc_boundary_t* b,
                      const ermc_model_t* m, const ermc_config_t* c, double t_max,
                      double qe, int64_t n, const int64_t* cells, const uint32_t* rays,
                      const double* dirs, ermc_ray_result_t* out, char* err, size_t len) {
  tables_t v;
  hier_t h;
  memset(&h, 0, sizeof h);
  ctx_t X;
  double* mem = NULL;
  int rc = 0;
  if (setup_ctx(&X, &v, &h, &mem, g, T, b, m, c, t_max, qe, err, len)) {
    free(mem);
    free_hier(&h);
    return 1;
  }
  const level_t* L = &h.lv[0];
  for (int64_t s = 0; s < n && !rc; ++s) {
    int64_t cc = cells[s];
    int i = (int)(cc / ((int64_t)L->n[1] * L->n[2]));
    int j = (int)((cc / L->n[2]) % L->n[1]);
    int k = (int)(cc % L->n[2]);
    ray_t ray;
    march_t mr;
    if ((rc = init_ray(&X, i, j, k, rays[s], c->seed, &ray, err, len))) break;
    if (dirs)
      for (int a = 0; a < 3; ++a) ray.dir[a] = dirs[3 * s + a];
    if ((rc = march(&X, ray, &mr, err, len))) break;
    ermc_ray_result_t* o = &out[s];
    memset(o, 0, sizeof *o);
    o->q_contribution = mr.q;
    o->weight_absorbed = mr.w_abs;
    o->weight_walls = mr.w_walls;
    o->weight_residual = mr.w_res;
    for (int a = 0; a < 3; ++a) o->dir[a] = ray.dir[a];
    o->prefactor = ray.prefactor;
    o->ib_source = ray.ib_source;
    o->steps = mr.steps;
    o->terminated_by = mr.term;
    o->reflections = mr.reflections;
    o->band = ray.band;
    o->quad = ray.quad;
    o->next_draw = ray.next_draw;
  }
  free(mem);
  free_hier(&h);
  return rc;
}

/* ------------------------------------------------------------ slab oracle */

double oracle_expint_e1(double x) {
  /* expint.cpp:10-37: series below 1, Lentz continued fraction above */
  if (x < 0.0) return NAN;
  if (x == 0.0) return kInfD;
  const double euler = 0.5772156649015328606;
  if (x <= 1.0) {
    double sum = 0.0, term = 1.0;
    for (int n = 1; n <= 60; ++n) {
      term *= -x / n;
      double add = -term / n;
      sum += add;
      if (fabs(add) < 1e-17 * fabs(sum)) break;
    }
    return -euler - log(x) + sum;
  }
  double bb = x + 1.0, cc = 1e308, dd = 1.0 / bb, hh = dd;
  for (int i = 1; i <= 200; ++i) {
    double a = -(double)i * i;
    bb += 2.0;
    dd = 1.0 / (a * dd + bb);
    cc = bb + a / cc;
    double del = cc * dd;
    hh *= del;
    if (fabs(del - 1.0) < 1e-16) break;
  }
  return hh * exp(-x);
}

double oracle_expint_e2(double x) {
  if (x == 0.0) return 1.0;
  return exp(-x) - x * oracle_expint_e1(x);
}

double oracle_expint_e3(double x) {
  if (x == 0.0) return 0.5;
  return 0.5 * (exp(-x) - x * oracle_expint_e2(x));
}

double oracle_profile(int profile, double t_const, double x) {
  /* cases.cpp:11-15 */
  switch (profile) {
    case ORACLE_PROFILE_LIN1: return 500.0 + 1000.0 * x;
    case ORACLE_PROFILE_LIN2: return 295.0 + 10.0 * x;
    case ORACLE_PROFILE_PARAB: return 500.0 - 2000.0 * x * x + 2000.0 * x;
    default: return t_const;
  }
}

typedef struct {
  int kind; /* 0: sigT4(x) E1(k|x0-x|), 1: sigT4 E2(k x), 2: sigT4 E2(k(L-x)) */
  int profile;
  double tc, kappa, x0, length;
} slab_f;

static double slab_eval(const slab_f* f, double x) {
  double t = oracle_profile(f->profile, f->tc, x);
  double s4 = sig4(t);
  if (f->kind == 0) return s4 * oracle_expint_e1(f->kappa * fabs(f->x0 - x));
  if (f->kind == 1) return s4 * oracle_expint_e2(f->kappa * x);
  return s4 * oracle_expint_e2(f->kappa * (f->length - x));
}

static const double kGl8x[8] = {-0.9602898564975363, -0.7966664774136267,
                                -0.5255324099163290, -0.1834346424956498,
                                0.1834346424956498,  0.5255324099163290,
                                0.7966664774136267,  0.9602898564975363};
static const double kGl8w[8] = {0.1012285362903763, 0.2223810344533745,
                                0.3137066458778873, 0.3626837833783620,
                                0.3626837833783620, 0.3137066458778873,
                                0.2223810344533745, 0.1012285362903763};

static double panel(const slab_f* f, double a, double b, int subdiv) {
  /* oracles.cpp:29-39 */
  double sum = 0.0, h = (b - a) / subdiv;
  for (int s = 0; s < subdiv; ++s) {
    double lo = a + s * h, mid = lo + 0.5 * h;
    for (int i = 0; i < 8; ++i) sum += kGl8w[i] * slab_eval(f, mid + 0.5 * h * kGl8x[i]);
  }
  return sum * 0.5 * h;
}

static double one_side(const slab_f* f, double from, double to, int refine) {
  double total = 0.0, len = fabs(to - from);
  if (len <= 0.0) return 0.0;
  double sign = to > from ? 1.0 : -1.0, hi = len;
  for (int d = 0; d < 44; ++d) {
    double lo = hi * 0.5, pa = from + sign * lo, pb = from + sign * hi;
    total += panel(f, pa < pb ? pa : pb, pa < pb ? pb : pa, refine);
    hi = lo;
  }
  return total;
}

static double graded(const slab_f* f, double a, double b, double s, int refine) {
  /* oracles.cpp:44-69 */
  if (b <= a) return 0.0;
  if (s <= a) return one_side(f, a, b, refine);
  if (s >= b) return one_side(f, b, a, refine);
  return one_side(f, s, a, refine) + one_side(f, s, b, refine);
}

int oracle_slab(double length, int profile, double tc, double kappa, double t_lo,
                double eps_lo, double t_hi, double eps_hi, const double* x, int nx,
                int refine, double* q, char* err, size_t len) {
  /* oracles.cpp:73-128 */
  if (length <= 0.0) {
    seterr(err, len, "slab_oracle: length must be positive");
    return 1;
  }
  double tau_l = kappa * length;
  double emit1 = eps_lo * kSigma * pow(t_lo, 4);
  double emit2 = eps_hi * kSigma * pow(t_hi, 4);
  double j1 = emit1, j2 = emit2;
  if (eps_lo < 1.0 || eps_hi < 1.0) {
    slab_f f1 = {1, profile, tc, kappa, 0.0, length};
    slab_f f2 = {2, profile, tc, kappa, 0.0, length};
    double hm1 = 2.0 * kappa * graded(&f1, 0.0, length, 0.0, refine);
    double hm2 = 2.0 * kappa * graded(&f2, 0.0, length, length, refine);
    for (int it = 0; it < 10000; ++it) {
      double n1 = emit1 + (1.0 - eps_lo) * (2.0 * j2 * oracle_expint_e3(tau_l) + hm1);
      double n2 = emit2 + (1.0 - eps_hi) * (2.0 * j1 * oracle_expint_e3(tau_l) + hm2);
      double change = fabs(n1 - j1) + fabs(n2 - j2);
      j1 = n1;
      j2 = n2;
      if (change < 1e-6 * (fabs(j1) + fabs(j2) + 1e-300)) break;
    }
  }
  for (int p = 0; p < nx; ++p) {
    double xp = x[p];
    if (xp < 0.0 || xp > length) {
      seterr(err, len, "slab_oracle: x outside slab");
      return 1;
    }
    slab_f fm = {0, profile, tc, kappa, xp, length};
    double medium = graded(&fm, 0.0, length, xp, refine);
    q[p] = kappa * (2.0 * j1 * oracle_expint_e2(kappa * xp) +
                    2.0 * j2 * oracle_expint_e2(kappa * (length - xp)) +
                    2.0 * kappa * medium - 4.0 * sig4(oracle_profile(profile, tc, xp)));
  }
  return 0;
}

/* ------------------------------------------------------------ kernel check */
/* C restatement of the fp64 lean kernel's expm1 (trace_fp64.cu,
 * expm1_lean) so tests can bound its distance to glibc's expm1 (the
 * reference's libm) on the CPU. Same operations, same fma() calls. */
double oracle_expm1_lean(double x) {
  static const double c[12] = {1.0 / 2, 1.0 / 6, 1.0 / 24, 1.0 / 120, 1.0 / 720,
                               1.0 / 5040, 1.0 / 40320, 1.0 / 362880, 1.0 / 3628800,
                               1.0 / 39916800, 1.0 / 479001600, 1.0 / 6227020800.0};
  if (!(x >= -40.0 && x <= 0.5)) {
    if (x < -40.0) return -1.0;
    return expm1(x);
  }
  const double magic = 6755399441055744.0;
  double t = fma(x, 1.4426950408889634074, magic);
  double j = t - magic;
  double r = fma(j, -6.93147180369123816490e-01, x);
  r = fma(j, -1.90821492927058770002e-10, r);
  double p = c[11];
  for (int i = 10; i >= 0; --i) p = fma(p, r, c[i]);
  double e = fma(r * r, p, r);
  long long ji = (long long)j;
  if (ji == 0) return e;
  uint64_t bits = (uint64_t)(ji + 1023) << 52;
  double sc;
  memcpy(&sc, &bits, sizeof sc);
  return fma(sc, e, sc - 1.0);
}

/* max |ulp| distance of oracle_expm1_lean to glibc expm1 over n stratified
 * samples of the march's arguments x = -kappa ds in [-40, 0]. */
double oracle_expm1_lean_max_ulp(long n, long* n_differ) {
  uint64_t s = 7;
  double worst = 0.0;
  long differ = 0;
  for (long i = 0; i < n; ++i) {
    s ^= s << 13;
    s ^= s >> 7;
    s ^= s << 17;
    double u = (double)(s >> 11) * 0x1p-53, x;
    switch (i % 5) {
      case 0: x = -u * 40; break;
      case 1: x = -u * 2; break;
      case 2: x = -u * 1e-3; break;
      case 3: x = -u * 1e-8; break;
      default: x = -exp(-u * 40); break;
    }
    double a = oracle_expm1_lean(x), b = expm1(x);
    if (a != b) {
      ++differ;
      double ulp = nextafter(fabs(b), 1.0 / 0.0) - fabs(b);
      double d = fabs(a - b) / ulp;
      if (d > worst) worst = d;
    }
  }
  if (n_differ) *n_differ = differ;
  return worst;
}
