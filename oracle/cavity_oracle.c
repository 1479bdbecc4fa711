/* cavity_oracle.c — TEST INFRASTRUCTURE ONLY. Never linked into, loaded by
 * or called from the product path (paper_2006_02602_b200/); only tests/,
 * __graft_entry__.smoke() and bench.py's CPU-baseline leg use it, as the
 * checker.
 *
 * A plain-C restatement of the reference's single-block hot path
 * (/root/reference/proj, abbreviated P/). Each function cites the reference
 * lines whose arithmetic it restates; floating-point operation order is kept
 * exactly (compiled with -ffp-contract=off like P/CMakeLists.txt:14), so the
 * results are bitwise those of the reference's scalar backend.
 *
 * Parity pinning: tests/test_oracle.py checks this restatement bitwise against
 * golden fixtures generated from the reference itself (tests/golden/, made by
 * tests/golden/make_golden.py through oracle/_ref/libcavity_ref.so) and, where
 * the reference library is present, directly against it. */
#define _POSIX_C_SOURCE 199309L
#include "cavity_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

static _Thread_local char g_err[512];

const char* oc_last_error(void) { return g_err; }

static int fail(int code, const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return code;
}

/* FluidParams defaults + for_rayleigh (P/include/cavity/solver.hpp:18-38,
 * P/src/solver.cpp:11-25); RunConfig/SolverConfig defaults
 * (P/include/cavity/util/config.hpp:15-34, solver.hpp:43-51). */
void oc_run_config_default(cav_run_config* c) {
  memset(c, 0, sizeof *c);
  c->nx = c->ny = c->nz = 32;
  c->np = 1;
  c->mode = CAV_MODE_3D;
  c->strategy = CAV_V3;
  c->steps = -1;
  cav_fluid_params* f = &c->fluid;
  f->rho = 1.0;
  f->nu = 1.5e-5;
  f->alpha = 1.5e-5 / 0.71;
  f->gravity[0] = 0.0;
  f->gravity[1] = 0.0;
  f->gravity[2] = -9.81;
  f->u_ref = 0.03;
  f->kappa = 0.01;
  f->t_hot = 300.5;
  f->t_cold = 299.5;
  f->t_inf = 300.0;
  f->length = 0.05;
  const double gmag =
      sqrt((f->gravity[0] * f->gravity[0] + f->gravity[1] * f->gravity[1]) + f->gravity[2] * f->gravity[2]);
  const double l3 = (f->length * f->length) * f->length;
  f->sigma = 1e5 * f->nu * f->alpha / (gmag * (f->t_hot - f->t_cold) * l3);
  c->cfl = 0.4;
  c->max_steps = 200000;
  c->conv_tol = 1e-8;
  c->rescale = 1;
  c->check_every = 10;
  c->timeout_ms = 20000.0;
  c->verify_tol = 1e-12;
}

/* make_stencil_params (P/src/solver.cpp:77-103). */
void oc_make_stencil_params(double dx, double dy, double dz, const cav_fluid_params* prm,
                            cav_stencil_params* s) {
  s->inv2dx = 1.0 / (2.0 * dx);
  s->inv2dy = 1.0 / (2.0 * dy);
  s->inv2dz = 1.0 / (2.0 * dz);
  s->invdx2 = 1.0 / (dx * dx);
  s->invdy2 = 1.0 / (dy * dy);
  s->invdz2 = 1.0 / (dz * dz);
  const double hx2 = dx * dx, hy2 = dy * dy, hz2 = dz * dz;
  s->invdx4 = 1.0 / (hx2 * hx2);
  s->invdy4 = 1.0 / (hy2 * hy2);
  s->invdz4 = 1.0 / (hz2 * hz2);
  s->kdx3 = prm->kappa * (hx2 * dx);
  s->kdy3 = prm->kappa * (hy2 * dy);
  s->kdz3 = prm->kappa * (hz2 * dz);
  s->u_ref = prm->u_ref;
  s->nu = prm->nu;
  s->alpha = prm->alpha;
  s->rho = prm->rho;
  s->inv_rho = 1.0 / prm->rho;
  s->sigma = prm->sigma;
  s->t_inf = prm->t_inf;
  s->gx = prm->gravity[0];
  s->gy = prm->gravity[1];
  s->gz = prm->gravity[2];
}

/* std::max(a, b) / std::min(a, b) semantics (first argument wins ties/NaN). */
static double smax(double a, double b) { return a < b ? b : a; }
static double smin(double a, double b) { return b < a ? b : a; }

/* One cell of residual_cell (P/src/kernels_cell.hpp:14-79), same op order. */
static void residual_one(const cav_field_ptrs* f, const cav_residual_ptrs* r, long c, long sj,
                         long sk, const cav_stencil_params* q) {
  const double *P = f->p, *U = f->u, *V = f->v, *W = f->w, *T = f->t;
  const double uc = U[c], vc = V[c], wc = W[c], tc = T[c];
  const double speed = sqrt((uc * uc + vc * vc) + wc * wc);
  const double b = smax(speed, q->u_ref);
  const double b2 = b * b;

  const double ux = (U[c + 1] - U[c - 1]) * q->inv2dx;
  const double uy = (U[c + sj] - U[c - sj]) * q->inv2dy;
  const double uz = (U[c + sk] - U[c - sk]) * q->inv2dz;
  const double vx = (V[c + 1] - V[c - 1]) * q->inv2dx;
  const double vy = (V[c + sj] - V[c - sj]) * q->inv2dy;
  const double vz = (V[c + sk] - V[c - sk]) * q->inv2dz;
  const double wx = (W[c + 1] - W[c - 1]) * q->inv2dx;
  const double wy = (W[c + sj] - W[c - sj]) * q->inv2dy;
  const double wz = (W[c + sk] - W[c - sk]) * q->inv2dz;
  const double tx = (T[c + 1] - T[c - 1]) * q->inv2dx;
  const double ty = (T[c + sj] - T[c - sj]) * q->inv2dy;
  const double tz = (T[c + sk] - T[c - sk]) * q->inv2dz;
  const double px = (P[c + 1] - P[c - 1]) * q->inv2dx;
  const double py = (P[c + sj] - P[c - sj]) * q->inv2dy;
  const double pz = (P[c + sk] - P[c - sk]) * q->inv2dz;

  const double dv = (ux + vy) + wz;
  const double p0 = P[c];
  const double fx = ((((P[c - 2] - 4.0 * P[c - 1]) + 6.0 * p0) - 4.0 * P[c + 1]) + P[c + 2]) * q->invdx4;
  const double fy =
      ((((P[c - 2 * sj] - 4.0 * P[c - sj]) + 6.0 * p0) - 4.0 * P[c + sj]) + P[c + 2 * sj]) * q->invdy4;
  const double fz =
      ((((P[c - 2 * sk] - 4.0 * P[c - sk]) + 6.0 * p0) - 4.0 * P[c + sk]) + P[c + 2 * sk]) * q->invdz4;
  const double dmp = b * ((q->kdx3 * fx + q->kdy3 * fy) + q->kdz3 * fz);
  r->p[c] = -b2 * (q->rho * dv + dmp);

  const double lu = ((U[c + 1] - 2.0 * uc) + U[c - 1]) * q->invdx2 +
                    ((U[c + sj] - 2.0 * uc) + U[c - sj]) * q->invdy2 +
                    ((U[c + sk] - 2.0 * uc) + U[c - sk]) * q->invdz2;
  const double lv = ((V[c + 1] - 2.0 * vc) + V[c - 1]) * q->invdx2 +
                    ((V[c + sj] - 2.0 * vc) + V[c - sj]) * q->invdy2 +
                    ((V[c + sk] - 2.0 * vc) + V[c - sk]) * q->invdz2;
  const double lw = ((W[c + 1] - 2.0 * wc) + W[c - 1]) * q->invdx2 +
                    ((W[c + sj] - 2.0 * wc) + W[c - sj]) * q->invdy2 +
                    ((W[c + sk] - 2.0 * wc) + W[c - sk]) * q->invdz2;
  const double cu = (uc * ux + vc * uy) + wc * uz;
  const double cv = (uc * vx + vc * vy) + wc * vz;
  const double cw = (uc * wx + vc * wy) + wc * wz;
  const double by = q->sigma * (tc - q->t_inf);
  r->u[c] = ((-cu - q->inv_rho * px) + q->nu * lu) + by * q->gx;
  r->v[c] = ((-cv - q->inv_rho * py) + q->nu * lv) + by * q->gy;
  r->w[c] = ((-cw - q->inv_rho * pz) + q->nu * lw) + by * q->gz;

  const double lt = ((T[c + 1] - 2.0 * tc) + T[c - 1]) * q->invdx2 +
                    ((T[c + sj] - 2.0 * tc) + T[c - sj]) * q->invdy2 +
                    ((T[c + sk] - 2.0 * tc) + T[c - sk]) * q->invdz2;
  const double ct = (uc * tx + vc * ty) + wc * tz;
  r->t[c] = -ct + q->alpha * lt;
}

/* residual_box_scalar (P/src/kernels_scalar.cpp:5-17). */
void oc_residual_box(const cav_field_ptrs* in, const cav_residual_ptrs* out, int X, int Y,
                     const cav_box* box, const cav_stencil_params* sp) {
  const long sj = X, sk = (long)X * Y;
  for (int k = box->lo[2]; k < box->hi[2]; ++k)
    for (int j = box->lo[1]; j < box->hi[1]; ++j)
      for (int i = box->lo[0]; i < box->hi[0]; ++i) residual_one(in, out, i + sj * j + sk * k, sj, sk, sp);
}

/* update_box_scalar (P/src/kernels_scalar.cpp:19-30). */
void oc_update_box(double* q, const double* r, double dt, int X, int Y, const cav_box* box) {
  const long sj = X, sk = (long)X * Y;
  for (int k = box->lo[2]; k < box->hi[2]; ++k)
    for (int j = box->lo[1]; j < box->hi[1]; ++j)
      for (int i = box->lo[0]; i < box->hi[0]; ++i) {
        const long c = i + sj * j + sk * k;
        q[c] = q[c] + dt * r[c];
      }
}

/* apply_boundary_conditions (P/src/solver.cpp:129-191): per wall face, the
 * two ghost layers at transverse interior positions. */
void oc_apply_bc(const cav_residual_ptrs* f, int nx, int ny, int nz, const int walls[6],
                 const cav_fluid_params* prm) {
  const int n[3] = {nx, ny, nz};
  const long X = nx + 4, Y = ny + 4;
  const long stride[3] = {1, X, X * Y};
  for (int fid = 0; fid < 6; ++fid) {
    if (!walls[fid]) continue;
    const int a = fid / 2, high = fid % 2;
    /* normal positions: ghost nearest the wall g0, outer ghost g1, interior i0..i2 */
    const int g1 = high ? n[a] + 3 : 0, g0 = high ? n[a] + 2 : 1;
    const int i0 = high ? n[a] + 1 : 2, i1 = high ? n[a] : 3, i2 = high ? n[a] - 1 : 4;
    const int a1 = a == 0 ? 1 : 0, a2 = a == 2 ? 1 : 2;
    const double tw = high ? prm->t_cold : prm->t_hot;
    const long s = stride[a];
    for (int q2 = 2; q2 < n[a2] + 2; ++q2)
      for (int q1 = 2; q1 < n[a1] + 2; ++q1) {
        const long base = q1 * stride[a1] + q2 * stride[a2];
        double* vel[3] = {f->u, f->v, f->w};
        for (int m = 0; m < 3; ++m) {
          vel[m][base + g0 * s] = -vel[m][base + i0 * s];
          vel[m][base + g1 * s] = -vel[m][base + i1 * s];
        }
        if (a == 0) {
          f->t[base + g0 * s] = 2.0 * tw - f->t[base + i0 * s];
          f->t[base + g1 * s] = 2.0 * tw - f->t[base + i1 * s];
        } else {
          f->t[base + g0 * s] = f->t[base + i0 * s];
          f->t[base + g1 * s] = f->t[base + i1 * s];
        }
        double* P = f->p;
        P[base + g0 * s] = (3.0 * P[base + i0 * s] - 3.0 * P[base + i1 * s]) + P[base + i2 * s];
        P[base + g1 * s] = (3.0 * P[base + g0 * s] - 3.0 * P[base + i0 * s]) + P[base + i1 * s];
      }
  }
}

/* compute_dt (P/src/solver.cpp:193-232): finiteness scan in P,U,V,W,T order,
 * then the CFL/viscous/thermal minimum. */
int oc_compute_dt(const cav_field_ptrs* f, int nx, int ny, int nz, double dx, double dy,
                  double dz, const cav_fluid_params* prm, double cfl, double* dt_out) {
  if (!(cfl > 0.0) || !isfinite(cfl)) {
    snprintf(g_err, sizeof g_err, "compute_dt: cfl must be positive, got %f", cfl);
    return CAV_EINVAL;
  }
  const long X = nx + 4, Y = ny + 4;
  const double* q[5] = {f->p, f->u, f->v, f->w, f->t};
  static const char* names[5] = {"p", "u", "v", "w", "T"};
  for (int v = 0; v < 5; ++v)
    for (int k = 2; k < nz + 2; ++k)
      for (int j = 2; j < ny + 2; ++j)
        for (int i = 2; i < nx + 2; ++i)
          if (!isfinite(q[v][i + X * (j + Y * k)])) {
            snprintf(g_err, sizeof g_err, "compute_dt: non-finite value in field %s", names[v]);
            return CAV_ERUNTIME;
          }
  double conv = INFINITY;
  for (int k = 2; k < nz + 2; ++k)
    for (int j = 2; j < ny + 2; ++j)
      for (int i = 2; i < nx + 2; ++i) {
        const long c = i + X * (j + Y * k);
        const double uc = f->u[c], vc = f->v[c], wc = f->w[c];
        const double b = smax(sqrt((uc * uc + vc * vc) + wc * wc), prm->u_ref);
        conv = smin(conv, dx / (fabs(uc) + b));
        conv = smin(conv, dy / (fabs(vc) + b));
        conv = smin(conv, dz / (fabs(wc) + b));
      }
  const double dmin = smin(smin(dx, dy), dz);
  const double visc = dmin * dmin / (6.0 * prm->nu);
  const double therm = dmin * dmin / (6.0 * prm->alpha);
  *dt_out = cfl * smin(smin(conv, visc), therm);
  return CAV_OK;
}

/* rescale_pressure (P/src/solver.cpp:248-257). */
void oc_rescale(double* p, int nx, int ny, int nz, double pc) {
  const long X = nx + 4, Y = ny + 4;
  for (int k = 2; k < nz + 2; ++k)
    for (int j = 2; j < ny + 2; ++j)
      for (int i = 2; i < nx + 2; ++i) p[i + X * (j + Y * k)] = p[i + X * (j + Y * k)] - pc;
}

/* ---- exact accumulator: restates ReproSum (P/include/cavity/util/repro_sum.hpp:19-173).
 * value*2^1140 in 35 little-endian u64 limbs, positive and negative halves. */
#define OC_LIMBS 35
typedef struct { uint64_t pos[OC_LIMBS], neg[OC_LIMBS]; } oc_acc;

static void limbs_add_shifted(uint64_t* L, uint64_t mant, int off) {
  int l = off >> 6;
  const unsigned __int128 wide = (unsigned __int128)mant << (off & 63);
  unsigned __int128 carry = (unsigned __int128)L[l] + (uint64_t)wide;
  L[l] = (uint64_t)carry;
  carry = (carry >> 64) + (uint64_t)(wide >> 64);
  for (++l; carry && l < OC_LIMBS; ++l) {
    carry += L[l];
    L[l] = (uint64_t)carry;
    carry >>= 64;
  }
}

static int acc_add(oc_acc* a, double x) { /* repro_sum.hpp:24-40 */
  if (!isfinite(x)) return fail(CAV_EINVAL, "repro_sum: non-finite term");
  if (x == 0.0) return CAV_OK;
  uint64_t bits;
  memcpy(&bits, &x, 8);
  const int e = (int)((bits >> 52) & 0x7FF);
  uint64_t m = bits & ((1ULL << 52) - 1);
  int off = 66; /* subnormal: m * 2^-1074 */
  if (e != 0) {
    m |= 1ULL << 52;
    off = e + 65; /* (m) * 2^(e-1075) */
  }
  limbs_add_shifted(bits >> 63 ? a->neg : a->pos, m, off);
  return CAV_OK;
}

static int limbs_cmp(const uint64_t* a, const uint64_t* b) {
  for (int i = OC_LIMBS - 1; i >= 0; --i)
    if (a[i] != b[i]) return a[i] > b[i] ? 1 : -1;
  return 0;
}

static int bit_at(const uint64_t* m, int b) { return (int)((m[b >> 6] >> (b & 63)) & 1); }

/* ReproSum::value (repro_sum.hpp:48-77): round-to-nearest-even of pos-neg. */
double oc_repro_value(const uint64_t* limbs70) {
  const uint64_t* pos = limbs70;
  const uint64_t* neg = limbs70 + OC_LIMBS;
  const int sign = limbs_cmp(pos, neg);
  if (sign == 0) return 0.0;
  const uint64_t* big = sign > 0 ? pos : neg;
  const uint64_t* small = sign > 0 ? neg : pos;
  uint64_t mag[OC_LIMBS];
  unsigned borrow = 0;
  for (int i = 0; i < OC_LIMBS; ++i) {
    const unsigned __int128 d = (unsigned __int128)big[i] - small[i] - borrow;
    mag[i] = (uint64_t)d;
    borrow = (unsigned)((d >> 64) & 1);
  }
  int top = -1;
  for (int i = OC_LIMBS - 1; i >= 0 && top < 0; --i)
    if (mag[i]) top = i * 64 + 63 - __builtin_clzll(mag[i]);
  uint64_t mant = 0;
  int e2;
  const int lo = top <= 52 ? 0 : top - 52;
  for (int b = top; b >= lo; --b) mant = (mant << 1) | (uint64_t)bit_at(mag, b);
  if (top <= 52) {
    e2 = -1140;
  } else {
    const int guard = bit_at(mag, top - 53);
    int sticky = 0;
    for (int b = top - 54; b >= 0 && !sticky; --b) sticky = bit_at(mag, b);
    if (guard && (sticky || (mant & 1))) {
      if (++mant == (1ULL << 53)) {
        mant >>= 1;
        ++top;
      }
    }
    e2 = top - 52 - 1140;
  }
  const double r = ldexp((double)mant, e2);
  return sign > 0 ? r : -r;
}

/* residual_norm_partials (P/src/solver.cpp:259-274): exact sums of fl(r*r). */
int oc_norm_partials(const cav_field_ptrs* r, int nx, int ny, int nz, uint64_t* out) {
  const long X = nx + 4, Y = ny + 4;
  const double* q[5] = {r->p, r->u, r->v, r->w, r->t};
  for (int v = 0; v < 5; ++v) {
    oc_acc acc;
    memset(&acc, 0, sizeof acc);
    for (int k = 2; k < nz + 2; ++k)
      for (int j = 2; j < ny + 2; ++j)
        for (int i = 2; i < nx + 2; ++i) {
          const double x = q[v][i + X * (j + Y * k)];
          const int st = acc_add(&acc, x * x);
          if (st) return st;
        }
    memcpy(out + 70 * v, acc.pos, sizeof acc.pos);
    memcpy(out + 70 * v + OC_LIMBS, acc.neg, sizeof acc.neg);
  }
  return CAV_OK;
}

/* face_interior_box / face_ghost_box (P/src/slab.cpp:21-49). */
int oc_face_box(int nx, int ny, int nz, int face, int depth, int ghost, cav_box* out) {
  const int n[3] = {nx, ny, nz};
  const int a = face / 2, high = face % 2;
  if (depth < 1 || depth > 2) return fail(CAV_EINVAL, "slab: depth must be 1..2");
  if (n[a] < depth) return fail(CAV_EINVAL, "slab: block too thin for requested depth");
  for (int x = 0; x < 3; ++x) {
    out->lo[x] = 2;
    out->hi[x] = n[x] + 2;
  }
  if (!ghost) {
    out->lo[a] = high ? n[a] + 2 - depth : 2;
    out->hi[a] = high ? n[a] + 2 : 2 + depth;
  } else {
    out->lo[a] = high ? n[a] + 2 : 2 - depth;
    out->hi[a] = high ? n[a] + 2 + depth : 2;
  }
  return CAV_OK;
}

/* copy_box_to / copy_box_from (P/src/slab.cpp:51-71): k, then j, then a
 * contiguous i-row. */
void oc_copy_box_to(const double* f, int X, int Y, const cav_box* b, double* out) {
  const int w = b->hi[0] - b->lo[0];
  for (int k = b->lo[2]; k < b->hi[2]; ++k)
    for (int j = b->lo[1]; j < b->hi[1]; ++j, out += w)
      memcpy(out, f + b->lo[0] + (long)X * (j + (long)Y * k), (size_t)w * 8);
}

void oc_copy_box_from(double* f, int X, int Y, const cav_box* b, const double* in) {
  const int w = b->hi[0] - b->lo[0];
  for (int k = b->lo[2]; k < b->hi[2]; ++k)
    for (int j = b->lo[1]; j < b->hi[1]; ++j, in += w)
      memcpy(f + b->lo[0] + (long)X * (j + (long)Y * k), in, (size_t)w * 8);
}

/* ---- serial run: rank_main's loop for np = 1 (P/src/runner.cpp:150-251),
 * results bitwise-equal for every decomposition (P/README.md:10-15). */
static double now_s(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

int oc_run_serial(const cav_run_config* cfg, const cav_case_options* opt, cav_case_result* out) {
  const cav_fluid_params* fl = &cfg->fluid;
  if (!(fl->rho > 0) || !(fl->nu > 0) || !(fl->alpha > 0) || !(fl->u_ref > 0) || !(fl->length > 0))
    return fail(CAV_EINVAL, "params: non-positive constant");
  const int nx = cfg->nx, ny = cfg->ny, nz = cfg->nz;
  if (nx < 5 || ny < 5 || nz < 5) return fail(CAV_EINVAL, "grid: minimum is 5 nodes per axis");
  const double dx = fl->length / (nx - 1), dy = fl->length / (ny - 1), dz = fl->length / (nz - 1);
  const long X = nx + 4, Y = ny + 4, S = X * Y * (nz + 4);
  double* mem = (double*)malloc(sizeof(double) * (size_t)S * 10);
  if (!mem) return fail(CAV_ELENGTH, "fieldset: allocation failed");
  double* F[5];
  double* R[5];
  for (int v = 0; v < 5; ++v) {
    F[v] = mem + v * S;
    R[v] = mem + (5 + v) * S;
  }
  /* allocate_fieldset zero-fills; initialize_fields (P/src/solver.cpp:292-298) */
  memset(mem, 0, sizeof(double) * (size_t)S * 10);
  for (long c = 0; c < S; ++c) F[4][c] = fl->t_inf;

  const cav_field_ptrs in = {F[0], F[1], F[2], F[3], F[4]};
  const cav_residual_ptrs fw = {F[0], F[1], F[2], F[3], F[4]};
  const cav_field_ptrs rin = {R[0], R[1], R[2], R[3], R[4]};
  const cav_residual_ptrs rout = {R[0], R[1], R[2], R[3], R[4]};
  cav_stencil_params sp;
  oc_make_stencil_params(dx, dy, dz, fl, &sp);
  const int walls[6] = {1, 1, 1, 1, 1, 1};
  const cav_box whole = {{2, 2, 2}, {nx + 2, ny + 2, nz + 2}};
  const long long N = (long long)nx * ny * nz;
  const long cidx = ((nx - 1) / 2 + 2) + X * (((ny - 1) / 2 + 2) + Y * ((nz - 1) / 2 + 2));

  const int fixed = cfg->steps >= 0;
  const long long target = fixed ? cfg->steps : cfg->max_steps;
  const int cadence = cfg->check_every > 1 ? cfg->check_every : 1;
  const int want_hist = opt->collect_history || cfg->monitor_every > 0;
  double peaks[5] = {0, 0, 0, 0, 0};
  int converged = 0, status = CAV_OK;
  long long it = 0, nh = 0;
  double t0 = 0.0, seconds = 0.0;
  uint64_t limbs[350];
  while (it < target) {
    ++it;
    if (it == 2) t0 = now_s();
    oc_apply_bc(&fw, nx, ny, nz, walls, fl);
    oc_residual_box(&in, &rout, (int)X, (int)Y, &whole, &sp);
    const int check = (!fixed || want_hist) && (it == 1 || it % cadence == 0);
    if (check) {
      status = oc_norm_partials(&rin, nx, ny, nz, limbs);
      if (status) break;
      double l2[5];
      for (int v = 0; v < 5; ++v) l2[v] = sqrt(oc_repro_value(limbs + 70 * v) / (double)N);
      if (nh < out->hist_capacity) {
        out->hist_iter[nh] = it;
        for (int v = 0; v < 5; ++v) out->hist_l2[5 * nh + v] = l2[v];
      }
      ++nh;
      if (!fixed) {
        double worst = 0.0;
        for (int v = 0; v < 5; ++v) {
          peaks[v] = smax(peaks[v], l2[v]);
          if (peaks[v] > 0.0) worst = smax(worst, l2[v] / peaks[v]);
        }
        converged = worst <= cfg->conv_tol;
      }
    }
    double dt;
    status = oc_compute_dt(&in, nx, ny, nz, dx, dy, dz, fl, cfg->cfl, &dt);
    if (status) break;
    for (int v = 0; v < 5; ++v) oc_update_box(F[v], R[v], dt, (int)X, (int)Y, &whole);
    if (cfg->rescale) oc_rescale(F[0], nx, ny, nz, F[0][cidx]);
    if (converged) break;
  }
  if (status) {
    char msg[512];
    snprintf(msg, sizeof msg, "iteration %lld: %s", it, g_err);
    snprintf(g_err, sizeof g_err, "%s", msg);
    free(mem);
    return CAV_ERUNTIME;
  }
  if (it >= 2) seconds = now_s() - t0;
  out->steps_marched = it;
  out->steps_timed = it > 1 ? it - 1 : 0;
  out->converged = converged;
  out->np = 1;
  out->dims[0] = out->dims[1] = out->dims[2] = 1;
  out->wall_time_s = seconds;
  out->ssspnt = (out->steps_timed > 0 && seconds > 0.0)
                    ? 1e-7 * (double)N * (double)out->steps_timed / seconds
                    : NAN;
  out->bytes_sent = 0;
  out->hist_count = nh;
  if (out->ledgers && out->ledger_capacity > 0) memset(out->ledgers, 0, sizeof(cav_ledger));
  if (out->fields) {
    for (int v = 0; v < 5; ++v) {
      double* dst = out->fields + (size_t)v * (size_t)N;
      for (int k = 2; k < nz + 2; ++k)
        for (int j = 2; j < ny + 2; ++j, dst += nx) memcpy(dst, F[v] + 2 + X * (j + Y * k), (size_t)nx * 8);
    }
  }
  free(mem);
  return CAV_OK;
}
