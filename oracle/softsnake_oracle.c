/*
 * softsnake_oracle.c — TEST INFRASTRUCTURE ONLY.
 *
 * A scalar, single-environment CPU restatement of the reference hot path
 * (arXiv:1904.02833 softsnake 0.1.0, /root/reference/pkg/src/softsnake).
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference leg may load it; the product (paper_1904_02833_b200)
 * never links or calls it.
 *
 * Every function cites the reference file:line it restates. Floating-point
 * expressions keep the reference's evaluation order (compiled with
 * -ffp-contract=off so no FMA contraction), except:
 *   - numpy `@` dot products (BLAS ddot) are summed sequentially;
 *   - numpy.linalg.inv (LAPACK) is replaced by Gauss-Jordan with partial
 *     pivoting;
 * both agree with the reference to a few ulp (pinned by tests/golden).
 * Row layout, family order and contact compaction are the reference's.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "../include/softsnake_b200.h"

#define PSI_TO_PA 6894.76 /* pneumatics.py:23 */

typedef struct or_sim {
  /* topology (owned copies) */
  int P, nb, ndof, bd0, nd, nt, na, nh, nw, nq, nch, links, has_strain;
  double *inv_mass, *body_mass, *body_inertia;
  int32_t *pairs, *dchan;
  double *rest, *dcomp;
  int32_t *tets;
  double *rest_inv, *tcomp;
  int32_t *apart, *abody;
  double *anchor, *acomp;
  int32_t *hba, *hbb;
  double *ha, *hb, *hax, *ht1, *ht2, *hcomp;
  int32_t *wbody;
  double *wrad, *waxis;
  int32_t *cparts; /* [nq] */
  ss_params p;
  /* derived (solver.py:179-255) */
  double h, gamma;
  int od, ot, oa, oh, ms;
  int32_t *idx_d, *idx_t, *idx_a, *idx_h;
  double *eh2, *eh2_diag, *dyn_static;
  int n_act;
  int32_t *act_rows, *act_ch;
  /* state */
  double *pos, *vel, *bpos, *bquat, *blin, *bang;
  double *lam_d, *lam_t, *lam_a, *lam_h;
  double *quats, *dirs, *scale, *live, *target, *press;
  double *warm;
  int32_t *warm_valid;
  double time;
  /* work */
  double *res_d, *vals_d, *res_t, *vals_t, *res_a, *vals_a, *res_h, *vals_h;
  double *w, *u, *minv_diag, *ang_inv, *ang;
  /* stats of the last frame */
  int contact_count, inverted, newton, pcr;
  double residual;
} or_sim;

/* ------------------------------------------------------------------ util */
static void* dup(const void* src, size_t bytes) {
  if (bytes == 0) return calloc(1, 8);
  void* d = malloc(bytes);
  if (src) memcpy(d, src, bytes); else memset(d, 0, bytes);
  return d;
}
/* numpy.maximum semantics: NaN in a propagates */
static double npmax(double a, double b) { return (a >= b || a != a) ? a : b; }
static double seqdot(const double* a, const double* b, int n) {
  double s = 0.0;
  for (int i = 0; i < n; ++i) s += a[i] * b[i];
  return s;
}

/* 3x3 inverse, Gauss-Jordan with partial pivoting (stands in for
 * np.linalg.inv at state.py:262). */
static void inv3(const double* A, double* X) {
  double a[3][6];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 6; ++j) a[i][j] = j < 3 ? A[3 * i + j] : (j - 3 == i ? 1.0 : 0.0);
  for (int c = 0; c < 3; ++c) {
    int piv = c;
    for (int r = c + 1; r < 3; ++r)
      if (fabs(a[r][c]) > fabs(a[piv][c])) piv = r;
    if (piv != c)
      for (int j = 0; j < 6; ++j) { double t = a[c][j]; a[c][j] = a[piv][j]; a[piv][j] = t; }
    double d = a[c][c];
    for (int j = 0; j < 6; ++j) a[c][j] /= d;
    for (int r = 0; r < 3; ++r) {
      if (r == c) continue;
      double f = a[r][c];
      for (int j = 0; j < 6; ++j) a[r][j] -= f * a[c][j];
    }
  }
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) X[3 * i + j] = a[i][j + 3];
}

/* numpy_backend.py:91-104 / numba_backend.py:123-134 (no renormalisation) */
static void quat_to_mat(const double* q, double* R) {
  double w = q[0], x = q[1], y = q[2], z = q[3];
  R[0] = 1.0 - 2.0 * (y * y + z * z);
  R[1] = 2.0 * (x * y - w * z);
  R[2] = 2.0 * (x * z + w * y);
  R[3] = 2.0 * (x * y + w * z);
  R[4] = 1.0 - 2.0 * (x * x + z * z);
  R[5] = 2.0 * (y * z - w * x);
  R[6] = 2.0 * (x * z - w * y);
  R[7] = 2.0 * (y * z + w * x);
  R[8] = 1.0 - 2.0 * (x * x + y * y);
}
/* state.py:44-51 rotation_matrix = quat_normalize (state.py:16-21) + matrix */
static void rotation_matrix(const double* q, double* R) {
  double n = sqrt(seqdot(q, q, 4));
  double qn[4] = {1.0, 0.0, 0.0, 0.0};
  if (!(n < 1e-12))
    for (int k = 0; k < 4; ++k) qn[k] = q[k] / n;
  quat_to_mat(qn, R);
}
static void matvec3(const double* R, const double* v, double* o) {
  for (int i = 0; i < 3; ++i) o[i] = R[3 * i] * v[0] + R[3 * i + 1] * v[1] + R[3 * i + 2] * v[2];
}
/* np.einsum("nij,nj->ni") / ("ni,ni->n") contract length 3 as (p0+p2)+p1 */
static void matvec3_es(const double* R, const double* v, double* o) {
  for (int i = 0; i < 3; ++i) o[i] = R[3 * i] * v[0] + R[3 * i + 2] * v[2] + R[3 * i + 1] * v[1];
}
static double dot3_es(const double* a, const double* b) { return a[0] * b[0] + a[2] * b[2] + a[1] * b[1]; }
static void cross3(const double* a, const double* b, double* o) {
  o[0] = a[1] * b[2] - a[2] * b[1];
  o[1] = a[2] * b[0] - a[0] * b[2];
  o[2] = a[0] * b[1] - a[1] * b[0];
}

/* ---------------------------------------------------- backend kernels */
/* numba_backend.py:31-40 */
void or_block_forward(const int32_t* idx, const double* vals, int n, int r, int k,
                      const double* u, double* out) {
  for (int e = 0; e < n; ++e)
    for (int i = 0; i < r; ++i) {
      double acc = 0.0;
      for (int j = 0; j < k; ++j) acc += vals[((size_t)e * r + i) * k + j] * u[idx[(size_t)e * k + j]];
      out[(size_t)e * r + i] = acc;
    }
}
/* numba_backend.py:43-52 */
void or_block_transpose(const int32_t* idx, const double* vals, int n, int r, int k,
                        const double* x, double* y) {
  for (int e = 0; e < n; ++e)
    for (int j = 0; j < k; ++j) {
      double acc = 0.0;
      for (int i = 0; i < r; ++i) acc += vals[((size_t)e * r + i) * k + j] * x[(size_t)e * r + i];
      y[idx[(size_t)e * k + j]] += acc;
    }
}
/* numba_backend.py:55-65 */
void or_block_rowdiag(const int32_t* idx, const double* vals, int n, int r, int k,
                      const double* md, double* out) {
  for (int e = 0; e < n; ++e)
    for (int i = 0; i < r; ++i) {
      double acc = 0.0;
      for (int j = 0; j < k; ++j) {
        double v = vals[((size_t)e * r + i) * k + j];
        acc += v * v * md[idx[(size_t)e * k + j]];
      }
      out[(size_t)e * r + i] = acc;
    }
}
/* numba_backend.py:68-82 */
void or_minv_apply(const double* md, const double* ang_inv, int nb, int bd0,
                   const double* u, double* out, int ndof) {
  for (int i = 0; i < ndof; ++i) out[i] = md[i] * u[i];
  for (int b = 0; b < nb; ++b) {
    int o = bd0 + 6 * b + 3;
    double w0 = u[o], w1 = u[o + 1], w2 = u[o + 2];
    const double* A = ang_inv + 9 * b;
    out[o] = A[0] * w0 + A[1] * w1 + A[2] * w2;
    out[o + 1] = A[3] * w0 + A[4] * w1 + A[5] * w2;
    out[o + 2] = A[6] * w0 + A[7] * w1 + A[8] * w2;
  }
}
/* numba_backend.py:85-94 */
void or_ereg_apply(const double* v6, const double* x, double* out, int n) {
  for (int e = 0; e < n; ++e)
    for (int i = 0; i < 6; ++i) {
      double acc = 0.0;
      for (int j = 0; j < 6; ++j) acc += v6[(size_t)e * 36 + 6 * i + j] * x[(size_t)e * 6 + j];
      out[(size_t)e * 6 + i] = acc;
    }
}
/* numba_backend.py:105-120 */
void or_eval_distance(const double* pos, const int32_t* pairs, const double* rest,
                      const double* scale, double* dirs, double* res, int n) {
  for (int e = 0; e < n; ++e) {
    int i = pairs[2 * e], j = pairs[2 * e + 1];
    double dx = pos[3 * i] - pos[3 * j];
    double dy = pos[3 * i + 1] - pos[3 * j + 1];
    double dz = pos[3 * i + 2] - pos[3 * j + 2];
    double ln = sqrt(dx * dx + dy * dy + dz * dz);
    if (ln > 1e-12) {
      dirs[3 * e] = dx / ln;
      dirs[3 * e + 1] = dy / ln;
      dirs[3 * e + 2] = dz / ln;
    }
    res[e] = ln - rest[e] * scale[e];
  }
}
/* numba_backend.py:137-312; returns the inverted count, writes the polar
 * iteration count per element to iters (may be NULL). */
int or_eval_tetra(const double* pos, const int32_t* tets, const double* rest_inv,
                  double* quats, double tol, int maxiter, double* out_res,
                  double* out_vals, int n, int32_t* iters) {
  int n_inv = 0;
  for (int e = 0; e < n; ++e) {
    const int32_t* tv = tets + 4 * e;
    const double* Ri = rest_inv + 9 * e;
    double Ds[9], F[9], R[9], S[9], K[9], Ki[9], wv[12];
    for (int a = 0; a < 3; ++a) {
      Ds[3 * a + 0] = pos[3 * tv[1] + a] - pos[3 * tv[0] + a];
      Ds[3 * a + 1] = pos[3 * tv[2] + a] - pos[3 * tv[0] + a];
      Ds[3 * a + 2] = pos[3 * tv[3] + a] - pos[3 * tv[0] + a];
    }
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) {
        double acc = 0.0;
        for (int k = 0; k < 3; ++k) acc += Ds[3 * i + k] * Ri[3 * k + j];
        F[3 * i + j] = acc;
      }
    double detF = F[0] * (F[4] * F[8] - F[5] * F[7]) - F[1] * (F[3] * F[8] - F[5] * F[6]) +
                  F[2] * (F[3] * F[7] - F[4] * F[6]);
    if (detF <= 0.0) n_inv++;
    double qw = quats[4 * e], qx = quats[4 * e + 1], qy = quats[4 * e + 2], qz = quats[4 * e + 3];
    int it;
    for (it = 0; it < maxiter; ++it) {
      double r[9];
      double qq[4] = {qw, qx, qy, qz};
      quat_to_mat(qq, r);
      double o0 = 0.0, o1 = 0.0, o2 = 0.0, tr = 0.0;
      for (int j = 0; j < 3; ++j) {
        double rc0 = r[j], rc1 = r[3 + j], rc2 = r[6 + j];
        double f0 = F[j], f1 = F[3 + j], f2 = F[6 + j];
        o0 += rc1 * f2 - rc2 * f1;
        o1 += rc2 * f0 - rc0 * f2;
        o2 += rc0 * f1 - rc1 * f0;
        tr += rc0 * f0 + rc1 * f1 + rc2 * f2;
      }
      double s = 1.0 / (fabs(tr) + 1e-9);
      o0 *= s; o1 *= s; o2 *= s;
      double wn = sqrt(o0 * o0 + o1 * o1 + o2 * o2);
      if (wn < tol) break;
      double half = 0.5 * wn;
      double cw = cos(half);
      double sw = sin(half) / wn;
      double dw = cw, dx = sw * o0, dy = sw * o1, dz = sw * o2;
      double nw = dw * qw - dx * qx - dy * qy - dz * qz;
      double nx = dw * qx + dx * qw + dy * qz - dz * qy;
      double ny = dw * qy - dx * qz + dy * qw + dz * qx;
      double nz = dw * qz + dx * qy - dy * qx + dz * qw;
      double qn = sqrt(nw * nw + nx * nx + ny * ny + nz * nz);
      qw = nw / qn; qx = nx / qn; qy = ny / qn; qz = nz / qn;
    }
    if (iters) iters[e] = it;
    quats[4 * e] = qw; quats[4 * e + 1] = qx; quats[4 * e + 2] = qy; quats[4 * e + 3] = qz;
    quat_to_mat(quats + 4 * e, R);
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) {
        double acc = 0.0;
        for (int k = 0; k < 3; ++k) acc += R[3 * k + i] * F[3 * k + j];
        S[3 * i + j] = acc;
      }
    for (int i = 0; i < 3; ++i)
      for (int j = i + 1; j < 3; ++j) {
        double mm = 0.5 * (S[3 * i + j] + S[3 * j + i]);
        S[3 * i + j] = mm; S[3 * j + i] = mm;
      }
    double* rs = out_res + 6 * e;
    rs[0] = S[0] - 1.0; rs[1] = S[4] - 1.0; rs[2] = S[8] - 1.0;
    rs[3] = S[5]; rs[4] = S[2]; rs[5] = S[1];
    double trS = S[0] + S[4] + S[8];
    for (int i = 0; i < 3; ++i) {
      for (int j = 0; j < 3; ++j) K[3 * i + j] = -S[3 * i + j];
      K[4 * i] += trS + 1e-14;
    }
    double detK = K[0] * (K[4] * K[8] - K[5] * K[7]) - K[1] * (K[3] * K[8] - K[5] * K[6]) +
                  K[2] * (K[3] * K[7] - K[4] * K[6]);
    if (fabs(detK) < 1e-30) detK = detK >= 0 ? 1e-30 : -1e-30;
    double id = 1.0 / detK;
    Ki[0] = (K[4] * K[8] - K[5] * K[7]) * id;
    Ki[1] = (K[2] * K[7] - K[1] * K[8]) * id;
    Ki[2] = (K[1] * K[5] - K[2] * K[4]) * id;
    Ki[3] = (K[5] * K[6] - K[3] * K[8]) * id;
    Ki[4] = (K[0] * K[8] - K[2] * K[6]) * id;
    Ki[5] = (K[2] * K[3] - K[0] * K[5]) * id;
    Ki[6] = (K[3] * K[7] - K[4] * K[6]) * id;
    Ki[7] = (K[1] * K[6] - K[0] * K[7]) * id;
    Ki[8] = (K[0] * K[4] - K[1] * K[3]) * id;
    for (int j = 0; j < 3; ++j) {
      wv[3 + j] = Ri[j];
      wv[6 + j] = Ri[3 + j];
      wv[9 + j] = Ri[6 + j];
      wv[j] = -(wv[3 + j] + wv[6 + j] + wv[9 + j]);
    }
    double* ov = out_vals + 72 * (size_t)e;
    for (int v = 0; v < 4; ++v)
      for (int a = 0; a < 3; ++a) {
        double G[9];
        for (int i = 0; i < 3; ++i)
          for (int j = 0; j < 3; ++j) G[3 * i + j] = R[3 * a + i] * wv[3 * v + j];
        double g0 = G[7] - G[5], g1 = G[2] - G[6], g2 = G[3] - G[1];
        double w0 = Ki[0] * g0 + Ki[1] * g1 + Ki[2] * g2;
        double w1 = Ki[3] * g0 + Ki[4] * g1 + Ki[5] * g2;
        double w2 = Ki[6] * g0 + Ki[7] * g1 + Ki[8] * g2;
        int col = 3 * v + a;
        double ws00 = -w2 * S[3] + w1 * S[6];
        double ws01 = -w2 * S[4] + w1 * S[7];
        double ws02 = -w2 * S[5] + w1 * S[8];
        double ws10 = w2 * S[0] - w0 * S[6];
        double ws11 = w2 * S[1] - w0 * S[7];
        double ws12 = w2 * S[2] - w0 * S[8];
        double ws20 = -w1 * S[0] + w0 * S[3];
        double ws21 = -w1 * S[1] + w0 * S[4];
        double ws22 = -w1 * S[2] + w0 * S[5];
        ov[0 * 12 + col] = G[0] - ws00;
        ov[1 * 12 + col] = G[4] - ws11;
        ov[2 * 12 + col] = G[8] - ws22;
        ov[3 * 12 + col] = 0.5 * (G[5] + G[7]) - 0.5 * (ws12 + ws21);
        ov[4 * 12 + col] = 0.5 * (G[2] + G[6]) - 0.5 * (ws02 + ws20);
        ov[5 * 12 + col] = 0.5 * (G[1] + G[3]) - 0.5 * (ws01 + ws10);
      }
  }
  return n_inv;
}

/* ------------------------------------------------------- construction */
void or_destroy(or_sim* s);

or_sim* or_create(const ss_topology* t, const ss_params* p) {
  or_sim* s = (or_sim*)calloc(1, sizeof(or_sim));
  s->P = t->num_particles; s->nb = t->num_bodies;
  s->ndof = 3 * s->P + 6 * s->nb; s->bd0 = 3 * s->P;
  s->nd = t->n_dist; s->nt = t->n_tet; s->na = t->n_attach; s->nh = t->n_hinge;
  s->nw = t->n_wheel; s->nch = t->n_channels; s->links = s->nch / 2;
  s->has_strain = t->has_strain;
  s->p = *p;
  int P = s->P, nb = s->nb, nd = s->nd, nt = s->nt, na = s->na, nh = s->nh, nw = s->nw;
  s->inv_mass = dup(t->inv_mass, 8 * (size_t)P);
  s->body_mass = dup(t->body_mass, 8 * (size_t)nb);
  s->body_inertia = dup(t->body_inertia, 72 * (size_t)nb);
  s->pairs = dup(t->dist_pairs, 8 * (size_t)nd);
  s->rest = dup(t->dist_rest, 8 * (size_t)nd);
  s->dcomp = dup(t->dist_compliance, 8 * (size_t)nd);
  s->dchan = dup(t->dist_channel, 4 * (size_t)nd);
  s->tets = dup(t->tets, 16 * (size_t)nt);
  s->rest_inv = dup(t->tet_rest_inv, 72 * (size_t)nt);
  s->tcomp = dup(t->tet_compliance, 288 * (size_t)nt);
  s->apart = dup(t->attach_particle, 4 * (size_t)na);
  s->abody = dup(t->attach_body, 4 * (size_t)na);
  s->anchor = dup(t->attach_anchor, 24 * (size_t)na);
  s->acomp = dup(t->attach_compliance, 8 * (size_t)na);
  s->hba = dup(t->hinge_body_a, 4 * (size_t)nh);
  s->hbb = dup(t->hinge_body_b, 4 * (size_t)nh);
  s->ha = dup(t->hinge_anchor_a, 24 * (size_t)nh);
  s->hb = dup(t->hinge_anchor_b, 24 * (size_t)nh);
  s->hax = dup(t->hinge_axis_a, 24 * (size_t)nh);
  s->ht1 = dup(t->hinge_tan1_b, 24 * (size_t)nh);
  s->ht2 = dup(t->hinge_tan2_b, 24 * (size_t)nh);
  s->hcomp = dup(t->hinge_compliance, 8 * (size_t)nh);
  s->wbody = dup(t->wheel_body, 4 * (size_t)nw);
  s->wrad = dup(t->wheel_radius, 8 * (size_t)nw);
  s->waxis = dup(t->wheel_axis, 24 * (size_t)nw);
  if (t->contact_particles) {
    s->nq = t->n_contact_particles;
    s->cparts = dup(t->contact_particles, 4 * (size_t)s->nq);
  } else {
    s->nq = P;
    s->cparts = (int32_t*)malloc(4 * (size_t)(P ? P : 1));
    for (int i = 0; i < P; ++i) s->cparts[i] = i;
  }
  /* solver.py:187-232 */
  s->h = p->dt / p->substeps;
  double h = s->h;
  double dmp = p->constraint_damping > 0.0 ? p->constraint_damping : 0.0;
  s->gamma = 1.0 / (1.0 + dmp);
  s->od = 0; s->ot = nd; s->oa = nd + 6 * nt; s->oh = s->oa + 3 * na; s->ms = s->oh + 5 * nh;
  s->idx_d = malloc(4 * (size_t)(6 * nd + 1));
  for (int e = 0; e < nd; ++e)
    for (int a = 0; a < 3; ++a) {
      s->idx_d[6 * e + a] = 3 * s->pairs[2 * e] + a;
      s->idx_d[6 * e + 3 + a] = 3 * s->pairs[2 * e + 1] + a;
    }
  s->idx_t = malloc(4 * (size_t)(12 * nt + 1));
  for (int e = 0; e < nt; ++e)
    for (int v = 0; v < 4; ++v)
      for (int a = 0; a < 3; ++a) s->idx_t[12 * e + 3 * v + a] = 3 * s->tets[4 * e + v] + a;
  s->idx_a = malloc(4 * (size_t)(9 * na + 1));
  for (int e = 0; e < na; ++e) {
    for (int a = 0; a < 3; ++a) s->idx_a[9 * e + a] = 3 * s->apart[e] + a;
    for (int a = 0; a < 6; ++a) s->idx_a[9 * e + 3 + a] = s->bd0 + 6 * s->abody[e] + a;
  }
  s->idx_h = malloc(4 * (size_t)(12 * nh + 1));
  for (int e = 0; e < nh; ++e)
    for (int a = 0; a < 6; ++a) {
      s->idx_h[12 * e + a] = s->bd0 + 6 * s->hba[e] + a;
      s->idx_h[12 * e + 6 + a] = s->bd0 + 6 * s->hbb[e] + a;
    }
  s->eh2 = malloc(8 * (size_t)(36 * nt + 1));
  s->eh2_diag = malloc(8 * (size_t)(6 * nt + 1));
  for (int e = 0; e < nt; ++e)
    for (int k = 0; k < 36; ++k) s->eh2[36 * e + k] = s->gamma * s->tcomp[36 * e + k] / (h * h);
  for (int e = 0; e < nt; ++e)
    for (int i = 0; i < 6; ++i) s->eh2_diag[6 * e + i] = s->eh2[36 * e + 7 * i];
  s->dyn_static = calloc((size_t)s->ms + 1, 8);
  for (int e = 0; e < nd; ++e) s->dyn_static[s->od + e] = s->gamma * s->dcomp[e] / (h * h);
  for (int e = 0; e < na; ++e)
    for (int i = 0; i < 3; ++i) s->dyn_static[s->oa + 3 * e + i] = s->gamma * s->acomp[e] / (h * h);
  for (int e = 0; e < nh; ++e)
    for (int i = 0; i < 5; ++i) s->dyn_static[s->oh + 5 * e + i] = s->gamma * s->hcomp[e] / (h * h);
  /* actuated rows solver.py:241-248 */
  s->act_rows = malloc(4 * (size_t)(nd + 1));
  s->act_ch = malloc(4 * (size_t)(nd + 1));
  s->n_act = 0;
  if (nd && s->nch && s->has_strain)
    for (int e = 0; e < nd; ++e)
      if (s->dchan[e] >= 0) { s->act_rows[s->n_act] = e; s->act_ch[s->n_act] = s->dchan[e]; s->n_act++; }
  /* state defaults */
  s->pos = calloc(3 * (size_t)P + 1, 8); s->vel = calloc(3 * (size_t)P + 1, 8);
  s->bpos = calloc(3 * (size_t)nb + 1, 8); s->bquat = calloc(4 * (size_t)nb + 1, 8);
  for (int b = 0; b < nb; ++b) s->bquat[4 * b] = 1.0;
  s->blin = calloc(3 * (size_t)nb + 1, 8); s->bang = calloc(3 * (size_t)nb + 1, 8);
  s->lam_d = calloc((size_t)nd + 1, 8); s->lam_t = calloc(6 * (size_t)nt + 1, 8);
  s->lam_a = calloc(3 * (size_t)na + 1, 8); s->lam_h = calloc(5 * (size_t)nh + 1, 8);
  s->quats = calloc(4 * (size_t)nt + 1, 8);
  for (int e = 0; e < nt; ++e) s->quats[4 * e] = 1.0;
  s->dirs = calloc(3 * (size_t)nd + 1, 8);
  for (int e = 0; e < nd; ++e) s->dirs[3 * e] = 1.0;
  s->scale = calloc((size_t)nd + 1, 8);
  for (int e = 0; e < nd; ++e) s->scale[e] = 1.0;
  s->live = calloc((size_t)s->nch + 1, 8); s->target = calloc((size_t)s->nch + 1, 8);
  for (int c = 0; c < s->nch; ++c) { s->live[c] = 1.0; s->target[c] = 1.0; }
  s->press = calloc((size_t)s->nch + 1, 8);
  s->warm = calloc(3 * (size_t)nw + 1, 8);
  s->warm_valid = calloc((size_t)nw + 1, 4);
  /* work */
  s->res_d = calloc((size_t)nd + 1, 8); s->vals_d = calloc(6 * (size_t)nd + 1, 8);
  s->res_t = calloc(6 * (size_t)nt + 1, 8); s->vals_t = calloc(72 * (size_t)nt + 1, 8);
  s->res_a = calloc(3 * (size_t)na + 1, 8); s->vals_a = calloc(27 * (size_t)na + 1, 8);
  s->res_h = calloc(5 * (size_t)nh + 1, 8); s->vals_h = calloc(60 * (size_t)nh + 1, 8);
  s->w = calloc((size_t)s->ndof + 1, 8); s->u = calloc((size_t)s->ndof + 1, 8);
  s->minv_diag = calloc((size_t)s->ndof + 1, 8);
  s->ang_inv = calloc(9 * (size_t)nb + 1, 8); s->ang = calloc(9 * (size_t)nb + 1, 8);
  return s;
}

void or_destroy(or_sim* s) {
  if (!s) return;
  void* ptrs[] = {s->inv_mass, s->body_mass, s->body_inertia, s->pairs, s->rest, s->dcomp, s->dchan,
                  s->tets, s->rest_inv, s->tcomp, s->apart, s->abody, s->anchor, s->acomp, s->hba,
                  s->hbb, s->ha, s->hb, s->hax, s->ht1, s->ht2, s->hcomp, s->wbody, s->wrad,
                  s->waxis, s->cparts, s->idx_d, s->idx_t, s->idx_a, s->idx_h, s->eh2, s->eh2_diag,
                  s->dyn_static, s->act_rows, s->act_ch, s->pos, s->vel, s->bpos, s->bquat, s->blin,
                  s->bang, s->lam_d, s->lam_t, s->lam_a, s->lam_h, s->quats, s->dirs, s->scale,
                  s->live, s->target, s->press, s->warm, s->warm_valid, s->res_d, s->vals_d,
                  s->res_t, s->vals_t, s->res_a, s->vals_a, s->res_h, s->vals_h, s->w, s->u,
                  s->minv_diag, s->ang_inv, s->ang};
  for (size_t i = 0; i < sizeof(ptrs) / sizeof(ptrs[0]); ++i) free(ptrs[i]);
  free(s);
}

/* state I/O in the reference shapes (single env) */
#define CP(dst, src, cnt) do { if (src) memcpy(dst, src, 8 * (size_t)(cnt)); } while (0)
void or_set_state(or_sim* s, const ss_state_view* v) {
  CP(s->pos, v->positions, 3 * s->P); CP(s->vel, v->velocities, 3 * s->P);
  CP(s->bpos, v->body_pos, 3 * s->nb); CP(s->bquat, v->body_quat, 4 * s->nb);
  CP(s->blin, v->body_lin_vel, 3 * s->nb); CP(s->bang, v->body_ang_vel, 3 * s->nb);
  CP(s->lam_d, v->lam_dist, s->nd); CP(s->lam_t, v->lam_tetra, 6 * s->nt);
  CP(s->lam_a, v->lam_attach, 3 * s->na); CP(s->lam_h, v->lam_hinge, 5 * s->nh);
  CP(s->quats, v->tet_quats, 4 * s->nt); CP(s->dirs, v->dist_dirs, 3 * s->nd);
  CP(s->scale, v->dist_scale, s->nd); CP(s->live, v->strain_live, s->nch);
  CP(s->target, v->strain_target, s->nch); CP(s->press, v->pressures, s->nch);
  CP(s->warm, v->warm, 3 * s->nw);
  if (v->warm_valid) memcpy(s->warm_valid, v->warm_valid, 4 * (size_t)s->nw);
  if (v->time) s->time = v->time[0];
}
void or_get_state(const or_sim* s, ss_state_view* v) {
  CP(v->positions, s->pos, 3 * s->P); CP(v->velocities, s->vel, 3 * s->P);
  CP(v->body_pos, s->bpos, 3 * s->nb); CP(v->body_quat, s->bquat, 4 * s->nb);
  CP(v->body_lin_vel, s->blin, 3 * s->nb); CP(v->body_ang_vel, s->bang, 3 * s->nb);
  CP(v->lam_dist, s->lam_d, s->nd); CP(v->lam_tetra, s->lam_t, 6 * s->nt);
  CP(v->lam_attach, s->lam_a, 3 * s->na); CP(v->lam_hinge, s->lam_h, 5 * s->nh);
  CP(v->tet_quats, s->quats, 4 * s->nt); CP(v->dist_dirs, s->dirs, 3 * s->nd);
  CP(v->dist_scale, s->scale, s->nd); CP(v->strain_live, s->live, s->nch);
  CP(v->strain_target, s->target, s->nch); CP(v->pressures, s->press, s->nch);
  CP(v->warm, s->warm, 3 * s->nw);
  if (v->warm_valid) memcpy(v->warm_valid, s->warm_valid, 4 * (size_t)s->nw);
  if (v->time) v->time[0] = s->time;
}
void or_get_stats(const or_sim* s, ss_env_stats* st) {
  st->newton_iterations = s->newton; st->pcr_iterations = s->pcr;
  st->contact_count = s->contact_count; st->inverted_tets = s->inverted;
  st->residual = s->residual;
  int fin = 1;
  for (int i = 0; i < 3 * s->P; ++i) if (!isfinite(s->pos[i])) fin = 0;
  st->finite = fin; st->_pad = 0;
}

/* ------------------------------------------------------------ pneumatics */
/* pneumatics.py:62-72 (Python min/max semantics) */
double or_update_pressure(double p, double target, double ki, double kd, double cap, double ps) {
  if (target > p) {
    double dp = (target - p) / ps;
    double a = p + ps * dp * dp * ki;
    return target < a ? target : a;
  }
  if (target < p) {
    double dec = p * kd;
    double m = cap < dec ? cap : dec;
    double r = p - m;
    return r > 0.0 ? r : 0.0;
  }
  return p;
}
/* pneumatics.py:102-116 + solver.py:274-282 */
static void tick_channels(or_sim* s, const double* cmd, int latency) {
  for (int i = 0; i < s->links; ++i) {
    double a = cmd[i], left = 0.0, right = 0.0;
    if (a > 0.0) right = a;
    else if (a < 0.0) left = -a;
    if (latency) {
      s->press[2 * i] = or_update_pressure(s->press[2 * i], left, s->p.k_inflate, s->p.k_deflate, s->p.deflate_cap, s->p.supply);
      s->press[2 * i + 1] = or_update_pressure(s->press[2 * i + 1], right, s->p.k_inflate, s->p.k_deflate, s->p.deflate_cap, s->p.supply);
    } else {
      s->press[2 * i] = left;
      s->press[2 * i + 1] = right;
    }
  }
}

/* ---------------------------------------------------------------- step */
typedef struct { const int32_t* idx; const double* vals; int off, n, r, k; } fam_t;

typedef struct {
  or_sim* s;
  fam_t* fams; int nf;
  const double* dyn; const double* act; int m;
  double* xa; double* y;
} apply_ctx;

/* solver.py:380-399 */
static void apply_a(apply_ctx* c, const double* x, double* y) {
  or_sim* s = c->s;
  int m = c->m;
  const double* xa = x;
  if (c->act) {
    for (int i = 0; i < m; ++i) c->xa[i] = x[i] * c->act[i];
    xa = c->xa;
  }
  memset(s->w, 0, 8 * (size_t)s->ndof);
  for (int f = 0; f < c->nf; ++f) {
    fam_t* F = c->fams + f;
    or_block_transpose(F->idx, F->vals, F->n, F->r, F->k, xa + F->off, s->w);
  }
  or_minv_apply(s->minv_diag, s->ang_inv, s->nb, s->bd0, s->w, s->u, s->ndof);
  for (int f = 0; f < c->nf; ++f) {
    fam_t* F = c->fams + f;
    or_block_forward(F->idx, F->vals, F->n, F->r, F->k, s->u, y + F->off);
  }
  for (int i = 0; i < m; ++i) y[i] += c->dyn[i] * xa[i];
  if (s->nt) {
    double tmp[6];
    for (int e = 0; e < s->nt; ++e) {
      or_ereg_apply(s->eh2 + 36 * (size_t)e, xa + s->ot + 6 * e, tmp, 1);
      for (int i = 0; i < 6; ++i) y[s->ot + 6 * e + i] += tmp[i];
    }
  }
  if (c->act)
    for (int i = 0; i < m; ++i) {
      y[i] *= c->act[i];
      y[i] += (1.0 - c->act[i]) * x[i];
    }
}

/* solver.py:51-92 (x0 = None). Returns the last history entry. */
static double pcr_solve(apply_ctx* c, const double* rhs, const double* diag, int iters, double* x) {
  int m = c->m;
  double* d = malloc(8 * (size_t)(m + 1));
  double* r = malloc(8 * (size_t)(m + 1));
  double* z = malloc(8 * (size_t)(m + 1));
  double* az = malloc(8 * (size_t)(m + 1));
  double* p = malloc(8 * (size_t)(m + 1));
  double* ap = malloc(8 * (size_t)(m + 1));
  for (int i = 0; i < m; ++i) {
    d[i] = diag[i] > 1e-300 ? diag[i] : 1.0;
    x[i] = 0.0;
    r[i] = rhs[i];
    z[i] = r[i] / d[i];
  }
  apply_a(c, z, az);
  memcpy(p, z, 8 * (size_t)m);
  memcpy(ap, az, 8 * (size_t)m);
  double rho = seqdot(z, az, m);
  double rz = seqdot(r, z, m);
  double hist = sqrt(0.0 > rz ? 0.0 : rz); /* Python max(rz, 0.0) */
  for (int it = 0; it < iters; ++it) {
    double den = 0.0;
    for (int i = 0; i < m; ++i) den += ap[i] * (ap[i] / d[i]);
    if (den <= 1e-300 || !isfinite(den)) continue;
    double alpha = rho / den;
    for (int i = 0; i < m; ++i) {
      x[i] += alpha * p[i];
      r[i] -= alpha * ap[i];
      z[i] = r[i] / d[i];
    }
    rz = seqdot(r, z, m);
    hist = sqrt(0.0 > rz ? 0.0 : rz);
    apply_a(c, z, az);
    double rho_new = seqdot(z, az, m);
    double beta = rho > 1e-300 ? rho_new / rho : 0.0;
    rho = rho_new;
    for (int i = 0; i < m; ++i) {
      p[i] = z[i] + beta * p[i];
      ap[i] = az[i] + beta * ap[i];
    }
  }
  free(d); free(r); free(z); free(az); free(p); free(ap);
  return hist;
}

/* state.py:246-268 */
static void build_mass_inverse(or_sim* s) {
  for (int i = 0; i < s->P; ++i)
    for (int a = 0; a < 3; ++a) s->minv_diag[3 * i + a] = s->inv_mass[i];
  for (int b = 0; b < s->nb; ++b) {
    double R[9], RI[9], iw[9];
    rotation_matrix(s->bquat + 4 * b, R);
    const double* I = s->body_inertia + 9 * b;
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) {
        double acc = 0.0;
        for (int k = 0; k < 3; ++k) acc += R[3 * i + k] * I[3 * k + j];
        RI[3 * i + j] = acc;
      }
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) {
        double acc = 0.0;
        for (int k = 0; k < 3; ++k) acc += RI[3 * i + k] * R[3 * j + k];
        iw[3 * i + j] = acc;
      }
    memcpy(s->ang + 9 * b, iw, 72);
    inv3(iw, s->ang_inv + 9 * b);
    int o = s->bd0 + 6 * b;
    double im = 1.0 / s->body_mass[b];
    for (int a = 0; a < 3; ++a) {
      s->minv_diag[o + a] = im;
      s->minv_diag[o + 3 + a] = s->ang_inv[9 * b + 4 * a];
    }
  }
}

typedef struct { int wheel; int index; double point[3]; double gap; } contact_t;

/* contact.py:62-93 (normal (0,0,1); the friction basis is contact.py:20-32
 * evaluated at that normal: t1=(1,0,0), t2=(0,1,0)) */
static int detect_contacts(or_sim* s, contact_t* out) {
  int nc = 0;
  double gh = s->p.ground_height, margin = s->p.contact_margin;
  for (int k = 0; k < s->nw; ++k) {
    int b = s->wbody[k];
    const double* c = s->bpos + 3 * b;
    double R[9], axis[3];
    rotation_matrix(s->bquat + 4 * b, R);
    matvec3(R, s->waxis + 3 * k, axis);
    double nd = 0.0 * axis[0] + 0.0 * axis[1] + 1.0 * axis[2];
    double d[3] = {0.0 - nd * axis[0], 0.0 - nd * axis[1], 1.0 - nd * axis[2]};
    double dn = sqrt(seqdot(d, d, 3));
    if (dn < 1e-9) {
      d[0] = 1.0 - axis[0] * axis[0];
      d[1] = 0.0 - axis[0] * axis[1];
      d[2] = 0.0 - axis[0] * axis[2];
      dn = sqrt(seqdot(d, d, 3));
    }
    for (int a = 0; a < 3; ++a) d[a] = d[a] / dn;
    double pt[3];
    for (int a = 0; a < 3; ++a) pt[a] = c[a] - s->wrad[k] * d[a];
    double gap = pt[2] - gh;
    if (gap < margin) {
      contact_t* ct = out + nc++;
      ct->wheel = 1; ct->index = b; ct->gap = gap;
      memcpy(ct->point, pt, 24);
    }
  }
  for (int q = 0; q < s->nq; ++q) {
    int i = s->cparts[q];
    if (s->pos[3 * i + 2] - gh < margin) {
      contact_t* ct = out + nc++;
      ct->wheel = 0; ct->index = i;
      memcpy(ct->point, s->pos + 3 * i, 24);
      ct->gap = ct->point[2] - gh;
    }
  }
  return nc;
}

/* constraints.py:220-237 */
static void eval_attach(or_sim* s) {
  for (int e = 0; e < s->na; ++e) {
    int b = s->abody[e], pi = s->apart[e];
    double R[9], rw[3];
    quat_to_mat(s->bquat + 4 * b, R);
    matvec3_es(R, s->anchor + 3 * e, rw);
    for (int a = 0; a < 3; ++a) s->res_a[3 * e + a] = s->bpos[3 * b + a] + rw[a] - s->pos[3 * pi + a];
    double* v = s->vals_a + 27 * e;
    memset(v, 0, 27 * 8);
    for (int a = 0; a < 3; ++a) { v[9 * a + a] = -1.0; v[9 * a + 3 + a] = 1.0; }
    v[0 * 9 + 7] = rw[2]; v[0 * 9 + 8] = -rw[1];
    v[1 * 9 + 6] = -rw[2]; v[1 * 9 + 8] = rw[0];
    v[2 * 9 + 6] = rw[1]; v[2 * 9 + 7] = -rw[0];
  }
}
/* constraints.py:312-349 */
static void eval_hinge(or_sim* s) {
  for (int e = 0; e < s->nh; ++e) {
    int ba = s->hba[e], bb = s->hbb[e];
    double Ra[9], Rb[9], ra[3], rb[3], na[3], t1[3], t2[3], c1[3], c2[3];
    quat_to_mat(s->bquat + 4 * ba, Ra);
    quat_to_mat(s->bquat + 4 * bb, Rb);
    matvec3_es(Ra, s->ha + 3 * e, ra);
    matvec3_es(Rb, s->hb + 3 * e, rb);
    matvec3_es(Ra, s->hax + 3 * e, na);
    matvec3_es(Rb, s->ht1 + 3 * e, t1);
    matvec3_es(Rb, s->ht2 + 3 * e, t2);
    double* rs = s->res_h + 5 * e;
    for (int a = 0; a < 3; ++a) rs[a] = s->bpos[3 * ba + a] + ra[a] - s->bpos[3 * bb + a] - rb[a];
    rs[3] = dot3_es(t1, na);
    rs[4] = dot3_es(t2, na);
    double* v = s->vals_h + 60 * e;
    memset(v, 0, 60 * 8);
    for (int a = 0; a < 3; ++a) { v[12 * a + a] = 1.0; v[12 * a + 6 + a] = -1.0; }
    v[0 * 12 + 4] = ra[2]; v[0 * 12 + 5] = -ra[1];
    v[1 * 12 + 3] = -ra[2]; v[1 * 12 + 5] = ra[0];
    v[2 * 12 + 3] = ra[1]; v[2 * 12 + 4] = -ra[0];
    v[0 * 12 + 10] = -rb[2]; v[0 * 12 + 11] = rb[1];
    v[1 * 12 + 9] = rb[2]; v[1 * 12 + 11] = -rb[0];
    v[2 * 12 + 9] = -rb[1]; v[2 * 12 + 10] = rb[0];
    cross3(na, t1, c1);
    cross3(na, t2, c2);
    for (int a = 0; a < 3; ++a) {
      v[3 * 12 + 3 + a] = c1[a]; v[3 * 12 + 9 + a] = -c1[a];
      v[4 * 12 + 3 + a] = c2[a]; v[4 * 12 + 9 + a] = -c2[a];
    }
  }
}

/* solver.py:537-544 */
static void apply_impulse(or_sim* s, double* v, fam_t* fams, int nf, const double* dlam) {
  memset(s->w, 0, 8 * (size_t)s->ndof);
  for (int f = 0; f < nf; ++f)
    or_block_transpose(fams[f].idx, fams[f].vals, fams[f].n, fams[f].r, fams[f].k, dlam + fams[f].off, s->w);
  or_minv_apply(s->minv_diag, s->ang_inv, s->nb, s->bd0, s->w, s->u, s->ndof);
  for (int i = 0; i < s->ndof; ++i) v[i] += s->u[i];
}

static void pack_static_lambda(const or_sim* s, double* out) {
  memcpy(out + s->od, s->lam_d, 8 * (size_t)s->nd);
  memcpy(out + s->ot, s->lam_t, 48 * (size_t)s->nt);
  memcpy(out + s->oa, s->lam_a, 24 * (size_t)s->na);
  memcpy(out + s->oh, s->lam_h, 40 * (size_t)s->nh);
}

/* solver.py:334-523 */
static void substep(or_sim* s) {
  const ss_params* cfg = &s->p;
  double h = s->h;
  int P = s->P, nb = s->nb, ndof = s->ndof;
  /* _slew_actuation  solver.py:284-292 */
  if (s->n_act) {
    double dmax = cfg->max_strain_rate * h;
    for (int c = 0; c < s->nch; ++c) {
      double d = s->target[c] - s->live[c];
      if (d < -dmax) d = -dmax;
      if (d > dmax) d = dmax;
      s->live[c] += d;
    }
    for (int k = 0; k < s->n_act; ++k) s->scale[s->act_rows[k]] = s->live[s->act_ch[k]];
  }
  build_mass_inverse(s);
  /* _predict_velocities  solver.py:316-332 */
  double* v = malloc(8 * (size_t)(ndof + 1));
  double hg[3] = {h * cfg->gravity[0], h * cfg->gravity[1], h * cfg->gravity[2]};
  for (int i = 0; i < P; ++i)
    for (int a = 0; a < 3; ++a) {
      double vi = s->vel[3 * i + a];
      v[3 * i + a] = s->inv_mass[i] > 0.0 ? vi + hg[a] : vi;
    }
  for (int b = 0; b < nb; ++b) {
    double* t = v + s->bd0 + 6 * b;
    const double* w = s->bang + 3 * b;
    double iww[3], tau[3], it[3];
    for (int a = 0; a < 3; ++a) t[a] = s->blin[3 * b + a] + hg[a];
    matvec3_es(s->ang + 9 * b, w, iww);
    cross3(w, iww, tau);
    for (int a = 0; a < 3; ++a) tau[a] = -tau[a];
    matvec3_es(s->ang_inv + 9 * b, tau, it);
    for (int a = 0; a < 3; ++a) t[3 + a] = w[a] + h * it[a];
  }
  /* contacts */
  contact_t* cts = malloc(sizeof(contact_t) * (size_t)(s->nw + s->nq + 1));
  int nc = cfg->ground_enabled ? detect_contacts(s, cts) : 0;
  double* lam_n = calloc((size_t)nc + 1, 8);
  double* lam_f = calloc(2 * (size_t)nc + 1, 8);
  for (int k = 0; k < nc; ++k)
    if (cts[k].wheel)
      for (int w = 0; w < s->nw; ++w)
        if (s->wbody[w] == cts[k].index && s->warm_valid[w]) {
          lam_n[k] = s->warm[3 * w];
          lam_f[2 * k] = s->warm[3 * w + 1];
          lam_f[2 * k + 1] = s->warm[3 * w + 2];
          break;
        }
  int oc = s->ms, of = oc + nc, m = of + 2 * nc;
  /* families  solver.py:354-367 */
  fam_t fams[6];
  int nf = 0;
  if (s->nd) fams[nf++] = (fam_t){s->idx_d, s->vals_d, s->od, s->nd, 1, 6};
  if (s->nt) fams[nf++] = (fam_t){s->idx_t, s->vals_t, s->ot, s->nt, 6, 12};
  if (s->na) fams[nf++] = (fam_t){s->idx_a, s->vals_a, s->oa, s->na, 3, 9};
  if (s->nh) fams[nf++] = (fam_t){s->idx_h, s->vals_h, s->oh, s->nh, 5, 12};
  int32_t* cdof = calloc(6 * (size_t)nc + 1, 4);
  double* nvals = calloc(6 * (size_t)nc + 1, 8);
  double* fvals = calloc(12 * (size_t)nc + 1, 8);
  double* gaps = calloc((size_t)nc + 1, 8);
  if (nc) {
    /* contact.py:183-215 */
    static const double n[3] = {0.0, 0.0, 1.0}, t1[3] = {1.0, 0.0, 0.0}, t2[3] = {0.0, 1.0, 0.0};
    for (int k = 0; k < nc; ++k) {
      contact_t* c = cts + k;
      gaps[k] = c->gap;
      if (c->wheel) {
        int b = c->index, o = s->bd0 + 6 * b;
        for (int j = 0; j < 6; ++j) cdof[6 * k + j] = o + j;
        double r[3], cr[3];
        for (int a = 0; a < 3; ++a) r[a] = c->point[a] - s->bpos[3 * b + a];
        cross3(r, n, cr);
        for (int a = 0; a < 3; ++a) { nvals[6 * k + a] = n[a]; nvals[6 * k + 3 + a] = cr[a]; }
        cross3(r, t1, cr);
        for (int a = 0; a < 3; ++a) { fvals[12 * k + a] = t1[a]; fvals[12 * k + 3 + a] = cr[a]; }
        cross3(r, t2, cr);
        for (int a = 0; a < 3; ++a) { fvals[12 * k + 6 + a] = t2[a]; fvals[12 * k + 9 + a] = cr[a]; }
      } else {
        int i = c->index;
        for (int a = 0; a < 3; ++a) cdof[6 * k + a] = 3 * i + a;
        for (int a = 0; a < 3; ++a) {
          nvals[6 * k + a] = n[a];
          fvals[12 * k + a] = t1[a];
          fvals[12 * k + 6 + a] = t2[a];
        }
      }
    }
    fams[nf++] = (fam_t){cdof, nvals, oc, nc, 1, 6};
    fams[nf++] = (fam_t){cdof, fvals, of, nc, 2, 6};
  }
  double* dyn = calloc((size_t)m + 1, 8);
  memcpy(dyn, s->dyn_static, 8 * (size_t)s->ms);
  for (int i = of; i < m; ++i) dyn[i] = cfg->friction_compliance / (h * h);
  double* act = NULL;
  if (nc) {
    act = malloc(8 * (size_t)m);
    for (int i = 0; i < m; ++i) act[i] = 1.0;
  }
  /* assembly  solver.py:405-436 */
  if (s->nd) or_eval_distance(s->pos, s->pairs, s->rest, s->scale, s->dirs, s->res_d, s->nd);
  for (int e = 0; e < s->nd; ++e)
    for (int a = 0; a < 3; ++a) {
      s->vals_d[6 * e + a] = s->dirs[3 * e + a];
      s->vals_d[6 * e + 3 + a] = -s->dirs[3 * e + a];
    }
  if (s->nt)
    s->inverted += or_eval_tetra(s->pos, s->tets, s->rest_inv, s->quats, 1e-12, 500, s->res_t, s->vals_t, s->nt, NULL);
  if (s->na) eval_attach(s);
  if (s->nh) eval_hinge(s);
  double* base_diag = malloc(8 * (size_t)(m + 1));
  for (int f = 0; f < nf; ++f)
    or_block_rowdiag(fams[f].idx, fams[f].vals, fams[f].n, fams[f].r, fams[f].k, s->minv_diag, base_diag + fams[f].off);
  for (int i = 0; i < 6 * s->nt; ++i) base_diag[s->ot + i] += s->eh2_diag[i];
  double* rhs = malloc(8 * (size_t)(m + 1));
  double* jv = malloc(8 * (size_t)(m + 1));
  double* lam = calloc((size_t)m + 1, 8);
  double* lam_before = malloc(8 * (size_t)(m + 1));
  double* diag = malloc(8 * (size_t)(m + 1));
  double* dl = malloc(8 * (size_t)(m + 1));
  double* a2 = calloc(2 * (size_t)nc + 1, 8);
  pack_static_lambda(s, lam);
  memcpy(lam + oc, lam_n, 8 * (size_t)nc);
  memcpy(lam + of, lam_f, 16 * (size_t)nc);
  apply_impulse(s, v, fams, nf, lam);
  apply_ctx ctx = {s, fams, nf, dyn, act, m, malloc(8 * (size_t)(m + 1)), NULL};
  double g = s->gamma;
  double tmp[6];
  for (int itn = 0; itn < cfg->newton_iters; ++itn) {
    for (int f = 0; f < nf; ++f)
      or_block_forward(fams[f].idx, fams[f].vals, fams[f].n, fams[f].r, fams[f].k, v, jv + fams[f].off);
    for (int e = 0; e < s->nd; ++e) {
      int i = s->od + e;
      rhs[i] = -(g * s->res_d[e] / h + jv[i] + dyn[i] * s->lam_d[e]);
    }
    for (int e = 0; e < s->nt; ++e) {
      or_ereg_apply(s->eh2 + 36 * (size_t)e, s->lam_t + 6 * e, tmp, 1);
      for (int k = 0; k < 6; ++k) {
        int i = s->ot + 6 * e + k;
        rhs[i] = -(g * s->res_t[6 * e + k] / h + jv[i] + tmp[k]);
      }
    }
    for (int e = 0; e < 3 * s->na; ++e) {
      int i = s->oa + e;
      rhs[i] = -(g * s->res_a[e] / h + jv[i] + dyn[i] * s->lam_a[e]);
    }
    for (int e = 0; e < 5 * s->nh; ++e) {
      int i = s->oh + e;
      rhs[i] = -(g * s->res_h[e] / h + jv[i] + dyn[i] * s->lam_h[e]);
    }
    for (int k = 0; k < nc; ++k) {
      /* fischer_burmeister  solver.py:36-48, 463-472 */
      double a = gaps[k] / h + jv[oc + k];
      double b = lam_n[k];
      double root = sqrt(a * a + b * b + cfg->fb_delta);
      double phi = a + b - root;
      double da = 1.0 - a / root;
      double db = 1.0 - b / root;
      if (da < cfg->fb_slope_min) da = cfg->fb_slope_min;
      else if (da > cfg->fb_slope_max) da = cfg->fb_slope_max;
      rhs[oc + k] = -phi / da;
      dyn[oc + k] = db / da;
      double on = (cfg->mu * npmax(lam_n[k], 0.0) > 0.0) ? 1.0 : 0.0;
      for (int t = 0; t < 2; ++t) {
        int i = of + 2 * k + t;
        a2[2 * k + t] = on;
        act[i] = on;
        rhs[i] = -(on * (jv[i] + dyn[i] * lam_f[2 * k + t]));
      }
    }
    for (int i = 0; i < m; ++i) {
      diag[i] = npmax(base_diag[i] + dyn[i], 1e-30);
    }
    for (int k = 0; k < 2 * nc; ++k)
      if (!(a2[k] > 0.0)) diag[of + k] = 1.0;
    s->residual = pcr_solve(&ctx, rhs, diag, cfg->pcr_iters, dl);
    s->pcr += cfg->pcr_iters;
    /* multiplier update  solver.py:487-509 */
    memcpy(lam_before, lam, 8 * (size_t)m);
    for (int e = 0; e < s->nd; ++e) s->lam_d[e] += dl[s->od + e];
    for (int e = 0; e < 6 * s->nt; ++e) s->lam_t[e] += dl[s->ot + e];
    for (int e = 0; e < 3 * s->na; ++e) s->lam_a[e] += dl[s->oa + e];
    for (int e = 0; e < 5 * s->nh; ++e) s->lam_h[e] += dl[s->oh + e];
    for (int k = 0; k < nc; ++k) {
      lam_n[k] += dl[oc + k];
      lam_f[2 * k] += dl[of + 2 * k];
      lam_f[2 * k + 1] += dl[of + 2 * k + 1];
    }
    /* FrictionState.project  contact.py:157-165 */
    for (int k = 0; k < nc; ++k) {
      lam_n[k] = npmax(lam_n[k], 0.0);
      double rad = cfg->mu * npmax(lam_n[k], 0.0);
      double f0 = lam_f[2 * k], f1 = lam_f[2 * k + 1];
      double nrm = sqrt(f0 * f0 + f1 * f1);
      if (nrm > rad) {
        double sc = nrm > 0.0 ? rad / nrm : 0.0;
        lam_f[2 * k] *= sc;
        lam_f[2 * k + 1] *= sc;
      }
    }
    pack_static_lambda(s, lam);
    memcpy(lam + oc, lam_n, 8 * (size_t)nc);
    memcpy(lam + of, lam_f, 16 * (size_t)nc);
    for (int i = 0; i < m; ++i) lam_before[i] = lam[i] - lam_before[i];
    apply_impulse(s, v, fams, nf, lam_before);
    s->newton++;
  }
  /* state.set_velocities + integrate_pose  state.py:155-160, 187-192 */
  for (int i = 0; i < 3 * P; ++i) s->vel[i] = v[i];
  for (int b = 0; b < nb; ++b)
    for (int a = 0; a < 3; ++a) {
      s->blin[3 * b + a] = v[s->bd0 + 6 * b + a];
      s->bang[3 * b + a] = v[s->bd0 + 6 * b + 3 + a];
    }
  for (int i = 0; i < 3 * P; ++i) s->pos[i] += h * s->vel[i];
  for (int i = 0; i < 3 * nb; ++i) s->bpos[i] += h * s->blin[i];
  /* quat_step  state.py:171-184 */
  double ch = 0.5 * h;
  for (int b = 0; b < nb; ++b) {
    double* q = s->bquat + 4 * b;
    const double* w = s->bang + 3 * b;
    double r0 = q[0] - ch * (w[0] * q[1] + w[1] * q[2] + w[2] * q[3]);
    double r1 = q[1] + ch * (w[0] * q[0] + w[1] * q[3] - w[2] * q[2]);
    double r2 = q[2] + ch * (-w[0] * q[3] + w[1] * q[0] + w[2] * q[1]);
    double r3 = q[3] + ch * (w[0] * q[2] - w[1] * q[1] + w[2] * q[0]);
    double nrm = sqrt(r0 * r0 + r1 * r1 + r2 * r2 + r3 * r3);
    q[0] = r0 / nrm; q[1] = r1 / nrm; q[2] = r2 / nrm; q[3] = r3 / nrm;
  }
  s->time += h;
  /* store_warm  contact.py:167-180 */
  for (int w = 0; w < s->nw; ++w) s->warm_valid[w] = 0;
  for (int k = 0; k < nc; ++k)
    if (cts[k].wheel)
      for (int w = 0; w < s->nw; ++w)
        if (s->wbody[w] == cts[k].index) {
          s->warm_valid[w] = 1;
          s->warm[3 * w] = lam_n[k];
          s->warm[3 * w + 1] = lam_f[2 * k];
          s->warm[3 * w + 2] = lam_f[2 * k + 1];
        }
  s->contact_count += nc;
  free(v); free(cts); free(lam_n); free(lam_f); free(cdof); free(nvals); free(fvals); free(gaps);
  free(dyn); free(act); free(base_diag); free(rhs); free(jv); free(lam); free(lam_before);
  free(diag); free(dl); free(a2); free(ctx.xa);
}

/* Simulator.step  solver.py:296-314 */
void or_step(or_sim* s, const double* commands, int latency) {
  if (commands && s->nch) tick_channels(s, commands, latency);
  if (s->n_act)
    for (int c = 0; c < s->nch; ++c) s->target[c] = 1.0 + s->press[c] * PSI_TO_PA / s->p.strain_youngs;
  s->contact_count = 0; s->inverted = 0; s->newton = 0; s->pcr = 0; s->residual = 0.0;
  for (int k = 0; k < s->p.substeps; ++k) substep(s);
}

/* several frames with per-frame commands [frames, links] */
void or_run(or_sim* s, const double* commands, int latency, int frames) {
  for (int f = 0; f < frames; ++f) or_step(s, commands ? commands + (size_t)f * s->links : NULL, latency);
}

int or_sizeof_state_view(void) { return (int)sizeof(ss_state_view); }
int or_sizeof_topology(void) { return (int)sizeof(ss_topology); }
int or_sizeof_params(void) { return (int)sizeof(ss_params); }
