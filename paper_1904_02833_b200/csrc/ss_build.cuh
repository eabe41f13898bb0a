// ss_build.cuh — the link mesh of the scene builder (snake.py:97-189,
// constraints.py:128-137) as per-element functions shared by the device
// builder (ss_api.cu: ss_build_links) and a host C++ compile of the same
// code (tests: tools/build_check). Every float result is bitwise the
// reference's numpy result:
//  * rest inverse: np.linalg.inv = LAPACK dgesv(D, I) in OpenBLAS 0.3.30
//    (the numpy wheel's scipy-openblas, SkylakeX kernels): left-looking
//    getf2 (gemv tails as an FMA dot then one subtraction, dscal by the
//    reciprocal pivot), then getrs = laswp + trsm (unit lower: rows 0-1
//    solved with contracted updates, row 2 by a gemm dot; upper: row 2,
//    rows 0-1 by a gemm product, then the contracted 2x2 solve), the
//    diagonal applied as packed reciprocals;
//  * np.linalg.det = sign * exp(sum log|u_ii|) (numpy's slogdet path) with
//    glibc's log/exp, which are correctly rounded here: they are evaluated
//    in double-double arithmetic and rounded once;
//  * the cable rest length np.linalg.norm = sqrt(ddot) with the ddot tail
//    loop FMA-contracted.
// Checked against the reference topology digests (tests/test_builder.py).
#pragma once
#include <math.h>

#ifdef __CUDACC__
#define SSB_FN __host__ __device__ inline
#else
#define SSB_FN static inline
#endif

// ---------------------------------------------------- double-double
struct ssb_dd {
  double hi, lo;
};
SSB_FN ssb_dd ssb_two_sum(double a, double b) {
  const double s = a + b;
  const double bb = s - a;
  return ssb_dd{s, (a - (s - bb)) + (b - bb)};
}
SSB_FN ssb_dd ssb_fast_two_sum(double a, double b) {
  const double s = a + b;
  return ssb_dd{s, b - (s - a)};
}
SSB_FN ssb_dd ssb_two_prod(double a, double b) {
  const double p = a * b;
  return ssb_dd{p, fma(a, b, -p)};
}
SSB_FN ssb_dd ssb_add(ssb_dd a, ssb_dd b) {
  ssb_dd s = ssb_two_sum(a.hi, b.hi);
  ssb_dd t = ssb_two_sum(a.lo, b.lo);
  s.lo += t.hi;
  s = ssb_fast_two_sum(s.hi, s.lo);
  s.lo += t.lo;
  return ssb_fast_two_sum(s.hi, s.lo);
}
SSB_FN ssb_dd ssb_mul(ssb_dd a, ssb_dd b) {
  ssb_dd p = ssb_two_prod(a.hi, b.hi);
  p.lo += a.hi * b.lo + a.lo * b.hi;
  return ssb_fast_two_sum(p.hi, p.lo);
}
SSB_FN ssb_dd ssb_mul_d(ssb_dd a, double b) {
  ssb_dd p = ssb_two_prod(a.hi, b);
  p.lo += a.lo * b;
  return ssb_fast_two_sum(p.hi, p.lo);
}

// exp(x) in double-double (relative error ~1e-31): x = k ln2 + r,
// exp(r / 16) by its Taylor series, squared four times
SSB_FN ssb_dd ssb_exp_dd(ssb_dd x) {
  const double ln2_hi = 6.93147180559945286227e-01, ln2_lo = 2.31904681384629955842e-17;
  const double k = rint(x.hi / ln2_hi);
  ssb_dd r = ssb_add(x, ssb_two_prod(-k, ln2_hi));
  r = ssb_add(r, ssb_two_prod(-k, ln2_lo));
  r.hi *= 0.0625;
  r.lo *= 0.0625;
  // Horner: 1 + r (1 + r/2 (1 + r/3 (... (1 + r/14))))
  ssb_dd s{1.0, 0.0};
  for (int n = 14; n >= 1; --n) {
    ssb_dd q = ssb_mul(s, r);
    // q / n in double-double
    const double qh = q.hi / n;
    ssb_dd back = ssb_two_prod(qh, (double)n);
    const double ql = ((q.hi - back.hi) - back.lo + q.lo) / n;
    s = ssb_add(ssb_dd{1.0, 0.0}, ssb_fast_two_sum(qh, ql));
  }
  for (int i = 0; i < 4; ++i) s = ssb_mul(s, s);
  const double sc = ldexp(1.0, (int)k);
  return ssb_dd{s.hi * sc, s.lo * sc};
}
// exp(x) rounded to nearest (round the double-double once)
SSB_FN double ssb_exp_cr(double x) {
  const ssb_dd e = ssb_exp_dd(ssb_dd{x, 0.0});
  return e.hi + e.lo;
}
// log(x) rounded to nearest: one Newton step y + x exp(-y) - 1 from the
// library log, in double-double
SSB_FN double ssb_log_cr(double x) {
  const double y0 = log(x);
  const ssb_dd e = ssb_exp_dd(ssb_dd{-y0, 0.0});
  ssb_dd t = ssb_mul_d(e, x);
  t = ssb_add(t, ssb_dd{-1.0, 0.0});
  const ssb_dd y = ssb_add(ssb_dd{y0, 0.0}, t);
  return y.hi + y.lo;
}

// ------------------------------------------------ 3x3 inverse + det
// D row-major [r][c]; X row-major inverse; returns np.linalg.det(D)
SSB_FN double ssb_inv_det3(const double* D, double* X) {
  double A[3][3];  // column-major like LAPACK: A[col][row]
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) A[c][r] = D[3 * r + c];
  int ipiv[3];
  for (int j = 0; j < 3; ++j) {
    double* b = A[j];
    for (int i = 0; i < j; ++i) {
      const int ip = ipiv[i];
      if (ip != i) {
        const double t = b[i];
        b[i] = b[ip];
        b[ip] = t;
      }
    }
    for (int i = 1; i < j; ++i) {
      double dot = A[0][i] * b[0];
      for (int k = 1; k < i; ++k) dot = fma(A[k][i], b[k], dot);
      b[i] -= dot;
    }
    if (j > 0)
      for (int r = j; r < 3; ++r) {
        double t = A[0][r] * b[0];
        for (int k = 1; k < j; ++k) t = fma(A[k][r], b[k], t);
        b[r] = b[r] - t;
      }
    int jp = j;
    double mx = fabs(b[j]);
    for (int r = j + 1; r < 3; ++r)
      if (fabs(b[r]) > mx) {
        mx = fabs(b[r]);
        jp = r;
      }
    ipiv[j] = jp;
    const double p = b[jp];
    if (jp != j)
      for (int c = 0; c <= j; ++c) {
        const double t = A[c][j];
        A[c][j] = A[c][jp];
        A[c][jp] = t;
      }
    const double rp = 1.0 / p;
    for (int r = j + 1; r < 3; ++r) b[r] = b[r] * rp;
  }
  const double i22 = 1.0 / A[2][2], i11 = 1.0 / A[1][1], i00 = 1.0 / A[0][0];
  for (int col = 0; col < 3; ++col) {
    double c[3] = {0.0, 0.0, 0.0};
    c[col] = 1.0;
    for (int i = 0; i < 3; ++i) {
      const int ip = ipiv[i];
      if (ip != i) {
        const double t = c[i];
        c[i] = c[ip];
        c[ip] = t;
      }
    }
    c[1] = fma(-c[0], A[0][1], c[1]);
    {
      double acc = A[0][2] * c[0];
      acc = fma(A[1][2], c[1], acc);
      c[2] = c[2] - acc;
    }
    c[2] = c[2] * i22;
    c[0] = c[0] - A[2][0] * c[2];
    c[1] = c[1] - A[2][1] * c[2];
    c[1] = c[1] * i11;
    c[0] = fma(-c[1], A[1][0], c[0]);
    c[0] = c[0] * i00;
    for (int r = 0; r < 3; ++r) X[3 * r + col] = c[r];
  }
  // numpy det: sign from the pivots and the diagonal, exp of the log sum
  double sign = 1.0, logdet = 0.0;
  for (int j = 0; j < 3; ++j) {
    if (ipiv[j] != j) sign = -sign;
    double u = A[j][j];
    if (u < 0) {
      sign = -sign;
      u = -u;
    }
    logdet += ssb_log_cr(u);
  }
  return sign * ssb_exp_cr(logdet);
}

// np.linalg.norm of a 3-vector: sqrt(ddot), tail loop contracted
SSB_FN double ssb_norm3(double x, double y, double z) {
  double d = x * x;
  d = fma(y, y, d);
  d = fma(z, z, d);
  return sqrt(d);
}

#ifdef __CUDACC__
// ------------------------------------------------------ device builder
// One grid per array family; every link of every snake at once (links are
// laid out consecutively, particle base = link * NP, snake.py:308-320).
struct SsbLink {
  int S, W, H, L;                  // grid nodes per link, links
  double dx, dy, dz, hw;           // steps, half width (snake.py:103-105, 113-114)
  double E, nu, rho;               // youngs, poisson, density
  double c_act, c_inext, c_struct; // cable compliances
  const double* origin;            // [L][3]
  const int* chan;                 // [L][2] left, right
  int NP, NT, NC;                  // per link
};
// snake.py:37-50 five-tet split (corner offsets di, dj, dk)
__constant__ int ssb_cell[2][5][4][3] = {
    {{{0, 0, 0}, {1, 0, 0}, {0, 1, 0}, {0, 0, 1}},
     {{1, 1, 0}, {0, 1, 0}, {1, 0, 0}, {1, 1, 1}},
     {{1, 0, 1}, {0, 0, 1}, {1, 1, 1}, {1, 0, 0}},
     {{0, 1, 1}, {1, 1, 1}, {0, 0, 1}, {0, 1, 0}},
     {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}, {1, 1, 1}}},
    {{{1, 0, 0}, {0, 0, 0}, {1, 1, 0}, {1, 0, 1}},
     {{0, 1, 0}, {1, 1, 0}, {0, 0, 0}, {0, 1, 1}},
     {{0, 0, 1}, {1, 0, 1}, {0, 1, 1}, {0, 0, 0}},
     {{1, 1, 1}, {0, 1, 1}, {1, 0, 1}, {1, 1, 0}},
     {{0, 0, 0}, {1, 1, 0}, {1, 0, 1}, {0, 1, 1}}}};

// rest position of local node (i, j, k) of link l: origin + [i dx, j dy - hw, k dz]
__device__ inline void ssb_pos(const SsbLink& g, int l, int i, int j, int k, double* x) {
  const double* o = g.origin + 3 * l;
  x[0] = o[0] + (double)i * g.dx;
  x[1] = o[1] + ((double)j * g.dy - g.hw);
  x[2] = o[2] + (double)k * g.dz;
}

__global__ void ssb_k_particles(const SsbLink g, double* pos) {
  const long n = (long)g.L * g.NP;
  for (long p = blockIdx.x * (long)blockDim.x + threadIdx.x; p < n; p += (long)gridDim.x * blockDim.x) {
    const int l = (int)(p / g.NP), q = (int)(p % g.NP);
    const int i = q / (g.W * g.H), j = (q / g.H) % g.W, k = q % g.H;
    ssb_pos(g, l, i, j, k, pos + 3 * p);
  }
}

// TetraElement.from_positions (constraints.py:128-137) + tetra_compliance
// (constraints.py:26-40); bad[0] counts degenerate tets
__global__ void ssb_k_tets(const SsbLink g, int* tets, double* rinv, double* vol, double* comp,
                           int* bad) {
  const long n = (long)g.L * g.NT;
  const int cw = g.W - 1, chh = g.H - 1;
  for (long t = blockIdx.x * (long)blockDim.x + threadIdx.x; t < n; t += (long)gridDim.x * blockDim.x) {
    const int l = (int)(t / g.NT), r = (int)(t % g.NT);
    const int cell = r / 5, s = r % 5;
    const int ci = cell / (cw * chh), cj = (cell / chh) % cw, ck = cell % chh;
    const int par = (ci + cj + ck) % 2;
    double x[4][3];
    for (int v = 0; v < 4; ++v) {
      const int i = ci + ssb_cell[par][s][v][0], j = cj + ssb_cell[par][s][v][1],
                k = ck + ssb_cell[par][s][v][2];
      tets[4 * t + v] = l * g.NP + (i * g.W + j) * g.H + k;
      ssb_pos(g, l, i, j, k, x[v]);
    }
    double D[9];
    for (int a = 0; a < 3; ++a)
      for (int c = 0; c < 3; ++c) D[3 * a + c] = x[c + 1][a] - x[0][a];
    double X[9];
    const double det = ssb_inv_det3(D, X);
    if (fabs(det) < 1e-18) atomicAdd(bad, 1);
    const double v6 = fabs(det) / 6.0;
    for (int q = 0; q < 9; ++q) rinv[9 * t + q] = X[q];
    vol[t] = v6;
    const double c = 1.0 / (v6 * g.E);
    const double nu = g.nu;
    double* C = comp + 36 * t;
    for (int q = 0; q < 36; ++q) C[q] = 0.0;
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) C[6 * a + b] = c * (a == b ? 1.0 : -nu);
    const double sh = c * (1.0 + nu);
    C[21] = sh;
    C[28] = sh;
    C[35] = sh;
  }
}

// lumped masses: rho V / 4 per tet corner, accumulated per node in tet order
// (snake.py:130, np.add.at); the cells around the node in lexicographic
// order, five tets each, give ascending tet ids
__global__ void ssb_k_masses(const SsbLink g, const double* vol, double* mass) {
  const long n = (long)g.L * g.NP;
  const int cw = g.W - 1, chh = g.H - 1;
  for (long p = blockIdx.x * (long)blockDim.x + threadIdx.x; p < n; p += (long)gridDim.x * blockDim.x) {
    const int l = (int)(p / g.NP), q = (int)(p % g.NP);
    const int i = q / (g.W * g.H), j = (q / g.H) % g.W, k = q % g.H;
    double m = 0.0;
    for (int ci = i - 1; ci <= i; ++ci) {
      if (ci < 0 || ci >= g.S - 1) continue;
      for (int cj = j - 1; cj <= j; ++cj) {
        if (cj < 0 || cj >= cw) continue;
        for (int ck = k - 1; ck <= k; ++ck) {
          if (ck < 0 || ck >= chh) continue;
          const int par = (ci + cj + ck) % 2;
          const int cell = (ci * cw + cj) * chh + ck;
          for (int s = 0; s < 5; ++s)
            for (int v = 0; v < 4; ++v)
              if (ci + ssb_cell[par][s][v][0] == i && cj + ssb_cell[par][s][v][1] == j &&
                  ck + ssb_cell[par][s][v][2] == k)
                m += g.rho * vol[(long)l * g.NT + 5 * cell + s] / 4.0;
        }
      }
    }
    mass[p] = m;
  }
}

// the cable list of one link in the reference order (snake.py:136-176):
// chamber cables, spine, perimeter rings, cross braces
__device__ inline void ssb_cable(const SsbLink& g, int l, int c, int* a, int* b, double* comp,
                                 int* kind, int* ch) {
  const int S = g.S, W = g.W, H = g.H;
  auto lid = [&](int i, int j, int k) { return (i * W + j) * H + k; };
  *ch = -1;
  if (c < 2 * H) {  // chambers: (j = 0, right), (j = W-1, left)
    const int side = c / H, k = c % H;
    const int j = side == 0 ? 0 : W - 1;
    *a = lid(0, j, k);
    *b = lid(S - 1, j, k);
    *comp = g.c_act;
    *kind = 1;
    *ch = side == 0 ? g.chan[2 * l + 1] : g.chan[2 * l];
    return;
  }
  c -= 2 * H;
  if (c < H * (S - 1)) {  // spine
    const int k = c / (S - 1), i = c % (S - 1), jc = W / 2;
    *a = lid(i, jc, k);
    *b = lid(i + 1, jc, k);
    *comp = g.c_inext;
    *kind = 2;
    return;
  }
  c -= H * (S - 1);
  const int per_ring = 2 * (W - 1) + 2 * (H - 1);
  const int n_ring = S - S / 3 - (S % 3 >= 2 ? 1 : 0);  // sections with i % 3 != 1
  if (c < n_ring * per_ring) {
    const int rs = c / per_ring;
    int q = c % per_ring;
    // the rs-th section with i % 3 != 1: 0, 2, 3, 5, 6, ...
    const int i = rs == 0 ? 0 : (rs % 2 == 1 ? 3 * ((rs + 1) / 2) - 1 : 3 * (rs / 2));
    *comp = g.c_struct;
    *kind = 0;
    if (q < 2 * (W - 1)) {
      const int k = q < W - 1 ? 0 : H - 1, j = q % (W - 1);
      *a = lid(i, j, k);
      *b = lid(i, j + 1, k);
    } else {
      q -= 2 * (W - 1);
      const int j = q < H - 1 ? 0 : W - 1, k = q % (H - 1);
      *a = lid(i, j, k);
      *b = lid(i, j, k + 1);
    }
    return;
  }
  c -= n_ring * per_ring;  // braces: 4 per section
  const int i = c / 4, q = c % 4;
  const int j0 = q < 2 ? 0 : W - 1, j1 = q < 2 ? 2 : W - 3;
  *comp = g.c_struct;
  *kind = 0;
  if (q % 2 == 0) {
    *a = lid(i, j0, 0);
    *b = lid(i, j1, H - 1);
  } else {
    *a = lid(i, j0, H - 1);
    *b = lid(i, j1, 0);
  }
}

__global__ void ssb_k_cables(const SsbLink g, int* pairs, double* rest, double* comp, int* kind,
                             int* chan, int* mounts) {
  const long n = (long)g.L * g.NC;
  for (long t = blockIdx.x * (long)blockDim.x + threadIdx.x; t < n; t += (long)gridDim.x * blockDim.x) {
    const int l = (int)(t / g.NC), c = (int)(t % g.NC);
    int a, b, kd, ch;
    double cp;
    ssb_cable(g, l, c, &a, &b, &cp, &kd, &ch);
    double xa[3], xb[3];
    ssb_pos(g, l, a / (g.W * g.H), (a / g.H) % g.W, a % g.H, xa);
    ssb_pos(g, l, b / (g.W * g.H), (b / g.H) % g.W, b % g.H, xb);
    pairs[2 * t] = l * g.NP + a;
    pairs[2 * t + 1] = l * g.NP + b;
    rest[t] = ssb_norm3(xa[0] - xb[0], xa[1] - xb[1], xa[2] - xb[2]);
    comp[t] = cp;
    kind[t] = kd;
    chan[t] = ch;
  }
  // frame mounts (snake.py:184-187): j in (0, W/2, W-1) x k in (0, H-1),
  // start face then end face; [L][2][6]
  for (long t = blockIdx.x * (long)blockDim.x + threadIdx.x; t < 12L * g.L; t += (long)gridDim.x * blockDim.x) {
    const int l = (int)(t / 12), face = (int)(t % 12) / 6, m = (int)(t % 6);
    const int js[3] = {0, g.W / 2, g.W - 1};
    const int j = js[m / 2], k = m % 2 == 0 ? 0 : g.H - 1;
    const int i = face == 0 ? 0 : g.S - 1;
    mounts[t] = l * g.NP + (i * g.W + j) * g.H + k;
  }
}
#endif
