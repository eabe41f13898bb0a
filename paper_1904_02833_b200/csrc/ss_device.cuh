// ss_device.cuh — data model and step kernels of the B200 soft-snake step.
//
// Layout: every per-environment array is [item][E] with the environment
// index innermost (E = padded env count). A CUDA block is W env-lanes x IL
// item-lanes (W*IL = 256, W = min(E, 32)), so with E >= 32 a warp covers
// 32 environments of ONE constraint: topology loads are warp-uniform
// broadcasts and every state/J load is a coalesced 256-byte line; with E = 1
// a warp covers 32 consecutive items of the single environment (item-major,
// still coalesced). One code path serves the batched and single-env cases.
//
// Arithmetic restates the reference (softsnake/solver.py, constraints.py,
// contact.py, state.py, kernels/numba_backend.py) with its evaluation order;
// the library is compiled with --fmad=false so no FMA contraction changes a
// rounding. Scatter-free J^T x: per DOF, an incidence list sorted in the
// reference's accumulation order (family order of solver.py:354-367, element
// ascending, column ascending; numba_backend.py:43-52) is gathered, so the
// sums are bitwise the numba block_transpose sums. PCR scalars are per
// environment, reduced deterministically (fixed tree + fixed block order).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#define DI __device__ __forceinline__
#define SS_PSI_TO_PA 6894.76  // pneumatics.py:23
#define SS_THREADS 256

// incidence families (code bits 29..31)
enum { F_DIST = 0, F_TET = 1, F_ATTP = 2, F_ATTB = 3, F_HINGE = 4, F_CN = 5, F_CF = 6 };

struct Dims {
  int E, W, lgW, tiles, n_real;
  int P, nb, ndof, bd0, nd, nt, na, nh, nw, nq, ns, nch, links;
  int ms, m, od, ot, oa, oh, on, of;
  int act_enabled;
  int tc_inbox, n_inc;  // tet column sums in incidence order (E = 1), incidences
};

struct Par {
  double h, gamma, hg[3], ground_h, margin, mu, fdyn, fb_delta, smin, smax, dmax;
  double youngs, ki, kd, cap, supply, half_h, dt;
  int newton, pcr, substeps, exact_j;
};

// scene topology, shared by every environment (item-indexed only)
struct Topo {
  const double *inv_mass, *body_inv_mass, *body_inertia;         // [P] [nb] [nb*9]
  const int *d_i, *d_j, *d_chan;                                  // [nd]
  const double *d_rest, *d_dyn;                                   // [nd]
  const int* t_idx;                                               // [4][nt]
  const double *t_rinv, *t_e3;                                    // [nt][10] (9 + pad) [3][nt]
  const int *a_p, *a_b;                                           // [na]
  const double *a_anc, *a_dyn;                                    // [3][na] [na]
  const int *h_a, *h_b;                                           // [nh]
  const double *h_anca, *h_ancb, *h_axa, *h_t1, *h_t2, *h_dyn;    // [3][nh] ... [nh]
  const int* w_body;                                              // [nw]
  const double *w_rad, *w_axis;                                   // [nw] [3][nw]
  const int* slot_part;                                           // [nq]
  const int *inc_ptr, *inc;                                       // [P+nb+1], codes
  const int2* inc_tet;                                            // [P] tet run [begin, end)
  const int* tdst;                                                // [nt][4] incidence of each tet vertex
};

// persistent per-environment state, [item][E]
struct State {
  double *pos, *vel;                    // [3P]
  double *bpos, *bquat, *blin, *bang;   // [3nb] [4nb] [3nb] [3nb]
  double* lam;                          // [ms] internal row order
  double *quat, *dirs, *scale;          // [4][nt] [3][nd] [nd]
  double *live, *target, *press;        // [nch]
  double* warm;                         // [3][nw]
  int* warm_valid;                      // [nw]
  double* time;                         // [1]
  // per-frame statistics (StepStats, solver.py:142-151), per env
  double* resid;                        // [1]
  int *nc_cnt, *inv_cnt, *nonfinite;    // [1]
  // on-device gait generator (snake.py:235-241): [6] = amplitude psi,
  // angular rate rad/s, phase offset, turn bias, time offset t0, links per
  // snake; gait_frame = frames stepped since ss_set_gait
  double* gait;                         // [6]
  int* gait_frame;                      // [1]
};

// per-substep workspace, [item][E]
struct Work {
  double *v, *u;            // [ndof]
  double* ang_inv;          // [9][nb]
  double* res;              // [ms] (tet rows unused: derived from S)
  double* tS;               // [6][nt] compact tet Jacobian sym(R^T F) (R from S.quat)
  double* tC;               // [12][nt] per-tet J^T x column sums (gather input)
  double* rw;               // [3][na]
  double* hJ;               // [60][nh]
  double* wJ;               // [18][nw]  normal(6), friction0(6), friction1(6)
  int* present;             // [ns]
  double *gap, *actf, *dynn; // [ns]
  double* lamc;             // [3ns] contact multipliers in contact-row order
  double* bdiag;            // [m]
  double *x, *r, *z, *p, *ap, *az, *d;  // [m]
  double* part;             // [gy_red][E]
  int* cnt;                 // [tiles]
  double *rho, *alpha, *beta;  // [E]
  double* alpha_prev;           // [E] alpha of the previous PCR iteration (deferred x update)
  int* last_step;               // [E] index of the last executed k_pcr_step (-1: none)
  int* broken;                  // [E]
  double* snap_rhs;             // [m] rhs of the last Newton pass (keep_matrix only)
  // k_jtg (persistent, tile-pipelined J^T z gather): ring of tet column sums
  // [JTG_RING][12][nt][32] and its counters ([0] queue head, then per tile
  // [tiles] P1 done, [tiles] P2 done); reset by a memset node per launch
  double* ring;
  int* jctr;
};

struct Ctx {
  Dims D;
  Par p;
  Topo T;
  State S;
  Work K;
};

// Programmatic dependent launch: every frame kernel may be launched before
// its predecessor on the stream has finished (ss_api.cu, SS_PDL); it waits
// here, before its first read, for the predecessor's memory to be visible
// (a no-op without PDL). Only the launch latency and the predecessor's tail
// overlap; no kernel reads anything before this point.
DI void pdl_wait() {
#ifndef SS_NO_PDL_TRIGGER
  // the next kernel may start launching once every CTA of this one has started
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
#endif
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
}

#define SETUP                                              \
  pdl_wait();                                              \
  const int E = c.D.E;                                     \
  const int lane = threadIdx.x & (c.D.W - 1);              \
  const int il = threadIdx.x >> c.D.lgW;                   \
  const int IL = blockDim.x >> c.D.lgW;                    \
  const int env = blockIdx.x * c.D.W + lane;               \
  (void)il;                                                \
  (void)IL;
#define FOR_ITEMS(it, n) for (int it = blockIdx.y * IL + il; it < (n); it += gridDim.y * IL)
#define IX(item) ((size_t)(item) * E + env)
// tet column sums tC: [12][nt][E] (a [nt][12] layout for E = 1 was tried:
// the gather did not speed up and the strided writes cost k_tet_jt 35%)
// Batched (E >= 32): [nt][12][E], a tet's 12 column sums are 12 consecutive
// env rows (contiguous 3 KB runs per tet: 0.5 ms/frame faster than [12][nt][E]
// at 1024 envs). Few env lanes: [12][nt][E], so consecutive tets of one env
// stay coalesced for k_tet_jt's stores (the tet-major order costs the 1M-tet
// scene 9%).
#define TCX(k, t) (E >= 32 ? ((size_t)(t) * 12 + (k)) * E + env : ((size_t)(k) * nt + (t)) * E + env)
// One large mesh (E = 1, c.D.tc_inbox): the column sums of tet t's vertex v
// are stored at that vertex's incidence k = tdst[4 t + v] of the J^T list,
// tC[4k .. 4k+2] (one 32-byte sector per incidence, 256-bit store): a node's
// tet run [inc_tet.x, inc_tet.y) is then consecutive sectors, read by the
// gather with 256-bit loads in the same order as before (same sums, bitwise).
// The scattered access moves from the gather's 8-byte reads (three
// component arrays, 1M tets apart) to k_tet_jt's full-sector writes.
DI void tc_st4(double* p, double a0, double a1, double a2) {
  asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(a0), "d"(a1), "d"(a2),
               "d"(0.0) : "memory");
}
// Streaming loads of data read once per launch (compact tet J, z rows,
// quaternions): read-only path without an L1 allocation, so the L1 keeps the
// gathered DOF vector u (each node line is read by ~12 tets).
// SS_NO_LDHINTS restores plain loads.
DI double ld_stream(const double* p) {
#ifdef SS_NO_LDHINTS
  return *p;
#else
  double v;
  asm("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
#endif
}
DI void tc_ld4(const double* p, double& a0, double& a1, double& a2) {
  double q[4];
  asm("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];" : "=d"(q[0]), "=d"(q[1]), "=d"(q[2]), "=d"(q[3])
      : "l"(p));
  a0 = q[0];
  a1 = q[1];
  a2 = q[2];
}
// the 3 column sums of (tet t, vertex v). IB: 1 inbox layout, 0 the TCX
// layout, -1 decided at run time (c.D.tc_inbox); the hot kernels are
// instantiated per layout so the batched path carries no inbox code.
template <int IB = -1>
DI void tc_put(const Ctx& c, int t, int v, int env, double a0, double a1, double a2) {
  const int E = c.D.E, nt = c.D.nt;
  const int mode = IB < 0 ? c.D.tc_inbox : IB;
  if (mode == 1) {
    tc_st4(c.K.tC + 4 * (size_t)__ldg(&c.T.tdst[4 * (size_t)t + v]), a0, a1, a2);
  } else if (mode == 2) {
    // batched incidence order: [n_inc][3][E], three 256-byte env lines per incidence
    double* p = c.K.tC + (size_t)__ldg(&c.T.tdst[4 * (size_t)t + v]) * 3 * E + env;
    p[0] = a0;
    p[E] = a1;
    p[2 * (size_t)E] = a2;
  } else {
    c.K.tC[TCX(3 * v, t)] = a0;
    c.K.tC[TCX(3 * v + 1, t)] = a1;
    c.K.tC[TCX(3 * v + 2, t)] = a2;
  }
}
template <int IB = -1>
DI void tc_put12(const Ctx& c, int t, int env, const double* col12) {
  if constexpr (IB == 0) {
    const int E = c.D.E, nt = c.D.nt;
#pragma unroll
    for (int k = 0; k < 12; ++k) c.K.tC[TCX(k, t)] = col12[k];
  } else {
#pragma unroll
    for (int v = 0; v < 4; ++v) tc_put<IB>(c, t, v, env, col12[3 * v], col12[3 * v + 1], col12[3 * v + 2]);
  }
}
// the 3 column sums of incidence k (= tet e's vertex v)
template <int IB = -1>
DI void tc_get(const Ctx& c, int k, int v, int e, int env, double& a0, double& a1, double& a2) {
  const int E = c.D.E, nt = c.D.nt;
  const int mode = IB < 0 ? c.D.tc_inbox : IB;
  if (mode == 1) {
    tc_ld4(c.K.tC + 4 * (size_t)k, a0, a1, a2);
  } else if (mode == 2) {
    const double* p = c.K.tC + (size_t)k * 3 * E + env;
    a0 = p[0];
    a1 = p[E];
    a2 = p[2 * (size_t)E];
  } else {
    a0 = c.K.tC[TCX(3 * v, e)];
    a1 = c.K.tC[TCX(3 * v + 1, e)];
    a2 = c.K.tC[TCX(3 * v + 2, e)];
  }
}

// ------------------------------------------------------------ small math
// numpy.maximum: NaN in a propagates
DI double npmax(double a, double b) { return (a >= b || a != a) ? a : b; }

// numpy_backend.py:91-104 (no renormalisation)
DI void quat_to_mat(double w, double x, double y, double z, double* R) {
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
// state.py:16-21,44-51 rotation_matrix (normalised)
DI void rot_normalized(const double* q, double* R) {
  double n = sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
  if (n < 1e-12) {
    quat_to_mat(1.0, 0.0, 0.0, 0.0, R);
  } else {
    quat_to_mat(q[0] / n, q[1] / n, q[2] / n, q[3] / n, R);
  }
}
// np.einsum("nij,nj->ni") contracts length 3 as (p0 + p2) + p1
DI void matvec_es(const double* R, const double* v, double* o) {
#pragma unroll
  for (int i = 0; i < 3; ++i) o[i] = R[3 * i] * v[0] + R[3 * i + 2] * v[2] + R[3 * i + 1] * v[1];
}
DI double dot_es(const double* a, const double* b) { return a[0] * b[0] + a[2] * b[2] + a[1] * b[1]; }
DI void matvec_seq(const double* R, const double* v, double* o) {
#pragma unroll
  for (int i = 0; i < 3; ++i) o[i] = R[3 * i] * v[0] + R[3 * i + 1] * v[1] + R[3 * i + 2] * v[2];
}
DI void cross3(const double* a, const double* b, double* o) {
  o[0] = a[1] * b[2] - a[2] * b[1];
  o[1] = a[2] * b[0] - a[0] * b[2];
  o[2] = a[0] * b[1] - a[1] * b[0];
}
// 3x3 inverse by Gauss-Jordan with partial pivoting (for np.linalg.inv, state.py:262)
DI void inv3(const double* A, double* X) {
  double a[3][6];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 6; ++j) a[i][j] = j < 3 ? A[3 * i + j] : (j - 3 == i ? 1.0 : 0.0);
#pragma unroll
  for (int col = 0; col < 3; ++col) {
    int piv = col;
    for (int r = col + 1; r < 3; ++r)
      if (fabs(a[r][col]) > fabs(a[piv][col])) piv = r;
    if (piv != col) {
#pragma unroll
      for (int j = 0; j < 6; ++j) {
        double t = a[col][j];
        a[col][j] = a[piv][j];
        a[piv][j] = t;
      }
    }
    double dd = a[col][col];
#pragma unroll
    for (int j = 0; j < 6; ++j) a[col][j] /= dd;
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      if (r == col) continue;
      double f = a[r][col];
#pragma unroll
      for (int j = 0; j < 6; ++j) a[r][j] -= f * a[col][j];
    }
  }
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) X[3 * i + j] = a[i][j + 3];
}

// pneumatics.py:62-72 (Python min/max semantics)
DI double update_pressure(double p, double target, const Par& P) {
  if (target > p) {
    double dp = (target - p) / P.supply;
    double a = p + P.supply * dp * dp * P.ki;
    return target < a ? target : a;
  }
  if (target < p) {
    double dec = p * P.kd;
    double mn = P.cap < dec ? P.cap : dec;
    double r = p - mn;
    return r > 0.0 ? r : 0.0;
  }
  return p;
}

// minv diagonal entry for a global DOF (state.py:246-268): particles
// inv_mass, bodies 1/m then diag(I_w^-1)
DI double minv_diag_of(const Ctx& c, int dof, int env) {
  const int E = c.D.E;
  if (dof < c.D.bd0) return c.T.inv_mass[dof / 3];
  int b = (dof - c.D.bd0) / 6, k = (dof - c.D.bd0) % 6;
  if (k < 3) return c.T.body_inv_mass[b];
  return c.K.ang_inv[IX((size_t)(4 * (k - 3)) * c.D.nb + b)];
}

// attachment J value (constraints.py:227-237): row i, column col of
// [-I3 | I3 | -skew(R r)]
DI double att_val(int i, int col, const double* rw) {
  if (col < 3) return col == i ? -1.0 : 0.0;
  if (col < 6) return col - 3 == i ? 1.0 : 0.0;
  int k = col - 6;
  if (i == 0) return k == 0 ? 0.0 : (k == 1 ? rw[2] : -rw[1]);
  if (i == 1) return k == 0 ? -rw[2] : (k == 1 ? 0.0 : rw[0]);
  return k == 0 ? rw[1] : (k == 1 ? -rw[0] : 0.0);
}

// ---------------------------------------------------- reduction helper
// Deterministic per-env block reduction of `val`, then "last block" combine
// over gridDim.y in fixed order. Returns true in the W threads of the last
// block with il == 0 and the total in *tot.
DI bool reduce_env(const Ctx& c, double val, double* tot) {
  SETUP
  __shared__ double red[SS_THREADS];
  __shared__ int amlast;
  red[threadIdx.x] = val;
  __syncthreads();
  for (int s = IL >> 1; s > 0; s >>= 1) {
    if (il < s) red[threadIdx.x] += red[threadIdx.x + s * c.D.W];
    __syncthreads();
  }
  if (il == 0) c.K.part[(size_t)blockIdx.y * E + env] = red[lane];
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = atomicAdd(&c.K.cnt[blockIdx.x], 1);
    amlast = (t == (int)gridDim.y - 1);
  }
  __syncthreads();
  if (!amlast) return false;
  if (threadIdx.x == 0) c.K.cnt[blockIdx.x] = 0;
  // the last block combines the gridDim.y partials with all its item lanes
  // (lane il sums rows il, il + IL, ... in order, then the same fixed tree)
  double s = 0.0;
  for (int y = il; y < (int)gridDim.y; y += IL) s += __ldcg(&c.K.part[(size_t)y * E + env]);
  red[threadIdx.x] = s;
  __syncthreads();
  for (int st = IL >> 1; st > 0; st >>= 1) {
    if (il < st) red[threadIdx.x] += red[threadIdx.x + st * c.D.W];
    __syncthreads();
  }
  if (il != 0) return false;
  *tot = red[lane];
  return true;
}

// ================================================================ frame
// Simulator.step head: ChannelBank.tick + _update_actuation
// (solver.py:296-301, pneumatics.py:102-116, solver.py:279-282)
// gait command of link i at frame f: clamp(sin(w t + alpha (i mod lps)) +
// bias, -1, 1) * A with t = t0 + f dt (snake.py:235-241, harness.py:190-192)
DI double gait_cmd(const Ctx& c, int env, int i) {
  const int E = c.D.E;
  const double A = c.S.gait[IX(0)], w = c.S.gait[IX(1)], al = c.S.gait[IX(2)];
  const double bias = c.S.gait[IX(3)], t0 = c.S.gait[IX(4)];
  const int lps = (int)c.S.gait[IX(5)];
  const double t = t0 + (double)c.S.gait_frame[env] * c.p.dt;
  const int k = lps > 0 ? i % lps : i;
  double raw = sin(w * t + al * (double)k) + bias;
  raw = raw < -1.0 ? -1.0 : (raw > 1.0 ? 1.0 : raw);
  return raw * A;
}

// gait: commands from the per-env generator instead of cmd (the frame
// counter advances in k_pre of the first substep, after every link read it)
__global__ void k_frame_begin(const Ctx c, const double* __restrict__ cmd, int has_cmd,
                              int latency, int gait) {
  SETUP
  const int n = c.D.links > 0 ? c.D.links : 1;
  FOR_ITEMS(i, n) {
    if (i == 0) {
      c.S.nc_cnt[env] = 0;
      c.S.inv_cnt[env] = 0;
      c.S.nonfinite[env] = 0;
    }
    if (i < c.D.links) {
      if (has_cmd || gait) {
        int ce = env < c.D.n_real ? env : 0;
        double a = gait ? gait_cmd(c, env, i) : cmd[(size_t)ce * c.D.links + i];
        double left = 0.0, right = 0.0;
        if (a > 0.0) right = a;
        else if (a < 0.0) left = -a;
        double* pl = &c.S.press[IX(2 * i)];
        double* pr = &c.S.press[IX(2 * i + 1)];
        if (latency) {
          *pl = update_pressure(*pl, left, c.p);
          *pr = update_pressure(*pr, right, c.p);
        } else {
          *pl = left;
          *pr = right;
        }
      }
      if (c.D.act_enabled) {
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          double pp = c.S.press[IX(2 * i + k)];
          c.S.target[IX(2 * i + k)] = 1.0 + pp * SS_PSI_TO_PA / c.p.youngs;
        }
      }
    }
  }
}

// Simulator.set_channel_targets (solver.py:274-277): the pneumatic tick
// alone (ChannelBank.tick, pneumatics.py:102-116), without the strain
// target update that step() does after it (_update_actuation)
__global__ void k_tick(const Ctx c, const double* __restrict__ cmd, int latency) {
  SETUP
  FOR_ITEMS(i, c.D.links) {
    const int ce = env < c.D.n_real ? env : 0;
    const double a = cmd[(size_t)ce * c.D.links + i];
    double left = 0.0, right = 0.0;
    if (a > 0.0) right = a;
    else if (a < 0.0) left = -a;
    double* pl = &c.S.press[IX(2 * i)];
    double* pr = &c.S.press[IX(2 * i + 1)];
    if (latency) {
      *pl = update_pressure(*pl, left, c.p);
      *pr = update_pressure(*pr, right, c.p);
    } else {
      *pl = left;
      *pr = right;
    }
  }
}

// =============================================================== substep
// _slew_actuation (solver.py:284-292), build_mass_inverse (state.py:246-268)
// and _predict_velocities (solver.py:316-332). Items: P particles, nb
// bodies, nch channels.
__global__ void k_pre(const Ctx c, int gait_tick) {
  SETUP
  const int P = c.D.P, nb = c.D.nb;
  if (gait_tick && blockIdx.y == 0 && il == 0) c.S.gait_frame[env] += 1;
  FOR_ITEMS(it, P + nb + c.D.nch) {
    if (it < P) {
      const bool live = c.T.inv_mass[it] > 0.0;
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        double vi = c.S.vel[IX(3 * it + a)];
        c.K.v[IX(3 * it + a)] = live ? vi + c.p.hg[a] : vi;
      }
    } else if (it < P + nb) {
      const int b = it - P;
      double q[4], R[9], RI[9], iw[9], Ai[9];
#pragma unroll
      for (int k = 0; k < 4; ++k) q[k] = c.S.bquat[IX(4 * b + k)];
      rot_normalized(q, R);
      const double* I = c.T.body_inertia + 9 * b;
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j)
          RI[3 * i + j] = R[3 * i] * I[j] + R[3 * i + 1] * I[3 + j] + R[3 * i + 2] * I[6 + j];
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j)
          iw[3 * i + j] = RI[3 * i] * R[3 * j] + RI[3 * i + 1] * R[3 * j + 1] + RI[3 * i + 2] * R[3 * j + 2];
      inv3(iw, Ai);
#pragma unroll
      for (int k = 0; k < 9; ++k) c.K.ang_inv[IX((size_t)k * nb + b)] = Ai[k];
      double w[3], iww[3], tau[3], t3[3];
#pragma unroll
      for (int a = 0; a < 3; ++a) w[a] = c.S.bang[IX(3 * b + a)];
      matvec_es(iw, w, iww);
      cross3(w, iww, tau);
#pragma unroll
      for (int a = 0; a < 3; ++a) tau[a] = -tau[a];
      matvec_es(Ai, tau, t3);
      const int o = c.D.bd0 + 6 * b;
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        c.K.v[IX(o + a)] = c.S.blin[IX(3 * b + a)] + c.p.hg[a];
        c.K.v[IX(o + 3 + a)] = w[a] + c.p.h * t3[a];
      }
    } else if (c.D.act_enabled) {
      const int ch = it - P - nb;
      double live = c.S.live[IX(ch)];
      double d = c.S.target[IX(ch)] - live;
      if (d < -c.p.dmax) d = -c.p.dmax;
      else if (d > c.p.dmax) d = c.p.dmax;
      c.S.live[IX(ch)] = live + d;
    }
  }
}

// detect_ground_contacts + FrictionState.for_contacts + contact_row_blocks
// + block_rowdiag of the contact families (contact.py:62-93, 135-149,
// 183-215; solver.py:421-424). One item per candidate slot: wheels first,
// then contact particles in order; present slots are the reference's
// compacted contact list in the same order.
__global__ void k_slots(const Ctx c) {
  SETUP
  const int nw = c.D.nw, ns = c.D.ns;
  FOR_ITEMS(s, ns) {
    double gap;
    int present;
    double nv[6], f0[6], f1[6], md[6];
    double lam_n = 0.0, lam_f0 = 0.0, lam_f1 = 0.0;
    if (s < nw) {
      const int b = c.T.w_body[s];
      double q[4], R[9], ax[3], al[3], ctr[3];
#pragma unroll
      for (int k = 0; k < 4; ++k) q[k] = c.S.bquat[IX(4 * b + k)];
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        ctr[a] = c.S.bpos[IX(3 * b + a)];
        al[a] = c.T.w_axis[a * nw + s];
      }
      rot_normalized(q, R);
      matvec_seq(R, al, ax);
      double nd = 0.0 * ax[0] + 0.0 * ax[1] + 1.0 * ax[2];
      double dv[3] = {0.0 - nd * ax[0], 0.0 - nd * ax[1], 1.0 - nd * ax[2]};
      double dn = sqrt(dv[0] * dv[0] + dv[1] * dv[1] + dv[2] * dv[2]);
      if (dn < 1e-9) {
        dv[0] = 1.0 - ax[0] * ax[0];
        dv[1] = 0.0 - ax[0] * ax[1];
        dv[2] = 0.0 - ax[0] * ax[2];
        dn = sqrt(dv[0] * dv[0] + dv[1] * dv[1] + dv[2] * dv[2]);
      }
      double pt[3], r[3], cr[3];
      const double rad = c.T.w_rad[s];
#pragma unroll
      for (int a = 0; a < 3; ++a) pt[a] = ctr[a] - rad * (dv[a] / dn);
      gap = pt[2] - c.p.ground_h;
      present = gap < c.p.margin;
#pragma unroll
      for (int a = 0; a < 3; ++a) r[a] = pt[a] - ctr[a];
      const double n[3] = {0.0, 0.0, 1.0}, t1[3] = {1.0, 0.0, 0.0}, t2[3] = {0.0, 1.0, 0.0};
      cross3(r, n, cr);
#pragma unroll
      for (int a = 0; a < 3; ++a) { nv[a] = n[a]; nv[3 + a] = cr[a]; }
      cross3(r, t1, cr);
#pragma unroll
      for (int a = 0; a < 3; ++a) { f0[a] = t1[a]; f0[3 + a] = cr[a]; }
      cross3(r, t2, cr);
#pragma unroll
      for (int a = 0; a < 3; ++a) { f1[a] = t2[a]; f1[3 + a] = cr[a]; }
#pragma unroll
      for (int k = 0; k < 6; ++k) {
        c.K.wJ[IX((size_t)k * nw + s)] = nv[k];
        c.K.wJ[IX((size_t)(6 + k) * nw + s)] = f0[k];
        c.K.wJ[IX((size_t)(12 + k) * nw + s)] = f1[k];
      }
      const int o = c.D.bd0 + 6 * b;
#pragma unroll
      for (int k = 0; k < 6; ++k) md[k] = minv_diag_of(c, o + k, env);
      if (present && c.S.warm_valid[IX(s)]) {
        lam_n = c.S.warm[IX(s)];
        lam_f0 = c.S.warm[IX(nw + s)];
        lam_f1 = c.S.warm[IX(2 * nw + s)];
      }
    } else {
      const int pi = c.T.slot_part[s - nw];
      gap = c.S.pos[IX(3 * pi + 2)] - c.p.ground_h;
      present = gap < c.p.margin;
#pragma unroll
      for (int k = 0; k < 6; ++k) { nv[k] = 0.0; f0[k] = 0.0; f1[k] = 0.0; }
      nv[2] = 1.0;
      f0[0] = 1.0;
      f1[1] = 1.0;
      const double mp = c.T.inv_mass[pi], m0 = c.T.inv_mass[0];
      md[0] = mp; md[1] = mp; md[2] = mp;
      md[3] = m0; md[4] = m0; md[5] = m0;   // padded columns point at DOF 0
    }
    double dn_ = 0.0, d0 = 0.0, d1 = 0.0;
#pragma unroll
    for (int k = 0; k < 6; ++k) {
      dn_ += nv[k] * nv[k] * md[k];
      d0 += f0[k] * f0[k] * md[k];
      d1 += f1[k] * f1[k] * md[k];
    }
    c.K.present[IX(s)] = present;
    c.K.gap[IX(s)] = gap;
    c.K.bdiag[IX(c.D.on + s)] = dn_;
    c.K.bdiag[IX(c.D.of + s)] = d0;
    c.K.bdiag[IX(c.D.of + ns + s)] = d1;
    c.K.lamc[IX(s)] = lam_n;
    c.K.lamc[IX(ns + s)] = lam_f0;
    c.K.lamc[IX(2 * ns + s)] = lam_f1;
    if (c.p.newton == 0 && s < nw) {
      // store_warm after an empty Newton loop (solver.py:522, contact.py:167-180);
      // otherwise k_newton_final's last pass stores it
      c.S.warm_valid[IX(s)] = present ? 1 : 0;
      c.S.warm[IX(s)] = lam_n;
      c.S.warm[IX(nw + s)] = lam_f0;
      c.S.warm[IX(2 * nw + s)] = lam_f1;
    }
    if (present) atomicAdd(&c.S.nc_cnt[env], 1);
  }
}

// ------------------------------------------------------------- tetra eval
// numba_backend.py:137-312. The Jacobian is never stored: an element keeps
// S = sym(R^T F) (6 doubles) beside its persistent quaternion; R and K^-1
// are rebuilt bitwise from them (tet_unpack), and tet_col() recomputes any
// column with the exact expressions of the reference, so every use sees
// the same bits the eval produced.

// compact tet Jacobian of one element in registers
struct TetC {
  double R[9], S[9], K[9];
};

// rest-inverse direction w_v (numba_backend.py:270-281)
DI void tet_wv(const double* Ri, int v, double* w) {
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    const double w0 = -(Ri[j] + Ri[3 + j] + Ri[6 + j]);
    w[j] = v == 0 ? w0 : (v == 1 ? Ri[j] : (v == 2 ? Ri[3 + j] : Ri[6 + j]));
  }
}

// column 3v+a of the 6x12 Jacobian (numba_backend.py:283-311)
DI void tet_col(const TetC& T, const double* wv, int a, double* o) {
  const double* R = T.R;
  const double* S = T.S;
  const double* Ki = T.K;
  double G[9];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) G[3 * i + j] = R[3 * a + i] * wv[j];
  const double g0 = G[7] - G[5], g1 = G[2] - G[6], g2 = G[3] - G[1];
  const double w0 = Ki[0] * g0 + Ki[1] * g1 + Ki[2] * g2;
  const double w1 = Ki[3] * g0 + Ki[4] * g1 + Ki[5] * g2;
  const double w2 = Ki[6] * g0 + Ki[7] * g1 + Ki[8] * g2;
  const double ws00 = -w2 * S[3] + w1 * S[6];
  const double ws01 = -w2 * S[4] + w1 * S[7];
  const double ws02 = -w2 * S[5] + w1 * S[8];
  const double ws10 = w2 * S[0] - w0 * S[6];
  const double ws11 = w2 * S[1] - w0 * S[7];
  const double ws12 = w2 * S[2] - w0 * S[8];
  const double ws20 = -w1 * S[0] + w0 * S[3];
  const double ws21 = -w1 * S[1] + w0 * S[4];
  const double ws22 = -w1 * S[2] + w0 * S[5];
  o[0] = G[0] - ws00;
  o[1] = G[4] - ws11;
  o[2] = G[8] - ws22;
  o[3] = 0.5 * (G[5] + G[7]) - 0.5 * (ws12 + ws21);
  o[4] = 0.5 * (G[2] + G[6]) - 0.5 * (ws02 + ws20);
  o[5] = 0.5 * (G[1] + G[3]) - 0.5 * (ws01 + ws10);
}

// polar decomposition + strain + K^-1; returns det(F) <= 0
// K^-1 with K = tr(S) I - S (+1e-14 on the diagonal), by cofactors
// (numba_backend.py:221-240). Pure function of S: the compact tet Jacobian
// stores S only and every consumer recomputes K^-1 bitwise.
DI void tet_kinv(const double* S, double* Ki) {
  const double trS = S[0] + S[4] + S[8];
  double K[9];
#pragma unroll
  for (int i = 0; i < 9; ++i) K[i] = -S[i];
  K[0] += trS + 1e-14;
  K[4] += trS + 1e-14;
  K[8] += trS + 1e-14;
  double detK = K[0] * (K[4] * K[8] - K[5] * K[7]) - K[1] * (K[3] * K[8] - K[5] * K[6]) +
                K[2] * (K[3] * K[7] - K[4] * K[6]);
  if (fabs(detK) < 1e-30) detK = detK >= 0 ? 1e-30 : -1e-30;
  const double id = 1.0 / detK;
  Ki[0] = (K[4] * K[8] - K[5] * K[7]) * id;
  Ki[1] = (K[2] * K[7] - K[1] * K[8]) * id;
  Ki[2] = (K[1] * K[5] - K[2] * K[4]) * id;
  Ki[3] = (K[5] * K[6] - K[3] * K[8]) * id;
  Ki[4] = (K[0] * K[8] - K[2] * K[6]) * id;
  Ki[5] = (K[2] * K[3] - K[0] * K[5]) * id;
  Ki[6] = (K[3] * K[7] - K[4] * K[6]) * id;
  Ki[7] = (K[1] * K[6] - K[0] * K[7]) * id;
  Ki[8] = (K[0] * K[4] - K[1] * K[3]) * id;
}

// the warm-started polar iteration (numba_backend.py:178-218) on q in place;
// returns the iteration count
DI int polar_iterate(const double* F, double* q, double tol, int maxiter, int* iters) {
  double qw = q[0], qx = q[1], qy = q[2], qz = q[3];
  int it = 0;
  for (; it < maxiter; ++it) {
    double r[9];
    quat_to_mat(qw, qx, qy, qz, r);
    double o0 = 0.0, o1 = 0.0, o2 = 0.0, tr = 0.0;
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const double rc0 = r[j], rc1 = r[3 + j], rc2 = r[6 + j];
      const double f0 = F[j], f1 = F[3 + j], f2 = F[6 + j];
      o0 += rc1 * f2 - rc2 * f1;
      o1 += rc2 * f0 - rc0 * f2;
      o2 += rc0 * f1 - rc1 * f0;
      tr += rc0 * f0 + rc1 * f1 + rc2 * f2;
    }
    const double s = 1.0 / (fabs(tr) + 1e-9);
    o0 *= s;
    o1 *= s;
    o2 *= s;
    const double wn = sqrt(o0 * o0 + o1 * o1 + o2 * o2);
    if (wn < tol) break;
    if (wn != wn) {
      // non-finite element (a diverged env): the reference keeps iterating to
      // maxiter and ends with a NaN quaternion; end there at once
      qw = qx = qy = qz = __longlong_as_double(0x7ff8000000000000ll);
      it = maxiter;
      break;
    }
    const double half = 0.5 * wn;
    double sh, cw;
    sincos(half, &sh, &cw);  // one shared argument reduction
    const double sw = sh / wn;
    const double dw = cw, dx = sw * o0, dy = sw * o1, dz = sw * o2;
    const double nw = dw * qw - dx * qx - dy * qy - dz * qz;
    const double nx = dw * qx + dx * qw + dy * qz - dz * qy;
    const double ny = dw * qy - dx * qz + dy * qw + dz * qx;
    const double nz = dw * qz + dx * qy - dy * qx + dz * qw;
    const double qn = sqrt(nw * nw + nx * nx + ny * ny + nz * nz);
    qw = nw / qn;
    qx = nx / qn;
    qy = ny / qn;
    qz = nz / qn;
  }
  if (iters) *iters = it;
  q[0] = qw; q[1] = qx; q[2] = qy; q[3] = qz;
  return it;
}

DI int tet_eval_core(const double* X, const double* Ri, double* q, double tol, int maxiter,
                     TetC& T, int* iters) {
  double F[9];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const double x0 = X[a];
    const double Ds0 = X[3 + a] - x0, Ds1 = X[6 + a] - x0, Ds2 = X[9 + a] - x0;
#pragma unroll
    for (int j = 0; j < 3; ++j) F[3 * a + j] = Ds0 * Ri[j] + Ds1 * Ri[3 + j] + Ds2 * Ri[6 + j];
  }
  const double detF = F[0] * (F[4] * F[8] - F[5] * F[7]) - F[1] * (F[3] * F[8] - F[5] * F[6]) +
                      F[2] * (F[3] * F[7] - F[4] * F[6]);
  int it = polar_iterate(F, q, tol, maxiter, iters);
  (void)it;
  const double qw = q[0], qx = q[1], qy = q[2], qz = q[3];
  double* R = T.R;
  double* S = T.S;
  quat_to_mat(qw, qx, qy, qz, R);
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) S[3 * i + j] = R[i] * F[j] + R[3 + i] * F[3 + j] + R[6 + i] * F[6 + j];
  {
    const double m01 = 0.5 * (S[1] + S[3]);
    S[1] = m01; S[3] = m01;
    const double m02 = 0.5 * (S[2] + S[6]);
    S[2] = m02; S[6] = m02;
    const double m12 = 0.5 * (S[5] + S[7]);
    S[5] = m12; S[7] = m12;
  }
  tet_kinv(S, T.K);
  return detF <= 0.0 ? 1 : 0;
}

// strain residual in Voigt order [xx yy zz yz xz xy] (numba_backend.py:241-246)
DI void tet_res(const TetC& T, double* r) {
  r[0] = T.S[0] - 1.0;
  r[1] = T.S[4] - 1.0;
  r[2] = T.S[8] - 1.0;
  r[3] = T.S[5];
  r[4] = T.S[2];
  r[5] = T.S[1];
}

// compact storage: S (6 unique, symmetrised explicitly in tet_eval_core).
// R = quat_to_mat(q) of the tet's persistent quaternion (tet_eval_core builds
// R from exactly that q) and K^-1 = tet_kinv(S) are recomputed bitwise on
// load: 10 doubles per tet read instead of 21.
DI void tet_store(const Ctx& c, int t, int env, const TetC& T) {
  const int E = c.D.E, nt = c.D.nt;
  const int sym[6] = {0, 4, 8, 5, 2, 1};
#pragma unroll
  for (int k = 0; k < 6; ++k) c.K.tS[IX(k * nt + t)] = T.S[sym[k]];
}
DI void tet_unpack(const double* q, const double* s, TetC& T) {
  quat_to_mat(q[0], q[1], q[2], q[3], T.R);
  // [0 1 2; 3 4 5; 6 7 8] <- (00 11 22 12 02 01)
  T.S[0] = s[0]; T.S[4] = s[1]; T.S[8] = s[2];
  T.S[5] = s[3]; T.S[7] = s[3];
  T.S[2] = s[4]; T.S[6] = s[4];
  T.S[1] = s[5]; T.S[3] = s[5];
  tet_kinv(T.S, T.K);
}
DI void tet_load(const Ctx& c, int t, int env, TetC& T) {
  const int E = c.D.E, nt = c.D.nt;
  double q[4], s[6];
#pragma unroll
  for (int k = 0; k < 4; ++k) q[k] = c.S.quat[IX(k * nt + t)];
#pragma unroll
  for (int k = 0; k < 6; ++k) s[k] = c.K.tS[IX(k * nt + t)];
  tet_unpack(q, s, T);
}
DI void tet_rinv(const Ctx& c, int t, double* Ri) {
  // one tet's rest inverse is 80 contiguous bytes: 5 broadcast 16-byte loads
  const double2* p = reinterpret_cast<const double2*>(c.T.t_rinv + 10 * (size_t)t);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const double2 v = __ldg(p + k);
    Ri[2 * k] = v.x;
    Ri[2 * k + 1] = v.y;
  }
  Ri[8] = __ldg(c.T.t_rinv + 10 * (size_t)t + 8);
}

// J^T x for one tet: the 12 column sums acc_j = sum_i J[i][j] x_i in the
// reference's accumulation order (numba_backend.py:43-52), written to tC
template <int IB = -1>
DI void tet_contrib(const Ctx& c, int t, int env, const TetC& T, const double* Ri,
                    const double* x6) {
  const int E = c.D.E, nt = c.D.nt;
  (void)E;
  (void)nt;
#pragma unroll 1
  for (int v = 0; v < 4; ++v) {
    double wv[3];
    tet_wv(Ri, v, wv);
    double acc3[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      double col[6];
      tet_col(T, wv, a, col);
      double acc = 0.0;
#pragma unroll
      for (int i = 0; i < 6; ++i) acc += col[i] * x6[i];
      acc3[a] = acc;
    }
    tc_put<IB>(c, t, v, env, acc3[0], acc3[1], acc3[2]);
  }
}

// J y for one tet: y_i = sum_j J[i][j] vec[idx_j] (numba_backend.py:31-40)
DI void tet_forward(const Ctx& c, int t, int env, const TetC& T, const double* Ri,
                    const double* vec, double* y) {
  const int E = c.D.E, nt = c.D.nt;
#pragma unroll
  for (int i = 0; i < 6; ++i) y[i] = 0.0;
#pragma unroll 1
  for (int v = 0; v < 4; ++v) {
    const int node = c.T.t_idx[v * nt + t];
    double wv[3];
    tet_wv(Ri, v, wv);
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const double uj = vec[IX(3 * node + a)];
      double col[6];
      tet_col(T, wv, a, col);
#pragma unroll
      for (int i = 0; i < 6; ++i) y[i] += col[i] * uj;
    }
  }
}

// ---- structured application of the same operator (default solver path)
// The 6x12 block is never materialised: with Z the symmetric matrix of a
// Voigt vector z (shear entries halved), N = Z S, n = K^-1 ax(N),
//   (J^T z)_{3v+a} = R_a . (Z w_v - n x w_v),
// and with L = sum_v u_v w_v^T, G = R^T L, w = K^-1 ax(G),
//   J u = voigt(sym(G) - sym(skew(w) S)).
// Algebraically identical to the columns of tet_col (numba_backend.py:283-311);
// only the association of the sums differs (~1e-16 relative), for ~5x fewer
// FP64 operations. ax(M) = (M21 - M12, M02 - M20, M10 - M01) as g in the ref.
// Structured tet operators (the default, non-bitwise mode): explicit fused
// multiply-adds (the file is built with --fmad=false so that every
// reference-order expression elsewhere keeps numba's rounding). dot3(a..) =
// a0 b0 + a1 b1 + a2 b2 as two FMAs.
DI double dot3(double a0, double b0, double a1, double b1, double a2, double b2) {
  return __fma_rn(a2, b2, __fma_rn(a1, b1, a0 * b0));
}

// J^T z of one tet as its 12 column sums: (J^T z)_{3v+a} = R_a . (Z w_v -
// n x w_v) with Z = sym-voigt(z), n = K^-1 ax(Z S)
DI void tet_jt_cols(const TetC& T, const double* Ri, const double* z, double* col12) {
  const double* S = T.S;
  const double* Ki = T.K;
  const double* R = T.R;
  const double Z00 = z[0], Z11 = z[1], Z22 = z[2];
  const double Z12 = 0.5 * z[3], Z02 = 0.5 * z[4], Z01 = 0.5 * z[5];
  const double N21 = dot3(Z02, S[1], Z12, S[4], Z22, S[7]);
  const double N12 = dot3(Z01, S[2], Z11, S[5], Z12, S[8]);
  const double N02 = dot3(Z00, S[2], Z01, S[5], Z02, S[8]);
  const double N20 = dot3(Z02, S[0], Z12, S[3], Z22, S[6]);
  const double N10 = dot3(Z01, S[0], Z11, S[3], Z12, S[6]);
  const double N01 = dot3(Z00, S[1], Z01, S[4], Z02, S[7]);
  const double m0 = N21 - N12, m1 = N02 - N20, m2 = N10 - N01;
  const double n0 = dot3(Ki[0], m0, Ki[1], m1, Ki[2], m2);
  const double n1 = dot3(Ki[3], m0, Ki[4], m1, Ki[5], m2);
  const double n2 = dot3(Ki[6], m0, Ki[7], m1, Ki[8], m2);
#pragma unroll
  for (int v = 0; v < 4; ++v) {
    double wv[3];
    tet_wv(Ri, v, wv);
    const double q0 = dot3(Z00, wv[0], Z01, wv[1], Z02, wv[2]) - __fma_rn(n1, wv[2], -n2 * wv[1]);
    const double q1 = dot3(Z01, wv[0], Z11, wv[1], Z12, wv[2]) - __fma_rn(n2, wv[0], -n0 * wv[2]);
    const double q2 = dot3(Z02, wv[0], Z12, wv[1], Z22, wv[2]) - __fma_rn(n0, wv[1], -n1 * wv[0]);
#pragma unroll
    for (int a = 0; a < 3; ++a) col12[3 * v + a] = dot3(R[3 * a], q0, R[3 * a + 1], q1, R[3 * a + 2], q2);
  }
}
template <int IB = -1>
DI void tet_contrib_fast(const Ctx& c, int t, int env, const TetC& T, const double* Ri,
                         const double* z) {
  const int E = c.D.E, nt = c.D.nt;
  double col12[12];
  tet_jt_cols(T, Ri, z, col12);
  if constexpr (IB == 0) {
#pragma unroll
    for (int k = 0; k < 12; ++k) c.K.tC[TCX(k, t)] = col12[k];
  } else {
    tc_put12<IB>(c, t, env, col12);
  }
}

// J u of one tet from its 4 node values uv[3v+a] (structured chain rule):
// voigt(sym(G) - sym(skew(K^-1 ax G) S)), G = R^T sum_v u_v w_v^T
DI void tet_forward_uv(const TetC& T, const double* Ri, const double* uv, double* y) {
  const double* R = T.R;
  const double* S = T.S;
  const double* Ki = T.K;
  double du[9];
#pragma unroll
  for (int v = 1; v < 4; ++v)
#pragma unroll
    for (int a = 0; a < 3; ++a) du[3 * (v - 1) + a] = uv[3 * v + a] - uv[a];
  // L_aj = sum_{v=1..3} (u_v - u_0)_a Ri[v-1][j]   (w_0 = -(w_1 + w_2 + w_3))
  double L[9];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int j = 0; j < 3; ++j) L[3 * a + j] = dot3(du[a], Ri[j], du[3 + a], Ri[3 + j], du[6 + a], Ri[6 + j]);
  double G[9];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) G[3 * i + j] = dot3(R[i], L[j], R[3 + i], L[3 + j], R[6 + i], L[6 + j]);
  const double g0 = G[7] - G[5], g1 = G[2] - G[6], g2 = G[3] - G[1];
  const double w0 = dot3(Ki[0], g0, Ki[1], g1, Ki[2], g2);
  const double w1 = dot3(Ki[3], g0, Ki[4], g1, Ki[5], g2);
  const double w2 = dot3(Ki[6], g0, Ki[7], g1, Ki[8], g2);
  const double ws00 = __fma_rn(w1, S[6], -w2 * S[3]);
  const double ws01 = __fma_rn(w1, S[7], -w2 * S[4]);
  const double ws02 = __fma_rn(w1, S[8], -w2 * S[5]);
  const double ws10 = __fma_rn(w2, S[0], -w0 * S[6]);
  const double ws11 = __fma_rn(w2, S[1], -w0 * S[7]);
  const double ws12 = __fma_rn(w2, S[2], -w0 * S[8]);
  const double ws20 = __fma_rn(w0, S[3], -w1 * S[0]);
  const double ws21 = __fma_rn(w0, S[4], -w1 * S[1]);
  const double ws22 = __fma_rn(w0, S[5], -w1 * S[2]);
  y[0] = G[0] - ws00;
  y[1] = G[4] - ws11;
  y[2] = G[8] - ws22;
  y[3] = 0.5 * ((G[5] + G[7]) - (ws12 + ws21));
  y[4] = 0.5 * ((G[2] + G[6]) - (ws02 + ws20));
  y[5] = 0.5 * ((G[1] + G[3]) - (ws01 + ws10));
}
DI void tet_node_vals(const Ctx& c, int t, int env, const double* vec, double* uv) {
  const int E = c.D.E, nt = c.D.nt;
#pragma unroll
  for (int v = 0; v < 4; ++v) {
    const int node = c.T.t_idx[v * nt + t];
#pragma unroll
    for (int a = 0; a < 3; ++a) uv[3 * v + a] = vec[IX(3 * node + a)];
  }
}
DI void tet_forward_fast(const Ctx& c, int t, int env, const TetC& T, const double* Ri,
                         const double* vec, double* y) {
  double uv[12];
  tet_node_vals(c, t, env, vec, uv);
  tet_forward_uv(T, Ri, uv, y);
}

// EXACT selects the materialised-column path (bitwise numba sums)
template <bool EXACT, int IB = -1>
DI void tet_jt(const Ctx& c, int t, int env, const TetC& T, const double* Ri, const double* x6) {
  if (EXACT) tet_contrib<IB>(c, t, env, T, Ri, x6);
  else tet_contrib_fast<IB>(c, t, env, T, Ri, x6);
}
template <bool EXACT>
DI void tet_j(const Ctx& c, int t, int env, const TetC& T, const double* Ri, const double* vec,
              double* y) {
  if (EXACT) tet_forward(c, t, env, T, Ri, vec, y);
  else tet_forward_fast(c, t, env, T, Ri, vec, y);
}

// The polar decomposition of TetraSet.eval alone (the warm-started
// quaternion iteration of numba_backend.py:178-218): a small-register kernel
// so the data-dependent FP64 loop runs at high occupancy; k_eval_tet then
// finds the converged quaternion and runs zero iterations (the same q, so
// R, S, the Jacobian and every result are bitwise those of the fused kernel).
#ifndef SS_POLAR_MINB
#define SS_POLAR_MINB 4
#endif
__global__ void __launch_bounds__(SS_THREADS, SS_POLAR_MINB) k_eval_polar(const Ctx c) {
  SETUP
  const int nt = c.D.nt;
  FOR_ITEMS(t, nt) {
    double X[12], Ri[9], q[4];
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int node = c.T.t_idx[v * nt + t];
#pragma unroll
      for (int a = 0; a < 3; ++a) X[3 * v + a] = c.S.pos[IX(3 * node + a)];
    }
    tet_rinv(c, t, Ri);
#pragma unroll
    for (int k = 0; k < 4; ++k) q[k] = c.S.quat[IX(k * nt + t)];
    double F[9];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const double x0 = X[a];
      const double Ds0 = X[3 + a] - x0, Ds1 = X[6 + a] - x0, Ds2 = X[9 + a] - x0;
#pragma unroll
      for (int j = 0; j < 3; ++j) F[3 * a + j] = Ds0 * Ri[j] + Ds1 * Ri[3 + j] + Ds2 * Ri[6 + j];
    }
    polar_iterate(F, q, 1e-12, 500, nullptr);
#pragma unroll
    for (int k = 0; k < 4; ++k) c.S.quat[IX(k * nt + t)] = q[k];
  }
}

// TetraSet.eval + its block_rowdiag + eh2 diag (solver.py:410-426), and
// the tet part of the initial impulse J^T lam (solver.py:428-436).
template <bool EXACT>
#ifdef SS_EVAL_MINB
#define SS_EVAL_MINB_LB __launch_bounds__(SS_THREADS, SS_EVAL_MINB)
#else
#define SS_EVAL_MINB_LB __launch_bounds__(SS_THREADS)
#endif
__global__ void SS_EVAL_MINB_LB k_eval_tet(const Ctx c, int polar_done) {
  SETUP
  const int nt = c.D.nt;
  FOR_ITEMS(t, nt) {
    double X[12], Ri[9], q[4], im[4];
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int node = c.T.t_idx[v * nt + t];
      im[v] = c.T.inv_mass[node];
#pragma unroll
      for (int a = 0; a < 3; ++a) X[3 * v + a] = c.S.pos[IX(3 * node + a)];
    }
    tet_rinv(c, t, Ri);
#pragma unroll
    for (int k = 0; k < 4; ++k) q[k] = c.S.quat[IX(k * nt + t)];
    TetC T;
    const int inv = tet_eval_core(X, Ri, q, 1e-12, polar_done ? 0 : 500, T, nullptr);
#pragma unroll
    for (int k = 0; k < 4; ++k) c.S.quat[IX(k * nt + t)] = q[k];
    tet_store(c, t, env, T);
    // block_rowdiag (numba_backend.py:55-65): acc_i = sum_j J_ij^2 minv_j
    double diag[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
#pragma unroll 1
    for (int v = 0; v < 4; ++v) {
      double wv[3];
      tet_wv(Ri, v, wv);
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        double col[6];
        tet_col(T, wv, a, col);
#pragma unroll
        for (int i = 0; i < 6; ++i) diag[i] += col[i] * col[i] * im[v];
      }
    }
    const double ed = c.T.t_e3[t], es = c.T.t_e3[2 * nt + t];
#pragma unroll
    for (int i = 0; i < 6; ++i) c.K.bdiag[IX(c.D.ot + i * nt + t)] = diag[i] + (i < 3 ? ed : es);
    double lam6[6];
#pragma unroll
    for (int i = 0; i < 6; ++i) lam6[i] = c.S.lam[IX(c.D.ot + i * nt + t)];
    tet_jt<EXACT>(c, t, env, T, Ri, lam6);
    if (inv) atomicAdd(&c.S.inv_cnt[env], 1);
  }
}

// DistanceSet.eval, AttachmentSet.eval, HingeSet.eval and their rowdiag
// (constraints.py:88-100, 220-237, 312-349; numba_backend.py:105-120)
__global__ void k_eval_misc(const Ctx c) {
  SETUP
  const int nd = c.D.nd, na = c.D.na, nh = c.D.nh, nb = c.D.nb;
  FOR_ITEMS(it, nd + na + nh) {
    if (it < nd) {
      const int d = it, i = c.T.d_i[d], j = c.T.d_j[d];
      double dx = c.S.pos[IX(3 * i)] - c.S.pos[IX(3 * j)];
      double dy = c.S.pos[IX(3 * i + 1)] - c.S.pos[IX(3 * j + 1)];
      double dz = c.S.pos[IX(3 * i + 2)] - c.S.pos[IX(3 * j + 2)];
      double ln = sqrt(dx * dx + dy * dy + dz * dz);
      double u0, u1, u2;
      if (ln > 1e-12) {
        u0 = dx / ln; u1 = dy / ln; u2 = dz / ln;
        c.S.dirs[IX(d)] = u0;
        c.S.dirs[IX(nd + d)] = u1;
        c.S.dirs[IX(2 * nd + d)] = u2;
      } else {
        u0 = c.S.dirs[IX(d)]; u1 = c.S.dirs[IX(nd + d)]; u2 = c.S.dirs[IX(2 * nd + d)];
      }
      double sc;
      const int ch = c.T.d_chan[d];
      if (c.D.act_enabled && ch >= 0) {
        sc = c.S.live[IX(ch)];
        c.S.scale[IX(d)] = sc;
      } else {
        sc = c.S.scale[IX(d)];
      }
      c.K.res[IX(c.D.od + d)] = ln - c.T.d_rest[d] * sc;
      const double mi = c.T.inv_mass[i], mj = c.T.inv_mass[j];
      const double nu0 = -u0, nu1 = -u1, nu2 = -u2;
      double acc = 0.0;
      acc += u0 * u0 * mi;
      acc += u1 * u1 * mi;
      acc += u2 * u2 * mi;
      acc += nu0 * nu0 * mj;
      acc += nu1 * nu1 * mj;
      acc += nu2 * nu2 * mj;
      c.K.bdiag[IX(c.D.od + d)] = acc;
    } else if (it < nd + na) {
      const int a = it - nd, b = c.T.a_b[a], pi = c.T.a_p[a];
      double R[9], anc[3], rw[3];
      quat_to_mat(c.S.bquat[IX(4 * b)], c.S.bquat[IX(4 * b + 1)], c.S.bquat[IX(4 * b + 2)],
                  c.S.bquat[IX(4 * b + 3)], R);
#pragma unroll
      for (int k = 0; k < 3; ++k) anc[k] = c.T.a_anc[k * na + a];
      matvec_es(R, anc, rw);
      double md[9];
      const double mp = c.T.inv_mass[pi];
      const int o = c.D.bd0 + 6 * b;
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        c.K.rw[IX(k * na + a)] = rw[k];
        c.K.res[IX(c.D.oa + k * na + a)] =
            c.S.bpos[IX(3 * b + k)] + rw[k] - c.S.pos[IX(3 * pi + k)];
        md[k] = mp;
      }
#pragma unroll
      for (int k = 0; k < 6; ++k) md[3 + k] = minv_diag_of(c, o + k, env);
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        double acc = 0.0;
#pragma unroll
        for (int col = 0; col < 9; ++col) {
          double v = att_val(i, col, rw);
          acc += v * v * md[col];
        }
        c.K.bdiag[IX(c.D.oa + i * na + a)] = acc;
      }
    } else {
      const int h = it - nd - na, ba = c.T.h_a[h], bb = c.T.h_b[h];
      double Ra[9], Rb[9], v3[3], ra[3], rb[3], na_[3], t1[3], t2[3], c1[3], c2[3];
      quat_to_mat(c.S.bquat[IX(4 * ba)], c.S.bquat[IX(4 * ba + 1)], c.S.bquat[IX(4 * ba + 2)],
                  c.S.bquat[IX(4 * ba + 3)], Ra);
      quat_to_mat(c.S.bquat[IX(4 * bb)], c.S.bquat[IX(4 * bb + 1)], c.S.bquat[IX(4 * bb + 2)],
                  c.S.bquat[IX(4 * bb + 3)], Rb);
#define LD3(src) for (int k = 0; k < 3; ++k) v3[k] = src[k * nh + h];
      LD3(c.T.h_anca) matvec_es(Ra, v3, ra);
      LD3(c.T.h_ancb) matvec_es(Rb, v3, rb);
      LD3(c.T.h_axa) matvec_es(Ra, v3, na_);
      LD3(c.T.h_t1) matvec_es(Rb, v3, t1);
      LD3(c.T.h_t2) matvec_es(Rb, v3, t2);
#undef LD3
#pragma unroll
      for (int k = 0; k < 3; ++k)
        c.K.res[IX(c.D.oh + k * nh + h)] =
            c.S.bpos[IX(3 * ba + k)] + ra[k] - c.S.bpos[IX(3 * bb + k)] - rb[k];
      c.K.res[IX(c.D.oh + 3 * nh + h)] = dot_es(t1, na_);
      c.K.res[IX(c.D.oh + 4 * nh + h)] = dot_es(t2, na_);
      double J[60];
#pragma unroll
      for (int k = 0; k < 60; ++k) J[k] = 0.0;
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        J[12 * a + a] = 1.0;
        J[12 * a + 6 + a] = -1.0;
      }
      J[0 * 12 + 4] = ra[2]; J[0 * 12 + 5] = -ra[1];
      J[1 * 12 + 3] = -ra[2]; J[1 * 12 + 5] = ra[0];
      J[2 * 12 + 3] = ra[1]; J[2 * 12 + 4] = -ra[0];
      J[0 * 12 + 10] = -rb[2]; J[0 * 12 + 11] = rb[1];
      J[1 * 12 + 9] = rb[2]; J[1 * 12 + 11] = -rb[0];
      J[2 * 12 + 9] = -rb[1]; J[2 * 12 + 10] = rb[0];
      cross3(na_, t1, c1);
      cross3(na_, t2, c2);
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        J[3 * 12 + 3 + a] = c1[a]; J[3 * 12 + 9 + a] = -c1[a];
        J[4 * 12 + 3 + a] = c2[a]; J[4 * 12 + 9 + a] = -c2[a];
      }
      double md[12];
#pragma unroll
      for (int k = 0; k < 6; ++k) {
        md[k] = minv_diag_of(c, c.D.bd0 + 6 * ba + k, env);
        md[6 + k] = minv_diag_of(c, c.D.bd0 + 6 * bb + k, env);
      }
#pragma unroll
      for (int i = 0; i < 5; ++i) {
        double acc = 0.0;
#pragma unroll
        for (int j = 0; j < 12; ++j) {
          double v = J[12 * i + j];
          c.K.hJ[IX((size_t)(12 * i + j) * nh + h)] = v;
          acc += v * v * md[j];
        }
        c.K.bdiag[IX(c.D.oh + i * nh + h)] = acc;
      }
    }
  }
}


// ------------------------------------------------------------ J^T gather
// mode 0 (apply_a, solver.py:380-387): w = J^T (act o x), u = M^-1 w.
// mode 1 (_apply_impulse, solver.py:537-544): v += M^-1 J^T x over the
// present contacts, friction rows regardless of the active set.
// xs: static rows [ms][E]; xc: contact rows [3 ns][E]; tets read their
// column sums from tC (written by the producing element kernel).
// One incidence (code = (fam<<29)|(v<<25)|e) of a particle's / a body's
// J^T list: its contribution to the DOF's w (block_transpose,
// numba_backend.py:43-52, per row); false when the row is inactive.
template <int IB = -1>
DI bool inc_particle(const Ctx& c, int k, int code, int mode, const double* __restrict__ xs,
                     const double* __restrict__ xc, int env, double& a0, double& a1,
                     double& a2) {
  const int E = c.D.E, nt = c.D.nt, na = c.D.na, ns = c.D.ns;
  (void)nt;
  const int fam = (int)((unsigned)code >> 29), v = (code >> 25) & 15, e = code & 0x1FFFFFF;
  if (fam == F_TET) {
    tc_get<IB>(c, k, v, e, env, a0, a1, a2);
  } else if (fam == F_DIST) {
    const int nd = c.D.nd;
    const double xr = xs[IX(c.D.od + e)];
    double d0 = c.S.dirs[IX(e)], d1 = c.S.dirs[IX(nd + e)], d2 = c.S.dirs[IX(2 * nd + e)];
    if (v) { d0 = -d0; d1 = -d1; d2 = -d2; }
    a0 = 0.0 + d0 * xr;
    a1 = 0.0 + d1 * xr;
    a2 = 0.0 + d2 * xr;
  } else if (fam == F_ATTP) {
    double x3[3];
    const double rw[3] = {0.0, 0.0, 0.0};
#pragma unroll
    for (int i = 0; i < 3; ++i) x3[i] = xs[IX(c.D.oa + i * na + e)];
    double acc[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      acc[a] = 0.0;
#pragma unroll
      for (int i = 0; i < 3; ++i) acc[a] += att_val(i, a, rw) * x3[i];
    }
    a0 = acc[0]; a1 = acc[1]; a2 = acc[2];
  } else {  // F_CN / F_CF on a particle slot: n = (0,0,1), t1 = (1,0,0), t2 = (0,1,0)
    const bool on = mode == 0 ? (fam == F_CN ? c.K.present[IX(e)] != 0 : c.K.actf[IX(e)] != 0.0)
                              : c.K.present[IX(e)] != 0;
    if (!on) return false;
    if (fam == F_CN) {
      const double xn = xc[IX(e)];
      a0 = 0.0 + 0.0 * xn;
      a1 = 0.0 + 0.0 * xn;
      a2 = 0.0 + 1.0 * xn;
    } else {
      const double xf0 = xc[IX(ns + e)], xf1 = xc[IX(2 * ns + e)];
      a0 = 0.0 + 1.0 * xf0;
      a0 += 0.0 * xf1;
      a1 = 0.0 + 0.0 * xf0;
      a1 += 1.0 * xf1;
      a2 = 0.0 + 0.0 * xf0;
      a2 += 0.0 * xf1;
    }
  }
  return true;
}
DI bool inc_body(const Ctx& c, int code, int mode, const double* __restrict__ xs,
                 const double* __restrict__ xc, int env, double* acc) {
  const int E = c.D.E, na = c.D.na, nh = c.D.nh, nw = c.D.nw, ns = c.D.ns;
  const int fam = (int)((unsigned)code >> 29), v = (code >> 25) & 15, e = code & 0x1FFFFFF;
  if (fam == F_ATTB) {
    double x3[3], rw[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      x3[i] = xs[IX(c.D.oa + i * na + e)];
      rw[i] = c.K.rw[IX(i * na + e)];
    }
#pragma unroll
    for (int kk = 0; kk < 6; ++kk) {
      acc[kk] = 0.0;
#pragma unroll
      for (int i = 0; i < 3; ++i) acc[kk] += att_val(i, 3 + kk, rw) * x3[i];
    }
  } else if (fam == F_HINGE) {
    double x5[5];
#pragma unroll
    for (int i = 0; i < 5; ++i) x5[i] = xs[IX(c.D.oh + i * nh + e)];
#pragma unroll
    for (int kk = 0; kk < 6; ++kk) {
      acc[kk] = 0.0;
#pragma unroll
      for (int i = 0; i < 5; ++i)
        acc[kk] += c.K.hJ[IX((size_t)(12 * i + 6 * v + kk) * nh + e)] * x5[i];
    }
  } else {  // wheel slot e (< nw)
    const bool on = mode == 0 ? (fam == F_CN ? c.K.present[IX(e)] != 0 : c.K.actf[IX(e)] != 0.0)
                              : c.K.present[IX(e)] != 0;
    if (!on) return false;
    if (fam == F_CN) {
      const double xn = xc[IX(e)];
#pragma unroll
      for (int kk = 0; kk < 6; ++kk) acc[kk] = 0.0 + c.K.wJ[IX((size_t)kk * nw + e)] * xn;
    } else {
      const double xf0 = xc[IX(ns + e)], xf1 = xc[IX(2 * ns + e)];
#pragma unroll
      for (int kk = 0; kk < 6; ++kk) {
        acc[kk] = 0.0 + c.K.wJ[IX((size_t)(6 + kk) * nw + e)] * xf0;
        acc[kk] += c.K.wJ[IX((size_t)(12 + kk) * nw + e)] * xf1;
      }
    }
  }
  return true;
}

#ifndef SS_GATHER_MINB
#define SS_GATHER_MINB 4
#endif
// minv_apply (numba_backend.py:68-82) of one body's w, stored (mode 0) or
// added to v (mode 1)
DI void gather_body_out(const Ctx& c, int b, int mode, const double* w, int env) {
  const int E = c.D.E;
  const double im = c.T.body_inv_mass[b];
  double u[6];
#pragma unroll
  for (int a = 0; a < 3; ++a) u[a] = im * w[a];
  const int nb = c.D.nb;
  double A[9];
#pragma unroll
  for (int k = 0; k < 9; ++k) A[k] = c.K.ang_inv[IX((size_t)k * nb + b)];
  u[3] = A[0] * w[3] + A[1] * w[4] + A[2] * w[5];
  u[4] = A[3] * w[3] + A[4] * w[4] + A[5] * w[5];
  u[5] = A[6] * w[3] + A[7] * w[4] + A[8] * w[5];
  const int o = c.D.bd0 + 6 * b;
  if (mode == 0) {
#pragma unroll
    for (int k = 0; k < 6; ++k) c.K.u[IX(o + k)] = u[k];
  } else {
#pragma unroll
    for (int k = 0; k < 6; ++k) c.K.v[IX(o + k)] += u[k];
  }
}

// SPLIT > 1 (structured mode, few env lanes): SPLIT adjacent item lanes
// share one DOF and walk every SPLIT-th incidence of its list, then combine
// with a fixed shuffle tree — the serial incidence walk of a lone env is
// latency-bound (one CTA column per 256 DOFs), this gives it SPLIT× the
// loads in flight. Not the reference's summation order (exact mode keeps
// SPLIT = 1).
// G = SPLIT | 16 * inbox layout
template <int G>
__global__ void __launch_bounds__(SS_THREADS, SS_GATHER_MINB) k_gather(const Ctx c, int mode,
                                                       const double* __restrict__ xs,
                                                       const double* __restrict__ xc) {
  constexpr int SPLIT = G & 15;
  constexpr int IB = G >> 4;
  SETUP
  const int P = c.D.P, nt = c.D.nt, na = c.D.na, nh = c.D.nh, nw = c.D.nw, ns = c.D.ns;
  if constexpr (SPLIT > 1) {
    (void)nt; (void)na; (void)nh; (void)nw; (void)ns;
    const int sub = il % SPLIT, ilg = il / SPLIT, ILg = IL / SPLIT;
    const int n_it = P + c.D.nb;
    // block-uniform trip count: every lane reaches the shuffles
    for (int it0 = blockIdx.y * ILg; it0 < n_it; it0 += gridDim.y * ILg) {
      const int it = it0 + ilg;
      double w[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
      if (it < n_it) {
        const int k0 = c.T.inc_ptr[it], k1 = c.T.inc_ptr[it + 1];
        if (it < P) {
          for (int k = k0 + sub; k < k1; k += SPLIT) {
            double a0, a1, a2;
            if (!inc_particle<IB>(c, k, c.T.inc[k], mode, xs, xc, env, a0, a1, a2)) continue;
            w[0] += a0;
            w[1] += a1;
            w[2] += a2;
          }
        } else {
          for (int k = k0 + sub; k < k1; k += SPLIT) {
            double acc[6];
            if (!inc_body(c, c.T.inc[k], mode, xs, xc, env, acc)) continue;
#pragma unroll
            for (int kk = 0; kk < 6; ++kk) w[kk] += acc[kk];
          }
        }
      }
#pragma unroll
      for (int off = SPLIT >> 1; off > 0; off >>= 1) {
#pragma unroll
        for (int kk = 0; kk < 6; ++kk) w[kk] += __shfl_xor_sync(0xffffffffu, w[kk], off * c.D.W);
      }
      if (it >= n_it || sub != 0) continue;
      if (it < P) {
        const double im = c.T.inv_mass[it];
        const double u0 = im * w[0], u1 = im * w[1], u2 = im * w[2];
        if (mode == 0) {
          c.K.u[IX(3 * it)] = u0;
          c.K.u[IX(3 * it + 1)] = u1;
          c.K.u[IX(3 * it + 2)] = u2;
        } else {
          c.K.v[IX(3 * it)] += u0;
          c.K.v[IX(3 * it + 1)] += u1;
          c.K.v[IX(3 * it + 2)] += u2;
        }
      } else {
        gather_body_out(c, it - P, mode, w, env);
      }
    }
  } else {
  FOR_ITEMS(it, P + c.D.nb) {
    const int k0 = c.T.inc_ptr[it], k1 = c.T.inc_ptr[it + 1];
    if (it < P) {
      double w0 = 0.0, w1 = 0.0, w2 = 0.0;
      // the list is sorted by family: [dist][tet][attach][contact normal][friction]
      const int2 tr = c.T.inc_tet[it];
#ifndef SS_GATHER_NO_FLAG_PREFETCH
      // a contact slot's flags (its last two entries) loaded now, so the slot's
      // test at the end of the walk does not wait a memory round trip
      int pf_slot = -1, pf_pres = 0;
      double pf_act = 0.0;
      if (k1 - k0 >= 2) {
        const int cl = c.T.inc[k1 - 1];
        if ((int)((unsigned)cl >> 29) == F_CF) {
          pf_slot = cl & 0x1FFFFFF;
          pf_pres = c.K.present[IX(pf_slot)];
          pf_act = c.K.actf[IX(pf_slot)];
        }
      }
#endif
      for (int k = k0; k < k1; ++k) {
        if (k == tr.x) {
          // tet run: column sums from tC, loads hoisted 4 incidences at a time
          const double* __restrict__ tC = c.K.tC;
#ifndef SS_GATHER_UNROLL
#define SS_GATHER_UNROLL 6
#endif
          constexpr int GU = SS_GATHER_UNROLL;
          for (; k + GU - 1 < tr.y; k += GU) {
            double a[3 * GU];
            if (IB == 1) {
#pragma unroll
              for (int j = 0; j < GU; ++j) tc_ld4(tC + 4 * (size_t)(k + j), a[3 * j], a[3 * j + 1], a[3 * j + 2]);
            } else if (IB == 2) {
              // incidence order: the run's addresses follow from k, no code lookup
              const double* p = tC + (size_t)k * 3 * E + env;
#pragma unroll
              for (int j = 0; j < 3 * GU; ++j) a[j] = p[(size_t)j * E];
            } else {
#pragma unroll
              for (int j = 0; j < GU; ++j) {
                const int code = c.T.inc[k + j];
                const int v = (code >> 25) & 15, e = code & 0x1FFFFFF;
                a[3 * j] = tC[TCX(3 * v, e)];
                a[3 * j + 1] = tC[TCX(3 * v + 1, e)];
                a[3 * j + 2] = tC[TCX(3 * v + 2, e)];
              }
            }
#pragma unroll
            for (int j = 0; j < GU; ++j) {
              w0 += a[3 * j];
              w1 += a[3 * j + 1];
              w2 += a[3 * j + 2];
            }
          }
          for (; k < tr.y; ++k) {
            const int code = c.T.inc[k];
            const int v = (code >> 25) & 15, e = code & 0x1FFFFFF;
            double a0, a1, a2;
            tc_get<IB>(c, k, v, e, env, a0, a1, a2);
            w0 += a0;
            w1 += a1;
            w2 += a2;
          }
          if (k >= k1) break;
        }
        const int code = c.T.inc[k];
        double a0, a1, a2;
#ifndef SS_GATHER_NO_FLAG_PREFETCH
        {
          const int fam = (int)((unsigned)code >> 29);
          if ((fam == F_CN || fam == F_CF) && (code & 0x1FFFFFF) == pf_slot) {
            // inc_particle's contact branch with the prefetched flags
            const bool on = mode == 0 ? (fam == F_CN ? pf_pres != 0 : pf_act != 0.0) : pf_pres != 0;
            if (!on) continue;
            const int e = pf_slot;
            if (fam == F_CN) {
              const double xn = xc[IX(e)];
              a0 = 0.0 + 0.0 * xn;
              a1 = 0.0 + 0.0 * xn;
              a2 = 0.0 + 1.0 * xn;
            } else {
              const double xf0 = xc[IX(ns + e)], xf1 = xc[IX(2 * ns + e)];
              a0 = 0.0 + 1.0 * xf0;
              a0 += 0.0 * xf1;
              a1 = 0.0 + 0.0 * xf0;
              a1 += 1.0 * xf1;
              a2 = 0.0 + 0.0 * xf0;
              a2 += 0.0 * xf1;
            }
            w0 += a0;
            w1 += a1;
            w2 += a2;
            continue;
          }
        }
#endif
        if (!inc_particle<IB>(c, k, code, mode, xs, xc, env, a0, a1, a2)) continue;
        w0 += a0;
        w1 += a1;
        w2 += a2;
      }
      const double im = c.T.inv_mass[it];
      const double u0 = im * w0, u1 = im * w1, u2 = im * w2;
      if (mode == 0) {
        c.K.u[IX(3 * it)] = u0;
        c.K.u[IX(3 * it + 1)] = u1;
        c.K.u[IX(3 * it + 2)] = u2;
      } else {
        c.K.v[IX(3 * it)] += u0;
        c.K.v[IX(3 * it + 1)] += u1;
        c.K.v[IX(3 * it + 2)] += u2;
      }
    } else {
      const int b = it - P;
      double w[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
      for (int k = k0; k < k1; ++k) {
        const int code = c.T.inc[k];
        double acc[6];
        if (!inc_body(c, code, mode, xs, xc, env, acc)) continue;
#pragma unroll
        for (int kk = 0; kk < 6; ++kk) w[kk] += acc[kk];
      }
      gather_body_out(c, b, mode, w, env);
    }
  }
  }
}

// ------------------------------- bulk-copy J^T x gather (one large mesh, E = 1)
// With the incidence-order column sums (tc_inbox) the tet runs of 32
// consecutive particles are ONE contiguous byte range of tC: [lo, hi) =
// [first particle's run start, last particle's run end) x 32 B. A warp takes
// 32 particles; lane 0 streams that range into a per-warp shared-memory ring
// in windows of SS_GB_WIN incidences with cp.async.bulk (TMA bulk copy,
// completion counted on an mbarrier), SS_GB_NBUF windows in flight; every
// lane then adds its own particle's entries from shared memory in incidence
// order. Each particle's sum is the same sequence of additions as k_gather's
// serial walk (non-tet entries before and after the run from global memory,
// as there), so u / v are bitwise k_gather<17>'s. The serial walk issued one
// scattered 32-byte load per incidence and lane; here the tC stream moves as
// 4 KB copies (1M-tet scene: 10.0 -> 8.6 ms/frame). Measured and not kept
// (profiles/r2_summary.md): whole-span buffers per warp (~20 KB, 9 warps/SM),
// chunk-pipelined double buffers with the non-tet operands of the next chunk
// in flight (5 warps/SM): 10.6-13.9 ms/frame — the walk needs the warps.
#ifndef SS_GB_WIN
#define SS_GB_WIN 128  // incidences per window (32 B each)
#endif
#ifndef SS_GB_NBUF
#define SS_GB_NBUF 2
#endif
#ifndef SS_GB_MINB
#define SS_GB_MINB 3
#endif
#define SS_GB_WARPS (SS_THREADS / 32)
constexpr size_t kGbSmem = (size_t)SS_GB_WARPS * SS_GB_NBUF * SS_GB_WIN * 32;

DI uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
DI void mbar_init(uint64_t* b, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(b)), "r"(count) : "memory");
}
DI bool mbar_try_wait(uint64_t* b, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      " selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_addr(b)), "r"(parity)
      : "memory");
  return ok != 0;
}
// lane 0 of a warp: arm the barrier for `bytes` and start the bulk copy
DI void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
               "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}

__global__ void __launch_bounds__(SS_THREADS, SS_GB_MINB) k_gather_bulk(const Ctx c, int mode,
                                                        const double* __restrict__ xs,
                                                        const double* __restrict__ xc) {
  pdl_wait();
  extern __shared__ __align__(128) double gb_smem[];
  __shared__ uint64_t gbar[SS_GB_WARPS][SS_GB_NBUF];
  const int E = 1, env = 0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int P = c.D.P;
  if (lane == 0) {
#pragma unroll
    for (int b = 0; b < SS_GB_NBUF; ++b) mbar_init(&gbar[warp][b], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  double* ring = gb_smem + (size_t)warp * SS_GB_NBUF * SS_GB_WIN * 4;
  const double* tC = c.K.tC;
  uint32_t phase = 0;  // bit b: parity of buffer b's next completion
  const int nchunks = (P + 31) >> 5;
  for (int ch = blockIdx.x * SS_GB_WARPS + warp; ch < nchunks; ch += gridDim.x * SS_GB_WARPS) {
    const int it = ch * 32 + lane;
    const bool act = it < P;
    int k0 = 0, k1 = 0;
    int2 tr = make_int2(-1, -1);
    if (act) {
      k0 = c.T.inc_ptr[it];
      k1 = c.T.inc_ptr[it + 1];
      tr = c.T.inc_tet[it];
    }
    const bool has_run = tr.x >= 0 && tr.y > tr.x;
    const int lo = __reduce_min_sync(0xffffffffu, has_run ? tr.x : INT_MAX);
    const int hi = __reduce_max_sync(0xffffffffu, has_run ? tr.y : INT_MIN);
    const int nwin = lo == INT_MAX ? 0 : (hi - lo + SS_GB_WIN - 1) / SS_GB_WIN;
    if (lane == 0) {
      for (int w = 0; w < SS_GB_NBUF && w < nwin; ++w) {
        const int wlo = lo + w * SS_GB_WIN, wn = min(SS_GB_WIN, hi - wlo);
        bulk_load(ring + (size_t)w * SS_GB_WIN * 4, tC + 4 * (size_t)wlo, 32u * wn, &gbar[warp][w]);
      }
    }
    double w0 = 0.0, w1 = 0.0, w2 = 0.0;
    double a0, a1, a2;
    // entries before the tet run (distance rows), while the first windows land
    const int kpre = has_run ? tr.x : k1;
    for (int k = k0; k < kpre; ++k) {
      if (!inc_particle<1>(c, k, c.T.inc[k], mode, xs, xc, env, a0, a1, a2)) continue;
      w0 += a0;
      w1 += a1;
      w2 += a2;
    }
    for (int w = 0; w < nwin; ++w) {
      const int b = w % SS_GB_NBUF;
      while (!mbar_try_wait(&gbar[warp][b], (phase >> b) & 1u)) {
      }
      phase ^= 1u << b;
      const int wlo = lo + w * SS_GB_WIN, whi = min(wlo + SS_GB_WIN, hi);
      if (has_run) {
        const double* sb = ring + (size_t)b * SS_GB_WIN * 4;
        const int ka = max(tr.x, wlo), kb = min(tr.y, whi);
        for (int k = ka; k < kb; ++k) {
          const double2 v01 = *reinterpret_cast<const double2*>(sb + 4 * (k - wlo));
          const double v2 = sb[4 * (k - wlo) + 2];
          w0 += v01.x;
          w1 += v01.y;
          w2 += v2;
        }
      }
      // the warp's generic-proxy reads of buffer b are done (syncwarp); the
      // fence orders them before the async-proxy refill (this window's
      // successor, or the next chunk's first windows)
      __syncwarp();
      if (lane == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        if (w + SS_GB_NBUF < nwin) {
          const int nlo = lo + (w + SS_GB_NBUF) * SS_GB_WIN, nn = min(SS_GB_WIN, hi - nlo);
          bulk_load(ring + (size_t)b * SS_GB_WIN * 4, tC + 4 * (size_t)nlo, 32u * nn,
                    &gbar[warp][b]);
        }
      }
    }
    if (!act) continue;
    for (int k = has_run ? tr.y : k1; k < k1; ++k) {
      if (!inc_particle<1>(c, k, c.T.inc[k], mode, xs, xc, env, a0, a1, a2)) continue;
      w0 += a0;
      w1 += a1;
      w2 += a2;
    }
    const double im = c.T.inv_mass[it];
    const double u0 = im * w0, u1 = im * w1, u2 = im * w2;
    if (mode == 0) {
      c.K.u[IX(3 * it)] = u0;
      c.K.u[IX(3 * it + 1)] = u1;
      c.K.u[IX(3 * it + 2)] = u2;
    } else {
      c.K.v[IX(3 * it)] += u0;
      c.K.v[IX(3 * it + 1)] += u1;
      c.K.v[IX(3 * it + 2)] += u2;
    }
  }
  // rigid bodies: k_gather's body walk
  for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < c.D.nb; b += gridDim.x * blockDim.x) {
    const int k0 = c.T.inc_ptr[P + b], k1 = c.T.inc_ptr[P + b + 1];
    double w[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    for (int k = k0; k < k1; ++k) {
      double acc[6];
      if (!inc_body(c, c.T.inc[k], mode, xs, xc, env, acc)) continue;
#pragma unroll
      for (int kk = 0; kk < 6; ++kk) w[kk] += acc[kk];
    }
    gather_body_out(c, b, mode, w, env);
  }
}

// ------------------------------------ persistent tile-pipelined J^T z gather
// k_tet_jt + k_gather<1> (mode 0) of one PCR iteration as ONE persistent
// launch over a queue of work items, per 32-env tile: P1(T) pieces compute
// the tet column sums of tile T into a ring slot, P2(T) pieces gather them
// per DOF (same code, same order: bitwise the two-kernel result). The queue
// interleaves tiles with a lag (P1(T + lag) before P2(T)), so a tile's
// column sums are read back a few microseconds after they are written and
// stay in L2 (the ring is an L2-persisting access window): the 24 doubles
// per tet of tC traffic leave HBM. Items are dequeued with an atomic head,
// so every item a CTA waits on is held by a running CTA (no deadlock under
// partial residency). Needs E % 32 == 0 (one tile = 32 env lanes).
#ifndef JTG_TETS
#define JTG_TETS 128   // tets per P1 piece (8 item lanes x 16)
#endif
#ifndef JTG_NODES
#define JTG_NODES 64   // DOFs (particles, then bodies) per P2 piece
#endif
struct JtgPlan {
  int tiles, n1, n2, lag, ring, n_items;
};
DI void jtg_decode(const JtgPlan& jp, int q, int& phase, int& T, int& piece) {
  // step s holds [P1(s) if s < tiles][P2(s - lag) if s >= lag]
  const int tl = jp.tiles, lag = jp.lag, n1 = jp.n1, n2 = jp.n2;
  // steps 0..lag-1 hold only P1 pieces
  const int head = lag * n1;
  if (q < head) {
    phase = 1; T = q / n1; piece = q % n1;
    return;
  }
  q -= head;
  const int mid = (tl - lag) * (n1 + n2);  // steps lag..tiles-1 hold both
  if (q < mid) {
    const int s = lag + q / (n1 + n2), r = q % (n1 + n2);
    if (r < n1) { phase = 1; T = s; piece = r; }
    else { phase = 2; T = s - lag; piece = r - n1; }
    return;
  }
  q -= mid;  // steps tiles..tiles+lag-1 hold only P2 pieces
  phase = 2; T = tl - lag + q / n2; piece = q % n2;
}
DI void jtg_wait(const int* ctr, int target) {
  if (threadIdx.x == 0) {
    while (*(volatile const int*)ctr < target) __nanosleep(32);
    __threadfence();
  }
  __syncthreads();
}
DI void jtg_signal(int* ctr) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(ctr, 1);
  }
}

#ifndef SS_JTG_MINB
#define SS_JTG_MINB 3
#endif
__global__ void __launch_bounds__(SS_THREADS, SS_JTG_MINB) k_jtg(const Ctx c, const JtgPlan jp) {
  pdl_wait();
  const int E = c.D.E, nt = c.D.nt, P = c.D.P, nb = c.D.nb;
  const int lane = threadIdx.x & 31, il = threadIdx.x >> 5;
  int* head = c.K.jctr;
  int* p1_done = c.K.jctr + 1;
  int* p2_done = c.K.jctr + 1 + jp.tiles;
  const double* __restrict__ xs = c.K.z;
  const double* __restrict__ xc = c.K.z + (size_t)c.D.ms * E;
  __shared__ int s_next;
  if (threadIdx.x == 0) s_next = atomicAdd(head, 1);
  for (;;) {
    __syncthreads();
    const int q = s_next;
    __syncthreads();
    if (q >= jp.n_items) return;
    // the next item is claimed now; its atomic overlaps this item's work
    if (threadIdx.x == 0) s_next = atomicAdd(head, 1);
    int phase, T, piece;
    jtg_decode(jp, q, phase, T, piece);
    const int env = T * 32 + lane;
    double* ring = c.K.ring + (size_t)(T % jp.ring) * 12 * nt * 32;
    if (phase == 1) {
      if (T >= jp.ring) jtg_wait(p2_done + T - jp.ring, jp.n2);  // ring slot free
      const int t0 = piece * JTG_TETS;
      for (int t = t0 + il; t < t0 + JTG_TETS && t < nt; t += 8) {
        double z6[6], Ri[9], col12[12];
#pragma unroll
        for (int i = 0; i < 6; ++i) z6[i] = c.K.z[IX(c.D.ot + i * nt + t)];
        TetC TT;
        tet_load(c, t, env, TT);
        tet_rinv(c, t, Ri);
        tet_jt_cols(TT, Ri, z6, col12);
#pragma unroll
        for (int k = 0; k < 12; ++k) ring[((size_t)k * nt + t) * 32 + lane] = col12[k];
      }
      jtg_signal(p1_done + T);
    } else {
      jtg_wait(p1_done + T, jp.n1);
      const int n0 = piece * JTG_NODES;
      for (int it = n0 + il; it < n0 + JTG_NODES && it < P + nb; it += 8) {
        const int k0 = c.T.inc_ptr[it], k1 = c.T.inc_ptr[it + 1];
        if (it < P) {
          double w0 = 0.0, w1 = 0.0, w2 = 0.0;
          const int2 tr = c.T.inc_tet[it];
          for (int k = k0; k < k1; ++k) {
            if (k == tr.x) {
              // loads hoisted 6 incidences at a time (k_gather's order of adds)
              constexpr int GU = 6;
              for (; k + GU - 1 < tr.y; k += GU) {
                double a[3 * GU];
#pragma unroll
                for (int j = 0; j < GU; ++j) {
                  const int code = c.T.inc[k + j];
                  const int v = (code >> 25) & 15, e = code & 0x1FFFFFF;
                  const double* rp = ring + ((size_t)(3 * v) * nt + e) * 32 + lane;
                  a[3 * j] = __ldcg(rp);
                  a[3 * j + 1] = __ldcg(rp + (size_t)nt * 32);
                  a[3 * j + 2] = __ldcg(rp + (size_t)2 * nt * 32);
                }
#pragma unroll
                for (int j = 0; j < GU; ++j) {
                  w0 += a[3 * j];
                  w1 += a[3 * j + 1];
                  w2 += a[3 * j + 2];
                }
              }
              for (; k < tr.y; ++k) {
                const int code = c.T.inc[k];
                const int v = (code >> 25) & 15, e = code & 0x1FFFFFF;
                const double* rp = ring + ((size_t)(3 * v) * nt + e) * 32 + lane;
                w0 += __ldcg(rp);
                w1 += __ldcg(rp + (size_t)nt * 32);
                w2 += __ldcg(rp + (size_t)2 * nt * 32);
              }
              if (k >= k1) break;
            }
            double a0, a1, a2;
            if (!inc_particle(c, k, c.T.inc[k], 0, xs, xc, env, a0, a1, a2)) continue;
            w0 += a0;
            w1 += a1;
            w2 += a2;
          }
          const double im = c.T.inv_mass[it];
          c.K.u[IX(3 * it)] = im * w0;
          c.K.u[IX(3 * it + 1)] = im * w1;
          c.K.u[IX(3 * it + 2)] = im * w2;
        } else {
          double w[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
          for (int k = k0; k < k1; ++k) {
            double acc[6];
            if (!inc_body(c, c.T.inc[k], 0, xs, xc, env, acc)) continue;
#pragma unroll
            for (int kk = 0; kk < 6; ++kk) w[kk] += acc[kk];
          }
          gather_body_out(c, it - P, 0, w, env);
        }
      }
      jtg_signal(p2_done + T);
    }
  }
}

// ------------------------------------------------ fused J^T z gather
// The PCR operator's J^T z -> u = M^-1 J^T z without the tet column sums in
// HBM (structured mode). Particles are partitioned into blocks (the snake:
// one block per link, no element spans two links); a CTA owns one block for
// FW env-lanes and accumulates the block's node sums in shared memory. Every
// element touching the block is scattered into them in a static schedule of
// conflict-free chunks (no two elements of a chunk share a node of the
// block; a barrier between chunks), families in the reference's order —
// distance rows, tets, attachments, contact normals, contact friction —
// so every node's sum is a fixed-order, deterministic sum of the same terms
// k_gather adds (per-term values bitwise equal; the order within a family
// is the chunk order instead of ascending element id). The tet terms are
// computed from z, the quaternion and S (tet_jt_cols) on the fly: 24 fewer
// doubles of HBM traffic per tet and PCR iteration than k_tet_jt writing tC
// and k_gather reading it back, and one launch fewer.
struct FusedPlan {
  int n_blocks;      // particle blocks (the body CTAs follow: blockIdx.y == n_blocks)
  int FW, FIL;       // env lanes x item lanes per CTA (FW * FIL = SS_THREADS); chunk <= FIL
  int nb_max;        // particles of the largest block (shared accumulator rows)
  const int* blk_p0;    // [n_blocks] first particle
  const int* blk_np;    // [n_blocks] particle count
  const int* blk_cptr;  // [n_blocks + 1] chunks of each block
  const int* chk;       // [n_chunks] family << 24 | element count; [n_chunks + 1] starts follow
  const int* elist;     // element ids (family-local), chunk after chunk
  const int2* enode;    // per elist entry: its 4 block-local particles, 16 bits each (0xFFFF: none)
  int sched_max;        // ints of the largest block's schedule (shared copy)
};

// raw loads of one element of a chunk (issued one chunk ahead)
struct FLoad {
  double x[16];
  int idx[4];
  int fam;
  int e;  // -1: no element for this thread
};

// sched (shared): [nch] headers, [nch] starts (block-relative), then per
// element its id and its packed particles (2 ints)
template <int FW>
DI void fused_load(const Ctx& c, const int* sched, int nch, int k, int il, int env, FLoad& L) {
  const int E = c.D.E, nt = c.D.nt, nd = c.D.nd, na = c.D.na, ns = c.D.ns;
  const int hdr = sched[k];
  L.fam = hdr >> 24;
  const int cnt = hdr & 0xFFFFFF;
  L.e = -1;
  if (il >= cnt) return;
  const int* el = sched + 2 * nch + 3 * (sched[nch + k] + il);
  const int e = el[0];
  const unsigned pk0 = (unsigned)el[1], pk1 = (unsigned)el[2];
  L.e = e;
  L.idx[0] = (int)(pk0 & 0xFFFF);
  L.idx[1] = (int)(pk0 >> 16);
  L.idx[2] = (int)(pk1 & 0xFFFF);
  L.idx[3] = (int)(pk1 >> 16);
  const double* __restrict__ xs = c.K.z;
  const double* __restrict__ xc = c.K.z + (size_t)c.D.ms * E;
  if (L.fam == F_TET) {
#pragma unroll
    for (int i = 0; i < 6; ++i) L.x[i] = xs[IX(c.D.ot + i * nt + e)];
#pragma unroll
    for (int q = 0; q < 4; ++q) L.x[6 + q] = c.S.quat[IX(q * nt + e)];
#pragma unroll
    for (int q = 0; q < 6; ++q) L.x[10 + q] = c.K.tS[IX(q * nt + e)];
  } else if (L.fam == F_DIST) {
    L.x[0] = xs[IX(c.D.od + e)];
    L.x[1] = c.S.dirs[IX(e)];
    L.x[2] = c.S.dirs[IX(nd + e)];
    L.x[3] = c.S.dirs[IX(2 * nd + e)];
  } else if (L.fam == F_ATTP) {
#pragma unroll
    for (int i = 0; i < 3; ++i) L.x[i] = xs[IX(c.D.oa + i * na + e)];
  } else {  // particle contact slot e
    L.x[0] = c.K.present[IX(e)] != 0 ? 1.0 : 0.0;
    L.x[1] = xc[IX(e)];
    L.x[2] = c.K.actf[IX(e)];
    L.x[3] = xc[IX(ns + e)];
    L.x[4] = xc[IX(2 * ns + e)];
  }
}

// one element's contribution to up to 4 particles (block-local; -1: none),
// per-term values exactly those of inc_particle
DI void fused_contrib(const Ctx& c, const FLoad& L, int* node, double* v) {
  node[0] = node[1] = node[2] = node[3] = 0xFFFF;
  if (L.e < 0) return;
  if (L.fam == F_TET) {
    TetC T;
    double Ri[9];
    tet_unpack(L.x + 6, L.x + 10, T);
    tet_rinv(c, L.e, Ri);
    tet_jt_cols(T, Ri, L.x, v);
#pragma unroll
    for (int k = 0; k < 4; ++k) node[k] = L.idx[k];
  } else if (L.fam == F_DIST) {
    const double xr = L.x[0], d0 = L.x[1], d1 = L.x[2], d2 = L.x[3];
    node[0] = L.idx[0];
    node[1] = L.idx[1];
    v[0] = 0.0 + d0 * xr;
    v[1] = 0.0 + d1 * xr;
    v[2] = 0.0 + d2 * xr;
    v[3] = 0.0 + (-d0) * xr;
    v[4] = 0.0 + (-d1) * xr;
    v[5] = 0.0 + (-d2) * xr;
  } else if (L.fam == F_ATTP) {
    const double rw[3] = {0.0, 0.0, 0.0};
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      double s_ = 0.0;
#pragma unroll
      for (int i = 0; i < 3; ++i) s_ += att_val(i, a, rw) * L.x[i];
      v[a] = s_;
    }
    node[0] = L.idx[0];
  } else {
    // contact slot: normal row (if present), then friction rows (if active);
    // as two terms added in that order (slot 0 and slot 1 of the same node)
    const double xn = L.x[1], xf0 = L.x[3], xf1 = L.x[4];
    if (L.x[0] != 0.0) {
      v[0] = 0.0 + 0.0 * xn;
      v[1] = 0.0 + 0.0 * xn;
      v[2] = 0.0 + 1.0 * xn;
      node[0] = L.idx[0];
    }
    if (L.x[2] != 0.0) {
      double a0 = 0.0 + 1.0 * xf0;
      a0 += 0.0 * xf1;
      double a1 = 0.0 + 0.0 * xf0;
      a1 += 1.0 * xf1;
      double a2 = 0.0 + 0.0 * xf0;
      a2 += 0.0 * xf1;
      v[3] = a0;
      v[4] = a1;
      v[5] = a2;
      node[1] = L.idx[0];
    }
  }
}

#ifndef SS_FUSED_MINB
#define SS_FUSED_MINB 2
#endif
template <int FW>
__global__ void __launch_bounds__(SS_THREADS, SS_FUSED_MINB) k_gather_fused(const Ctx c, const FusedPlan fp) {
  pdl_wait();
  extern __shared__ double fsm[];
  constexpr int FIL = SS_THREADS / FW;
  const int E = c.D.E;
  const int lane = threadIdx.x % FW, il = threadIdx.x / FW;
  const int env = blockIdx.x * FW + lane;
  const int P = c.D.P;
  if ((int)blockIdx.y >= fp.n_blocks) {
    // bodies (k_gather<1> body branch)
    const double* __restrict__ xs = c.K.z;
    const double* __restrict__ xc = c.K.z + (size_t)c.D.ms * E;
    for (int b = il; b < c.D.nb; b += FIL) {
      const int it = P + b;
      const int k0 = c.T.inc_ptr[it], k1 = c.T.inc_ptr[it + 1];
      double w[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
      for (int k = k0; k < k1; ++k) {
        double acc[6];
        if (!inc_body(c, c.T.inc[k], 0, xs, xc, env, acc)) continue;
#pragma unroll
        for (int kk = 0; kk < 6; ++kk) w[kk] += acc[kk];
      }
      gather_body_out(c, b, 0, w, env);
    }
    return;
  }
  const int blk = blockIdx.y;
  const int p0 = fp.blk_p0[blk], np = fp.blk_np[blk];
  double* acc = fsm;  // [np * 3][FW]
  int* sched = reinterpret_cast<int*>(fsm + (size_t)fp.nb_max * 3 * FW);
  for (int k = threadIdx.x; k < np * 3 * FW; k += SS_THREADS) acc[k] = 0.0;
  const int c0 = fp.blk_cptr[blk], c1 = fp.blk_cptr[blk + 1], nch = c1 - c0;
  {
    // this block's schedule into shared memory (headers, starts, elements)
    const int n_all = fp.blk_cptr[fp.n_blocks];
    const int s_0 = fp.chk[n_all + c0];
    const int s_1 = fp.chk[n_all + c1];
    for (int k = threadIdx.x; k < nch; k += SS_THREADS) {
      sched[k] = fp.chk[c0 + k];
      sched[nch + k] = fp.chk[n_all + c0 + k] - s_0;
    }
    int* el = sched + 2 * nch;
    for (int k = threadIdx.x; k < s_1 - s_0; k += SS_THREADS) {
      const int2 pk = fp.enode[s_0 + k];
      el[3 * k] = fp.elist[s_0 + k];
      el[3 * k + 1] = pk.x;
      el[3 * k + 2] = pk.y;
    }
  }
  __syncthreads();
  FLoad L;
  if (nch > 0) fused_load<FW>(c, sched, nch, 0, il, env, L);
  for (int k = 0; k < nch; ++k) {
    int node[4];
    double v[12];
    fused_contrib(c, L, node, v);
    if (k + 1 < nch) fused_load<FW>(c, sched, nch, k + 1, il, env, L);  // in flight over the adds
    __syncthreads();  // the previous chunk's adds are done
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int n = node[k];
      if (n >= np) continue;  // 0xFFFF: no particle of this block
      double* a = acc + (size_t)(3 * n) * FW + lane;
      a[0] += v[3 * k];
      a[FW] += v[3 * k + 1];
      a[2 * FW] += v[3 * k + 2];
    }
  }
  __syncthreads();
  for (int n = il; n < np; n += FIL) {
    const int it = p0 + n;
    const double im = c.T.inv_mass[it];
    c.K.u[IX(3 * it)] = im * acc[(3 * n) * FW + lane];
    c.K.u[IX(3 * it + 1)] = im * acc[(3 * n + 1) * FW + lane];
    c.K.u[IX(3 * it + 2)] = im * acc[(3 * n + 2) * FW + lane];
  }
}

// --------------------------------------------------------------- J rows
// block_forward of each family on a DOF vector vec ([ndof][E]);
// numba_backend.py:31-40 order (j ascending from acc = 0).
DI double row_dist(const Ctx& c, int d, const double* vec, int env) {
  const int E = c.D.E, nd = c.D.nd;
  const int i = c.T.d_i[d], j = c.T.d_j[d];
  const double u0 = c.S.dirs[IX(d)], u1 = c.S.dirs[IX(nd + d)], u2 = c.S.dirs[IX(2 * nd + d)];
  double acc = 0.0;
  acc += u0 * vec[IX(3 * i)];
  acc += u1 * vec[IX(3 * i + 1)];
  acc += u2 * vec[IX(3 * i + 2)];
  acc += -u0 * vec[IX(3 * j)];
  acc += -u1 * vec[IX(3 * j + 1)];
  acc += -u2 * vec[IX(3 * j + 2)];
  return acc;
}
DI void rows_att(const Ctx& c, int a, const double* vec, int env, double* y) {
  const int E = c.D.E, na = c.D.na;
  const int pi = c.T.a_p[a], o = c.D.bd0 + 6 * c.T.a_b[a];
  double uu[9], rw[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    uu[k] = vec[IX(3 * pi + k)];
    rw[k] = c.K.rw[IX(k * na + a)];
  }
#pragma unroll
  for (int k = 0; k < 6; ++k) uu[3 + k] = vec[IX(o + k)];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    double acc = 0.0;
#pragma unroll
    for (int j = 0; j < 9; ++j) acc += att_val(i, j, rw) * uu[j];
    y[i] = acc;
  }
}
DI void rows_hinge(const Ctx& c, int h, const double* vec, int env, double* y) {
  const int E = c.D.E, nh = c.D.nh;
  const int oa = c.D.bd0 + 6 * c.T.h_a[h], ob = c.D.bd0 + 6 * c.T.h_b[h];
  double uu[12];
#pragma unroll
  for (int k = 0; k < 6; ++k) {
    uu[k] = vec[IX(oa + k)];
    uu[6 + k] = vec[IX(ob + k)];
  }
#pragma unroll
  for (int i = 0; i < 5; ++i) {
    double acc = 0.0;
#pragma unroll
    for (int j = 0; j < 12; ++j) acc += c.K.hJ[IX((size_t)(12 * i + j) * nh + h)] * uu[j];
    y[i] = acc;
  }
}
// contact slot rows (normal, friction0, friction1) for a present slot
DI void rows_slot(const Ctx& c, int s, const double* vec, int env, double* y) {
  const int E = c.D.E, nw = c.D.nw;
  if (s < nw) {
    const int o = c.D.bd0 + 6 * c.T.w_body[s];
    double uu[6];
#pragma unroll
    for (int k = 0; k < 6; ++k) uu[k] = vec[IX(o + k)];
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      double acc = 0.0;
#pragma unroll
      for (int k = 0; k < 6; ++k) acc += c.K.wJ[IX((size_t)(6 * r + k) * nw + s)] * uu[k];
      y[r] = acc;
    }
  } else {
    const int pi = c.T.slot_part[s - nw];
    const double x0 = vec[IX(3 * pi)], x1 = vec[IX(3 * pi + 1)], x2 = vec[IX(3 * pi + 2)];
    const double z0 = vec[IX(0)];
    // padded columns 3..5 reference DOF 0 with zero values (contact.py:210-214)
    double a = 0.0;
    a += 0.0 * x0; a += 0.0 * x1; a += 1.0 * x2; a += 0.0 * z0; a += 0.0 * z0; a += 0.0 * z0;
    y[0] = a;
    a = 0.0;
    a += 1.0 * x0; a += 0.0 * x1; a += 0.0 * x2; a += 0.0 * z0; a += 0.0 * z0; a += 0.0 * z0;
    y[1] = a;
    a = 0.0;
    a += 0.0 * x0; a += 1.0 * x1; a += 0.0 * x2; a += 0.0 * z0; a += 0.0 * z0; a += 0.0 * z0;
    y[2] = a;
  }
}

// isotropic E_tet row products (ereg_apply, numba_backend.py:85-94; the
// zero entries of the Voigt pattern contribute exact zeros)
DI void ereg6(double ed, double eo, double es, const double* x, double* o) {
  o[0] = 0.0 + ed * x[0]; o[0] += eo * x[1]; o[0] += eo * x[2];
  o[1] = 0.0 + eo * x[0]; o[1] += ed * x[1]; o[1] += eo * x[2];
  o[2] = 0.0 + eo * x[0]; o[2] += eo * x[1]; o[2] += ed * x[2];
  o[3] = 0.0 + es * x[3];
  o[4] = 0.0 + es * x[4];
  o[5] = 0.0 + es * x[5];
}

// Rows owned by element item `it` (dist 1, tet 6, attach 3, hinge 5, slot 3
// when present, else 0) for this env.
DI int item_rows(const Ctx& c, int it, int env, int* rows) {
  const int E = c.D.E;
  const int nd = c.D.nd, nt = c.D.nt, na = c.D.na, nh = c.D.nh, ns = c.D.ns;
  if (it < nd) {
    rows[0] = c.D.od + it;
    return 1;
  }
  it -= nd;
  if (it < nt) {
#pragma unroll
    for (int i = 0; i < 6; ++i) rows[i] = c.D.ot + i * nt + it;
    return 6;
  }
  it -= nt;
  if (it < na) {
#pragma unroll
    for (int i = 0; i < 3; ++i) rows[i] = c.D.oa + i * na + it;
    return 3;
  }
  it -= na;
  if (it < nh) {
#pragma unroll
    for (int i = 0; i < 5; ++i) rows[i] = c.D.oh + i * nh + it;
    return 5;
  }
  it -= nh;
  if (!c.K.present[IX(it)]) return 0;
  rows[0] = c.D.on + it;
  rows[1] = c.D.of + it;
  rows[2] = c.D.of + ns + it;
  return 3;
}

// one item of the Newton head (k_newton_rhs): jv = J v, rhs, FB, active
// set, diagonal, z = r/d, x = 0, and the tet column sums of J^T z
template <bool EXACT>
DI void rhs_item(const Ctx& c, int it, int env) {
  const int E = c.D.E;
  const int nd = c.D.nd, nt = c.D.nt, na = c.D.na, nh = c.D.nh, ns = c.D.ns;
  const double g = c.p.gamma, h = c.p.h;
  const double* v = c.K.v;
#define SETROW(row, rhsv, diagv)                            \
  {                                                         \
    const double dg_ = (diagv);                             \
    const double d_ = dg_ > 1e-300 ? dg_ : 1.0;             \
    const double r_ = (rhsv);                               \
    c.K.r[IX(row)] = r_;                                    \
    c.K.d[IX(row)] = d_;                                    \
    c.K.z[IX(row)] = r_ / d_;                               \
    c.K.x[IX(row)] = 0.0;                                   \
  }
  if (it < nd) {
    const int row = c.D.od + it;
    const double jv = row_dist(c, it, v, env);
    const double dyn = c.T.d_dyn[it];
    SETROW(row, -(g * c.K.res[IX(row)] / h + jv + dyn * c.S.lam[IX(row)]),
           npmax(c.K.bdiag[IX(row)] + dyn, 1e-30));
  } else if (it < nd + nt) {
    const int t = it - nd;
    TetC T;
    double Ri[9], jv[6], lm[6], el[6], rs[6], z6[6];
    tet_load(c, t, env, T);
    tet_rinv(c, t, Ri);
    tet_j<EXACT>(c, t, env, T, Ri, v, jv);
    tet_res(T, rs);
#pragma unroll
    for (int i = 0; i < 6; ++i) lm[i] = c.S.lam[IX(c.D.ot + i * nt + t)];
    ereg6(c.T.t_e3[t], c.T.t_e3[nt + t], c.T.t_e3[2 * nt + t], lm, el);
#pragma unroll
    for (int i = 0; i < 6; ++i) {
      const int row = c.D.ot + i * nt + t;
      const double dg = npmax(c.K.bdiag[IX(row)] + 0.0, 1e-30);
      const double d = dg > 1e-300 ? dg : 1.0;
      const double r = -(g * rs[i] / h + jv[i] + el[i]);
      z6[i] = r / d;
      c.K.r[IX(row)] = r;
      c.K.d[IX(row)] = d;
      c.K.z[IX(row)] = z6[i];
      c.K.x[IX(row)] = 0.0;
    }
    tet_jt<EXACT>(c, t, env, T, Ri, z6);
  } else if (it < nd + nt + na) {
    const int a = it - nd - nt;
    double jv[3];
    rows_att(c, a, v, env, jv);
    const double dyn = c.T.a_dyn[a];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      const int row = c.D.oa + i * na + a;
      SETROW(row, -(g * c.K.res[IX(row)] / h + jv[i] + dyn * c.S.lam[IX(row)]),
             npmax(c.K.bdiag[IX(row)] + dyn, 1e-30));
    }
  } else if (it < nd + nt + na + nh) {
    const int hh = it - nd - nt - na;
    double jv[5];
    rows_hinge(c, hh, v, env, jv);
    const double dyn = c.T.h_dyn[hh];
#pragma unroll
    for (int i = 0; i < 5; ++i) {
      const int row = c.D.oh + i * nh + hh;
      SETROW(row, -(g * c.K.res[IX(row)] / h + jv[i] + dyn * c.S.lam[IX(row)]),
             npmax(c.K.bdiag[IX(row)] + dyn, 1e-30));
    }
  } else {
    const int s = it - nd - nt - na - nh;
    if (!c.K.present[IX(s)]) {
      c.K.actf[IX(s)] = 0.0;
      return;
    }
    const int rn = c.D.on + s, rf0 = c.D.of + s, rf1 = c.D.of + ns + s;
    double jv[3];
    rows_slot(c, s, v, env, jv);
    const double ln = c.K.lamc[IX(s)];
    const double a = c.K.gap[IX(s)] / h + jv[0];
    const double b = ln;
    const double root = sqrt(a * a + b * b + c.p.fb_delta);
    const double phi = a + b - root;
    double da = 1.0 - a / root;
    const double db = 1.0 - b / root;
    if (da < c.p.smin) da = c.p.smin;
    else if (da > c.p.smax) da = c.p.smax;
    const double dynn = db / da;
    c.K.dynn[IX(s)] = dynn;
    SETROW(rn, -phi / da, npmax(c.K.bdiag[IX(rn)] + dynn, 1e-30));
    const double on = (c.p.mu * npmax(ln, 0.0) > 0.0) ? 1.0 : 0.0;
    c.K.actf[IX(s)] = on;
    const double fd = c.p.fdyn;
    const double lf0 = c.K.lamc[IX(ns + s)], lf1 = c.K.lamc[IX(2 * ns + s)];
    SETROW(rf0, -on * (jv[1] + fd * lf0),
           on > 0.0 ? npmax(c.K.bdiag[IX(rf0)] + fd, 1e-30) : 1.0);
    SETROW(rf1, -on * (jv[2] + fd * lf1),
           on > 0.0 ? npmax(c.K.bdiag[IX(rf1)] + fd, 1e-30) : 1.0);
  }
#undef SETROW
}

// Newton head: jv = J v, velocity-level rhs, FB rows, friction active set,
// Jacobi diagonal; PCR setup r = rhs, z = r/d, x = 0, and the tet column
// sums of J^T z for the first apply (solver.py:439-478, 36-48, 62-70;
// contact.py:151-155). Also resets the per-env PCR scalars.
template <bool EXACT>
// 2 CTAs/SM (<= 128 registers): 164 -> 128 registers, 32 B spill, 9.5 -> 6.0 ms/frame
#ifndef SS_RHS_MINB
#define SS_RHS_MINB 2
#endif
#define SS_RHS_MINB_LB __launch_bounds__(SS_THREADS, SS_RHS_MINB)
__global__ void SS_RHS_MINB_LB k_newton_rhs(const Ctx c) {
  SETUP
  const int nd = c.D.nd, nt = c.D.nt, na = c.D.na, nh = c.D.nh, ns = c.D.ns;
  const double g = c.p.gamma, h = c.p.h;
  const double* v = c.K.v;
  (void)g; (void)h; (void)v; (void)nd; (void)nt; (void)na; (void)nh; (void)ns;
  FOR_ITEMS(it, nd + nt + na + nh + ns) {
    if (it == 0) {
      c.K.broken[env] = 0;
      c.K.beta[env] = 0.0;
      c.K.last_step[env] = -1;
    }
    rhs_item<EXACT>(c, it, env);
  }
}

// az = A z rows (apply_a second half, solver.py:388-399) + rho partial z.az.
// setup != 0: rho = z.az (pcr_solve setup, solver.py:70-73); else
// beta = rho_new / rho (solver.py:87-89). Absent contact slots are skipped.
template <bool EXACT>
#ifndef SS_APPLY_MINB
#define SS_APPLY_MINB 2
#endif
__global__ void __launch_bounds__(SS_THREADS, SS_APPLY_MINB) k_apply_rows(const Ctx c, int setup) {
  SETUP
  const int nd = c.D.nd, nt = c.D.nt, na = c.D.na, nh = c.D.nh, ns = c.D.ns;
  const double* u = c.K.u;
  const double* z = c.K.z;
  double part = 0.0;
  // structured mode: the next tet item's node ids are fetched one item ahead,
  // so its gathered u loads issue with the quaternion / S / z loads instead of
  // after a dependent index load
  int pf_t = -1, pf_n0 = 0, pf_n1 = 0, pf_n2 = 0, pf_n3 = 0;
  FOR_ITEMS(it, nd + nt + na + nh + ns) {
    if (it < nd) {
      const int row = c.D.od + it;
      const double zr = z[IX(row)];
      const double az = row_dist(c, it, u, env) + c.T.d_dyn[it] * zr;
      c.K.az[IX(row)] = az;
      part += zr * az;
    } else if (it < nd + nt) {
      const int t = it - nd;
      TetC T;
      double Ri[9], y[6], zz[6], ez[6];
      if (EXACT) {
        tet_load(c, t, env, T);
        tet_rinv(c, t, Ri);
        tet_j<EXACT>(c, t, env, T, Ri, u, y);
#pragma unroll
        for (int i = 0; i < 6; ++i) zz[i] = z[IX(c.D.ot + i * nt + t)];
      } else {
        // every load of the tet issued before any arithmetic (one memory
        // round trip per item instead of three); 32-bit element offsets
        // stepped by the row stride nt*E (fewer integer instructions per
        // address than the 64-bit IX products)
        double q[4], sv[6], uv[12];
        int nid[4];
        if (pf_t == t) {
          nid[0] = pf_n0; nid[1] = pf_n1; nid[2] = pf_n2; nid[3] = pf_n3;
        } else {
#pragma unroll
          for (int v = 0; v < 4; ++v) nid[v] = c.T.t_idx[v * nt + t];
        }
        const unsigned uE = (unsigned)E;
        const unsigned ntE = (unsigned)nt * uE;
        const unsigned tb = (unsigned)t * uE + (unsigned)env;
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const double* up = u + ((unsigned)(3 * nid[v]) * uE + (unsigned)env);
#pragma unroll
          for (int a = 0; a < 3; ++a) uv[3 * v + a] = up[a * uE];
        }
        {
          const double* qp = c.S.quat + tb;
#pragma unroll
          for (int k = 0; k < 4; ++k) q[k] = qp[k * ntE];
          const double* sp = c.K.tS + tb;
#pragma unroll
          for (int k = 0; k < 6; ++k) sv[k] = sp[k * ntE];
          const double* zp = z + ((unsigned)c.D.ot * uE + tb);
#pragma unroll
          for (int i = 0; i < 6; ++i) zz[i] = zp[i * ntE];
        }
        tet_rinv(c, t, Ri);
        const int tn = t + gridDim.y * IL;
        if (tn < nt) {
          pf_t = tn;
          pf_n0 = c.T.t_idx[tn];
          pf_n1 = c.T.t_idx[nt + tn];
          pf_n2 = c.T.t_idx[2 * nt + tn];
          pf_n3 = c.T.t_idx[3 * nt + tn];
        }
        tet_unpack(q, sv, T);
        tet_forward_uv(T, Ri, uv, y);
      }
      ereg6(c.T.t_e3[t], c.T.t_e3[nt + t], c.T.t_e3[2 * nt + t], zz, ez);
      {
        const unsigned uE = (unsigned)E;
        const unsigned ntE = (unsigned)nt * uE;
        double* ap = c.K.az + ((unsigned)c.D.ot * uE + (unsigned)t * uE + (unsigned)env);
#pragma unroll
        for (int i = 0; i < 6; ++i) {
          const double az = y[i] + ez[i];
          ap[i * ntE] = az;
          part += zz[i] * az;
        }
      }
    } else if (it < nd + nt + na) {
      const int a = it - nd - nt;
      double y[3];
      rows_att(c, a, u, env, y);
      const double dyn = c.T.a_dyn[a];
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        const int row = c.D.oa + i * na + a;
        const double zr = z[IX(row)];
        const double az = y[i] + dyn * zr;
        c.K.az[IX(row)] = az;
        part += zr * az;
      }
    } else if (it < nd + nt + na + nh) {
      const int hh = it - nd - nt - na;
      double y[5];
      rows_hinge(c, hh, u, env, y);
      const double dyn = c.T.h_dyn[hh];
#pragma unroll
      for (int i = 0; i < 5; ++i) {
        const int row = c.D.oh + i * nh + hh;
        const double zr = z[IX(row)];
        const double az = y[i] + dyn * zr;
        c.K.az[IX(row)] = az;
        part += zr * az;
      }
    } else {
      const int s = it - nd - nt - na - nh;
      if (!c.K.present[IX(s)]) continue;
      const int rn = c.D.on + s, rf0 = c.D.of + s, rf1 = c.D.of + ns + s;
      const double zn = z[IX(rn)], z0 = z[IX(rf0)], z1 = z[IX(rf1)];
      double y[3];
      rows_slot(c, s, u, env, y);
      const double an = y[0] + c.K.dynn[IX(s)] * zn;
      double a0 = z0, a1 = z1;
      if (c.K.actf[IX(s)] != 0.0) {
        a0 = y[1] + c.p.fdyn * z0;
        a1 = y[2] + c.p.fdyn * z1;
      }
      c.K.az[IX(rn)] = an;
      c.K.az[IX(rf0)] = a0;
      c.K.az[IX(rf1)] = a1;
      part += zn * an;
      part += z0 * a0;
      part += z1 * a1;
    }
  }
  double tot;
  if (reduce_env(c, part, &tot)) {
    if (setup) {
      c.K.rho[env] = tot;
    } else if (!c.K.broken[env]) {
      const double rho = c.K.rho[env];
      c.K.beta[env] = rho > 1e-300 ? tot / rho : 0.0;
      c.K.rho[env] = tot;
    }
  }
}

// k_apply_rows (structured mode) with the tet operands staged through shared
// memory by cp.async: the quaternion, S and z of a thread's NEXT tet item
// (16 doubles) are copied asynchronously into the other half of a per-thread
// double buffer while the current item computes, so the loads of two items
// are in flight per thread without holding them in registers (the kernel is
// bound by memory-level parallelism at 16 warps/SM). The first tet item's
// copy is issued at kernel start and overlaps the distance rows. Same
// arithmetic in the same order per thread: bitwise k_apply_rows<false>.
DI void cp_async8(double* smem_dst, const double* gsrc) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gsrc) : "memory");
}
DI void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
DI void cp_async_wait1() { asm volatile("cp.async.wait_group 1;\n" ::: "memory"); }
DI void cp_async_wait0() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

#ifndef SS_APPLYA_MINB
#define SS_APPLYA_MINB 2
#endif
#ifndef SS_APPLYA_STAGES
#define SS_APPLYA_STAGES 2
#endif
template <int N>
DI void cp_async_wait_n() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }
__global__ void __launch_bounds__(SS_THREADS, SS_APPLYA_MINB) k_apply_rows_async(const Ctx c,
                                                                                 int setup) {
  SETUP
  extern __shared__ double abuf[];  // [SS_APPLYA_STAGES][16][SS_THREADS]
  constexpr int NST = SS_APPLYA_STAGES;
  const int nd = c.D.nd, nt = c.D.nt, na = c.D.na, nh = c.D.nh, ns = c.D.ns;
  const double* u = c.K.u;
  const double* z = c.K.z;
  const int stride = gridDim.y * IL;
  auto stage_tet = [&](int t, int st) {
    double* b = abuf + (size_t)st * 16 * SS_THREADS + threadIdx.x;
#pragma unroll
    for (int k = 0; k < 4; ++k) cp_async8(b + k * SS_THREADS, c.S.quat + IX(k * nt + t));
#pragma unroll
    for (int k = 0; k < 6; ++k) cp_async8(b + (4 + k) * SS_THREADS, c.K.tS + IX(k * nt + t));
#pragma unroll
    for (int i = 0; i < 6; ++i) cp_async8(b + (10 + i) * SS_THREADS, z + IX(c.D.ot + i * nt + t));
  };
  // the first NST-1 tet items of this thread, staged now (overlap the distance rows)
  int stg = 0;
  int it_pf;  // the next tet item to stage
  {
    int it0 = blockIdx.y * IL + il;
    if (it0 < nd) it0 += ((nd - it0 + stride - 1) / stride) * stride;
    it_pf = it0;
    for (int q = 0; q < NST - 1; ++q) {
      if (it_pf < nd + nt) stage_tet(it_pf - nd, q);
      cp_async_commit();
      it_pf += stride;
    }
  }
  double part = 0.0;
  int pf_t = -1, pf_n0 = 0, pf_n1 = 0, pf_n2 = 0, pf_n3 = 0;
  FOR_ITEMS(it, nd + nt + na + nh + ns) {
    if (it < nd) {
      const int row = c.D.od + it;
      const double zr = z[IX(row)];
      const double az = row_dist(c, it, u, env) + c.T.d_dyn[it] * zr;
      c.K.az[IX(row)] = az;
      part += zr * az;
    } else if (it < nd + nt) {
      const int t = it - nd;
      double Ri[9], y[6], zz[6], ez[6], uv[12];
      int nid[4];
      if (pf_t == t) {
        nid[0] = pf_n0; nid[1] = pf_n1; nid[2] = pf_n2; nid[3] = pf_n3;
      } else {
#pragma unroll
        for (int v = 0; v < 4; ++v) nid[v] = c.T.t_idx[v * nt + t];
      }
#pragma unroll
      for (int v = 0; v < 4; ++v)
#pragma unroll
        for (int a = 0; a < 3; ++a) uv[3 * v + a] = u[IX(3 * nid[v] + a)];
      tet_rinv(c, t, Ri);
      const int tn = t + stride;
      if (tn < nt) {
        pf_t = tn;
        pf_n0 = c.T.t_idx[tn];
        pf_n1 = c.T.t_idx[nt + tn];
        pf_n2 = c.T.t_idx[2 * nt + tn];
        pf_n3 = c.T.t_idx[3 * nt + tn];
      }
      {
        int sn = stg + NST - 1;
        if (sn >= NST) sn -= NST;
        if (it_pf < nd + nt) stage_tet(it_pf - nd, sn);
        cp_async_commit();
        it_pf += stride;
      }
      cp_async_wait_n<NST - 1>();  // this item's stage has landed
      const double* b = abuf + (size_t)stg * 16 * SS_THREADS + threadIdx.x;
      double q[4], sv[6];
#pragma unroll
      for (int k = 0; k < 4; ++k) q[k] = b[k * SS_THREADS];
#pragma unroll
      for (int k = 0; k < 6; ++k) sv[k] = b[(4 + k) * SS_THREADS];
#pragma unroll
      for (int i = 0; i < 6; ++i) zz[i] = b[(10 + i) * SS_THREADS];
      stg = stg + 1 == NST ? 0 : stg + 1;
      TetC T;
      tet_unpack(q, sv, T);
      tet_forward_uv(T, Ri, uv, y);
      ereg6(c.T.t_e3[t], c.T.t_e3[nt + t], c.T.t_e3[2 * nt + t], zz, ez);
#pragma unroll
      for (int i = 0; i < 6; ++i) {
        const double az = y[i] + ez[i];
        c.K.az[IX(c.D.ot + i * nt + t)] = az;
        part += zz[i] * az;
      }
    } else if (it < nd + nt + na) {
      const int a = it - nd - nt;
      double y[3];
      rows_att(c, a, u, env, y);
      const double dyn = c.T.a_dyn[a];
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        const int row = c.D.oa + i * na + a;
        const double zr = z[IX(row)];
        const double az = y[i] + dyn * zr;
        c.K.az[IX(row)] = az;
        part += zr * az;
      }
    } else if (it < nd + nt + na + nh) {
      const int hh = it - nd - nt - na;
      double y[5];
      rows_hinge(c, hh, u, env, y);
      const double dyn = c.T.h_dyn[hh];
#pragma unroll
      for (int i = 0; i < 5; ++i) {
        const int row = c.D.oh + i * nh + hh;
        const double zr = z[IX(row)];
        const double az = y[i] + dyn * zr;
        c.K.az[IX(row)] = az;
        part += zr * az;
      }
    } else {
      const int s = it - nd - nt - na - nh;
      if (!c.K.present[IX(s)]) continue;
      const int rn = c.D.on + s, rf0 = c.D.of + s, rf1 = c.D.of + ns + s;
      const double zn = z[IX(rn)], z0 = z[IX(rf0)], z1 = z[IX(rf1)];
      double y[3];
      rows_slot(c, s, u, env, y);
      const double an = y[0] + c.K.dynn[IX(s)] * zn;
      double a0 = z0, a1 = z1;
      if (c.K.actf[IX(s)] != 0.0) {
        a0 = y[1] + c.p.fdyn * z0;
        a1 = y[2] + c.p.fdyn * z1;
      }
      c.K.az[IX(rn)] = an;
      c.K.az[IX(rf0)] = a0;
      c.K.az[IX(rf1)] = a1;
      part += zn * an;
      part += z0 * a0;
      part += z1 * a1;
    }
  }
  cp_async_wait0();
  double tot;
  if (reduce_env(c, part, &tot)) {
    if (setup) {
      c.K.rho[env] = tot;
    } else if (!c.K.broken[env]) {
      const double rho = c.K.rho[env];
      c.K.beta[env] = rho > 1e-300 ? tot / rho : 0.0;
      c.K.rho[env] = tot;
    }
  }
}

// Tet mapping of the two-warp kernels: a pair of warps takes one tet for 32
// env lanes (W == 32) or 32 consecutive tets of the single env (W == 1).
// Every thread of a pair runs the same trip count (tw_act masks the tail), so
// the pair's named barriers always see both warps.
#define TW_SETUP                                                              \
  const int tw_slot = threadIdx.x & 31;                                       \
  const int pair = (threadIdx.x >> 5) >> 1, role = (threadIdx.x >> 5) & 1;     \
  const int tw_mul = c.D.W == 1 ? 32 : 1;                                     \
  const int tw_base = (blockIdx.y * 4 + pair) * tw_mul;                        \
  const int tw_off = c.D.W == 1 ? tw_slot : 0;                                \
  const int tw_stride = gridDim.y * 4 * tw_mul;

// k_apply_rows (structured mode, E >= 32) with each tet split over TWO warps
// of the same 32 envs: warp A (even item lane) loads the 4 nodes' u, the
// rest-shape inverse and the quaternion and forms G = R^T sum_v u_v w_v^T;
// warp B (odd item lane) loads S, z and E_tet, forms K^-1, takes G through
// shared memory (one named barrier per warp pair and item, G double
// buffered) and finishes w = K^-1 ax(G), J u = voigt(sym(G) - sym(skew(w) S)),
// az and the rho partial. The same operations as tet_forward_uv (every az
// bitwise equal); half the live registers per thread, so three CTAs per SM
// (24 warps) instead of two keep more loads in flight. The rho partials are
// summed over a different thread assignment (rounding-level differences).
#ifndef SS_APPLY2_MINB
#define SS_APPLY2_MINB 3
#endif
DI void named_bar(int id, int count) { asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(count) : "memory"); }

__global__ void __launch_bounds__(SS_THREADS, SS_APPLY2_MINB) k_apply_rows2(const Ctx c, int setup) {
  SETUP
  __shared__ double gsh[4][2][9][32];  // [pair][buffer][G entry][env lane]
  const int nd = c.D.nd, nt = c.D.nt, na = c.D.na, nh = c.D.nh, ns = c.D.ns;
  const double* u = c.K.u;
  const double* z = c.K.z;
  TW_SETUP
  const unsigned uE = (unsigned)E;
  const unsigned ntE = (unsigned)nt * uE;
  double part = 0.0;
  int buf = 0;
  const int tstride = tw_stride;
#ifndef SS_APPLY2_NO_NIDPF
  // warp A: the next item's node ids one item ahead
  int nid_n[4] = {0, 0, 0, 0};
  {
    const int t0 = tw_base + tw_off;
    if (role == 0 && t0 < nt) {
#pragma unroll
      for (int v = 0; v < 4; ++v) nid_n[v] = c.T.t_idx[v * nt + t0];
    }
  }
#endif
  // ---- tets: item lanes paired
  for (int tw_t = tw_base; tw_t < nt; tw_t += tw_stride) {
    const int t = tw_t + tw_off;
    const bool tw_act = t < nt;
    const int tc = tw_act ? t : nt - 1;  // tail lanes load a valid tet, store nothing
    const unsigned tb = (unsigned)tc * uE + (unsigned)env;
    double* g = &gsh[pair][buf][0][tw_slot];
    if (role == 0) {
      double uv[12], q[4], Ri[9];
      int nid[4];
#ifndef SS_APPLY2_NO_NIDPF
#pragma unroll
      for (int v = 0; v < 4; ++v) nid[v] = nid_n[v];
      if (t + tstride < nt) {
#pragma unroll
        for (int v = 0; v < 4; ++v) nid_n[v] = c.T.t_idx[v * nt + t + tstride];
      }
#else
#pragma unroll
      for (int v = 0; v < 4; ++v) nid[v] = c.T.t_idx[v * nt + tc];
#endif
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const double* up = u + ((unsigned)(3 * nid[v]) * uE + (unsigned)env);
#pragma unroll
        for (int a = 0; a < 3; ++a) uv[3 * v + a] = up[a * uE];
      }
      const double* qp = c.S.quat + tb;
#pragma unroll
      for (int k = 0; k < 4; ++k) q[k] = ld_stream(qp + k * ntE);
      tet_rinv(c, tc, Ri);
      // tet_forward_uv, first half: du, L, G
      double du[9];
#pragma unroll
      for (int v = 1; v < 4; ++v)
#pragma unroll
        for (int a = 0; a < 3; ++a) du[3 * (v - 1) + a] = uv[3 * v + a] - uv[a];
      double L[9];
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int j = 0; j < 3; ++j)
          L[3 * a + j] = dot3(du[a], Ri[j], du[3 + a], Ri[3 + j], du[6 + a], Ri[6 + j]);
      double R[9];
      quat_to_mat(q[0], q[1], q[2], q[3], R);
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j)
          g[(3 * i + j) * 32] = dot3(R[i], L[j], R[3 + i], L[3 + j], R[6 + i], L[6 + j]);
      named_bar(1 + pair, 64);
    } else {
      double sv[6], zz[6];
      const double* sp = c.K.tS + tb;
#pragma unroll
      for (int k = 0; k < 6; ++k) sv[k] = ld_stream(sp + k * ntE);
      const double* zp = z + ((unsigned)c.D.ot * uE + tb);
#pragma unroll
      for (int i = 0; i < 6; ++i) zz[i] = ld_stream(zp + i * ntE);
      const double ed = c.T.t_e3[tc], eo = c.T.t_e3[nt + tc], es = c.T.t_e3[2 * nt + tc];
      double S[9], Ki[9];
      S[0] = sv[0]; S[4] = sv[1]; S[8] = sv[2];
      S[5] = sv[3]; S[7] = sv[3];
      S[2] = sv[4]; S[6] = sv[4];
      S[1] = sv[5]; S[3] = sv[5];
      tet_kinv(S, Ki);
      named_bar(1 + pair, 64);
      double G[9];
#pragma unroll
      for (int k = 0; k < 9; ++k) G[k] = g[k * 32];
      // tet_forward_uv, second half
      const double g0 = G[7] - G[5], g1 = G[2] - G[6], g2 = G[3] - G[1];
      const double w0 = dot3(Ki[0], g0, Ki[1], g1, Ki[2], g2);
      const double w1 = dot3(Ki[3], g0, Ki[4], g1, Ki[5], g2);
      const double w2 = dot3(Ki[6], g0, Ki[7], g1, Ki[8], g2);
      const double ws00 = __fma_rn(w1, S[6], -w2 * S[3]);
      const double ws01 = __fma_rn(w1, S[7], -w2 * S[4]);
      const double ws02 = __fma_rn(w1, S[8], -w2 * S[5]);
      const double ws10 = __fma_rn(w2, S[0], -w0 * S[6]);
      const double ws11 = __fma_rn(w2, S[1], -w0 * S[7]);
      const double ws12 = __fma_rn(w2, S[2], -w0 * S[8]);
      const double ws20 = __fma_rn(w0, S[3], -w1 * S[0]);
      const double ws21 = __fma_rn(w0, S[4], -w1 * S[1]);
      const double ws22 = __fma_rn(w0, S[5], -w1 * S[2]);
      double y[6], ez[6];
      y[0] = G[0] - ws00;
      y[1] = G[4] - ws11;
      y[2] = G[8] - ws22;
      y[3] = 0.5 * ((G[5] + G[7]) - (ws12 + ws21));
      y[4] = 0.5 * ((G[2] + G[6]) - (ws02 + ws20));
      y[5] = 0.5 * ((G[1] + G[3]) - (ws01 + ws10));
      ereg6(ed, eo, es, zz, ez);
      double* ap = c.K.az + ((unsigned)c.D.ot * uE + tb);
      if (tw_act) {
#pragma unroll
        for (int i = 0; i < 6; ++i) {
          const double az = y[i] + ez[i];
          ap[i * ntE] = az;
          part += zz[i] * az;
        }
      }
    }
    buf ^= 1;
  }
  // ---- every other item (distance, attachment, hinge, contact slot rows)
  const int n_other = nd + na + nh + ns;
  for (int q2 = blockIdx.y * IL + il; q2 < n_other; q2 += gridDim.y * IL) {
    int it = q2 < nd ? q2 : q2 + nt;
    if (it < nd) {
      const int row = c.D.od + it;
      const double zr = z[IX(row)];
      const double az = row_dist(c, it, u, env) + c.T.d_dyn[it] * zr;
      c.K.az[IX(row)] = az;
      part += zr * az;
    } else if (it < nd + nt + na) {
      const int a = it - nd - nt;
      double y[3];
      rows_att(c, a, u, env, y);
      const double dyn = c.T.a_dyn[a];
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        const int row = c.D.oa + i * na + a;
        const double zr = z[IX(row)];
        const double az = y[i] + dyn * zr;
        c.K.az[IX(row)] = az;
        part += zr * az;
      }
    } else if (it < nd + nt + na + nh) {
      const int hh = it - nd - nt - na;
      double y[5];
      rows_hinge(c, hh, u, env, y);
      const double dyn = c.T.h_dyn[hh];
#pragma unroll
      for (int i = 0; i < 5; ++i) {
        const int row = c.D.oh + i * nh + hh;
        const double zr = z[IX(row)];
        const double az = y[i] + dyn * zr;
        c.K.az[IX(row)] = az;
        part += zr * az;
      }
    } else {
      const int s = it - nd - nt - na - nh;
      if (!c.K.present[IX(s)]) continue;
      const int rn = c.D.on + s, rf0 = c.D.of + s, rf1 = c.D.of + ns + s;
      const double zn = z[IX(rn)], z0 = z[IX(rf0)], z1 = z[IX(rf1)];
      double y[3];
      rows_slot(c, s, u, env, y);
      const double an = y[0] + c.K.dynn[IX(s)] * zn;
      double a0 = z0, a1 = z1;
      if (c.K.actf[IX(s)] != 0.0) {
        a0 = y[1] + c.p.fdyn * z0;
        a1 = y[2] + c.p.fdyn * z1;
      }
      c.K.az[IX(rn)] = an;
      c.K.az[IX(rf0)] = a0;
      c.K.az[IX(rf1)] = a1;
      part += zn * an;
      part += z0 * a0;
      part += z1 * a1;
    }
  }
  double tot;
  if (reduce_env(c, part, &tot)) {
    if (setup) {
      c.K.rho[env] = tot;
    } else if (!c.K.broken[env]) {
      const double rho = c.K.rho[env];
      c.K.beta[env] = rho > 1e-300 ? tot / rho : 0.0;
      c.K.rho[env] = tot;
    }
  }
}

// k_apply_rows2 with the streaming tet operands moved by the Tensor Memory
// Accelerator. A CTA's four warp pairs take four consecutive tets of the
// same 32 env lanes per iteration, so the quaternion rows [4][nt][E], the
// compact J [6][nt][E] and the tet rows of z [6][nt][E] of one iteration are
// three 3-D boxes {32 envs, 4 tets, 4/6 rows} (16 KB): thread 0 issues them
// with cp.async.bulk.tensor (one CUtensorMap per field and wave, created at
// ss_create) SS_APPLY3_NST iterations ahead into a shared-memory ring; a
// stage's arrival completes its `full` mbarrier (transaction bytes), and
// every warp arrives on its `empty` mbarrier once its operands are in
// registers, which lets thread 0 refill it. The warps no longer wait a
// global round trip for q, S, z; only the gathered u (L1/L2) stays on the
// load path. Arithmetic, order and stores are k_apply_rows2's (az bitwise,
// rho bitwise the two-warp kernel's: same thread assignment).
#ifndef SS_APPLY3_NST
#define SS_APPLY3_NST 2
#endif
#ifndef SS_APPLY3_MINB
#define SS_APPLY3_MINB 3
#endif
struct TmApply {
  CUtensorMap q, s, z;
};
constexpr int kA3Box = 16 * 4 * 32;  // doubles per stage: q(4) S(6) z(6) rows x 4 tets x 32 lanes
constexpr size_t kA3Smem = (size_t)SS_APPLY3_NST * kA3Box * 8;
DI void tma_load_3d(void* dst, const CUtensorMap* map, int x, int y, int z, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_addr(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_addr(bar))
      : "memory");
}
DI void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(b)) : "memory");
}
DI void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(b)),
               "r"(bytes)
               : "memory");
}

__global__ void __launch_bounds__(SS_THREADS, SS_APPLY3_MINB) k_apply_rows3(
    const Ctx c, int setup, const __grid_constant__ TmApply tm) {
  SETUP
  __shared__ double gsh[4][2][9][32];  // [pair][buffer][G entry][env lane]
  __shared__ uint64_t full[SS_APPLY3_NST], empty[SS_APPLY3_NST];
  extern __shared__ __align__(128) double a3[];
  const int nd = c.D.nd, nt = c.D.nt, na = c.D.na, nh = c.D.nh, ns = c.D.ns;
  const double* u = c.K.u;
  const double* z = c.K.z;
  TW_SETUP
  const unsigned uE = (unsigned)E;
  double part = 0.0;
  int buf = 0;
  const int tstride = tw_stride;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int s = 0; s < SS_APPLY3_NST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], SS_THREADS / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // CTA-uniform trip count (every warp arrives on every stage's empty barrier)
  const int t_cta = blockIdx.y * 4;
  const int niter = nt > t_cta ? (nt - t_cta + tstride - 1) / tstride : 0;
  const int env0 = blockIdx.x * 32;
  auto issue = [&](int j) {
    const int s = j % SS_APPLY3_NST;
    double* st = a3 + (size_t)s * kA3Box;
    const int t0 = t_cta + j * tstride;
    mbar_expect_tx(&full[s], kA3Box * 8);
    tma_load_3d(st, &tm.q, env0, t0, 0, &full[s]);
    tma_load_3d(st + 512, &tm.s, env0, t0, 0, &full[s]);
    tma_load_3d(st + 1280, &tm.z, env0, t0, 0, &full[s]);
  };
  if (threadIdx.x == 0) {
    for (int j = 0; j < SS_APPLY3_NST && j < niter; ++j) issue(j);
  }
  // warp A: the next item's node ids one item ahead
  int nid_n[4] = {0, 0, 0, 0};
  {
    const int t0 = tw_base + tw_off;
    if (role == 0 && t0 < nt) {
#pragma unroll
      for (int v = 0; v < 4; ++v) nid_n[v] = c.T.t_idx[v * nt + t0];
    }
  }
  for (int j = 0; j < niter; ++j) {
    if (threadIdx.x == 0 && j >= 1 && j - 1 + SS_APPLY3_NST < niter) {
      // refill the stage every warp released in iteration j - 1
      const int sp = (j - 1) % SS_APPLY3_NST;
      while (!mbar_try_wait(&empty[sp], (uint32_t)(((j - 1) / SS_APPLY3_NST) & 1))) {
      }
      issue(j - 1 + SS_APPLY3_NST);
    }
    const int t = t_cta + pair + j * tstride;
    const bool tw_act = t < nt;
    const int tc = tw_act ? t : nt - 1;
    const int s = j % SS_APPLY3_NST;
    const double* st = a3 + (size_t)s * kA3Box;
    while (!mbar_try_wait(&full[s], (uint32_t)((j / SS_APPLY3_NST) & 1))) {
    }
    double* g = &gsh[pair][buf][0][tw_slot];
    if (role == 0) {
      double uv[12], q[4], Ri[9];
      int nid[4];
#pragma unroll
      for (int v = 0; v < 4; ++v) nid[v] = nid_n[v];
      if (t + tstride < nt) {
#pragma unroll
        for (int v = 0; v < 4; ++v) nid_n[v] = c.T.t_idx[v * nt + t + tstride];
      }
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const double* up = u + ((unsigned)(3 * nid[v]) * uE + (unsigned)env);
#pragma unroll
        for (int a = 0; a < 3; ++a) uv[3 * v + a] = up[a * uE];
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) q[k] = st[(k * 4 + pair) * 32 + tw_slot];
      __syncwarp();
      if (tw_slot == 0) mbar_arrive(&empty[s]);
      tet_rinv(c, tc, Ri);
      double du[9];
#pragma unroll
      for (int v = 1; v < 4; ++v)
#pragma unroll
        for (int a = 0; a < 3; ++a) du[3 * (v - 1) + a] = uv[3 * v + a] - uv[a];
      double L[9];
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int jj = 0; jj < 3; ++jj)
          L[3 * a + jj] = dot3(du[a], Ri[jj], du[3 + a], Ri[3 + jj], du[6 + a], Ri[6 + jj]);
      double R[9];
      quat_to_mat(q[0], q[1], q[2], q[3], R);
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int jj = 0; jj < 3; ++jj)
          g[(3 * i + jj) * 32] = dot3(R[i], L[jj], R[3 + i], L[3 + jj], R[6 + i], L[6 + jj]);
      named_bar(1 + pair, 64);
    } else {
      double sv[6], zz[6];
#pragma unroll
      for (int k = 0; k < 6; ++k) sv[k] = st[512 + (k * 4 + pair) * 32 + tw_slot];
#pragma unroll
      for (int i = 0; i < 6; ++i) zz[i] = st[1280 + (i * 4 + pair) * 32 + tw_slot];
      __syncwarp();
      if (tw_slot == 0) mbar_arrive(&empty[s]);
      const double ed = c.T.t_e3[tc], eo = c.T.t_e3[nt + tc], es = c.T.t_e3[2 * nt + tc];
      double S[9], Ki[9];
      S[0] = sv[0]; S[4] = sv[1]; S[8] = sv[2];
      S[5] = sv[3]; S[7] = sv[3];
      S[2] = sv[4]; S[6] = sv[4];
      S[1] = sv[5]; S[3] = sv[5];
      tet_kinv(S, Ki);
      named_bar(1 + pair, 64);
      double G[9];
#pragma unroll
      for (int k = 0; k < 9; ++k) G[k] = g[k * 32];
      const double g0 = G[7] - G[5], g1 = G[2] - G[6], g2 = G[3] - G[1];
      const double w0 = dot3(Ki[0], g0, Ki[1], g1, Ki[2], g2);
      const double w1 = dot3(Ki[3], g0, Ki[4], g1, Ki[5], g2);
      const double w2 = dot3(Ki[6], g0, Ki[7], g1, Ki[8], g2);
      const double ws00 = __fma_rn(w1, S[6], -w2 * S[3]);
      const double ws01 = __fma_rn(w1, S[7], -w2 * S[4]);
      const double ws02 = __fma_rn(w1, S[8], -w2 * S[5]);
      const double ws10 = __fma_rn(w2, S[0], -w0 * S[6]);
      const double ws11 = __fma_rn(w2, S[1], -w0 * S[7]);
      const double ws12 = __fma_rn(w2, S[2], -w0 * S[8]);
      const double ws20 = __fma_rn(w0, S[3], -w1 * S[0]);
      const double ws21 = __fma_rn(w0, S[4], -w1 * S[1]);
      const double ws22 = __fma_rn(w0, S[5], -w1 * S[2]);
      double y[6], ez[6];
      y[0] = G[0] - ws00;
      y[1] = G[4] - ws11;
      y[2] = G[8] - ws22;
      y[3] = 0.5 * ((G[5] + G[7]) - (ws12 + ws21));
      y[4] = 0.5 * ((G[2] + G[6]) - (ws02 + ws20));
      y[5] = 0.5 * ((G[1] + G[3]) - (ws01 + ws10));
      ereg6(ed, eo, es, zz, ez);
      const unsigned tb = (unsigned)tc * uE + (unsigned)env;
      double* ap = c.K.az + ((unsigned)c.D.ot * uE + tb);
      const unsigned ntE = (unsigned)nt * uE;
      if (tw_act) {
#pragma unroll
        for (int i = 0; i < 6; ++i) {
          const double az = y[i] + ez[i];
          ap[i * ntE] = az;
          part += zz[i] * az;
        }
      }
    }
    buf ^= 1;
  }
  // ---- every other item (distance, attachment, hinge, contact slot rows)
  const int n_other = nd + na + nh + ns;
  for (int q2 = blockIdx.y * IL + il; q2 < n_other; q2 += gridDim.y * IL) {
    int it = q2 < nd ? q2 : q2 + nt;
    if (it < nd) {
      const int row = c.D.od + it;
      const double zr = z[IX(row)];
      const double az = row_dist(c, it, u, env) + c.T.d_dyn[it] * zr;
      c.K.az[IX(row)] = az;
      part += zr * az;
    } else if (it < nd + nt + na) {
      const int a = it - nd - nt;
      double y[3];
      rows_att(c, a, u, env, y);
      const double dyn = c.T.a_dyn[a];
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        const int row = c.D.oa + i * na + a;
        const double zr = z[IX(row)];
        const double az = y[i] + dyn * zr;
        c.K.az[IX(row)] = az;
        part += zr * az;
      }
    } else if (it < nd + nt + na + nh) {
      const int hh = it - nd - nt - na;
      double y[5];
      rows_hinge(c, hh, u, env, y);
      const double dyn = c.T.h_dyn[hh];
#pragma unroll
      for (int i = 0; i < 5; ++i) {
        const int row = c.D.oh + i * nh + hh;
        const double zr = z[IX(row)];
        const double az = y[i] + dyn * zr;
        c.K.az[IX(row)] = az;
        part += zr * az;
      }
    } else {
      const int s = it - nd - nt - na - nh;
      if (!c.K.present[IX(s)]) continue;
      const int rn = c.D.on + s, rf0 = c.D.of + s, rf1 = c.D.of + ns + s;
      const double zn = z[IX(rn)], z0 = z[IX(rf0)], z1 = z[IX(rf1)];
      double y[3];
      rows_slot(c, s, u, env, y);
      const double an = y[0] + c.K.dynn[IX(s)] * zn;
      double a0 = z0, a1 = z1;
      if (c.K.actf[IX(s)] != 0.0) {
        a0 = y[1] + c.p.fdyn * z0;
        a1 = y[2] + c.p.fdyn * z1;
      }
      c.K.az[IX(rn)] = an;
      c.K.az[IX(rf0)] = a0;
      c.K.az[IX(rf1)] = a1;
      part += zn * an;
      part += z0 * a0;
      part += z1 * a1;
    }
  }
  double tot;
  if (reduce_env(c, part, &tot)) {
    if (setup) {
      c.K.rho[env] = tot;
    } else if (!c.K.broken[env]) {
      const double rho = c.K.rho[env];
      c.K.beta[env] = rho > 1e-300 ? tot / rho : 0.0;
      c.K.rho[env] = tot;
    }
  }
}

// Row-wise iteration over the m rows of an env: static rows always, contact
// rows only when their slot is present (absent slots do not exist in the
// reference's compacted system). Returns false for an absent contact row.
DI bool row_live(const Ctx& c, int row, int env) {
  if (row < c.D.ms) return true;
  const int E = c.D.E;
  int s = row - c.D.ms;
  s = s < c.D.ns ? s : (s < 2 * c.D.ns ? s - c.D.ns : s - 2 * c.D.ns);
  return c.K.present[IX(s)] != 0;
}

// p = z + beta p, ap = az + beta ap (setup: copies), then den = ap.(ap/d)
// and alpha = rho/den with the breakdown guard (solver.py:71-81, 90-91).
// Element-owned rows, all loads of an element issued before its stores.
// Structured mode (!EXACT) stores apd = ap/d in the ap buffer instead of ap
// (ap_prev = apd_prev * d when needed): the step then needs neither ap nor d.
template <bool EXACT>
// structured mode pinned to 3 CTAs/SM (<= 85 registers; at 85 registers and 2
// CTAs/SM the kernel takes 33.5 instead of 28.9 ms/frame)
__global__ void __launch_bounds__(SS_THREADS, EXACT ? 2 : 3) k_pcr_dir(const Ctx c, int setup) {
  SETUP
  const bool brk = c.K.broken[env] != 0;
  const double beta = c.K.beta[env];
  const int n_el = c.D.nd + c.D.nt + c.D.na + c.D.nh + c.D.ns;
  double* __restrict__ P_ = c.K.p;
  double* __restrict__ AP = c.K.ap;
  const double* __restrict__ Z = c.K.z;
  const double* __restrict__ AZ = c.K.az;
  const double* __restrict__ Dg = c.K.d;
  double part = 0.0;
  FOR_ITEMS(it, n_el) {
    int rows[6];
    const int nr = item_rows(c, it, env, rows);
    double zr[6], azr[6], pr[6], apr[6], dr[6];
#pragma unroll
    for (int q = 0; q < 6; ++q) {
      if (q < nr) {
        const size_t o = IX(rows[q]);
        if (EXACT) zr[q] = Z[o];
        azr[q] = AZ[o];
        dr[q] = Dg[o];
        if (!setup) {
          if (EXACT) pr[q] = P_[o];
          apr[q] = AP[o];
        }
      }
    }
#pragma unroll
    for (int q = 0; q < 6; ++q) {
      if (q < nr) {
        const size_t o = IX(rows[q]);
        double ap;
        if (setup) {
          if (EXACT) P_[o] = zr[q];
          ap = azr[q];
        } else if (!brk) {
          if (EXACT) P_[o] = zr[q] + beta * pr[q];
          ap = azr[q] + beta * (EXACT ? apr[q] : apr[q] * dr[q]);
        } else {
          ap = EXACT ? apr[q] : apr[q] * dr[q];
        }
        const double apd = ap / dr[q];
        if (!brk || setup) AP[o] = EXACT ? ap : apd;
        part += ap * apd;
      }
    }
  }
  double den;
  if (reduce_env(c, part, &den)) {
    if (!c.K.broken[env]) {
      if (den <= 1e-300 || !isfinite(den)) {
        c.K.broken[env] = 1;
      } else {
        c.K.alpha_prev[env] = c.K.alpha[env];
        c.K.alpha[env] = c.K.rho[env] / den;
      }
    }
  }
}

// k_pcr_dir (structured mode) over rows instead of elements: every row is
// independent (ap = az + beta ap_prev, apd = ap/d, den += ap apd; absent
// contact rows skipped), so a thread keeps DIR_UNROLL rows' loads in flight
// with few registers and the grid holds more warps. Same per-row values as
// k_pcr_dir<false>; den is summed over another thread assignment.
#ifndef SS_DIR2_MINB
#define SS_DIR2_MINB 4
#endif
#ifndef DIR_UNROLL
#define DIR_UNROLL 4
#endif
__global__ void __launch_bounds__(SS_THREADS, SS_DIR2_MINB) k_pcr_dir_rows(const Ctx c, int setup) {
  SETUP
  const bool brk = c.K.broken[env] != 0;
  const double beta = c.K.beta[env];
  const int m = c.D.m;
  double* __restrict__ AP = c.K.ap;
  const double* __restrict__ AZ = c.K.az;
  const double* __restrict__ Dg = c.K.d;
  const int stride = gridDim.y * IL;
  double part = 0.0;
  for (int r0 = blockIdx.y * IL + il; r0 < m; r0 += DIR_UNROLL * stride) {
    double az[DIR_UNROLL], dg[DIR_UNROLL], apo[DIR_UNROLL];
    bool live[DIR_UNROLL];
#pragma unroll
    for (int q = 0; q < DIR_UNROLL; ++q) {
      const int row = r0 + q * stride;
      live[q] = row < m && row_live(c, row, env);
      if (live[q]) {
        const size_t o = IX(row);
        az[q] = AZ[o];
        dg[q] = Dg[o];
        if (!setup) apo[q] = AP[o];
      }
    }
#pragma unroll
    for (int q = 0; q < DIR_UNROLL; ++q) {
      if (!live[q]) continue;
      const size_t o = IX(r0 + q * stride);
      double ap;
      if (setup) ap = az[q];
      else if (!brk) ap = az[q] + beta * (apo[q] * dg[q]);
      else ap = apo[q] * dg[q];
      const double apd = ap / dg[q];
      if (!brk || setup) AP[o] = apd;
      part += ap * apd;
    }
  }
  double den;
  if (reduce_env(c, part, &den)) {
    if (!c.K.broken[env]) {
      if (den <= 1e-300 || !isfinite(den)) {
        c.K.broken[env] = 1;
      } else {
        c.K.alpha_prev[env] = c.K.alpha[env];
        c.K.alpha[env] = c.K.rho[env] / den;
      }
    }
  }
}

// x += alpha p, r -= alpha ap, z = r/d (solver.py:81-84); element-owned
// rows, loads before stores. Structured mode (!EXACT) keeps no r vector (it
// is d z by definition) and reads apd = ap/d from k_pcr_dir: z -= alpha apd
// carries the same recurrence one rounding apart per row, and the pass moves
// 6 row vectors (x p z apd in, x z out) instead of 8; k_newton_final takes
// r = d z for the residual.
// Structured mode also forms the search direction here, p = z + beta p
// (p = z on the first iteration; solver.py:90-91), from the z it already
// reads, instead of in k_pcr_dir: the same value bitwise, two row vectors
// fewer per iteration (k_pcr_dir no longer reads z, p or writes p).
template <bool EXACT>
#ifndef SS_STEP_MINB
#define SS_STEP_MINB 3
#endif
__global__ void __launch_bounds__(SS_THREADS, EXACT ? 2 : SS_STEP_MINB) k_pcr_step(const Ctx c, int k) {
  SETUP
  if (c.K.broken[env]) return;  // the reference skips the whole iteration
  const bool first = k == 0;
  // structured mode defers x: an even iteration leaves x alone, the next
  // (odd) one applies both, x = (x + alpha_prev p_old) + alpha p_new — the
  // reference's two updates in the reference's order (bitwise the same x),
  // with one x read/write per two iterations; k_newton_final applies a
  // pending even update (last_step)
  const bool upd_x = EXACT || (k & 1);
  const double alpha = c.K.alpha[env];
  const double beta = c.K.beta[env];
  const double alpha_prev = EXACT ? 0.0 : c.K.alpha_prev[env];
  if (!EXACT && blockIdx.y == 0 && il == 0) c.K.last_step[env] = k;
  const int n_el = c.D.nd + c.D.nt + c.D.na + c.D.nh + c.D.ns;
  double* __restrict__ X_ = c.K.x;
  double* __restrict__ R_ = c.K.r;
  double* __restrict__ Z_ = c.K.z;
  double* __restrict__ P_ = c.K.p;
  const double* __restrict__ AP = c.K.ap;
  const double* __restrict__ Dg = c.K.d;
  FOR_ITEMS(it, n_el) {
    int rows[6];
    const int nr = item_rows(c, it, env, rows);
    double xr[6], pr[6], rr[6], apr[6], dr[6];
#pragma unroll
    for (int q = 0; q < 6; ++q) {
      if (q < nr) {
        const size_t o = IX(rows[q]);
        if (upd_x) xr[q] = X_[o];
        if (EXACT || !first) pr[q] = P_[o];
        rr[q] = EXACT ? R_[o] : Z_[o];
        apr[q] = AP[o];
        if (EXACT) dr[q] = Dg[o];
      }
    }
#pragma unroll
    for (int q = 0; q < 6; ++q) {
      if (q < nr) {
        const size_t o = IX(rows[q]);
        if (EXACT) {
          X_[o] = xr[q] + alpha * pr[q];
          const double r = rr[q] - alpha * apr[q];
          R_[o] = r;
          Z_[o] = r / dr[q];
        } else {
          const double pn = first ? rr[q] : rr[q] + beta * pr[q];  // rr holds z here
          P_[o] = pn;
          if (upd_x) X_[o] = (xr[q] + alpha_prev * pr[q]) + alpha * pn;
          Z_[o] = rr[q] - alpha * apr[q];
        }
      }
    }
  }
}

// k_pcr_step + k_tet_jt in one pass (structured mode, E >= 32): a tet's 6
// rows are stepped by warp A (x, p, z, ap/d in; x, p, z out), which hands the
// new z to warp B through shared memory (named barrier per warp pair, double
// buffered); B loads the quaternion, S and the rest-shape inverse and writes
// the tet's 12 column sums of J^T z. The same operations as the two kernels
// (bitwise the same x, p, z and tC), without re-reading the tet rows of z and
// with one launch fewer per PCR iteration. Broken envs skip every store (the
// reference skips the whole iteration; tC keeps the previous pass).
#ifndef SS_STEPJT_MINB
#define SS_STEPJT_MINB 3
#endif
__global__ void __launch_bounds__(SS_THREADS, SS_STEPJT_MINB) k_step_jt(const Ctx c, int k) {
  SETUP
  __shared__ double zsh[4][2][6][32];  // [pair][buffer][row][env lane]
  const bool brk = c.K.broken[env] != 0;
  const bool first = k == 0;
  const bool upd_x = (k & 1) != 0;
  const double alpha = c.K.alpha[env];
  const double beta = c.K.beta[env];
  const double alpha_prev = c.K.alpha_prev[env];
  if (!brk && blockIdx.y == 0 && il == 0) c.K.last_step[env] = k;
  const int nd = c.D.nd, nt = c.D.nt, na = c.D.na, nh = c.D.nh, ns = c.D.ns;
  double* __restrict__ X_ = c.K.x;
  double* __restrict__ Z_ = c.K.z;
  double* __restrict__ P_ = c.K.p;
  const double* __restrict__ AP = c.K.ap;
  const int pair = il >> 1, role = il & 1;
  const unsigned uE = (unsigned)E;
  const unsigned ntE = (unsigned)nt * uE;
  int buf = 0;
  for (int t = blockIdx.y * (IL >> 1) + pair; t < nt; t += gridDim.y * (IL >> 1)) {
    double* zs = &zsh[pair][buf][0][lane];
    if (role == 0) {
      const unsigned ob = (unsigned)c.D.ot * uE + (unsigned)t * uE + (unsigned)env;
      double xr[6], pr[6], rr[6], apr[6];
#pragma unroll
      for (int q = 0; q < 6; ++q) {
        const unsigned o = ob + q * ntE;
        if (upd_x) xr[q] = X_[o];
        if (!first) pr[q] = P_[o];
        rr[q] = Z_[o];
        apr[q] = AP[o];
      }
#pragma unroll
      for (int q = 0; q < 6; ++q) {
        const unsigned o = ob + q * ntE;
        const double pn = first ? rr[q] : rr[q] + beta * pr[q];
        const double zn = rr[q] - alpha * apr[q];
        if (!brk) {
          P_[o] = pn;
          if (upd_x) X_[o] = (xr[q] + alpha_prev * pr[q]) + alpha * pn;
          Z_[o] = zn;
        }
        zs[q * 32] = zn;
      }
      named_bar(1 + pair, 64);
    } else {
      TetC T;
      double Ri[9];
      tet_load(c, t, env, T);
      tet_rinv(c, t, Ri);
      named_bar(1 + pair, 64);
      if (!brk) {
        double z6[6], col12[12];
#pragma unroll
        for (int q = 0; q < 6; ++q) z6[q] = zs[q * 32];
        tet_jt_cols(T, Ri, z6, col12);
        tc_put12(c, t, env, col12);
      }
    }
    buf ^= 1;
  }
  if (brk) return;  // after the last named barrier of this thread's pair
  const int n_other = nd + na + nh + ns;
  for (int q2 = blockIdx.y * IL + il; q2 < n_other; q2 += gridDim.y * IL) {
    const int it = q2 < nd ? q2 : q2 + nt;
    int rows[6];
    const int nr = item_rows(c, it, env, rows);
    double xr[6], pr[6], rr[6], apr[6];
#pragma unroll
    for (int q = 0; q < 6; ++q) {
      if (q < nr) {
        const size_t o = IX(rows[q]);
        if (upd_x) xr[q] = X_[o];
        if (!first) pr[q] = P_[o];
        rr[q] = Z_[o];
        apr[q] = AP[o];
      }
    }
#pragma unroll
    for (int q = 0; q < 6; ++q) {
      if (q < nr) {
        const size_t o = IX(rows[q]);
        const double pn = first ? rr[q] : rr[q] + beta * pr[q];
        P_[o] = pn;
        if (upd_x) X_[o] = (xr[q] + alpha_prev * pr[q]) + alpha * pn;
        Z_[o] = rr[q] - alpha * apr[q];
      }
    }
  }
}

// tet column sums of J^T z for the next apply (after k_pcr_step);
// M = EXACT | 2 * inbox layout
#ifndef SS_TETJT_MINB
#define SS_TETJT_MINB 3
#endif
template <int M>
__global__ void __launch_bounds__(SS_THREADS, (M & 1) ? 2 : SS_TETJT_MINB) k_tet_jt(const Ctx c) {
  constexpr bool EXACT = (M & 1) != 0;
  constexpr int IB = (M >> 1) & 3;
  SETUP
  if (c.K.broken[env]) return;  // z unchanged: tC from the previous pass is still valid
  const int nt = c.D.nt;
  FOR_ITEMS(t, nt) {
    double z6[6], Ri[9];
#pragma unroll
    for (int i = 0; i < 6; ++i) z6[i] = c.K.z[IX(c.D.ot + i * nt + t)];
    TetC T;
    tet_load(c, t, env, T);
    tet_rinv(c, t, Ri);
    tet_jt<EXACT, IB>(c, t, env, T, Ri, z6);
  }
}

// one item of the Newton tail (k_newton_final): the last PCR step of its
// rows, lam += dl with the contact projection, dlam, the tet column sums of
// J^T dlam; r.z of its rows added to part
struct FinalArgs {
  bool step, pend, first;
  int last;
  double alpha, beta, alpha_pend;
};
template <bool EXACT>
DI void final_item(const Ctx& c, int it, int env, const FinalArgs& F, double& part) {
  const int E = c.D.E;
  const int nd = c.D.nd, nt = c.D.nt, na = c.D.na, nh = c.D.nh, ns = c.D.ns, nw = c.D.nw;
  (void)na;
  const bool step = F.step, pend = F.pend, first = F.first;
  const int last = F.last;
  const double alpha = F.alpha, beta = F.beta, alpha_pend = F.alpha_pend;
  int rows[6];
  const int nr = item_rows(c, it, env, rows);
  // one pass per row: only dl survives into the multiplier update (the
  // two-pass load-all-then-compute form spilled the loaded rows at 128
  // registers, and each spill store waited on its load)
  double dl[6];
#pragma unroll
  for (int q = 0; q < 6; ++q) {
    if (q < nr) {
      const size_t o = IX(rows[q]);
      double x = c.K.x[o], z = c.K.z[o];
      double r = EXACT ? c.K.r[o] : 0.0;
      const double dq = (step || !EXACT) ? c.K.d[o] : 1.0;
      const double po = (!EXACT && (pend || (step && !first))) ? c.K.p[o] : 0.0;
      if (pend) x += alpha_pend * po;
      if (step) {
        double pq;
        if (EXACT) pq = c.K.p[o];
        else pq = first ? z : z + beta * po;  // the direction as k_pcr_step forms it
        const double apq = c.K.ap[o];
        x += alpha * pq;
        if (EXACT) {
          r -= alpha * apq;
          z = r / dq;
        } else {
          z -= alpha * apq;  // the ap buffer holds ap/d (k_pcr_dir)
        }
      }
      if (!EXACT) r = dq * z;  // structured mode keeps r = d z implicit
      part += r * z;
      dl[q] = x;
    }
  }
  if (it < nd + nt + na + nh) {
    double d6[6];
#pragma unroll
    for (int q = 0; q < 6; ++q) {
      if (q >= nr) break;
      const size_t o = IX(rows[q]);
      const double l0 = c.S.lam[o];
      const double l1 = l0 + dl[q];
      c.S.lam[o] = l1;
      d6[q] = l1 - l0;
      c.K.az[o] = d6[q];
    }
    if (it >= nd && it < nd + nt) {
      const int t = it - nd;
      TetC T;
      double Ri[9];
      tet_load(c, t, env, T);
      tet_rinv(c, t, Ri);
      tet_jt<EXACT>(c, t, env, T, Ri, d6);
    }
  } else {
    const int s = it - nd - nt - na - nh;
    double n1 = 0.0, a1 = 0.0, b1 = 0.0;
    if (nr) {
      const int rn = c.D.on + s, rf0 = c.D.of + s, rf1 = c.D.of + ns + s;
      const double n0 = c.K.lamc[IX(s)], a0 = c.K.lamc[IX(ns + s)], b0 = c.K.lamc[IX(2 * ns + s)];
      n1 = n0 + dl[0];
      a1 = a0 + dl[1];
      b1 = b0 + dl[2];
      n1 = npmax(n1, 0.0);
      const double rad = c.p.mu * npmax(n1, 0.0);
      const double nrm = sqrt(a1 * a1 + b1 * b1);
      if (nrm > rad) {
        const double sc = nrm > 0.0 ? rad / nrm : 0.0;
        a1 *= sc;
        b1 *= sc;
      }
      c.K.lamc[IX(s)] = n1;
      c.K.lamc[IX(ns + s)] = a1;
      c.K.lamc[IX(2 * ns + s)] = b1;
      c.K.az[IX(rn)] = n1 - n0;
      c.K.az[IX(rf0)] = a1 - a0;
      c.K.az[IX(rf1)] = b1 - b0;
    }
    if (last && s < nw) {
      c.S.warm_valid[IX(s)] = nr ? 1 : 0;
      c.S.warm[IX(s)] = n1;
      c.S.warm[IX(nw + s)] = a1;
      c.S.warm[IX(2 * nw + s)] = b1;
    }
  }
}

// Last PCR step fused with the Newton multiplier update (solver.py:81-85,
// 487-509; contact.py:157-165): dl = x + alpha p, lam += dl, contact
// projection, dlam = lam_after - lam_before into az (rows) and the tet
// column sums of J^T dlam; residual sqrt(max(r.z, 0)) of the solve; on the
// last Newton pass store_warm (contact.py:167-180). do_step = 0 when
// pcr_iters == 0.
template <bool EXACT>
// 2 CTAs/SM (<= 128 registers): 216 -> 128 registers, 7.8 -> 6.6 ms/frame
#ifndef SS_FINAL_MINB
#define SS_FINAL_MINB 2
#endif
#define SS_FINAL_MINB_LB __launch_bounds__(SS_THREADS, SS_FINAL_MINB)
__global__ void SS_FINAL_MINB_LB k_newton_final(const Ctx c, int do_step, int last,
                                                 int first) {
  SETUP
  const bool step = do_step && !c.K.broken[env];
  const double alpha = c.K.alpha[env];
  const double beta = c.K.beta[env];
  // a deferred x update of the last executed (even) k_pcr_step: its alpha is
  // alpha_prev after a further k_pcr_dir, alpha after a breakdown
  const int ls = EXACT ? -1 : c.K.last_step[env];
  const bool pend = ls >= 0 && !(ls & 1);
  const double alpha_pend = pend ? (step ? c.K.alpha_prev[env] : alpha) : 0.0;
  const int nd = c.D.nd, nt = c.D.nt, na = c.D.na, nh = c.D.nh, ns = c.D.ns, nw = c.D.nw;
  const int n_el = nd + nt + na + nh + ns;
  double part = 0.0;
  FinalArgs FA{step, pend, first != 0, last, alpha, beta, alpha_pend};
  (void)nw; (void)na; (void)nh; (void)ns; (void)nd; (void)nt;
  FOR_ITEMS(it, n_el) {
    final_item<EXACT>(c, it, env, FA, part);
  }
  double rz;
  if (reduce_env(c, part, &rz)) c.S.resid[env] = sqrt(0.0 > rz ? 0.0 : rz);
}

// k_newton_rhs / k_newton_final (structured mode, E >= 32) with each tet
// split over two warps of the same 32 envs, as k_apply_rows2: the same
// expressions as tet_forward_uv / tet_res / tet_jt_cols (bitwise the same
// rows and column sums), half the live registers per thread.
#ifndef SS_NEWTON2_MINB
#define SS_NEWTON2_MINB 3
#endif
template <int IB>
__global__ void __launch_bounds__(SS_THREADS, SS_NEWTON2_MINB) k_newton_rhs2(const Ctx c) {
  SETUP
  __shared__ double gsh[4][9][32];   // G (A -> B)
  __shared__ double zsh[4][9][32];   // z6 and n (B -> A)
  const int nd = c.D.nd, nt = c.D.nt, na = c.D.na, nh = c.D.nh, ns = c.D.ns;
  const double gm = c.p.gamma, h = c.p.h;
  const double* v = c.K.v;
  if (blockIdx.y == 0 && il == 0) {
    c.K.broken[env] = 0;
    c.K.beta[env] = 0.0;
    c.K.last_step[env] = -1;
  }
  TW_SETUP
  const unsigned uE = (unsigned)E;
  const unsigned ntE = (unsigned)nt * uE;
  for (int tw_t = tw_base; tw_t < nt; tw_t += tw_stride) {
    const int t = tw_t + tw_off;
    const bool tw_act = t < nt;
    const int tc = tw_act ? t : nt - 1;  // tail lanes load a valid tet, store nothing
    const unsigned tb = (unsigned)tc * uE + (unsigned)env;
    double* g = &gsh[pair][0][tw_slot];
    double* zs = &zsh[pair][0][tw_slot];
    if (role == 0) {
      int nid[4];
#pragma unroll
      for (int vv = 0; vv < 4; ++vv) nid[vv] = c.T.t_idx[vv * nt + tc];
      double uv[12], q[4], Ri[9];
#pragma unroll
      for (int vv = 0; vv < 4; ++vv) {
        const double* up = v + ((unsigned)(3 * nid[vv]) * uE + (unsigned)env);
#pragma unroll
        for (int a = 0; a < 3; ++a) uv[3 * vv + a] = up[a * uE];
      }
      const double* qp = c.S.quat + tb;
#pragma unroll
      for (int k = 0; k < 4; ++k) q[k] = qp[k * ntE];
      tet_rinv(c, tc, Ri);
      double du[9];
#pragma unroll
      for (int vv = 1; vv < 4; ++vv)
#pragma unroll
        for (int a = 0; a < 3; ++a) du[3 * (vv - 1) + a] = uv[3 * vv + a] - uv[a];
      double L[9];
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int j = 0; j < 3; ++j)
          L[3 * a + j] = dot3(du[a], Ri[j], du[3 + a], Ri[3 + j], du[6 + a], Ri[6 + j]);
      double R[9];
      quat_to_mat(q[0], q[1], q[2], q[3], R);
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j)
          g[(3 * i + j) * 32] = dot3(R[i], L[j], R[3 + i], L[3 + j], R[6 + i], L[6 + j]);
      named_bar(1 + pair, 64);  // G ready
      named_bar(1 + pair, 64);  // z6, n ready
      // tet_jt_cols, per-vertex part
      const double Z00 = zs[0], Z11 = zs[32], Z22 = zs[64];
      const double Z12 = 0.5 * zs[96], Z02 = 0.5 * zs[128], Z01 = 0.5 * zs[160];
      const double n0 = zs[192], n1 = zs[224], n2 = zs[256];
#pragma unroll
      for (int vv = 0; vv < 4; ++vv) {
        double wv[3];
        tet_wv(Ri, vv, wv);
        const double q0 = dot3(Z00, wv[0], Z01, wv[1], Z02, wv[2]) - __fma_rn(n1, wv[2], -n2 * wv[1]);
        const double q1 = dot3(Z01, wv[0], Z11, wv[1], Z12, wv[2]) - __fma_rn(n2, wv[0], -n0 * wv[2]);
        const double q2 = dot3(Z02, wv[0], Z12, wv[1], Z22, wv[2]) - __fma_rn(n0, wv[1], -n1 * wv[0]);
        if (tw_act)
          tc_put<IB>(c, t, vv, env, dot3(R[0], q0, R[1], q1, R[2], q2),
                 dot3(R[3], q0, R[4], q1, R[5], q2), dot3(R[6], q0, R[7], q1, R[8], q2));
      }
    } else {
      double sv[6], lm[6], bd[6];
      const double* sp = c.K.tS + tb;
#pragma unroll
      for (int k = 0; k < 6; ++k) sv[k] = sp[k * ntE];
      const unsigned ob = (unsigned)c.D.ot * uE + tb;
#pragma unroll
      for (int i = 0; i < 6; ++i) lm[i] = c.S.lam[ob + i * ntE];
#pragma unroll
      for (int i = 0; i < 6; ++i) bd[i] = c.K.bdiag[ob + i * ntE];
      const double ed = c.T.t_e3[tc], eo = c.T.t_e3[nt + tc], es = c.T.t_e3[2 * nt + tc];
      double S[9], Ki[9];
      S[0] = sv[0]; S[4] = sv[1]; S[8] = sv[2];
      S[5] = sv[3]; S[7] = sv[3];
      S[2] = sv[4]; S[6] = sv[4];
      S[1] = sv[5]; S[3] = sv[5];
      tet_kinv(S, Ki);
      named_bar(1 + pair, 64);  // G ready
      double G[9];
#pragma unroll
      for (int k = 0; k < 9; ++k) G[k] = g[k * 32];
      // tet_forward_uv, second half: jv = J v
      const double g0 = G[7] - G[5], g1 = G[2] - G[6], g2 = G[3] - G[1];
      const double w0 = dot3(Ki[0], g0, Ki[1], g1, Ki[2], g2);
      const double w1 = dot3(Ki[3], g0, Ki[4], g1, Ki[5], g2);
      const double w2 = dot3(Ki[6], g0, Ki[7], g1, Ki[8], g2);
      const double ws00 = __fma_rn(w1, S[6], -w2 * S[3]);
      const double ws01 = __fma_rn(w1, S[7], -w2 * S[4]);
      const double ws02 = __fma_rn(w1, S[8], -w2 * S[5]);
      const double ws10 = __fma_rn(w2, S[0], -w0 * S[6]);
      const double ws11 = __fma_rn(w2, S[1], -w0 * S[7]);
      const double ws12 = __fma_rn(w2, S[2], -w0 * S[8]);
      const double ws20 = __fma_rn(w0, S[3], -w1 * S[0]);
      const double ws21 = __fma_rn(w0, S[4], -w1 * S[1]);
      const double ws22 = __fma_rn(w0, S[5], -w1 * S[2]);
      double jv[6];
      jv[0] = G[0] - ws00;
      jv[1] = G[4] - ws11;
      jv[2] = G[8] - ws22;
      jv[3] = 0.5 * ((G[5] + G[7]) - (ws12 + ws21));
      jv[4] = 0.5 * ((G[2] + G[6]) - (ws02 + ws20));
      jv[5] = 0.5 * ((G[1] + G[3]) - (ws01 + ws10));
      // tet_res (numba_backend.py:241-246)
      double rs[6];
      rs[0] = S[0] - 1.0;
      rs[1] = S[4] - 1.0;
      rs[2] = S[8] - 1.0;
      rs[3] = S[5];
      rs[4] = S[2];
      rs[5] = S[1];
      double el[6], z6[6];
      ereg6(ed, eo, es, lm, el);
#pragma unroll
      for (int i = 0; i < 6; ++i) {
        const double dg = npmax(bd[i] + 0.0, 1e-30);
        const double d = dg > 1e-300 ? dg : 1.0;
        const double r = -(gm * rs[i] / h + jv[i] + el[i]);
        z6[i] = r / d;
        const unsigned o = ob + i * ntE;
        if (tw_act) {
          c.K.r[o] = r;
          c.K.d[o] = d;
          c.K.z[o] = z6[i];
          c.K.x[o] = 0.0;
        }
      }
      // tet_jt_cols, shared part: n = K^-1 ax(Z S)
      const double Z00 = z6[0], Z11 = z6[1], Z22 = z6[2];
      const double Z12 = 0.5 * z6[3], Z02 = 0.5 * z6[4], Z01 = 0.5 * z6[5];
      const double N21 = dot3(Z02, S[1], Z12, S[4], Z22, S[7]);
      const double N12 = dot3(Z01, S[2], Z11, S[5], Z12, S[8]);
      const double N02 = dot3(Z00, S[2], Z01, S[5], Z02, S[8]);
      const double N20 = dot3(Z02, S[0], Z12, S[3], Z22, S[6]);
      const double N10 = dot3(Z01, S[0], Z11, S[3], Z12, S[6]);
      const double N01 = dot3(Z00, S[1], Z01, S[4], Z02, S[7]);
      const double m0 = N21 - N12, m1 = N02 - N20, m2 = N10 - N01;
#pragma unroll
      for (int i = 0; i < 6; ++i) zs[i * 32] = z6[i];
      zs[192] = dot3(Ki[0], m0, Ki[1], m1, Ki[2], m2);
      zs[224] = dot3(Ki[3], m0, Ki[4], m1, Ki[5], m2);
      zs[256] = dot3(Ki[6], m0, Ki[7], m1, Ki[8], m2);
      named_bar(1 + pair, 64);  // z6, n ready
    }
  }
  const int n_other = nd + na + nh + ns;
  for (int q2 = blockIdx.y * IL + il; q2 < n_other; q2 += gridDim.y * IL) {
    const int it = q2 < nd ? q2 : q2 + nt;
    rhs_item<false>(c, it, env);
  }
}

template <int IB>
__global__ void __launch_bounds__(SS_THREADS, SS_NEWTON2_MINB) k_newton_final2(const Ctx c, int do_step,
                                                                               int last, int first) {
  SETUP
  __shared__ double dsh[4][6][32];  // dlam of the tet rows (A -> B)
  const bool step = do_step && !c.K.broken[env];
  const double alpha = c.K.alpha[env];
  const double beta = c.K.beta[env];
  const int ls = c.K.last_step[env];
  const bool pend = ls >= 0 && !(ls & 1);
  const double alpha_pend = pend ? (step ? c.K.alpha_prev[env] : alpha) : 0.0;
  const int nd = c.D.nd, nt = c.D.nt, na = c.D.na, nh = c.D.nh, ns = c.D.ns;
  const FinalArgs FA{step, pend, first != 0, last, alpha, beta, alpha_pend};
  TW_SETUP
  const unsigned uE = (unsigned)E;
  const unsigned ntE = (unsigned)nt * uE;
  double part = 0.0;
  for (int tw_t = tw_base; tw_t < nt; tw_t += tw_stride) {
    const int t = tw_t + tw_off;
    const bool tw_act = t < nt;
    const int tc = tw_act ? t : nt - 1;  // tail lanes load a valid tet, store nothing
    double* ds = &dsh[pair][0][tw_slot];
    if (role == 0) {
      const unsigned ob = (unsigned)c.D.ot * uE + (unsigned)tc * uE + (unsigned)env;
#pragma unroll
      for (int q = 0; q < 6; ++q) {
        const unsigned o = ob + q * ntE;
        double x = c.K.x[o], z = c.K.z[o];
        const double dq = c.K.d[o];
        const double po = (pend || (step && !FA.first)) ? c.K.p[o] : 0.0;
        if (pend) x += alpha_pend * po;
        if (step) {
          const double pq = FA.first ? z : z + beta * po;
          const double apq = c.K.ap[o];
          x += alpha * pq;
          z -= alpha * apq;
        }
        const double r = dq * z;
        const double l0 = c.S.lam[o];
        const double l1 = l0 + x;
        const double d6 = l1 - l0;
        if (tw_act) {
          part += r * z;
          c.S.lam[o] = l1;
          c.K.az[o] = d6;
        }
        ds[q * 32] = d6;
      }
      named_bar(1 + pair, 64);
    } else {
      TetC T;
      double Ri[9];
      tet_load(c, tc, env, T);
      tet_rinv(c, tc, Ri);
      named_bar(1 + pair, 64);
      double d6[6], col12[12];
#pragma unroll
      for (int q = 0; q < 6; ++q) d6[q] = ds[q * 32];
      tet_jt_cols(T, Ri, d6, col12);
      if (tw_act) tc_put12<IB>(c, t, env, col12);
    }
    named_bar(1 + pair, 64);  // ds consumed before the next item overwrites it
  }
  const int n_other = nd + na + nh + ns;
  for (int q2 = blockIdx.y * IL + il; q2 < n_other; q2 += gridDim.y * IL) {
    const int it = q2 < nd ? q2 : q2 + nt;
    final_item<false>(c, it, env, FA, part);
  }
  double rz;
  if (reduce_env(c, part, &rz)) c.S.resid[env] = sqrt(0.0 > rz ? 0.0 : rz);
}

// set_velocities + integrate_pose + quat_step (state.py:155-160, 171-192)
__global__ void k_integrate(const Ctx c) {
  SETUP
  const int P = c.D.P;
  const double h = c.p.h;
  FOR_ITEMS(it, P + c.D.nb) {
    if (it == 0) c.S.time[env] = c.S.time[env] + h;
    if (it < P) {
      bool bad = false;
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        const double vv = c.K.v[IX(3 * it + a)];
        c.S.vel[IX(3 * it + a)] = vv;
        const double x = c.S.pos[IX(3 * it + a)] + h * vv;
        c.S.pos[IX(3 * it + a)] = x;
        bad |= !isfinite(x);
      }
      if (bad) c.S.nonfinite[env] = 1;
    } else {
      const int b = it - P, o = c.D.bd0 + 6 * b;
      double w[3];
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        const double lv = c.K.v[IX(o + a)];
        w[a] = c.K.v[IX(o + 3 + a)];
        c.S.blin[IX(3 * b + a)] = lv;
        c.S.bang[IX(3 * b + a)] = w[a];
        c.S.bpos[IX(3 * b + a)] = c.S.bpos[IX(3 * b + a)] + h * lv;
      }
      double q[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) q[k] = c.S.bquat[IX(4 * b + k)];
      const double ch = c.p.half_h;
      const double r0 = q[0] - ch * (w[0] * q[1] + w[1] * q[2] + w[2] * q[3]);
      const double r1 = q[1] + ch * (w[0] * q[0] + w[1] * q[3] - w[2] * q[2]);
      const double r2 = q[2] + ch * (-w[0] * q[3] + w[1] * q[0] + w[2] * q[1]);
      const double r3 = q[3] + ch * (w[0] * q[2] - w[1] * q[1] + w[2] * q[0]);
      const double nrm = sqrt(r0 * r0 + r1 * r1 + r2 * r2 + r3 * r3);
      c.S.bquat[IX(4 * b)] = r0 / nrm;
      c.S.bquat[IX(4 * b + 1)] = r1 / nrm;
      c.S.bquat[IX(4 * b + 2)] = r2 / nrm;
      c.S.bquat[IX(4 * b + 3)] = r3 / nrm;
    }
  }
}

// center_of_mass (state.py:285-292), one thread per env (readback only)
// mass-weighted centre of mass (state.py:285-292). Block = L env lanes x
// (256/L) particle groups; group g sums particles g, g+G, ... and the groups
// are combined in a fixed order (deterministic for any env count).
__global__ void __launch_bounds__(256) k_com(const Ctx c, int env0, int n, double* out) {
  __shared__ double sh[4][256];
  const int L = c.D.W, G = 256 / L;
  const int lane = threadIdx.x % L, g = threadIdx.x / L;
  const int e = blockIdx.x * L + lane;
  const int env = env0 + (e < n ? e : 0), E = c.D.E;
  double tot = 0.0, cx = 0.0, cy = 0.0, cz = 0.0;
  for (int i = g; i < c.D.P; i += G) {
    const double im = c.T.inv_mass[i];
    if (!(im > 0.0)) continue;
    const double m = 1.0 / im;
    tot += m;
    cx += m * c.S.pos[IX(3 * i)];
    cy += m * c.S.pos[IX(3 * i + 1)];
    cz += m * c.S.pos[IX(3 * i + 2)];
  }
  sh[0][threadIdx.x] = tot;
  sh[1][threadIdx.x] = cx;
  sh[2][threadIdx.x] = cy;
  sh[3][threadIdx.x] = cz;
  __syncthreads();
  for (int h = G / 2; h > 0; h >>= 1) {
    if (g < h)
      for (int k = 0; k < 4; ++k) sh[k][threadIdx.x] += sh[k][threadIdx.x + h * L];
    __syncthreads();
  }
  if (g != 0 || e >= n) return;
  tot = sh[0][lane];
  cx = sh[1][lane];
  cy = sh[2][lane];
  cz = sh[3][lane];
  for (int b = 0; b < c.D.nb; ++b) {
    const double m = 1.0 / c.T.body_inv_mass[b];
    tot += m;
    cx += m * c.S.bpos[IX(3 * b)];
    cy += m * c.S.bpos[IX(3 * b + 1)];
    cz += m * c.S.bpos[IX(3 * b + 2)];
  }
  out[3 * e] = cx / tot;
  out[3 * e + 1] = cy / tot;
  out[3 * e + 2] = cz / tot;
}

// Per-env rollout observables for the batched harness (snake.py:208-232,
// state.py:271-292): out[env] = [com(3), kinetic energy, yaw of every body
// (nb)]. Same lane x group layout and fixed combine order as k_com.
__global__ void __launch_bounds__(256) k_observe(const Ctx c, int env0, int n, double* out) {
  __shared__ double sh[5][256];
  const int L = c.D.W, G = 256 / L;
  const int lane = threadIdx.x % L, g = threadIdx.x / L;
  const int e = blockIdx.x * L + lane;
  const int env = env0 + (e < n ? e : 0), E = c.D.E;
  double tot = 0.0, cx = 0.0, cy = 0.0, cz = 0.0, ke = 0.0;
  for (int i = g; i < c.D.P; i += G) {
    const double im = c.T.inv_mass[i];
    if (!(im > 0.0)) continue;
    const double m = 1.0 / im;
    tot += m;
    cx += m * c.S.pos[IX(3 * i)];
    cy += m * c.S.pos[IX(3 * i + 1)];
    cz += m * c.S.pos[IX(3 * i + 2)];
    const double v0 = c.S.vel[IX(3 * i)], v1 = c.S.vel[IX(3 * i + 1)], v2 = c.S.vel[IX(3 * i + 2)];
    ke += m * (v0 * v0 + v1 * v1 + v2 * v2);
  }
  sh[0][threadIdx.x] = tot;
  sh[1][threadIdx.x] = cx;
  sh[2][threadIdx.x] = cy;
  sh[3][threadIdx.x] = cz;
  sh[4][threadIdx.x] = ke;
  __syncthreads();
  for (int h = G / 2; h > 0; h >>= 1) {
    if (g < h)
      for (int k = 0; k < 5; ++k) sh[k][threadIdx.x] += sh[k][threadIdx.x + h * L];
    __syncthreads();
  }
  if (g != 0 || e >= n) return;
  tot = sh[0][lane];
  cx = sh[1][lane];
  cy = sh[2][lane];
  cz = sh[3][lane];
  ke = 0.5 * sh[4][lane];
  const int nb = c.D.nb;
  double* o = out + (size_t)e * (4 + nb);
  for (int b = 0; b < nb; ++b) {
    const double m = 1.0 / c.T.body_inv_mass[b];
    tot += m;
    cx += m * c.S.bpos[IX(3 * b)];
    cy += m * c.S.bpos[IX(3 * b + 1)];
    cz += m * c.S.bpos[IX(3 * b + 2)];
    double qw = c.S.bquat[IX(4 * b)], qx = c.S.bquat[IX(4 * b + 1)];
    double qy = c.S.bquat[IX(4 * b + 2)], qz = c.S.bquat[IX(4 * b + 3)];
    const double qn = sqrt(qw * qw + qx * qx + qy * qy + qz * qz);
    qw /= qn; qx /= qn; qy /= qn; qz /= qn;
    double R[9];
    quat_to_mat(qw, qx, qy, qz, R);
    const double lv0 = c.S.blin[IX(3 * b)], lv1 = c.S.blin[IX(3 * b + 1)], lv2 = c.S.blin[IX(3 * b + 2)];
    const double w0 = c.S.bang[IX(3 * b)], w1 = c.S.bang[IX(3 * b + 1)], w2 = c.S.bang[IX(3 * b + 2)];
    // body-frame omega = R^T w; 0.5 w^T (R I R^T) w
    const double b0 = R[0] * w0 + R[3] * w1 + R[6] * w2;
    const double b1 = R[1] * w0 + R[4] * w1 + R[7] * w2;
    const double b2 = R[2] * w0 + R[5] * w1 + R[8] * w2;
    const double* I = c.T.body_inertia + 9 * b;
    const double i0 = I[0] * b0 + I[1] * b1 + I[2] * b2;
    const double i1 = I[3] * b0 + I[4] * b1 + I[5] * b2;
    const double i2 = I[6] * b0 + I[7] * b1 + I[8] * b2;
    ke += 0.5 * m * (lv0 * lv0 + lv1 * lv1 + lv2 * lv2) + 0.5 * (b0 * i0 + b1 * i1 + b2 * i2);
    o[4 + b] = atan2(R[3], R[0]);  // heading of the body x axis (snake.py:185-188)
  }
  o[0] = cx / tot;
  o[1] = cy / tot;
  o[2] = cz / tot;
  o[3] = ke;
}

// System inspection (solver.py:511-518 snapshot, 548-575 last_system): the
// last substep's Newton system of env lane `env` in the reference's block
// layout. Static rows are permuted to the reference row order; contact
// slots stay uncompacted (the host compacts present slots in slot order,
// which is the reference's contact order). Items: nd + nt + na + nh + ns
// elements, then P + nb mass-inverse nodes.
struct SysOut {
  double *dist_v, *tet_v, *att_v, *hinge_v, *slot_v;  // [nd][6] [nt][72] [na][27] [nh][60] [ns][18]
  int *dist_i, *tet_i, *att_i, *hinge_i, *slot_i, *slot_p;  // [nd][6] [nt][12] [na][9] [nh][12] [ns][6] [ns]
  double *rhs_s, *dyn_s, *rhs_c, *dyn_c;  // [ms] [ms] [ns][3] [ns][3]
  double *minv_d, *ang;                   // [ndof] [nb][9]
};
__global__ void k_export_system(const Ctx c, int env, SysOut o) {
  const int E = c.D.E;
  const int nd = c.D.nd, nt = c.D.nt, na = c.D.na, nh = c.D.nh, ns = c.D.ns, nw = c.D.nw;
  const int bd0 = c.D.bd0, n_el = nd + nt + na + nh + ns;
  const int ot_ref = nd, oa_ref = nd + 6 * nt, oh_ref = oa_ref + 3 * na;
  const double* snap = c.K.snap_rhs;
  for (int it = blockIdx.x * blockDim.x + threadIdx.x; it < n_el + c.D.P + c.D.nb;
       it += gridDim.x * blockDim.x) {
    if (it < nd) {
      const int d = it, i = c.T.d_i[d], j = c.T.d_j[d];
      for (int a = 0; a < 3; ++a) {
        const double u = c.S.dirs[IX(a * nd + d)];
        o.dist_v[6 * d + a] = u;
        o.dist_v[6 * d + 3 + a] = -u;
        o.dist_i[6 * d + a] = 3 * i + a;
        o.dist_i[6 * d + 3 + a] = 3 * j + a;
      }
      o.rhs_s[d] = snap[IX(c.D.od + d)];
      o.dyn_s[d] = c.T.d_dyn[d];
    } else if (it < nd + nt) {
      const int t = it - nd;
      TetC T;
      double Ri[9];
      tet_load(c, t, env, T);
      tet_rinv(c, t, Ri);
      for (int v = 0; v < 4; ++v) {
        double wv[3];
        tet_wv(Ri, v, wv);
        const int node = c.T.t_idx[v * nt + t];
        for (int a = 0; a < 3; ++a) {
          double col[6];
          tet_col(T, wv, a, col);
          for (int i = 0; i < 6; ++i) o.tet_v[72 * (size_t)t + 12 * i + 3 * v + a] = col[i];
          o.tet_i[12 * (size_t)t + 3 * v + a] = 3 * node + a;
        }
      }
      for (int i = 0; i < 6; ++i) {
        o.rhs_s[ot_ref + 6 * t + i] = snap[IX(c.D.ot + i * nt + t)];
        o.dyn_s[ot_ref + 6 * t + i] = 0.0;  // E_tet enters as 6x6 blocks
      }
    } else if (it < nd + nt + na) {
      const int a = it - nd - nt;
      double rw[3];
      for (int k = 0; k < 3; ++k) rw[k] = c.K.rw[IX(k * na + a)];
      for (int i = 0; i < 3; ++i) {
        for (int j = 0; j < 9; ++j) o.att_v[27 * a + 9 * i + j] = att_val(i, j, rw);
        o.rhs_s[oa_ref + 3 * a + i] = snap[IX(c.D.oa + i * na + a)];
        o.dyn_s[oa_ref + 3 * a + i] = c.T.a_dyn[a];
      }
      for (int k = 0; k < 3; ++k) o.att_i[9 * a + k] = 3 * c.T.a_p[a] + k;
      for (int k = 0; k < 6; ++k) o.att_i[9 * a + 3 + k] = bd0 + 6 * c.T.a_b[a] + k;
    } else if (it < nd + nt + na + nh) {
      const int h = it - nd - nt - na;
      for (int i = 0; i < 5; ++i) {
        for (int j = 0; j < 12; ++j) o.hinge_v[60 * h + 12 * i + j] = c.K.hJ[IX((size_t)(12 * i + j) * nh + h)];
        o.rhs_s[oh_ref + 5 * h + i] = snap[IX(c.D.oh + i * nh + h)];
        o.dyn_s[oh_ref + 5 * h + i] = c.T.h_dyn[h];
      }
      for (int k = 0; k < 6; ++k) {
        o.hinge_i[12 * h + k] = bd0 + 6 * c.T.h_a[h] + k;
        o.hinge_i[12 * h + 6 + k] = bd0 + 6 * c.T.h_b[h] + k;
      }
    } else if (it < n_el) {
      const int sl = it - nd - nt - na - nh;
      const int pres = c.K.present[IX(sl)] != 0;
      o.slot_p[sl] = pres;
      double* v = o.slot_v + 18 * (size_t)sl;
      int* ix = o.slot_i + 6 * sl;
      if (sl < nw) {
        const int ob = bd0 + 6 * c.T.w_body[sl];
        for (int k = 0; k < 6; ++k) ix[k] = ob + k;
        for (int r = 0; r < 3; ++r)
          for (int k = 0; k < 6; ++k) v[6 * r + k] = c.K.wJ[IX((size_t)(6 * r + k) * nw + sl)];
      } else {
        // particle contact: 3 DOFs, columns 3..5 padded with DOF 0 (contact.py:208-214)
        const int pi = c.T.slot_part[sl - nw];
        for (int k = 0; k < 6; ++k) ix[k] = k < 3 ? 3 * pi + k : 0;
        for (int k = 0; k < 18; ++k) v[k] = 0.0;
        v[2] = 1.0;       // normal (0, 0, 1)
        v[6 + 0] = 1.0;   // t1 (1, 0, 0)
        v[12 + 1] = 1.0;  // t2 (0, 1, 0)
      }
      o.rhs_c[3 * sl] = pres ? snap[IX(c.D.on + sl)] : 0.0;
      o.rhs_c[3 * sl + 1] = pres ? snap[IX(c.D.of + sl)] : 0.0;
      o.rhs_c[3 * sl + 2] = pres ? snap[IX(c.D.of + ns + sl)] : 0.0;
      o.dyn_c[3 * sl] = pres ? c.K.dynn[IX(sl)] : 0.0;
      o.dyn_c[3 * sl + 1] = c.p.fdyn;
      o.dyn_c[3 * sl + 2] = c.p.fdyn;
    } else if (it < n_el + c.D.P) {
      const int i = it - n_el;
      for (int a = 0; a < 3; ++a) o.minv_d[3 * i + a] = c.T.inv_mass[i];
    } else {
      const int b = it - n_el - c.D.P;
      for (int a = 0; a < 3; ++a) {
        o.minv_d[bd0 + 6 * b + a] = c.T.body_inv_mass[b];
        o.minv_d[bd0 + 6 * b + 3 + a] = 0.0;  // angular block in ang
      }
      for (int k = 0; k < 9; ++k) o.ang[9 * b + k] = c.K.ang_inv[IX((size_t)k * c.D.nb + b)];
    }
  }
}

// Episode reset (per-env initial-state replication and
// perturbation on the device): write the captured template env into the listed
// lanes of one wave. noise_sigma > 0 adds a deterministic N(0, sigma^2) draw
// per (seed, global env, element) — a counter hash, so an env's perturbation
// does not depend on which other envs reset with it; pinned particles
// (inv_mass 0) are never moved (mask).
DI unsigned long long ss_mix64(unsigned long long z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
DI double ss_gauss(unsigned long long seed, unsigned long long env, unsigned long long k) {
  const unsigned long long h1 = ss_mix64(seed ^ ss_mix64(env * 0x100000001B3ull + k));
  const unsigned long long h2 = ss_mix64(h1 ^ 0xD1B54A32D192ED03ull);
  const double u1 = ((h1 >> 11) + 1.0) * (1.0 / 9007199254740993.0);  // (0, 1]
  const double u2 = (h2 >> 11) * (1.0 / 9007199254740992.0);          // [0, 1)
  return sqrt(-2.0 * log(u1)) * cospi(2.0 * u2);
}
template <typename T>
__global__ void k_reset_field(T* dst, const T* src, const int* lanes, const int* envs, int n, int A,
                              int B, int swap, int E, double sigma, unsigned long long seed,
                              int salt, const double* mask) {
  const size_t K = (size_t)A * B;
  for (size_t g = blockIdx.x * (size_t)blockDim.x + threadIdx.x; g < K * n;
       g += (size_t)gridDim.x * blockDim.x) {
    const int j = (int)(g / K);
    const size_t k = g % K;
    const size_t a = k / B, b = k % B;
    const size_t item = swap ? b * A + a : k;
    T v = src[k];
    if (sigma > 0.0 && (!mask || mask[a] > 0.0))
      v = (T)((double)v + sigma * ss_gauss(seed, (unsigned long long)envs[j],
                                            ((unsigned long long)salt << 40) | k));
    dst[item * E + lanes[j]] = v;
  }
}

// host env-major [n][A*B] <-> device [item][E] (item = swap ? b*A+a : a*B+b).
// Scatter also replicates env 0 into the padding lanes [n_real, E).
template <typename T>
__global__ void k_scatter(T* dst, const T* src, int n, int A, int B, int swap, int E, int env0,
                          int n_real) {
  const size_t K = (size_t)A * B;
  const size_t tot = K * E;
  for (size_t g = blockIdx.x * (size_t)blockDim.x + threadIdx.x; g < tot;
       g += (size_t)gridDim.x * blockDim.x) {
    const int e = (int)(g % E);
    const size_t k = g / E;
    int se;
    if (e >= env0 && e < env0 + n) se = e - env0;
    else if (env0 == 0 && e >= n_real) se = 0;
    else continue;
    const size_t a = k / B, b = k % B;
    const size_t item = swap ? b * A + a : k;
    dst[item * E + e] = src[(size_t)se * K + k];
  }
}
template <typename T>
__global__ void k_gather_state(T* dst, const T* src, int n, int A, int B, int swap, int E,
                               int env0) {
  const size_t K = (size_t)A * B;
  const size_t tot = K * n;
  for (size_t g = blockIdx.x * (size_t)blockDim.x + threadIdx.x; g < tot;
       g += (size_t)gridDim.x * blockDim.x) {
    const int e = (int)(g / K);
    const size_t k = g % K;
    const size_t a = k / B, b = k % B;
    const size_t item = swap ? b * A + a : k;
    dst[g] = src[item * E + env0 + e];
  }
}
