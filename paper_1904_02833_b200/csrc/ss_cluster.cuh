// ss_cluster.cuh — cluster-resident Newton solver (one environment per
// thread-block cluster).
//
// The whole Newton loop of a substep (solver.py:428-509: initial impulse,
// newton_iters x {rhs, pcr_solve, multiplier update + projection, impulse})
// runs inside ONE kernel launch in which a cluster of C CTAs (C <= 16,
// one CTA per SM) owns one environment. The environment's elements and
// DOF nodes are partitioned over the C CTAs (contiguous mesh slabs); every
// PCR row vector, the compact tet Jacobians, the per-element J^T column
// sums and the DOF vectors live in shared memory for the whole solve. The
// node gather (J^T x, in the reference accumulation order) and the element
// forward products (J u) only read local shared memory: every cross-CTA
// transfer is a DSMEM *store* pushed by the producer before a cluster
// barrier (column sums into per-incidence inbox slots of the node owner, in
// the reference accumulation order; updated DOF values into halo copies of
// the consumer CTAs; reduction partials into every peer). The per-env PCR
// dot products are fixed-order trees combined across the cluster in rank
// order (identical in every CTA, deterministic). HBM is
// touched only to load the substep inputs and store the results, so the
// 160 PCR iterations of a frame run at on-chip bandwidth.
#pragma once
#include <cooperative_groups.h>

#include "ss_device.cuh"

namespace cg = cooperative_groups;

#define CL_THREADS 512
#define CL_MAXC 16

// contrib families (gather entry bits 23..25)
enum { CF_TET = 0, CF_DIST = 1, CF_ATT = 2, CF_HINGE = 3, CF_SLOT = 4 };

struct ClPlan {
  int C;                                    // CTAs per cluster
  int MT, MD, MA, MH, MS, MP, MB, MW;       // per-CTA maxima of each family / node kind
                                            // (MW: wheel slots, the first local slots)
  int NR, ME, MN, MDOFX, MIN;               // rows, elements, owned nodes, owned+halo DOFs, inbox
  // shared-memory offsets (doubles)
  int oZ, oP, oAP, oAZ, oD;                 // row vectors [NR] (x, r live in registers)
  int oJR, oJS, oJK;                        // compact tet J [9][MT] [6][MT] [6][MT]
  int oRi, oE3;                             // tet rest-shape inverse [9][MT], E_tet [3][MT]
  int oIn;                                  // inbox: per owned node, one 3/6-vector per incidence
  int oDir, oRw, oHJ, oWJ;                  // [3][MD] [3][MA] [60][MH] [18][MW]
  int oPres, oGap, oLc, oAct, oDyn, oBdn, oBdf;  // slots [MS] ... lamc [3][MS], bdf [2][MS]
  int oResD, oResA, oResH;                  // [MD] [3][MA] [5][MH]
  int oU, oV, oAng;                         // [MDOFX] (owned then halo DOFs) x2, [9][MB]
  int oRed;                                 // reduction partials [16][C]
  int smem_doubles;
  int G;               // clusters per environment (multi-cluster plans: one per component)
  double* xbuf;        // [xn][G][4] 16-byte tagged words: cluster partials of every reduction (G > 1)
  int* xcnt;           // [0] cross-cluster error flag (sticky)
  int xn;
  long long* dbg;      // optional phase timestamps (nullptr = off)
  const int* cnt;      // [C][8]: nT nD nA nH nS nP nB -
  const int* elem;     // [C][ME]    family-local global index of each local element
  const int* eref;     // [C][ME][4] local U/V offsets of the element's nodes
  const int* dest;     // [C][ME][4] inbox destinations: owner << 24 | inbox offset
  const int* node;     // [C][MN]    global node of each owned node: particle id, or P + body
  const int* in_ptr;   // [C][MN+1]  inbox offset of each owned node's first incidence
  const int* hp_ptr;   // [C][MN+1]  halo pushes of each owned node
  const int* hpush;    // consumer << 24 | consumer U/V offset
};

struct ClSmem {
  double* b;             // this CTA's shared memory base
  double* const* peer;   // shared-memory table of every CTA's base (incl. self)
};

// The fixed shuffle-down tree over 32 lanes (lane i < n holds src[i], the
// rest 0) evaluated by one thread for lane 0: the same additions in the
// same order as __shfl_down_sync with offsets 16..1, depth 5 (n <= 16).
DI double cl_tree16(const double* src, int n) {
  double v[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = (i < n ? src[i] : 0.0) + 0.0;  // offset 16: zeros
#pragma unroll
  for (int o = 8; o > 0; o >>= 1) {
#pragma unroll
    for (int i = 0; i < o; ++i) v[i] += v[i + o];
  }
  return v[0];
}

// Cluster-wide deterministic sums of N values (the same result in every
// CTA): per-warp shuffle trees (N independent chains), the CL_THREADS/32 warp
// partials combined by N*C threads at once — thread (q, dst) evaluates value
// q's warp tree and pushes the CTA partial to slot (slot + q) mod 16 of CTA
// dst — then the C partials combined by the same tree. The sums are bitwise
// those of the former shuffle-tree implementation (warp 0 reducing, then
// broadcasting).
// Exchange: each partial travels as ONE 16-byte DSMEM store {value, tag}
// (tag = this launch's reduction count, from 1; every CTA zeroes its box at
// kernel start, before the first cluster barrier) and the consumer threads
// poll their own box until every source's tag is present — no cluster
// barrier (tools/micro/cluster_sync.cu: sum3 with the barrier 3.5k cycles,
// tagged polling 1.9k). Slot reuse is safe: a CTA writes reduction r + 2
// only after finishing r + 1, which needs every CTA's r + 1 partial, which
// each CTA sends only after reading its r values. SS_CL_BARRIER_SUM keeps the
// barrier exchange (single doubles, [16][C] box).
template <int N>
DI void cl_cluster_sumN(const ClPlan& L, const ClSmem& S, const double* v, int slot,
                        double* scratch, double* out) {
  constexpr int NW = CL_THREADS >> 5;
  double w[N];
#pragma unroll
  for (int q = 0; q < N; ++q) w[q] = v[q];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
    for (int q = 0; q < N; ++q) w[q] += __shfl_down_sync(0xffffffffu, w[q], o);
  }
  const int wi = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) {
#pragma unroll
    for (int q = 0; q < N; ++q) scratch[q * NW + wi] = w[q];
  }
  __syncthreads();
  const int rank = (int)cg::this_cluster().block_rank();
  static_assert(NW == 16, "warp tree over 16 warp partials");
#ifdef SS_CL_BARRIER_SUM
  if ((int)threadIdx.x < N * L.C) {
    const int q = threadIdx.x / L.C, dst = threadIdx.x - q * L.C;
    S.peer[dst][L.oRed + ((slot + q) & 15) * L.C + rank] = cl_tree16(scratch + q * NW, NW);
  }
  cg::this_cluster().sync();
  if ((int)threadIdx.x < N) {
    const int q = threadIdx.x;
    scratch[48 + q] = cl_tree16(S.b + L.oRed + ((slot + q) & 15) * L.C, L.C);
  }
  __syncthreads();
#else
  const double tag = scratch[60] + 1.0;  // reductions of this launch so far + 1
  if ((int)threadIdx.x < N * L.C) {
    const int q = threadIdx.x / L.C, dst = threadIdx.x - q * L.C;
    const double t = cl_tree16(scratch + q * NW, NW);
    double* bx = S.peer[dst] + L.oRed + 2 * (((slot + q) & 15) * L.C + rank);
    *reinterpret_cast<double2*>(bx) = make_double2(t, tag);
  }
  if ((int)threadIdx.x < N * L.C) {
    const int q = threadIdx.x / L.C, src = threadIdx.x - q * L.C;
    const unsigned a = (unsigned)__cvta_generic_to_shared(S.b + L.oRed +
                                                         2 * (((slot + q) & 15) * L.C + src));
    double val, g;
    const long long t0 = clock64();
    while (true) {
      asm volatile("ld.volatile.shared.v2.f64 {%0, %1}, [%2];" : "=d"(val), "=d"(g) : "r"(a) : "memory");
      if (g == tag) break;
      if (clock64() - t0 > (1LL << 32)) {  // never when every CTA runs: flag, do not hang
        if (L.xcnt) L.xcnt[0] = 3;
        break;
      }
    }
    scratch[64 + 16 * q + src] = val;
  }
  __syncthreads();
  if ((int)threadIdx.x < N) {
    const int q = threadIdx.x;
    scratch[48 + q] = cl_tree16(scratch + 64 + 16 * q, L.C);
  }
  if (threadIdx.x == 0) scratch[60] = tag;
  __syncthreads();
#endif
#pragma unroll
  for (int q = 0; q < N; ++q) out[q] = scratch[48 + q];
}
DI double cl_cluster_sum(const ClPlan& L, const ClSmem& S, double v, int slot, double* scratch) {
  double o;
  cl_cluster_sumN<1>(L, S, &v, slot, scratch, &o);
  return o;
}
DI void cl_cluster_sum3(const ClPlan& L, const ClSmem& S, const double* v, int slot,
                        double* scratch, double* out) {
  cl_cluster_sumN<3>(L, S, v, slot, scratch, out);
}

// Multi-cluster environments (G > 1): the per-cluster totals v[0..n) (equal in
// every CTA of a cluster) are combined across the G clusters through global
// memory, flag-in-data: rank 0 of each cluster stores every total as one
// 16-byte word {lo, tag, hi, tag} (tag = reduction index + 1; the buffer is
// zeroed per launch), and in every CTA one thread per (cluster, total) polls
// that word until both tags are present — 8-byte halves are single-copy
// atomic, so a word with both tags holds both halves of the total — then the
// partials are added in cluster order (the same sum everywhere,
// deterministic). One L2 round trip, no fences, no atomics. The wait is
// bounded: a missing cluster (never the case when all are co-resident, which
// ss_create checks) ends it after ~2^32 cycles with an error flag instead of
// a hang.
constexpr int kClMaxGroups = 16;  // scratch[64 + 4 g + q] holds cluster g's totals
constexpr int kClXWords = 4;      // 16-byte words per (reduction, cluster)
DI void cl_xsum(const ClPlan& L, int grp, int rank, int& seq, double* v, int n, double* scratch) {
  if (L.G <= 1) return;
  const int r = seq++;
  if (r >= L.xn) {  // more reductions than the plan sized for: flag, never hang
    if (threadIdx.x == 0) L.xcnt[0] = 2;
    return;
  }
  const unsigned tag = (unsigned)r + 1u;
  uint4* slots = reinterpret_cast<uint4*>(L.xbuf) + (size_t)r * L.G * kClXWords;
  if (rank == 0 && (int)threadIdx.x < n) {
    const int q = threadIdx.x;
    const unsigned long long bits = (unsigned long long)__double_as_longlong(v[q]);
    uint4* w = slots + grp * kClXWords + q;
    asm volatile("st.relaxed.gpu.global.v4.b32 [%0], {%1, %2, %3, %4};" ::"l"(w),
                 "r"((unsigned)bits), "r"(tag), "r"((unsigned)(bits >> 32)), "r"(tag)
                 : "memory");
  }
  if ((int)threadIdx.x < L.G * n) {
    const int g = threadIdx.x / n, q = threadIdx.x % n;
    const uint4* w = slots + g * kClXWords + q;
    unsigned a, b, c, d;
    const long long t0 = clock64();
    while (true) {
      asm volatile("ld.relaxed.gpu.global.v4.b32 {%0, %1, %2, %3}, [%4];"
                   : "=r"(a), "=r"(b), "=r"(c), "=r"(d) : "l"(w) : "memory");
      if (b == tag && d == tag) break;
      if (clock64() - t0 > (1LL << 32)) {
        L.xcnt[0] = 1;
        break;
      }
    }
    scratch[64 + 4 * g + q] = __longlong_as_double((long long)(((unsigned long long)c << 32) | a));
  }
  __syncthreads();
  for (int q = 0; q < n; ++q) {
    double t = 0.0;
    for (int g = 0; g < L.G; ++g) t += scratch[64 + 4 * g + q];
    v[q] = t;
  }
  __syncthreads();
}

// ------------------------------------------------------------ node gather
// One thread per (owned node, axis): particles 3 threads each, bodies 6.
struct ClMn {
  int k0, k1, hp0, hp1, lb, base, a, width;  // inbox range, halo range, body slot, DOF base
  double im;
};

// w_a = sum of the node's inbox column a (incidence column sums stored by the
// element owners in the reference accumulation order), u = M^-1 w
// (numba_backend.py:68-82; body angular rows use all three angular sums);
// mode 0: U = u, mode 1: V += u; the value is pushed to every halo copy.
DI void cl_gather(const ClPlan& L, const ClSmem& S, bool has, const ClMn& mn, int mode) {
  if (!has) return;
  const double* sb = S.b;
  const int arr = mode == 0 ? L.oU : L.oV;
  double u;
  if (mn.width == 3 || mn.a < 3) {
    double w = 0.0;
    for (int k = mn.k0 + mn.a; k < mn.k1; k += mn.width) w += sb[k];
    u = mn.im * w;
  } else {
    double w3 = 0.0, w4 = 0.0, w5 = 0.0;
    for (int k = mn.k0; k < mn.k1; k += 6) {
      w3 += sb[k + 3];
      w4 += sb[k + 4];
      w5 += sb[k + 5];
    }
    const double* A = sb + L.oAng;
    const int i = mn.a - 3, MB = L.MB, lb = mn.lb;
    u = A[(3 * i) * MB + lb] * w3 + A[(3 * i + 1) * MB + lb] * w4 + A[(3 * i + 2) * MB + lb] * w5;
  }
  double* dst = S.b + arr + mn.base + mn.a;
  const double val = mode == 0 ? u : *dst + u;
  *dst = val;
  for (int q = mn.hp0; q < mn.hp1; ++q) {
    const int hp = L.hpush[q];
    S.peer[(unsigned)hp >> 24][arr + (hp & 0xFFFFFF) + mn.a] = val;
  }
}

// push n values to an inbox destination (owner << 24 | offset), negated if neg
DI void cl_put(const ClSmem& S, const ClPlan& L, int dst, const double* v, int n, bool neg = false) {
  double* p = S.peer[(unsigned)dst >> 24] + L.oIn + (dst & 0xFFFFFF);
  for (int k = 0; k < n; ++k) p[k] = neg ? -v[k] : v[k];
}

// row index of family-local row i of local element le
DI int cl_row_t(const ClPlan& L, int i, int le) { return i * L.MT + le; }
DI int cl_row_d(const ClPlan& L, int le) { return 6 * L.MT + le; }
DI int cl_row_a(const ClPlan& L, int i, int le) { return 6 * L.MT + L.MD + i * L.MA + le; }
DI int cl_row_h(const ClPlan& L, int i, int le) { return 6 * L.MT + L.MD + 3 * L.MA + i * L.MH + le; }
DI int cl_row_s(const ClPlan& L, int k, int le) {
  return 6 * L.MT + L.MD + 3 * L.MA + 5 * L.MH + k * L.MS + le;
}

// node DOF values of an element (local U/V copy: owned or halo)
DI const double* cl_dofp(const ClSmem& S, int ref, int arr) { return S.b + arr + ref; }

// local tet compact J from shared memory
DI void cl_tet_load(const ClPlan& L, const double* sb, int lt, TetC& T) {
#pragma unroll
  for (int k = 0; k < 9; ++k) T.R[k] = sb[L.oJR + k * L.MT + lt];
  double s[6], q[6];
#pragma unroll
  for (int k = 0; k < 6; ++k) {
    s[k] = sb[L.oJS + k * L.MT + lt];
    q[k] = sb[L.oJK + k * L.MT + lt];
  }
  T.S[0] = s[0]; T.S[4] = s[1]; T.S[8] = s[2];
  T.S[5] = s[3]; T.S[7] = s[3];
  T.S[2] = s[4]; T.S[6] = s[4];
  T.S[1] = s[5]; T.S[3] = s[5];
  T.K[0] = q[0]; T.K[4] = q[1]; T.K[8] = q[2];
  T.K[5] = q[3]; T.K[7] = q[3];
  T.K[2] = q[4]; T.K[6] = q[4];
  T.K[1] = q[5]; T.K[3] = q[5];
}

// J^T x of one tet into its 12 column sums (structured or materialised)
template <bool EXACT>
DI void cl_tet_jt(const TetC& T, const double* Ri, const double* x6, double* col12) {
  if (EXACT) {
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      double wv[3];
      tet_wv(Ri, v, wv);
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        double col[6];
        tet_col(T, wv, a, col);
        double acc = 0.0;
#pragma unroll
        for (int i = 0; i < 6; ++i) acc += col[i] * x6[i];
        col12[3 * v + a] = acc;
      }
    }
  } else {
    tet_jt_cols(T, Ri, x6, col12);
  }
}

// J u of one tet (u: 4 nodes x 3 gathered through the element refs)
template <bool EXACT>
DI void cl_tet_j(const TetC& T, const double* Ri, const double* uu, double* y) {
  if (EXACT) {
#pragma unroll
    for (int i = 0; i < 6; ++i) y[i] = 0.0;
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      double wv[3];
      tet_wv(Ri, v, wv);
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        double col[6];
        tet_col(T, wv, a, col);
#pragma unroll
        for (int i = 0; i < 6; ++i) y[i] += col[i] * uu[3 * v + a];
      }
    }
    return;
  }
  tet_forward_uv(T, Ri, uu, y);
}

// ---------------------------------------------------------------- family
// Element enumeration of a CTA: [tets][dist][attach][hinge][slots].
struct ClEl {
  int fam, le, g;  // family, family-local index, global index
};
// Per-thread element state, loaded once per kernel (a thread owns at most
// one element for the whole solve): identity, node offsets, inbox
// destinations, and the tet's rest-shape inverse and E_tet scalars.
struct ClMe {
  ClEl el;
  int ref[4], dst[4];
  double dyn;  // compliance term of distance / attachment / hinge rows
};
DI ClEl cl_el(const ClPlan& L, int rank, int e) {
  const int* cnt = L.cnt + 8 * rank;
  ClEl r;
  r.g = L.elem[(size_t)rank * L.ME + e];
  int b = 0;
  if (e < (b += cnt[0])) { r.fam = CF_TET; r.le = e; return r; }
  if (e < (b + cnt[1])) { r.fam = CF_DIST; r.le = e - b; return r; }
  b += cnt[1];
  if (e < (b + cnt[2])) { r.fam = CF_ATT; r.le = e - b; return r; }
  b += cnt[2];
  if (e < (b + cnt[3])) { r.fam = CF_HINGE; r.le = e - b; return r; }
  b += cnt[3];
  r.fam = CF_SLOT;
  r.le = e - b;
  return r;
}
DI int cl_nel(const ClPlan& L, int rank) {
  const int* cnt = L.cnt + 8 * rank;
  return cnt[0] + cnt[1] + cnt[2] + cnt[3] + cnt[4];
}

// rows of a local element: row q = base + q * stride for q < n (absent
// contact slots have none). Arithmetic, so no per-thread arrays are needed.
struct ClRows {
  int base, stride, n;
  DI int at(int q) const { return base + q * stride; }
};
DI ClRows cl_rows(const ClPlan& L, const double* sb, const ClEl& el) {
  switch (el.fam) {
    case CF_TET: return {cl_row_t(L, 0, el.le), L.MT, 6};
    case CF_DIST: return {cl_row_d(L, el.le), 1, 1};
    case CF_ATT: return {cl_row_a(L, 0, el.le), L.MA, 3};
    case CF_HINGE: return {cl_row_h(L, 0, el.le), L.MH, 5};
    default: return {cl_row_s(L, 0, el.le), L.MS, sb[L.oPres + el.le] == 0.0 ? 0 : 3};
  }
}

// Column sums J^T x of one element (per-row values xr[]) pushed to the
// inbox slots of its nodes. mode 0: apply_a masking (inactive friction ->
// 0); mode 1: impulse (present contacts, all rows). Absent slots push zeros.
template <bool EXACT>
DI void cl_contrib(const Ctx& c, const ClPlan& L, const ClSmem& S, const ClMe& me,
                   const double* xr, int mode) {
  const double* sb = S.b;
  const ClEl& el = me.el;
  const int* dst = me.dst;
  switch (el.fam) {
    case CF_TET: {
      TetC T;
      double col12[12], Ri[9];
      cl_tet_load(L, sb, el.le, T);
#pragma unroll
      for (int k = 0; k < 9; ++k) Ri[k] = sb[L.oRi + k * L.MT + el.le];
      cl_tet_jt<EXACT>(T, Ri, xr, col12);
#pragma unroll
      for (int v = 0; v < 4; ++v) cl_put(S, L, dst[v], col12 + 3 * v, 3);
      break;
    }
    case CF_DIST: {
      // +dir on the first particle, -dir on the second ((-d)*x == -(d*x))
      double a[3];
#pragma unroll
      for (int k = 0; k < 3; ++k) a[k] = 0.0 + sb[L.oDir + k * L.MD + el.le] * xr[0];
      cl_put(S, L, dst[0], a, 3);
      cl_put(S, L, dst[1], a, 3, true);
      break;
    }
    case CF_ATT: {
      double rw[3], col[9];
#pragma unroll
      for (int i = 0; i < 3; ++i) rw[i] = sb[L.oRw + i * L.MA + el.le];
#pragma unroll
      for (int j = 0; j < 9; ++j) {
        double acc = 0.0;
#pragma unroll
        for (int i = 0; i < 3; ++i) acc += att_val(i, j, rw) * xr[i];
        col[j] = acc;
      }
      cl_put(S, L, dst[0], col, 3);
      cl_put(S, L, dst[1], col + 3, 6);
      break;
    }
    case CF_HINGE: {
      double col[12];
#pragma unroll
      for (int j = 0; j < 12; ++j) {
        double acc = 0.0;
#pragma unroll
        for (int i = 0; i < 5; ++i) acc += sb[L.oHJ + (12 * i + j) * L.MH + el.le] * xr[i];
        col[j] = acc;
      }
      cl_put(S, L, dst[0], col, 6);
      cl_put(S, L, dst[1], col + 6, 6);
      break;
    }
    default: {
      const int ls = el.le;
      const bool pres = sb[L.oPres + ls] != 0.0;
      const bool fon = mode == 0 ? sb[L.oAct + ls] != 0.0 : true;
      const bool wheel = el.g < c.D.nw;
      double nv[6], f0[6], f1[6];
      if (wheel) {
#pragma unroll
        for (int k = 0; k < 6; ++k) {
          nv[k] = sb[L.oWJ + k * L.MW + ls];
          f0[k] = sb[L.oWJ + (6 + k) * L.MW + ls];
          f1[k] = sb[L.oWJ + (12 + k) * L.MW + ls];
        }
      } else {
#pragma unroll
        for (int k = 0; k < 6; ++k) { nv[k] = 0.0; f0[k] = 0.0; f1[k] = 0.0; }
        nv[2] = 1.0;
        f0[0] = 1.0;
        f1[1] = 1.0;
      }
      double cn[6], cf[6];
#pragma unroll
      for (int k = 0; k < 6; ++k) {
        cn[k] = pres ? 0.0 + nv[k] * xr[0] : 0.0;
        cf[k] = 0.0;
        if (pres && fon) {
          cf[k] = 0.0 + f0[k] * xr[1];
          cf[k] += f1[k] * xr[2];
        }
      }
      const int nd = wheel ? 6 : 3;
      cl_put(S, L, dst[0], cn, nd);
      cl_put(S, L, dst[1], cf, nd);
      break;
    }
  }
}

// J y rows of one element for a node vector at shared offset `arr` (U or V)
template <bool EXACT>
DI int cl_forward(const Ctx& c, const ClPlan& L, const ClSmem& S, const ClMe& me, int arr,
                  double* y) {
  const ClEl& el = me.el;
  const int* ref = me.ref;
  const double* sb = S.b;
  switch (el.fam) {
    case CF_TET: {
      double uu[12];
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const double* p = cl_dofp(S, ref[v], arr);
        uu[3 * v] = p[0];
        uu[3 * v + 1] = p[1];
        uu[3 * v + 2] = p[2];
      }
      TetC T;
      double Ri[9];
      cl_tet_load(L, sb, el.le, T);
#pragma unroll
      for (int k = 0; k < 9; ++k) Ri[k] = sb[L.oRi + k * L.MT + el.le];
      cl_tet_j<EXACT>(T, Ri, uu, y);
      return 6;
    }
    case CF_DIST: {
      const double* pi = cl_dofp(S, ref[0], arr);
      const double* pj = cl_dofp(S, ref[1], arr);
      const double u0 = sb[L.oDir + el.le], u1 = sb[L.oDir + L.MD + el.le],
                   u2 = sb[L.oDir + 2 * L.MD + el.le];
      double acc = 0.0;
      acc += u0 * pi[0];
      acc += u1 * pi[1];
      acc += u2 * pi[2];
      acc += -u0 * pj[0];
      acc += -u1 * pj[1];
      acc += -u2 * pj[2];
      y[0] = acc;
      return 1;
    }
    case CF_ATT: {
      const double* pp = cl_dofp(S, ref[0], arr);
      const double* pb = cl_dofp(S, ref[1], arr);
      double uu[9], rw[3];
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        uu[k] = pp[k];
        rw[k] = sb[L.oRw + k * L.MA + el.le];
      }
#pragma unroll
      for (int k = 0; k < 6; ++k) uu[3 + k] = pb[k];
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        double acc = 0.0;
#pragma unroll
        for (int j = 0; j < 9; ++j) acc += att_val(i, j, rw) * uu[j];
        y[i] = acc;
      }
      return 3;
    }
    case CF_HINGE: {
      const double* pa = cl_dofp(S, ref[0], arr);
      const double* pb = cl_dofp(S, ref[1], arr);
      double uu[12];
#pragma unroll
      for (int k = 0; k < 6; ++k) {
        uu[k] = pa[k];
        uu[6 + k] = pb[k];
      }
#pragma unroll
      for (int i = 0; i < 5; ++i) {
        double acc = 0.0;
#pragma unroll
        for (int j = 0; j < 12; ++j) acc += sb[L.oHJ + (12 * i + j) * L.MH + el.le] * uu[j];
        y[i] = acc;
      }
      return 5;
    }
    default: {
      const int ls = el.le;
      if (sb[L.oPres + ls] == 0.0) return 0;
      const double* p = cl_dofp(S, ref[0], arr);
      if (el.g < c.D.nw) {
#pragma unroll
        for (int r = 0; r < 3; ++r) {
          double acc = 0.0;
#pragma unroll
          for (int k = 0; k < 6; ++k) acc += sb[L.oWJ + (6 * r + k) * L.MW + ls] * p[k];
          y[r] = acc;
        }
      } else {
        // padded columns reference DOF 0 (contact.py:210-214): particle 0's x
        // particle 0 (padded columns): local, or read from its owner CTA
        const int r1 = ref[1];
        const double* p0 = r1 >= 0 ? cl_dofp(S, r1, arr)
                                   : S.peer[(unsigned)(-1 - r1) >> 24] + arr + ((-1 - r1) & 0xFFFFFF);
        const double x0 = p[0], x1 = p[1], x2 = p[2], z0 = p0[0];
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
      return 3;
    }
  }
}

// global static-row index of row i of element el (internal row layout)
DI int cl_grow(const Ctx& c, const ClEl& el, int i) {
  switch (el.fam) {
    case CF_TET: return c.D.ot + i * c.D.nt + el.g;
    case CF_DIST: return c.D.od + el.g;
    case CF_ATT: return c.D.oa + i * c.D.na + el.g;
    default: return c.D.oh + i * c.D.nh + el.g;
  }
}

// Row scaling by the Jacobi diagonal: EXACT divides like the reference
// (z = r/d); the structured mode keeps 1/d in the row vector and multiplies
// (one rounding of 1/d, <= 1 ulp per quotient, ~20x fewer FP64 operations).
template <bool EXACT>
DI double cl_dstore(double d) { return EXACT ? d : 1.0 / d; }
template <bool EXACT>
DI double cl_ddiv(double x, double dstored) { return EXACT ? x / dstored : x * dstored; }

// ===================================================================
// The Newton loop of one substep for one environment per cluster:
// grid.x = C * E, cluster (C,1,1), CL_THREADS threads, dynamic smem.
// Thread roles: element phases (one local element per thread), row phases
// (thread t owns rows t + j*CL_THREADS, j < CL_RPT; x and r of its rows live
// in registers for the whole solve), node phases (one (node, axis) per
// thread). Dead rows (absent contact slots, family padding) stay exactly 0.
#define CL_RPT 5
#define CL_STAMP(id)                                                                    \
  do {                                                                                  \
    if (L.dbg && blockIdx.x < 16 && threadIdx.x == 0 && itn == 1 && k == 3)             \
      L.dbg[16 * blockIdx.x + (id)] = clock64();                                        \
  } while (0)

template <bool EXACT>
__global__ void __launch_bounds__(CL_THREADS, 1) k_newton_cluster(const Ctx c, const ClPlan L) {
  pdl_wait();
  extern __shared__ __align__(16) double sm_[];
  __shared__ double scratch[64 + 4 * kClMaxGroups];
  __shared__ double* peers[CL_MAXC];
  cg::cluster_group cl = cg::this_cluster();
  const int rank = (int)cl.block_rank();
  // multi-cluster plans: G clusters per env, plan tables indexed by the
  // env-local CTA index (cluster grp, rank within it)
  const int gcta = blockIdx.x % (L.C * L.G);
  const int grp = gcta / L.C;
  const int env = blockIdx.x / (L.C * L.G);
  int xseq = 0;  // cross-cluster reduction sequence of this launch
  const int E = c.D.E;
  const int tid = threadIdx.x;
  if (tid < L.C) peers[tid] = cl.map_shared_rank(sm_, tid);
  ClSmem S;
  S.b = sm_;
  S.peer = peers;
  double* sb = sm_;
  const int* cnt = L.cnt + 8 * gcta;
  const int nEl = cl_nel(L, gcta);
  const int nP = cnt[5], nB = cnt[6];
  const double g = c.p.gamma, h = c.p.h;

  // ---- per-thread element state
  const bool has_el = tid < nEl;
  ClMe me;
  if (has_el) {
    me.el = cl_el(L, gcta, tid);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      me.ref[q] = L.eref[((size_t)gcta * L.ME + tid) * 4 + q];
      me.dst[q] = L.dest[((size_t)gcta * L.ME + tid) * 4 + q];
    }
    me.dyn = 0.0;
    if (me.el.fam == CF_DIST) me.dyn = c.T.d_dyn[me.el.g];
    else if (me.el.fam == CF_ATT) me.dyn = c.T.a_dyn[me.el.g];
    else if (me.el.fam == CF_HINGE) me.dyn = c.T.h_dyn[me.el.g];
  }
  // ---- per-thread (node, axis) state
  const bool has_na = tid < 3 * nP + 6 * nB;
  ClMn mn;
  if (has_na) {
    int n;
    if (tid < 3 * nP) {
      n = tid / 3;
      mn.a = tid % 3;
      mn.width = 3;
      mn.base = 3 * n;
      mn.lb = -1;
      mn.im = c.T.inv_mass[L.node[(size_t)gcta * L.MN + n]];
    } else {
      const int q = tid - 3 * nP;
      n = nP + q / 6;
      mn.a = q % 6;
      mn.width = 6;
      mn.lb = q / 6;
      mn.base = 3 * nP + 6 * mn.lb;
      mn.im = c.T.body_inv_mass[L.node[(size_t)gcta * L.MN + n] - c.D.P];
    }
    const int* iptr = L.in_ptr + (size_t)gcta * (L.MN + 1);
    const int* hptr = L.hp_ptr + (size_t)gcta * (L.MN + 1);
    mn.k0 = L.oIn + iptr[n];
    mn.k1 = L.oIn + iptr[n + 1];
    mn.hp0 = hptr[n];
    mn.hp1 = hptr[n + 1];
  }

  // ---- reduction box and counter (cl_cluster_sumN): zeroed before the first
  // cluster barrier, so no tag of an earlier launch is ever read
  for (int r = tid; r < 32 * L.C; r += CL_THREADS) sb[L.oRed + r] = 0.0;
  if (tid == 0) scratch[60] = 0.0;
  // ---- dead rows = 0 (d = 1): init every row, elements overwrite theirs
  for (int r = tid; r < L.NR; r += CL_THREADS) {
    sb[L.oZ + r] = 0.0;
    sb[L.oP + r] = 0.0;
    sb[L.oAP + r] = 0.0;
    sb[L.oAZ + r] = 0.0;
    sb[L.oD + r] = 1.0;
  }
  // ---- load substep inputs into shared memory
  if (has_el) {
    const ClEl& el = me.el;
    switch (el.fam) {
      case CF_TET: {
        const int nt = c.D.nt, t = el.g;
        TetC T;
        tet_load(c, t, env, T);  // R, K^-1 rebuilt from q and S
        const int sym[6] = {0, 4, 8, 5, 2, 1};
#pragma unroll
        for (int k = 0; k < 9; ++k) {
          sb[L.oJR + k * L.MT + el.le] = T.R[k];
          sb[L.oRi + k * L.MT + el.le] = c.T.t_rinv[10 * (size_t)t + k];
        }
#pragma unroll
        for (int k = 0; k < 6; ++k) {
          sb[L.oJS + k * L.MT + el.le] = T.S[sym[k]];
          sb[L.oJK + k * L.MT + el.le] = T.K[sym[k]];
        }
#pragma unroll
        for (int k = 0; k < 3; ++k) sb[L.oE3 + k * L.MT + el.le] = c.T.t_e3[k * nt + t];
        break;
      }
      case CF_DIST:
#pragma unroll
        for (int a = 0; a < 3; ++a) sb[L.oDir + a * L.MD + el.le] = c.S.dirs[IX(a * c.D.nd + el.g)];
        sb[L.oResD + el.le] = c.K.res[IX(c.D.od + el.g)];
        break;
      case CF_ATT:
#pragma unroll
        for (int i = 0; i < 3; ++i) {
          sb[L.oRw + i * L.MA + el.le] = c.K.rw[IX(i * c.D.na + el.g)];
          sb[L.oResA + i * L.MA + el.le] = c.K.res[IX(c.D.oa + i * c.D.na + el.g)];
        }
        break;
      case CF_HINGE:
        for (int k = 0; k < 60; ++k) sb[L.oHJ + k * L.MH + el.le] = c.K.hJ[IX((size_t)k * c.D.nh + el.g)];
#pragma unroll
        for (int i = 0; i < 5; ++i) sb[L.oResH + i * L.MH + el.le] = c.K.res[IX(c.D.oh + i * c.D.nh + el.g)];
        break;
      default: {
        const int s = el.g, ls = el.le, ns = c.D.ns;
        sb[L.oPres + ls] = c.K.present[IX(s)] ? 1.0 : 0.0;
        sb[L.oGap + ls] = c.K.gap[IX(s)];
#pragma unroll
        for (int k = 0; k < 3; ++k) sb[L.oLc + k * L.MS + ls] = c.K.lamc[IX(k * ns + s)];
        sb[L.oBdn + ls] = c.K.bdiag[IX(c.D.on + s)];
        sb[L.oBdf + ls] = c.K.bdiag[IX(c.D.of + s)];
        sb[L.oBdf + L.MS + ls] = c.K.bdiag[IX(c.D.of + ns + s)];
        if (s < c.D.nw)
          for (int k = 0; k < 18; ++k) sb[L.oWJ + k * L.MW + ls] = c.K.wJ[IX((size_t)k * c.D.nw + s)];
        break;
      }
    }
  }
  for (int n = tid; n < nP + nB; n += CL_THREADS) {
    const int gn = L.node[(size_t)gcta * L.MN + n];
    if (n < nP) {
#pragma unroll
      for (int a = 0; a < 3; ++a) sb[L.oV + 3 * n + a] = c.K.v[IX(3 * gn + a)];
    } else {
      const int lb = n - nP, gb = gn - c.D.P, o = c.D.bd0 + 6 * gb;
#pragma unroll
      for (int k = 0; k < 6; ++k) sb[L.oV + 3 * nP + 6 * lb + k] = c.K.v[IX(o + k)];
#pragma unroll
      for (int k = 0; k < 9; ++k) sb[L.oAng + k * L.MB + lb] = c.K.ang_inv[IX((size_t)k * c.D.nb + gb)];
    }
  }
  __syncthreads();
  // halo copies of V (owners push their loaded values)
  if (has_na) {
    const double val = sb[L.oV + mn.base + mn.a];
    for (int q = mn.hp0; q < mn.hp1; ++q) {
      const int hp = L.hpush[q];
      S.peer[(unsigned)hp >> 24][L.oV + (hp & 0xFFFFFF) + mn.a] = val;
    }
  }

  // ---- initial impulse v = vt + M^-1 J^T lam (solver.py:428-436)
  if (has_el) {
    const ClEl& el = me.el;
    double xr[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    if (el.fam == CF_SLOT) {
#pragma unroll
      for (int k = 0; k < 3; ++k) xr[k] = sb[L.oLc + k * L.MS + el.le];
    } else {
      const int nr = el.fam == CF_TET ? 6 : el.fam == CF_DIST ? 1 : el.fam == CF_ATT ? 3 : 5;
#pragma unroll
      for (int i = 0; i < 6; ++i)
        if (i < nr) xr[i] = c.S.lam[IX(cl_grow(c, el, i))];
    }
    cl_contrib<EXACT>(c, L, S, me, xr, 1);
  }
  cl.sync();
  cl_gather(L, S, has_na, mn, 1);
  cl.sync();

  int rslot = 0;  // rotating reduction slot (16 slots: rewritten only 15 barriers later)
  double resid = 0.0;
  double xr_[CL_RPT], rr_[CL_RPT];  // x and r of this thread's rows
  for (int itn = 0; itn < c.p.newton; ++itn) {
    const bool lastn = itn == c.p.newton - 1;
    // ---- rhs, FB, active set, diagonal; z = r/d; r -> AZ scratch; J^T z
    if (has_el) {
      const ClEl& el = me.el;
      const ClRows R = cl_rows(L, sb, el);
      double jv[6];
      if (R.n) cl_forward<EXACT>(c, L, S, me, L.oV, jv);
      double zr[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
      if (el.fam == CF_TET) {
        TetC T;
        cl_tet_load(L, sb, el.le, T);
        double rs[6], lm[6], el6[6];
        tet_res(T, rs);
#pragma unroll
        for (int i = 0; i < 6; ++i) lm[i] = c.S.lam[IX(cl_grow(c, el, i))];
        ereg6(sb[L.oE3 + el.le], sb[L.oE3 + L.MT + el.le], sb[L.oE3 + 2 * L.MT + el.le], lm, el6);
#pragma unroll
        for (int i = 0; i < 6; ++i) {
          const double dg = npmax(c.K.bdiag[IX(cl_grow(c, el, i))] + 0.0, 1e-30);
          const double d = dg > 1e-300 ? dg : 1.0;
          const double r = -(g * rs[i] / h + jv[i] + el6[i]);
          const double ds = cl_dstore<EXACT>(d);
          zr[i] = cl_ddiv<EXACT>(r, ds);
          sb[L.oAZ + R.at(i)] = r;
          sb[L.oD + R.at(i)] = ds;
          sb[L.oZ + R.at(i)] = zr[i];
        }
      } else if (el.fam != CF_SLOT) {
        const double dyn = me.dyn;
#pragma unroll
        for (int i = 0; i < 5; ++i) {
          if (i >= R.n) break;
          const int gr = cl_grow(c, el, i);
          const double res = el.fam == CF_DIST ? sb[L.oResD + el.le]
                           : el.fam == CF_ATT ? sb[L.oResA + i * L.MA + el.le]
                                              : sb[L.oResH + i * L.MH + el.le];
          const double dg = npmax(c.K.bdiag[IX(gr)] + dyn, 1e-30);
          const double d = dg > 1e-300 ? dg : 1.0;
          const double r = -(g * res / h + jv[i] + dyn * c.S.lam[IX(gr)]);
          const double ds = cl_dstore<EXACT>(d);
          zr[i] = cl_ddiv<EXACT>(r, ds);
          sb[L.oAZ + R.at(i)] = r;
          sb[L.oD + R.at(i)] = ds;
          sb[L.oZ + R.at(i)] = zr[i];
        }
      } else if (R.n) {
        const int ls = el.le;
        const double ln = sb[L.oLc + ls];
        const double a = sb[L.oGap + ls] / h + jv[0];
        const double b = ln;
        const double root = sqrt(a * a + b * b + c.p.fb_delta);
        const double phi = a + b - root;
        double da = 1.0 - a / root;
        const double db = 1.0 - b / root;
        if (da < c.p.smin) da = c.p.smin;
        else if (da > c.p.smax) da = c.p.smax;
        const double dynn = db / da;
        sb[L.oDyn + ls] = dynn;
        const double on = (c.p.mu * npmax(ln, 0.0) > 0.0) ? 1.0 : 0.0;
        sb[L.oAct + ls] = on;
        const double fd = c.p.fdyn;
        double rr[3], dd[3];
        rr[0] = -phi / da;
        {
          const double dg = npmax(sb[L.oBdn + ls] + dynn, 1e-30);
          dd[0] = dg > 1e-300 ? dg : 1.0;
        }
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          rr[1 + k] = -on * (jv[1 + k] + fd * sb[L.oLc + (1 + k) * L.MS + ls]);
          const double dg = on > 0.0 ? npmax(sb[L.oBdf + k * L.MS + ls] + fd, 1e-30) : 1.0;
          dd[1 + k] = dg > 1e-300 ? dg : 1.0;
        }
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          const double ds = cl_dstore<EXACT>(dd[k]);
          zr[k] = cl_ddiv<EXACT>(rr[k], ds);
          sb[L.oAZ + R.at(k)] = rr[k];
          sb[L.oD + R.at(k)] = ds;
          sb[L.oZ + R.at(k)] = zr[k];
        }
      } else {
        sb[L.oAct + el.le] = 0.0;
      }
      cl_contrib<EXACT>(c, L, S, me, zr, 0);
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < CL_RPT; ++j) {
      const int row = tid + j * CL_THREADS;
      xr_[j] = 0.0;
      rr_[j] = row < L.NR ? sb[L.oAZ + row] : 0.0;
    }
    bool broken = false;
    double rho = 0.0, alpha = 0.0, beta = 0.0;
    // Structured mode: one cluster reduction per PCR iteration. The apply
    // phase also sums s1 = az.D^-1 az and s2 = az.D^-1 ap_prev, so
    // den = ap.D^-1 ap with ap = az + beta ap_prev follows as
    // s1 + 2 beta s2 + beta^2 den_prev (same recurrence, solver.py:71-91;
    // 5e-14 relative per frame against the reference order, measured with
    // the reference's own pcr_solve patched), and the p/ap update, the step
    // and z = r/d run as one row pass.
    bool stepped = false;
    if (!EXACT) {
      double den = 0.0;
      for (int k = 0; k < c.p.pcr; ++k) {
        CL_STAMP(0);
        if (k > 0 && has_el) {
          const ClEl& el = me.el;
          const ClRows R = cl_rows(L, sb, el);
          double zr[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
#pragma unroll
          for (int q = 0; q < 6; ++q) {
            if (q >= R.n) break;
            zr[q] = sb[L.oZ + R.at(q)];
          }
          cl_contrib<EXACT>(c, L, S, me, zr, 0);
        }
        CL_STAMP(1);
        if (L.dbg) {  // stamps: every warp of the CTA done
          __syncthreads();
          CL_STAMP(10);
        }
        cl.sync();                            // column sums of J^T z visible
        CL_STAMP(2);
        cl_gather(L, S, has_na, mn, 0);       // U = M^-1 J^T z (+ halo pushes)
        CL_STAMP(3);
        if (L.dbg) {
          __syncthreads();
          CL_STAMP(11);
        }
        cl.sync();                            // U visible
        CL_STAMP(4);
        double part[3] = {0.0, 0.0, 0.0};
        auto acc = [&](int row, double zr, double az) {
          part[0] += zr * az;
          const double di = sb[L.oD + row];
          part[1] += az * (az * di);
          if (k > 0) part[2] += az * (sb[L.oAP + row] * di);
        };
        if (has_el) {
          const ClEl& el = me.el;
          const ClRows R = cl_rows(L, sb, el);
          const int nr = R.n;
          double y[6];
          if (nr) cl_forward<EXACT>(c, L, S, me, L.oU, y);
          if (!nr) {
          } else if (el.fam == CF_TET) {
            double zz[6], ez[6];
#pragma unroll
            for (int i = 0; i < 6; ++i) zz[i] = sb[L.oZ + R.at(i)];
            ereg6(sb[L.oE3 + el.le], sb[L.oE3 + L.MT + el.le], sb[L.oE3 + 2 * L.MT + el.le], zz, ez);
#pragma unroll
            for (int i = 0; i < 6; ++i) {
              const double az = y[i] + ez[i];
              sb[L.oAZ + R.at(i)] = az;
              acc(R.at(i), zz[i], az);
            }
          } else if (el.fam == CF_SLOT) {
            const int ls = el.le;
            const double zn = sb[L.oZ + R.at(0)], z0 = sb[L.oZ + R.at(1)], z1 = sb[L.oZ + R.at(2)];
            const double an = y[0] + sb[L.oDyn + ls] * zn;
            double a0 = z0, a1 = z1;
            if (sb[L.oAct + ls] != 0.0) {
              a0 = y[1] + c.p.fdyn * z0;
              a1 = y[2] + c.p.fdyn * z1;
            }
            sb[L.oAZ + R.at(0)] = an;
            sb[L.oAZ + R.at(1)] = a0;
            sb[L.oAZ + R.at(2)] = a1;
            acc(R.at(0), zn, an);
            acc(R.at(1), z0, a0);
            acc(R.at(2), z1, a1);
          } else {
            const double dyn = me.dyn;
#pragma unroll
            for (int i = 0; i < 5; ++i) {
              if (i >= nr) break;
              const double zr = sb[L.oZ + R.at(i)];
              const double az = y[i] + dyn * zr;
              sb[L.oAZ + R.at(i)] = az;
              acc(R.at(i), zr, az);
            }
          }
        }
        CL_STAMP(5);
        if (L.dbg) {
          __syncthreads();
          CL_STAMP(12);
        }
        double tot[3];
        cl_cluster_sum3(L, S, part, rslot, scratch, tot);
        cl_xsum(L, grp, rank, xseq, tot, 3, scratch);
        rslot = (rslot + 3) & 15;
        CL_STAMP(6);
        if (k == 0) {
          rho = tot[0];
          beta = 0.0;
          den = tot[1];
        } else {
          beta = rho > 1e-300 ? tot[0] / rho : 0.0;
          rho = tot[0];
          den = tot[1] + 2.0 * beta * tot[2] + beta * beta * den;
        }
        if (den <= 1e-300 || !isfinite(den)) {
          broken = true;  // the reference skips every remaining iteration
          break;
        }
        alpha = rho / den;
        // p = z + beta p, ap = az + beta ap, x += alpha p, r -= alpha ap, z = r/d
#pragma unroll
        for (int j = 0; j < CL_RPT; ++j) {
          const int row = tid + j * CL_THREADS;
          if (row < L.NR) {
            const double pn = k == 0 ? sb[L.oZ + row] : sb[L.oZ + row] + beta * sb[L.oP + row];
            const double apn = k == 0 ? sb[L.oAZ + row] : sb[L.oAZ + row] + beta * sb[L.oAP + row];
            sb[L.oP + row] = pn;
            sb[L.oAP + row] = apn;
            xr_[j] += alpha * pn;
            rr_[j] -= alpha * apn;
            sb[L.oZ + row] = cl_ddiv<EXACT>(rr_[j], sb[L.oD + row]);
          }
        }
        __syncthreads();
        CL_STAMP(7);
        CL_STAMP(8);
      }
      stepped = true;
    } else {
    for (int k = 0; k < c.p.pcr; ++k) {
        CL_STAMP(0);
        if (k > 0 && !broken) {
          // x += alpha p, r -= alpha ap, z = r/d (row-parallel), then J^T z
  #pragma unroll
          for (int j = 0; j < CL_RPT; ++j) {
            const int row = tid + j * CL_THREADS;
            if (row < L.NR) {
              xr_[j] += alpha * sb[L.oP + row];
              rr_[j] -= alpha * sb[L.oAP + row];
              sb[L.oZ + row] = cl_ddiv<EXACT>(rr_[j], sb[L.oD + row]);
            }
          }
          __syncthreads();
          if (has_el) {
            const ClEl& el = me.el;
            const ClRows R = cl_rows(L, sb, el);
            double zr[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
  #pragma unroll
            for (int q = 0; q < 6; ++q) {
              if (q >= R.n) break;
              zr[q] = sb[L.oZ + R.at(q)];
            }
            cl_contrib<EXACT>(c, L, S, me, zr, 0);
          }
        }
        CL_STAMP(1);
        if (!(k > 0 && broken)) {
          cl.sync();                            // column sums of J^T z visible
          CL_STAMP(2);
          cl_gather(L, S, has_na, mn, 0);       // U = M^-1 J^T z (+ halo pushes)
          CL_STAMP(3);
          cl.sync();                            // U visible
          CL_STAMP(4);
        }
        // az = J u + dyn z + E z; rho = z.az (element-parallel)
        double part = 0.0;
        if (!broken && has_el) {
          const ClEl& el = me.el;
          const ClRows R = cl_rows(L, sb, el);
          const int nr = R.n;
          double y[6];
          if (nr) cl_forward<EXACT>(c, L, S, me, L.oU, y);
          if (!nr) {
          } else if (el.fam == CF_TET) {
            double zz[6], ez[6];
  #pragma unroll
            for (int i = 0; i < 6; ++i) zz[i] = sb[L.oZ + R.at(i)];
            ereg6(sb[L.oE3 + el.le], sb[L.oE3 + L.MT + el.le], sb[L.oE3 + 2 * L.MT + el.le], zz, ez);
  #pragma unroll
            for (int i = 0; i < 6; ++i) {
              const double az = y[i] + ez[i];
              sb[L.oAZ + R.at(i)] = az;
              part += zz[i] * az;
            }
          } else if (el.fam == CF_SLOT) {
            const int ls = el.le;
            const double zn = sb[L.oZ + R.at(0)], z0 = sb[L.oZ + R.at(1)], z1 = sb[L.oZ + R.at(2)];
            const double an = y[0] + sb[L.oDyn + ls] * zn;
            double a0 = z0, a1 = z1;
            if (sb[L.oAct + ls] != 0.0) {
              a0 = y[1] + c.p.fdyn * z0;
              a1 = y[2] + c.p.fdyn * z1;
            }
            sb[L.oAZ + R.at(0)] = an;
            sb[L.oAZ + R.at(1)] = a0;
            sb[L.oAZ + R.at(2)] = a1;
            part += zn * an;
            part += z0 * a0;
            part += z1 * a1;
          } else {
            const double dyn = me.dyn;
  #pragma unroll
            for (int i = 0; i < 5; ++i) {
              if (i >= nr) break;
              const double zr = sb[L.oZ + R.at(i)];
              const double az = y[i] + dyn * zr;
              sb[L.oAZ + R.at(i)] = az;
              part += zr * az;
            }
          }
        }
        CL_STAMP(5);
        double rho_new = cl_cluster_sum(L, S, part, rslot, scratch);
        cl_xsum(L, grp, rank, xseq, &rho_new, 1, scratch);
        rslot = (rslot + 1) & 15;
        CL_STAMP(6);
        if (!broken) {
          if (k == 0) {
            rho = rho_new;
          } else {
            beta = rho > 1e-300 ? rho_new / rho : 0.0;
            rho = rho_new;
          }
        }
        // p = z + beta p, ap = az + beta ap; den = ap.(ap/d) (row-parallel)
        double dpart = 0.0;
  #pragma unroll
        for (int j = 0; j < CL_RPT; ++j) {
          const int row = tid + j * CL_THREADS;
          if (row < L.NR) {
            double ap;
            if (k == 0) {
              sb[L.oP + row] = sb[L.oZ + row];
              ap = sb[L.oAZ + row];
              sb[L.oAP + row] = ap;
            } else if (!broken) {
              sb[L.oP + row] = sb[L.oZ + row] + beta * sb[L.oP + row];
              ap = sb[L.oAZ + row] + beta * sb[L.oAP + row];
              sb[L.oAP + row] = ap;
            } else {
              ap = sb[L.oAP + row];
            }
            dpart += ap * cl_ddiv<EXACT>(ap, sb[L.oD + row]);
          }
        }
        CL_STAMP(7);
        double den = cl_cluster_sum(L, S, dpart, rslot, scratch);
        cl_xsum(L, grp, rank, xseq, &den, 1, scratch);
        rslot = (rslot + 1) & 15;
        CL_STAMP(8);
        if (!broken) {
          if (den <= 1e-300 || !isfinite(den)) broken = true;
          else alpha = rho / den;
        }
      }
    }
    // ---- last PCR step (row-parallel): dl = x + alpha p -> AZ scratch, r.z
    double rzp = 0.0;
    const bool step = c.p.pcr > 0 && !broken && !stepped;
#pragma unroll
    for (int j = 0; j < CL_RPT; ++j) {
      const int row = tid + j * CL_THREADS;
      if (row < L.NR) {
        double x = xr_[j], r = rr_[j], z = sb[L.oZ + row];
        if (step) {
          x += alpha * sb[L.oP + row];
          r -= alpha * sb[L.oAP + row];
          z = cl_ddiv<EXACT>(r, sb[L.oD + row]);
        }
        rzp += r * z;
        sb[L.oAZ + row] = x;
      }
    }
    __syncthreads();
    // ---- multiplier update + projection + dlam column sums (element-parallel)
    if (has_el) {
      const ClEl& el = me.el;
      const ClRows R = cl_rows(L, sb, el);
      const int nr = R.n;
      double dlam[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
      if (el.fam != CF_SLOT) {
#pragma unroll
        for (int q = 0; q < 6; ++q) {
          if (q >= nr) break;
          const size_t gi = IX(cl_grow(c, el, q));
          const double l0 = c.S.lam[gi];
          const double l1 = l0 + sb[L.oAZ + R.at(q)];
          c.S.lam[gi] = l1;
          dlam[q] = l1 - l0;
        }
      } else {
        const int ls = el.le, s = el.g;
        double n1 = 0.0, a1 = 0.0, b1 = 0.0;
        if (nr) {
          const double n0 = sb[L.oLc + ls], a0 = sb[L.oLc + L.MS + ls], b0 = sb[L.oLc + 2 * L.MS + ls];
          n1 = n0 + sb[L.oAZ + R.at(0)];
          a1 = a0 + sb[L.oAZ + R.at(1)];
          b1 = b0 + sb[L.oAZ + R.at(2)];
          n1 = npmax(n1, 0.0);
          const double rad = c.p.mu * npmax(n1, 0.0);
          const double nrm = sqrt(a1 * a1 + b1 * b1);
          if (nrm > rad) {
            const double sc = nrm > 0.0 ? rad / nrm : 0.0;
            a1 *= sc;
            b1 *= sc;
          }
          sb[L.oLc + ls] = n1;
          sb[L.oLc + L.MS + ls] = a1;
          sb[L.oLc + 2 * L.MS + ls] = b1;
          dlam[0] = n1 - n0;
          dlam[1] = a1 - a0;
          dlam[2] = b1 - b0;
        }
        if (lastn) {
          const int ns = c.D.ns, nw = c.D.nw;
#pragma unroll
          for (int k = 0; k < 3; ++k) c.K.lamc[IX(k * ns + s)] = sb[L.oLc + k * L.MS + ls];
          if (s < nw) {
            c.S.warm_valid[IX(s)] = nr ? 1 : 0;
            c.S.warm[IX(s)] = n1;
            c.S.warm[IX(nw + s)] = a1;
            c.S.warm[IX(2 * nw + s)] = b1;
          }
        }
      }
      cl_contrib<EXACT>(c, L, S, me, dlam, 1);
    }
    double rz = cl_cluster_sum(L, S, rzp, rslot, scratch);
    cl_xsum(L, grp, rank, xseq, &rz, 1, scratch);
    rslot = (rslot + 1) & 15;
    resid = sqrt(0.0 > rz ? 0.0 : rz);
    // the reduction's cluster barrier also published the dlam column sums
    cl_gather(L, S, has_na, mn, 1);  // v += M^-1 J^T dlam (+ halo pushes)
    cl.sync();
  }

  // ---- write back
  for (int n = tid; n < nP + nB; n += CL_THREADS) {
    const int gn = L.node[(size_t)gcta * L.MN + n];
    if (n < nP) {
#pragma unroll
      for (int a = 0; a < 3; ++a) c.K.v[IX(3 * gn + a)] = sb[L.oV + 3 * n + a];
    } else {
      const int lb = n - nP, o = c.D.bd0 + 6 * (gn - c.D.P);
#pragma unroll
      for (int k = 0; k < 6; ++k) c.K.v[IX(o + k)] = sb[L.oV + 3 * nP + 6 * lb + k];
    }
  }
  if (gcta == 0 && tid == 0) c.S.resid[env] = resid;
  cl.sync();  // no CTA may exit while peers can still access its shared memory
}
