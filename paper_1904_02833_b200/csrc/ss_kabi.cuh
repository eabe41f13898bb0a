// ss_kabi.cuh — kernel-level ABI: one entry point per reference backend
// function (kernels/numba_backend.py) with the same argument meaning, on
// device pointers in the reference's AoS shapes. Used for per-kernel
// parity; the batched step uses the fused kernels of ss_device.cuh.
#pragma once
#include "ss_device.cuh"

// numba_backend.py:31-40 — one thread per (element, row)
__global__ void kk_block_forward(const int* idx, const double* vals, int n, int r, int k,
                                 const double* u, double* out) {
  const long g = blockIdx.x * (long)blockDim.x + threadIdx.x;
  if (g >= (long)n * r) return;
  const long e = g / r;
  double acc = 0.0;
  for (int j = 0; j < k; ++j) acc += vals[g * k + j] * u[idx[e * k + j]];
  out[g] = acc;
}

// numba_backend.py:43-52 — scatter-free: the (element, column) pairs are
// stably sorted by target DOF (ssk_block_transpose: CSR transpose, keys =
// dof_idx, values = e*k + j ascending), so one thread per DOF walks exactly
// its own entries in the serial scatter's order: bitwise the reference sum
// at O(n k) work instead of a full scan per DOF.
__device__ __forceinline__ long kk_lower_bound(const int* a, long n, int key) {
  long lo = 0, hi = n;
  while (lo < hi) {
    const long mid = (lo + hi) >> 1;
    if (a[mid] < key) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}
__global__ void kk_iota(int* v, long n) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x)
    v[i] = (int)i;
}
__global__ void kk_block_transpose(const int* skey, const int* sval, long nk, const double* vals,
                                   int r, int k, const double* x, double* y, int ndof) {
  const int d = blockIdx.x * blockDim.x + threadIdx.x;
  if (d >= ndof) return;
  const long b = kk_lower_bound(skey, nk, d), e_ = kk_lower_bound(skey, nk, d + 1);
  double acc_y = y[d];
  for (long s = b; s < e_; ++s) {
    const long ej = sval[s];
    const long e = ej / k;
    const int j = (int)(ej % k);
    double acc = 0.0;
    for (int i = 0; i < r; ++i) acc += vals[(e * r + i) * k + j] * x[e * r + i];
    acc_y += acc;
  }
  y[d] = acc_y;
}

// numba_backend.py:55-65
__global__ void kk_block_rowdiag(const int* idx, const double* vals, int n, int r, int k,
                                 const double* md, double* out) {
  const long g = blockIdx.x * (long)blockDim.x + threadIdx.x;
  if (g >= (long)n * r) return;
  const long e = g / r;
  double acc = 0.0;
  for (int j = 0; j < k; ++j) {
    const double v = vals[g * k + j];
    acc += v * v * md[idx[e * k + j]];
  }
  out[g] = acc;
}

// numba_backend.py:68-82
__global__ void kk_minv_apply(const double* md, const double* ang_inv, int nb, int bd0,
                              const double* u, double* out, int ndof) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= ndof) return;
  double o = md[i] * u[i];
  if (i >= bd0) {
    const int b = (i - bd0) / 6, k = (i - bd0) % 6;
    if (b < nb && k >= 3) {
      const int base = bd0 + 6 * b + 3;
      const double* A = ang_inv + 9 * b + 3 * (k - 3);
      o = A[0] * u[base] + A[1] * u[base + 1] + A[2] * u[base + 2];
    }
  }
  out[i] = o;
}

// numba_backend.py:85-94
__global__ void kk_ereg_apply(const double* v6, const double* x, double* out, int n) {
  const long g = blockIdx.x * (long)blockDim.x + threadIdx.x;
  if (g >= (long)n * 6) return;
  const long e = g / 6;
  const int i = g % 6;
  double acc = 0.0;
  for (int j = 0; j < 6; ++j) acc += v6[e * 36 + 6 * i + j] * x[e * 6 + j];
  out[g] = acc;
}

// numba_backend.py:97-102 — single block, fixed tree order
__global__ void kk_dot(const double* a, const double* b, int n, double* out) {
  __shared__ double red[256];
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s += a[i] * b[i];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[0] = red[0];
}

// numba_backend.py:105-120
__global__ void kk_eval_distance(const double* pos, const int* pairs, const double* rest,
                                 const double* scale, double* dirs, double* res, int n) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n) return;
  const int i = pairs[2 * e], j = pairs[2 * e + 1];
  const double dx = pos[3 * i] - pos[3 * j];
  const double dy = pos[3 * i + 1] - pos[3 * j + 1];
  const double dz = pos[3 * i + 2] - pos[3 * j + 2];
  const double ln = sqrt(dx * dx + dy * dy + dz * dz);
  if (ln > 1e-12) {
    dirs[3 * e] = dx / ln;
    dirs[3 * e + 1] = dy / ln;
    dirs[3 * e + 2] = dz / ln;
  }
  res[e] = ln - rest[e] * scale[e];
}

// numba_backend.py:137-312 — one thread per element; J written from the
// same tet_col() the batched solver recomputes with
__global__ void kk_eval_tetra(const double* pos, const int* tets, const double* rest_inv,
                              double* quats, double tol, int maxiter, double* out_res,
                              double* out_vals, int n, int* n_inv) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n) return;
  double X[12], Ri[9], q[4];
  for (int v = 0; v < 4; ++v) {
    const int node = tets[4 * e + v];
    for (int a = 0; a < 3; ++a) X[3 * v + a] = pos[3 * node + a];
  }
  for (int k = 0; k < 9; ++k) Ri[k] = rest_inv[9 * (long)e + k];
  for (int k = 0; k < 4; ++k) q[k] = quats[4 * (long)e + k];
  TetC T;
  const int inv = tet_eval_core(X, Ri, q, tol, maxiter, T, nullptr);
  for (int k = 0; k < 4; ++k) quats[4 * (long)e + k] = q[k];
  double r6[6];
  tet_res(T, r6);
  for (int i = 0; i < 6; ++i) out_res[6 * (long)e + i] = r6[i];
  for (int v = 0; v < 4; ++v) {
    double wv[3];
    tet_wv(Ri, v, wv);
    for (int a = 0; a < 3; ++a) {
      double col[6];
      tet_col(T, wv, a, col);
      for (int i = 0; i < 6; ++i) out_vals[72 * (long)e + 12 * i + 3 * v + a] = col[i];
    }
  }
  if (inv) atomicAdd(n_inv, 1);
}
