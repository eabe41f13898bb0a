// ss_api.cu — C ABI of libsoftsnake_b200.so (include/softsnake_b200.h).
//
// Host side: topology preprocessing (row layout, incidence lists in the
// reference accumulation order, compliance pattern), device memory, the
// per-frame launch sequence captured once into a CUDA graph, state I/O.
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <nvtx3/nvToolsExt.h>

#include <cub/device/device_radix_sort.cuh>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <functional>
#include <vector>

#include "../../include/softsnake_b200.h"
#include "ss_build.cuh"
#include "ss_cluster.cuh"
#include "ss_device.cuh"
#include "ss_kabi.cuh"

namespace {

thread_local std::string g_err;

// NVTX range for the duration of a scope (frames, waves, builder phases;
// inside a graph replay the kernels themselves carry no host ranges)
struct NvtxRange {
  bool on;
  explicit NvtxRange(const char* name, bool on_ = true) : on(on_) {
    if (on) nvtxRangePushA(name);
  }
  ~NvtxRange() {
    if (on) nvtxRangePop();
  }
};

int fail(int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define CK(call)                                                                    \
  do {                                                                              \
    cudaError_t e_ = (call);                                                        \
    if (e_ != cudaSuccess)                                                          \
      return fail(SS_ECUDA, "%s failed: %s", #call, cudaGetErrorString(e_));        \
  } while (0)

// Debug (SS_GUARD=1): every array is followed by a guard band filled with
// 0xA5 at creation; ss_check_guards reports bytes that changed (an
// out-of-bounds write past some array). compute-sanitizer is not available
// on the GPU pool, so this and SS_POISON (workspace filled with NaN bytes
// instead of zeros: a read-before-write shows up as a changed result) are
// the memcheck / initcheck stand-ins (tests/test_gpu_guard.py).
thread_local size_t g_guard = 0;
thread_local std::vector<std::pair<char*, size_t>>* g_spans = nullptr;

// bump allocator over one cudaMalloc
struct Arena {
  char* base = nullptr;
  size_t cap = 0, off = 0;
  template <typename T>
  T* take(size_t n) {
    const size_t data = n * sizeof(T);
    size_t bytes = ((data + 255) / 256) * 256;
    if (bytes == 0) bytes = 256;
    bytes += g_guard;
    T* p = reinterpret_cast<T*>(base ? base + off : nullptr);
    if (base && g_guard && g_spans) g_spans->push_back({base + off + data, bytes - data});
    off += bytes;
    return p;
  }
};

}  // namespace

struct GridCaps {
  long stream = 148 * 32;  // PCR step, tet J^T z, element kernels without reduction
  long eval = 148 * 8;     // per-substep eval / integrate kernels
  long reduce = 148 * 2;   // per-env reduction kernels: one resident wave
  long gather = 148 * 8;   // per-DOF gather: one resident wave
  long dir = 148 * 2;      // k_pcr_dir: its own resident wave (lighter than apply)
};
struct ss_handle {
  int device = 0;
  cudaStream_t stream = nullptr;
  Ctx c{};                 // wave 0 (shared dims, topology, workspace)
  // waves: persistent state of wave w lives in its own block; the workspace
  // is shared and the waves of a frame run back to back on the stream
  int n_waves = 1;
  std::vector<Ctx> wave;   // per-wave contexts (State pointers, real lanes)
  std::vector<std::vector<cudaGraphExec_t>> wave_graphs;  // [wave][key]
  int gy_red = 1;   // apply / final grid rows (partials per env)
  int gy_dir = 1;   // k_pcr_dir grid rows
  void* topo_mem = nullptr;
  void* state_mem = nullptr;
  void* work_mem = nullptr;
  size_t bytes = 0;
  double* d_cmd = nullptr;      // [n_real * links] (one frame)
  double* d_stage = nullptr;    // staging for state I/O
  size_t stage_bytes = 0;
  int launches = 0;
  // cluster-resident Newton solver (0 = streaming kernels)
  int use_cluster = 0;
  GridCaps caps;
  // item lanes per DOF in the J^T gather (1: serial walk in reference order;
  // 2/4/8: split walk for few env lanes, structured mode only; SS_GATHER_SPLIT)
  int gather_split = 1;
  // concurrent lanes: waves alternate between n_lanes workspaces / streams so
  // two waves' kernels overlap (SS_LANES=2)
  int n_lanes = 1;
  int n_work = 1;  // workspace blocks: n_lanes, or one per wave with keep_matrix
  static constexpr int kMaxLanes = 4;
  cudaStream_t lane_stream[kMaxLanes] = {nullptr, nullptr, nullptr, nullptr};
  cudaEvent_t ev_fork = nullptr, ev_join[kMaxLanes] = {nullptr, nullptr, nullptr, nullptr};
  int keep = 0;  // keep_matrix: snapshot the last Newton rhs each frame
  char* d_init = nullptr;  // reset template: one env's state, packed per field
  ClPlan plan{};
  void* plan_mem = nullptr;
  void* xmem = nullptr;     // cross-cluster reduction buffers (multi-cluster plans)
  // fused J^T z gather of the PCR loop (k_gather_fused; structured mode)
  int fused = 0;
  FusedPlan fplan{};
  void* fplan_mem = nullptr;
  size_t fused_smem = 0;
  int fused_chunks = 0;
  int apply_async = 0;       // k_apply_rows_async (cp.async-staged tet operands)
  int jtg_grid = 0;          // k_jtg persistent grid (resident CTAs)
  int pdl = 0;               // programmatic dependent launch of the frame kernels (SS_PDL)
  int apply2 = 0;            // k_apply_rows2 (tet split over two warps; SS_APPLY2)
  int gy_red2 = 1;           // its grid rows (one resident wave)
  int dir2 = 0;              // k_pcr_dir_rows (row-wise, SS_DIR2)
  int polar_split = 0;       // k_eval_polar before k_eval_tet (SS_POLAR_SPLIT)
  int polar_narrow = 0;      // one env, small mesh: 32-thread CTAs for k_eval_polar (SS_POLAR_NARROW)
  int stepjt = 0;            // k_step_jt (step + tet J^T z in one pass; SS_STEPJT)
  int newton2 = 0;           // k_newton_rhs2 / k_newton_final2 (SS_NEWTON2)
  int gy_dir2 = 1;
  int apply3 = 0;            // k_apply_rows3 (TMA-staged tet operands; SS_APPLY3)
  std::vector<TmApply> tm_apply;  // its tensor maps, per wave
  int gather_bulk = 0;       // k_gather_bulk (one large mesh: TMA bulk-copied tC; SS_GATHER_BULK)
  int gbulk_grid = 0;
  JtgPlan jplan{};           // k_jtg plan (fixed at ss_create)
  size_t apply_async_smem = 0;
  std::vector<std::pair<char*, size_t>> guards;  // SS_GUARD spans
};

namespace {

// ------------------------------------------------------------ launch grid
dim3 grid_items(const Dims& D, long n, long cap_blocks) {
  const long IL = SS_THREADS >> D.lgW;
  long gy = (n + IL - 1) / IL;
  if (gy < 1) gy = 1;
  long cap = cap_blocks / D.tiles;
  if (cap < 1) cap = 1;
  if (gy > cap) gy = cap;
  if (gy > 65535) gy = 65535;
  return dim3(D.tiles, (unsigned)gy);
}
// grid caps (CTAs of 256 threads); SS_STREAM_BLOCKS / SS_REDUCE_BLOCKS
// override them at ss_create for tuning
long env_long(const char* name, long dflt) {
  const char* v = getenv(name);
  return v && *v ? atol(v) : dflt;
}
// layout of the tet column sums tC: 0 tet-major ([nt][12][E] batched, [12][nt]
// few lanes), 1 one large mesh in incidence order (a 32-byte sector per
// incidence), 2 batched incidence order ([n_inc][3][E]: a DOF's tet run is
// consecutive env lines, gathered without code lookups). The opt-in
// experimental J^T kernels assume layout 0.
int tc_mode(const Dims& D) {
  if (D.E == 1 && env_long("SS_TC_INBOX", 1)) return 1;
  if (D.W == 32 && env_long("SS_TC_INBOX2", 1) && !env_long("SS_FUSED", 0) &&
      !env_long("SS_JTG", 0) && !env_long("SS_STEPJT", 0))
    return 2;
  return 0;
}

// Measured on the 1024-env snake (tools/grid_sweep.sh): the PCR row/element
// kernels gain from 16 CTAs per SM-slot of grid (more independent blocks in
// flight: k_pcr_step 49.3 -> 45.1 ms/frame), the reducing kernels from
// exactly one resident wave (no tail wave: k_apply_rows 37.8 -> 35.5), the
// gather and eval kernels are best at 8 per SM.
// occupancy-derived caps of this device; SS_*_BLOCKS override them
GridCaps grid_caps(int device) {
  GridCaps g;
  int sms = 148, occ_a = 2, occ_d = 2, occ_g = 4;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_a, k_apply_rows<false>, SS_THREADS, 0);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_d, k_pcr_dir<false>, SS_THREADS, 0);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_g, k_gather<1>, SS_THREADS, 0);
  g.stream = env_long("SS_STREAM_BLOCKS", 32L * sms);
  g.eval = env_long("SS_EVAL_BLOCKS", 8L * sms);
  g.reduce = env_long("SS_REDUCE_BLOCKS", (long)sms * std::max(1, occ_a));
  g.gather = env_long("SS_GATHER_BLOCKS", (long)sms * std::max(1, occ_g));
  g.dir = env_long("SS_DIR_BLOCKS", (long)sms * std::max(1, occ_d));
  return g;
}

// kernel names for the profiler (ss_profile_frames)
const char* const kKernelNames[] = {"k_frame_begin", "k_pre",        "k_slots",    "k_eval_tet",
                                    "k_eval_misc",   "k_gather",     "k_newton_rhs", "k_apply_rows",
                                    "k_pcr_dir",     "k_pcr_step",   "k_newton_final", "k_integrate",
                                    "k_tet_jt",      "k_newton_cluster", "k_gather_fused",
                                    "k_apply_rows_async", "k_jtg", "k_apply_rows2",
                                    "k_pcr_dir_rows", "k_eval_polar", "k_step_jt",
                                    "k_newton_rhs2", "k_newton_final2", "k_gather_bulk", "k_apply_rows3"};
constexpr int kNumKernels = 25;
struct Prof {
  std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> ev;
};
int kid(const char* name) {
  for (int i = 0; i < kNumKernels; ++i) {
    const size_t n = strlen(kKernelNames[i]);
    if (!strncmp(name, kKernelNames[i], n) && (name[n] == 0 || name[n] == '<')) return i;
  }
  return -1;
}

#define LAUNCH(kern, grid, ...) LAUNCH_SM(kern, grid, 0, __VA_ARGS__)
#define LAUNCH_SM(kern, grid, smem, ...)                                 \
  do {                                                                   \
    cudaEvent_t e0_ = nullptr, e1_ = nullptr;                            \
    if (prof) {                                                          \
      cudaEventCreate(&e0_);                                             \
      cudaEventCreate(&e1_);                                             \
      cudaEventRecord(e0_, st);                                          \
    }                                                                    \
    if (H->pdl) {                                                        \
      cudaLaunchConfig_t cfg_ = {};                                      \
      cudaLaunchAttribute at_[1];                                        \
      at_[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;    \
      at_[0].val.programmaticStreamSerializationAllowed = 1;             \
      cfg_.attrs = at_;                                                  \
      cfg_.numAttrs = 1;                                                 \
      cfg_.gridDim = grid;                                               \
      cfg_.blockDim = blk;                                               \
      cfg_.dynamicSmemBytes = smem;                                      \
      cfg_.stream = st;                                                  \
      CK(cudaLaunchKernelEx(&cfg_, kern, __VA_ARGS__));                  \
    } else {                                                             \
      kern<<<grid, blk, smem, st>>>(__VA_ARGS__);                        \
    }                                                                    \
    if (prof) {                                                          \
      cudaEventRecord(e1_, st);                                          \
      prof->ev.push_back({kid(#kern), {e0_, e1_}});                      \
    }                                                                    \
    ++n;                                                                 \
  } while (0)

// 3-D tensor map of a [K][nt][E] double field (env innermost) with
// {32 envs, 4 tets, K rows} boxes (k_apply_rows3)
static int make_tmap3(CUtensorMap* m, const double* base, int E, int nt, int K) {
  static PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  if (!enc) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        !fn)
      return -1;
    enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  cuuint64_t dims[3] = {(cuuint64_t)E, (cuuint64_t)nt, (cuuint64_t)K};
  cuuint64_t strides[2] = {(cuuint64_t)E * 8, (cuuint64_t)nt * E * 8};
  cuuint32_t box[3] = {32, 4, (cuuint32_t)K};
  cuuint32_t es[3] = {1, 1, 1};
  const CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(base), dims,
                         strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : -1;
}

// grid rows of k_apply_rows2 / k_newton_final2 and k_pcr_dir_rows: one
// resident wave at their occupancy (the partial buffer is sized for them)
static void set_gy2(ss_handle* H, const Dims& D) {
  int occ_a = 3, occ_d = 4, sms = 148;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_a, k_apply_rows2, SS_THREADS, 0);
  if (env_long("SS_APPLY3", 0)) {  // k_apply_rows3 shares the grid: its residency bounds it
    int occ_a3 = occ_a;
    cudaFuncSetAttribute(k_apply_rows3, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kA3Smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_a3, k_apply_rows3, SS_THREADS, kA3Smem);
    occ_a = std::min(occ_a, std::max(1, occ_a3));
  }
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_d, k_pcr_dir_rows, SS_THREADS, 0);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, H->device);
  const long rows_el = ((long)D.nd + D.nt + D.na + D.nh + D.ns + 3) / 4;  // tet pairs bound
  const long rows_m = ((long)D.m + 7) / 8;
  long a = std::max(1L, (long)sms * std::max(1, occ_a) / std::max(1, D.tiles));
  long d = std::max(1L, (long)sms * std::max(1, occ_d) / std::max(1, D.tiles));
  a = std::min(a, std::max(1L, rows_el));
  d = std::min(d, std::max(1L, rows_m));
  H->gy_red2 = (int)std::min(env_long("SS_APPLY2_GY", a), 65535L);
  H->gy_dir2 = (int)std::min(env_long("SS_DIR2_GY", d), 65535L);
}

// ------------------------------------------------------ k_jtg plan
static int jtg_ring_slots() { return (int)std::max(2L, env_long("SS_JTG_RING", 3)); }
static int jtg_lag() { return (int)std::max(1L, env_long("SS_JTG_LAG", 2)); }
static bool jtg_wanted(const ss_handle* H, const Dims& D) {
  // opt-in (SS_JTG=1): starved of ready work items at L2-sized rings — 1024 envs:
  // 76-171 ms/frame against 46.5 for k_tet_jt + k_gather (profiles/r2_summary.md)
  return env_long("SS_JTG", 0) && !H->c.p.exact_j && !H->use_cluster && D.nt > 0 &&
         D.E >= 64 && D.E % 32 == 0;
}
static JtgPlan jtg_plan(const Dims& D) {
  JtgPlan jp;
  jp.tiles = D.E / 32;
  jp.n1 = (D.nt + JTG_TETS - 1) / JTG_TETS;
  jp.n2 = (D.P + D.nb + JTG_NODES - 1) / JTG_NODES;
  jp.lag = std::min(jtg_lag(), jp.tiles);
  jp.ring = std::max(jtg_ring_slots(), jp.lag + 1);
  jp.n_items = jp.tiles * (jp.n1 + jp.n2);
  return jp;
}

// Enqueue one frame (Simulator.step, solver.py:296-314) on the stream.
// With prof, every launch is bracketed by CUDA events (eager, not graphed).
// EX: materialised-column tet Jacobian (bitwise numba sums) instead of the
// structured application (default).
template <bool EX>
int enqueue_frame_t(ss_handle* H, const Ctx& c, const double* d_cmd, int has_cmd, int latency,
                    int* nl, Prof* prof, const TmApply* tma) {
  const Dims& D = c.D;
  cudaStream_t st = H->stream;
  const dim3 blk(SS_THREADS);
  int n = 0;
  const long n_el = (long)D.nd + D.nt + D.na + D.nh + D.ns;
  const dim3 g_links = grid_items(D, D.links > 0 ? D.links : 1, H->caps.eval);
  const dim3 g_pre = grid_items(D, D.P + D.nb + D.nch, H->caps.eval);
  const dim3 g_slots = grid_items(D, D.ns, H->caps.eval);
  const dim3 g_eval = grid_items(D, D.nt, H->caps.eval);
  const dim3 g_polar = grid_items(D, D.nt, H->caps.stream);
  const dim3 g_tet = grid_items(D, D.nt, H->caps.stream);
  const dim3 g_misc = grid_items(D, D.nd + D.na + D.nh, H->caps.eval);
  int gsp = EX ? 1 : H->gather_split;  // the split walk changes the summation order
  if (gsp == 0) {
    const long lanes = H->caps.gather * (long)SS_THREADS;
    gsp = 4;
    while (gsp > 1 && (long)(D.P + D.nb) * gsp * D.E > lanes) gsp >>= 1;
  }
  while (gsp > 1 && gsp * D.W > 32) gsp >>= 1;  // a DOF's lanes stay in one warp
  const dim3 g_gather = grid_items(D, (long)(D.P + D.nb) * gsp, H->caps.gather);
  const dim3 g_el = grid_items(D, n_el, H->caps.stream);
  const dim3 g_red(D.tiles, H->gy_red);
  const dim3 g_red2(D.tiles, H->gy_red2);
  const dim3 g_dir2(D.tiles, H->gy_dir2);
  const dim3 g_dir(D.tiles, H->gy_dir);
  const dim3 g_int = grid_items(D, D.P + D.nb, H->caps.eval);
  const double* xs_lam = c.S.lam;
  const double* xc_lam = c.K.lamc;
  const double* xs_z = c.K.z;
  const double* xc_z = c.K.z + (size_t)D.ms * D.E;
  const double* xs_dl = c.K.az;
  const double* xc_dl = c.K.az + (size_t)D.ms * D.E;
  // tet column sums in incidence order (one large mesh): separate
  // instantiations of the kernels that write or read them
  const bool ib = D.tc_inbox == 1;
  const bool ib2 = D.tc_inbox == 2;
#define GATHER(mode, xs, xc)                                           \
  do {                                                                 \
    if (ib) {                                                          \
      if (gsp == 1 && H->gather_bulk)                                  \
        LAUNCH_SM(k_gather_bulk, dim3(H->gbulk_grid), kGbSmem, c, mode, xs, xc); \
      else if (gsp == 8) LAUNCH(k_gather<24>, g_gather, c, mode, xs, xc); \
      else if (gsp == 4) LAUNCH(k_gather<20>, g_gather, c, mode, xs, xc); \
      else if (gsp == 2) LAUNCH(k_gather<18>, g_gather, c, mode, xs, xc); \
      else LAUNCH(k_gather<17>, g_gather, c, mode, xs, xc);               \
    } else if (ib2) {                                                  \
      LAUNCH(k_gather<33>, g_gather, c, mode, xs, xc);                   \
    } else {                                                           \
      if (gsp == 8) LAUNCH(k_gather<8>, g_gather, c, mode, xs, xc);       \
      else if (gsp == 4) LAUNCH(k_gather<4>, g_gather, c, mode, xs, xc);  \
      else if (gsp == 2) LAUNCH(k_gather<2>, g_gather, c, mode, xs, xc);  \
      else LAUNCH(k_gather<1>, g_gather, c, mode, xs, xc);                \
    }                                                                  \
  } while (0)
  // has_cmd: 0 no commands, 1 commands in d_cmd, 2 on-device gait generator
  const int gait = has_cmd == 2 ? 1 : 0;
  LAUNCH(k_frame_begin, g_links, c, d_cmd, has_cmd == 1 ? 1 : 0, latency, gait);
  for (int sub = 0; sub < c.p.substeps; ++sub) {
    // NVTX groups (eager profiled frames): substep > assembly / newton > pcr
    NvtxRange nv_sub("substep", prof != nullptr);
    NvtxRange* nv_asm = new NvtxRange("assembly: pre, contacts, eval", prof != nullptr);
    LAUNCH(k_pre, g_pre, c, gait && sub == 0 ? 1 : 0);
    if (D.ns) LAUNCH(k_slots, g_slots, c);
    if (D.nt && H->polar_split) {
      if (H->polar_narrow) {
        // one env: one warp per CTA, so the data-dependent polar loops of a
        // small mesh spread over every SM instead of ~17 full CTAs
        const dim3 blk(32);
        LAUNCH(k_eval_polar, dim3(D.tiles, (D.nt + 31) / 32), c);
      } else {
        LAUNCH(k_eval_polar, g_polar, c);
      }
    }
    if (D.nt) LAUNCH(k_eval_tet<EX>, g_eval, c, H->polar_split);  // + tet J^T lam
    if (D.nd + D.na + D.nh) LAUNCH(k_eval_misc, g_misc, c);
    if (H->use_cluster) {
      // whole Newton loop, one environment per cluster (ss_cluster.cuh)
      cudaEvent_t e0_ = nullptr, e1_ = nullptr;
      if (prof) {
        cudaEventCreate(&e0_);
        cudaEventCreate(&e1_);
        cudaEventRecord(e0_, st);
      }
      cudaLaunchConfig_t cfg = {};
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = H->plan.C;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      cfg.blockDim = dim3(CL_THREADS);
      cfg.gridDim = dim3(H->plan.C * H->plan.G * D.E);
      cfg.dynamicSmemBytes = 8 * (size_t)H->plan.smem_doubles;
      cfg.stream = st;
      if (H->plan.G > 1)  // cross-cluster tagged words of this launch
        CK(cudaMemsetAsync(H->plan.xbuf, 0, (size_t)H->plan.xn * H->plan.G * kClXWords * 16, st));
      CK(cudaLaunchKernelEx(&cfg, k_newton_cluster<EX>, c, H->plan));
      if (prof) {
        cudaEventRecord(e1_, st);
        prof->ev.push_back({kid("k_newton_cluster"), {e0_, e1_}});
      }
      ++n;
      LAUNCH(k_integrate, g_int, c);
      delete nv_asm;
      continue;
    }
    GATHER(1, xs_lam, xc_lam);  // v = vt + M^-1 J^T lam
    delete nv_asm;
    nv_asm = nullptr;
    for (int it = 0; it < c.p.newton; ++it) {
      NvtxRange nv_newton("newton", prof != nullptr);
      if (!EX && H->newton2) {
        if (ib) LAUNCH(k_newton_rhs2<1>, g_el, c);
        else if (ib2) LAUNCH(k_newton_rhs2<2>, g_el, c);
        else LAUNCH(k_newton_rhs2<0>, g_el, c);
      }
      else LAUNCH(k_newton_rhs<EX>, g_el, c);  // + tet J^T z0
      if (H->keep && sub == c.p.substeps - 1 && it == c.p.newton - 1)
        CK(cudaMemcpyAsync(c.K.snap_rhs, c.K.r, 8 * (size_t)D.m * D.E, cudaMemcpyDeviceToDevice,
                           st));  // the snapshot's rhs (solver.py:515)
      if (c.p.pcr > 0) {
        NvtxRange nv_pcr("pcr_solve", prof != nullptr);
        GATHER(0, xs_z, xc_z);
#define DIR(setup_)                                                          \
  do {                                                                       \
    if (!EX && H->dir2)                                                      \
      LAUNCH(k_pcr_dir_rows, g_dir2, c, setup_);                             \
    else                                                                     \
      LAUNCH(k_pcr_dir<EX>, g_dir, c, setup_);                               \
  } while (0)
#define APPLY(setup_)                                                        \
  do {                                                                       \
    if (!EX && tma)                                                          \
      LAUNCH_SM(k_apply_rows3, g_red2, kA3Smem, c, setup_, *tma);            \
    else if (!EX && H->apply2)                                               \
      LAUNCH(k_apply_rows2, g_red2, c, setup_);                              \
    else if (!EX && H->apply_async)                                          \
      LAUNCH_SM(k_apply_rows_async, g_red, H->apply_async_smem, c, setup_);  \
    else                                                                     \
      LAUNCH(k_apply_rows<EX>, g_red, c, setup_);                            \
  } while (0)
        APPLY(1);
        DIR(1);
        for (int k = 0; k + 1 < c.p.pcr; ++k) {
          if (!EX && H->stepjt) {
            // step + tet column sums in one pass, then the DOF gather
            LAUNCH(k_step_jt, g_el, c, k);
            GATHER(0, xs_z, xc_z);
          } else {
          LAUNCH(k_pcr_step<EX>, g_el, c, k);
          if (!EX && H->fused) {
            const dim3 g_fu(D.E / H->fplan.FW, H->fplan.n_blocks + 1);
            const size_t sm = H->fused_smem;
            switch (H->fplan.FW) {
              case 1: LAUNCH_SM(k_gather_fused<1>, g_fu, sm, c, H->fplan); break;
              case 2: LAUNCH_SM(k_gather_fused<2>, g_fu, sm, c, H->fplan); break;
              case 4: LAUNCH_SM(k_gather_fused<4>, g_fu, sm, c, H->fplan); break;
              default: LAUNCH_SM(k_gather_fused<8>, g_fu, sm, c, H->fplan); break;
            }
          } else if (!EX && c.K.ring) {
            // persistent tile-pipelined J^T gather (k_jtg): counters reset first
            const JtgPlan& jp = H->jplan;
            CK(cudaMemsetAsync(c.K.jctr, 0, sizeof(int) * (1 + 2 * (size_t)jp.tiles), st));
            LAUNCH(k_jtg, dim3(H->jtg_grid), c, jp);
          } else {
            if (D.nt && ib) LAUNCH(k_tet_jt<EX ? 3 : 2>, g_tet, c);
            else if (D.nt && ib2) LAUNCH(k_tet_jt<EX ? 5 : 4>, g_tet, c);
            else if (D.nt) LAUNCH(k_tet_jt<EX ? 1 : 0>, g_tet, c);
            GATHER(0, xs_z, xc_z);
          }
          }
          APPLY(0);
          DIR(0);
        }
      }
      if (!EX && H->newton2 && ib)
        LAUNCH(k_newton_final2<1>, g_red2, c, c.p.pcr > 0 ? 1 : 0, it == c.p.newton - 1 ? 1 : 0,
               c.p.pcr == 1 ? 1 : 0);
      else if (!EX && H->newton2 && ib2)
        LAUNCH(k_newton_final2<2>, g_red2, c, c.p.pcr > 0 ? 1 : 0, it == c.p.newton - 1 ? 1 : 0,
               c.p.pcr == 1 ? 1 : 0);
      else if (!EX && H->newton2)
        LAUNCH(k_newton_final2<0>, g_red2, c, c.p.pcr > 0 ? 1 : 0, it == c.p.newton - 1 ? 1 : 0,
               c.p.pcr == 1 ? 1 : 0);
      else
        LAUNCH(k_newton_final<EX>, g_red, c, c.p.pcr > 0 ? 1 : 0, it == c.p.newton - 1 ? 1 : 0,
               c.p.pcr == 1 ? 1 : 0);
      GATHER(1, xs_dl, xc_dl);  // v += M^-1 J^T dlam
    }
    LAUNCH(k_integrate, g_int, c);
  }
  if (nl) *nl = n;
  CK(cudaGetLastError());
  return SS_OK;
}
#undef LAUNCH
#undef LAUNCH_SM
#undef APPLY
#undef DIR

int enqueue_frame(ss_handle* H, int w, int has_cmd, int latency, int* nl, Prof* prof = nullptr) {
  const Ctx& c = H->wave[w];
  const double* d_cmd = H->d_cmd + (size_t)w * H->c.D.E * std::max(1, H->c.D.links);
  const TmApply* tma = H->apply3 ? &H->tm_apply[w] : nullptr;
  return H->c.p.exact_j ? enqueue_frame_t<true>(H, c, d_cmd, has_cmd, latency, nl, prof, tma)
                        : enqueue_frame_t<false>(H, c, d_cmd, has_cmd, latency, nl, prof, tma);
}

int get_graph(ss_handle* H, int w, int has_cmd, int latency, cudaGraphExec_t* out) {
  const int key = 2 * has_cmd + (latency ? 1 : 0);
  cudaGraphExec_t& slot = H->wave_graphs[w][key];
  if (slot) {
    *out = slot;
    return SS_OK;
  }
  cudaGraph_t g;
  CK(cudaStreamBeginCapture(H->stream, cudaStreamCaptureModeThreadLocal));
  int nl = 0;
  int rc = enqueue_frame(H, w, has_cmd, latency, &nl);
  cudaError_t e = cudaStreamEndCapture(H->stream, &g);
  if (rc) return rc;
  if (e != cudaSuccess) return fail(SS_ECUDA, "graph capture failed: %s", cudaGetErrorString(e));
  CK(cudaGraphInstantiate(&slot, g, 0));
  CK(cudaGraphDestroy(g));
  H->launches = nl;
  *out = slot;
  return SS_OK;
}

// state field table: (device base, A, B, swap, is_int)
struct Field {
  void* dev;
  int A, B, swap, is_int;
  void* host;
};

void state_fields(ss_handle* H, int w, const ss_state_view* v, Field* f, int* nf) {
  const Dims& D = H->c.D;
  const State& S = H->wave[w].S;
  const size_t E = D.E;
  int k = 0;
  auto add = [&](void* dev, int A, int B, int swap, int is_int, void* host) {
    f[k++] = Field{dev, A, B, swap, is_int, host};
  };
  add(S.pos, D.P, 3, 0, 0, v->positions);
  add(S.vel, D.P, 3, 0, 0, v->velocities);
  add(S.bpos, D.nb, 3, 0, 0, v->body_pos);
  add(S.bquat, D.nb, 4, 0, 0, v->body_quat);
  add(S.blin, D.nb, 3, 0, 0, v->body_lin_vel);
  add(S.bang, D.nb, 3, 0, 0, v->body_ang_vel);
  add(S.lam + (size_t)D.od * E, D.nd, 1, 0, 0, v->lam_dist);
  add(S.lam + (size_t)D.ot * E, D.nt, 6, 1, 0, v->lam_tetra);
  add(S.lam + (size_t)D.oa * E, D.na, 3, 1, 0, v->lam_attach);
  add(S.lam + (size_t)D.oh * E, D.nh, 5, 1, 0, v->lam_hinge);
  add(S.quat, D.nt, 4, 1, 0, v->tet_quats);
  add(S.dirs, D.nd, 3, 1, 0, v->dist_dirs);
  add(S.scale, D.nd, 1, 0, 0, v->dist_scale);
  add(S.live, D.nch, 1, 0, 0, v->strain_live);
  add(S.target, D.nch, 1, 0, 0, v->strain_target);
  add(S.press, D.nch, 1, 0, 0, v->pressures);
  add(S.warm, D.nw, 3, 1, 0, v->warm);
  add(S.warm_valid, D.nw, 1, 0, 1, v->warm_valid);
  add(S.time, 1, 1, 0, 0, v->time);
  *nf = k;
}

__global__ void k_fill(double* p, size_t n, double val) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x)
    p[i] = val;
}

}  // namespace

// ------------------------------------------------------ fused gather plan
// Particle blocks for k_gather_fused: runs of consecutive particles of one
// tet-connected component (a snake link), split evenly when a run exceeds
// the shared-memory budget or when too few CTAs would run. Per block, the
// elements touching it are packed greedily (ascending id) into chunks of at
// most FIL elements with no particle of the block twice in a chunk, family
// by family in the reference's accumulation order (solver.py:354-367).
static int plan_fused(ss_handle* H, const Dims& D, const int* tets, const std::vector<int>& d_i,
                      const std::vector<int>& d_j, const std::vector<int>& a_p,
                      const std::vector<int>& slot_part) {
  // off by default: bitwise-different order and latency-bound (r2 measurements:
  // 42-47 ms/frame vs 46.7 for k_tet_jt + k_gather at 1024 envs)
  const long mode = env_long("SS_FUSED", 0);  // -1 auto, 0 off, 1 on
  H->fused = 0;
  if (mode == 0 || D.nt == 0 || H->c.p.exact_j || H->use_cluster) return SS_OK;
  const int FW = (int)std::min<long>(env_long("SS_FUSED_W", 8), D.E);
  if (FW != 1 && FW != 2 && FW != 4 && FW != 8) return fail(SS_EINVAL, "SS_FUSED_W must be 1/2/4/8");
  if (mode < 0 && D.E < 8) return SS_OK;  // few env lanes: the split gather / cluster plans
  const int FIL = SS_THREADS / FW;
  const int tiles_f = D.E / FW;
  const long smem_cap = env_long("SS_FUSED_SMEM", 72 * 1024);
  const int nb_cap = (int)(smem_cap / 8 / FW / 3);
  if (nb_cap < 16) return SS_OK;
  // components of the tet graph (union-find)
  std::vector<int> par(D.P);
  for (int i = 0; i < D.P; ++i) par[i] = i;
  auto root = [&](int x) {
    while (par[x] != x) x = par[x] = par[par[x]];
    return x;
  };
  for (int t = 0; t < D.nt; ++t)
    for (int v = 1; v < 4; ++v) {
      const int ra = root(tets[4 * (size_t)t]), rb = root(tets[4 * (size_t)t + v]);
      if (ra != rb) par[std::max(ra, rb)] = std::min(ra, rb);
    }
  const int want_blocks = (148 + tiles_f - 1) / tiles_f;
  const int nb_target = std::max(16, (D.P + want_blocks - 1) / want_blocks);
  std::vector<int> bp0, bnp;
  for (int p = 0; p < D.P;) {
    int q = p + 1;
    const int r = root(p);
    while (q < D.P && root(q) == r) ++q;
    const int len = q - p;
    const int lim = std::min(nb_cap, std::max(nb_target, std::min(len, nb_cap)));
    const int parts = (len + lim - 1) / lim;
    for (int k = 0; k < parts; ++k) {
      const int x0 = p + (int)((long)len * k / parts), x1 = p + (int)((long)len * (k + 1) / parts);
      bp0.push_back(x0);
      bnp.push_back(x1 - x0);
    }
    p = q;
  }
  const int nbk = (int)bp0.size();
  int nb_max = 0;
  for (int x : bnp) nb_max = std::max(nb_max, x);
  std::vector<int> blk_of(D.P);
  for (int b = 0; b < nbk; ++b)
    for (int n = 0; n < bnp[b]; ++n) blk_of[bp0[b] + n] = b;
  // per block, per family: the elements touching it (ascending) and their particles
  struct Elem { int e; int nodes[4]; };
  std::vector<std::vector<Elem>> fam_el[4];  // dist, tet, attach, contact slot
  for (auto& f : fam_el) f.assign(nbk, {});
  auto add = [&](int f, int e, std::initializer_list<int> nodes) {
    Elem el{e, {-1, -1, -1, -1}};
    int k = 0;
    for (int n : nodes) el.nodes[k++] = n;
    int seen[4] = {-1, -1, -1, -1}, ns_ = 0;
    for (int n : nodes) {
      const int b = blk_of[n];
      bool dup = false;
      for (int j = 0; j < ns_; ++j) dup |= seen[j] == b;
      if (dup) continue;
      seen[ns_++] = b;
      fam_el[f][b].push_back(el);
    }
  };
  for (int e = 0; e < D.nd; ++e) add(0, e, {d_i[e], d_j[e]});
  for (int e = 0; e < D.nt; ++e)
    add(1, e, {tets[4 * (size_t)e], tets[4 * (size_t)e + 1], tets[4 * (size_t)e + 2], tets[4 * (size_t)e + 3]});
  for (int e = 0; e < D.na; ++e) add(2, e, {a_p[e]});
  // a particle contact slot adds its normal row, then its friction rows
  // (one element: the reference's CN-before-CF order per particle)
  for (int s = D.nw; s < D.ns; ++s) add(3, s, {slot_part[s - D.nw]});
  const int fam_code[4] = {F_DIST, F_TET, F_ATTP, F_CN};
  std::vector<int> cptr(1, 0), hdr, start, elist;
  std::vector<int2> enode;
  int sched_max = 0;
  std::vector<int> deg(D.P, 0);
  for (int b = 0; b < nbk; ++b) {
    const int el_b0 = (int)elist.size();
    for (int f = 0; f < 4; ++f) {
      // conflict-free packing into as few, as even chunks as possible: the
      // elements on the most-shared particles first, each into the smallest
      // open chunk it does not conflict with (at least max-degree chunks)
      const auto& els = fam_el[f][b];
      for (const Elem& el : els)
        for (int n : el.nodes)
          if (n >= 0) ++deg[n];
      int kmin = (int)((els.size() + FIL - 1) / FIL);
      for (const Elem& el : els)
        for (int n : el.nodes)
          if (n >= 0 && blk_of[n] == b) kmin = std::max(kmin, deg[n]);
      std::vector<int> order(els.size());
      std::vector<long> key(els.size(), 0);
      for (size_t i = 0; i < els.size(); ++i) {
        order[i] = (int)i;
        for (int n : els[i].nodes)
          if (n >= 0 && blk_of[n] == b) key[i] += deg[n];
      }
      std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return key[x] > key[y]; });
      std::vector<std::vector<int>> chunks(kmin);
      std::vector<std::vector<char>> used(kmin, std::vector<char>(bnp[b], 0));
      for (int i : order) {
        const Elem& el = els[i];
        int best = -1;
        for (size_t k = 0; k < chunks.size(); ++k) {
          if ((int)chunks[k].size() >= FIL) continue;
          bool ok = true;
          for (int n : el.nodes)
            if (n >= 0 && blk_of[n] == b && used[k][n - bp0[b]]) ok = false;
          if (ok && (best < 0 || chunks[k].size() < chunks[best].size())) best = (int)k;
        }
        if (best < 0) {
          best = (int)chunks.size();
          chunks.emplace_back();
          used.emplace_back(bnp[b], 0);
        }
        chunks[best].push_back(i);
        for (int n : el.nodes)
          if (n >= 0 && blk_of[n] == b) used[best][n - bp0[b]] = 1;
      }
      for (const Elem& el : els)
        for (int n : el.nodes)
          if (n >= 0) deg[n] = 0;
      for (auto& ck : chunks) std::sort(ck.begin(), ck.end());
      for (auto& ck : chunks) {
        if (ck.empty()) continue;
        hdr.push_back((fam_code[f] << 24) | (int)ck.size());
        start.push_back((int)elist.size());
        for (int i : ck) {
          // the element's particles in this block, block-local (0xFFFF: outside)
          const Elem* el = &els[i];
          const int e = el->e;
          unsigned q[4];
          for (int j = 0; j < 4; ++j) {
            const int n = el->nodes[j];
            q[j] = (n >= 0 && blk_of[n] == b) ? (unsigned)(n - bp0[b]) : 0xFFFFu;
          }
          elist.push_back(e);
          enode.push_back(make_int2((int)(q[0] | (q[1] << 16)), (int)(q[2] | (q[3] << 16))));
        }
      }
    }
    cptr.push_back((int)hdr.size());
    sched_max = std::max(sched_max, 2 * (cptr[b + 1] - cptr[b]) + 3 * ((int)elist.size() - el_b0));
  }
  start.push_back((int)elist.size());  // [n_chunks + 1] starts
  std::vector<int> chk(hdr);
  chk.insert(chk.end(), start.begin(), start.end());
  // device copy
  std::vector<int> enode_i(2 * enode.size());
  for (size_t i = 0; i < enode.size(); ++i) {
    enode_i[2 * i] = enode[i].x;
    enode_i[2 * i + 1] = enode[i].y;
  }
  std::vector<int>* arrs[] = {&bp0, &bnp, &cptr, &chk, &elist, &enode_i};
  size_t bytes = 0;
  for (auto* x : arrs) bytes += ((4 * std::max<size_t>(x->size(), 1) + 255) / 256) * 256;
  CK(cudaMalloc(&H->fplan_mem, bytes));
  const int* dp[6];
  {
    char* q = (char*)H->fplan_mem;
    for (int i = 0; i < 6; ++i) {
      dp[i] = (const int*)q;
      if (!arrs[i]->empty())
        CK(cudaMemcpy(q, arrs[i]->data(), 4 * arrs[i]->size(), cudaMemcpyHostToDevice));
      q += ((4 * std::max<size_t>(arrs[i]->size(), 1) + 255) / 256) * 256;
    }
  }
  FusedPlan& F = H->fplan;
  F.n_blocks = nbk;
  F.FW = FW;
  F.FIL = FIL;
  F.nb_max = nb_max;
  F.blk_p0 = dp[0];
  F.blk_np = dp[1];
  F.blk_cptr = dp[2];
  F.chk = dp[3];
  F.elist = dp[4];
  F.enode = reinterpret_cast<const int2*>(dp[5]);
  F.sched_max = sched_max;
  H->fused_smem = 8 * (size_t)nb_max * 3 * FW + 4 * (size_t)sched_max;
  if (H->fused_smem > 200 * 1024) return SS_OK;  // schedule too large for shared memory: unfused
  H->fused_chunks = (int)hdr.size();
  cudaError_t e = cudaSuccess;
  switch (FW) {
    case 1: e = cudaFuncSetAttribute(k_gather_fused<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)H->fused_smem); break;
    case 2: e = cudaFuncSetAttribute(k_gather_fused<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)H->fused_smem); break;
    case 4: e = cudaFuncSetAttribute(k_gather_fused<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)H->fused_smem); break;
    default: e = cudaFuncSetAttribute(k_gather_fused<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)H->fused_smem); break;
  }
  if (e != cudaSuccess) return fail(SS_ECUDA, "fused gather smem attribute: %s", cudaGetErrorString(e));
  H->fused = 1;
  return SS_OK;
}

// ------------------------------------------------------ cluster plan
// Partition of one environment over the C CTAs of a cluster (contiguous tet
// ranges = mesh slabs; every other element follows its first node). Each
// CTA gets: its element list, the local U/V layout (owned DOFs, then halo
// copies of the foreign nodes its elements touch), an inbox slot per
// incidence of every owned node in the reference accumulation order (the
// same sorted incidence lists as the streaming path), the inbox destination
// of every column block its elements produce, and the halo push lists.
struct PlanBuild {
  int C;
  std::vector<int> own_t, own_d, own_a, own_h, own_s, own_p, own_b;  // owner CTA
  std::vector<int> loc_t, loc_d, loc_a, loc_h, loc_s, loc_p, loc_b;  // family-local index
  std::vector<std::vector<int>> Lt, Ld, La, Lh, Ls, Lp, Lb;          // per CTA lists
  std::vector<std::vector<int>> halo;  // per CTA: halo nodes (global node id: p or P+b)
  std::vector<int> in_size;            // per CTA inbox doubles
  ClPlan P;
  size_t smem_bytes;
};

// comp (optional, multi-cluster plans): the connected component of every
// node (particles, then P + body), G groups of C CTAs, group k owning
// component k; without it one group of C CTAs owns the whole scene.
static void plan_partition(PlanBuild& B, const Dims& D, const std::vector<int>& d_i,
                           const std::vector<int>& d_j, const std::vector<int>& tets,
                           const std::vector<int>& a_p, const std::vector<int>& a_b,
                           const std::vector<int>& h_a, const std::vector<int>& h_b,
                           const std::vector<int>& w_body, const std::vector<int>& slot_part,
                           const std::vector<int>& inc_ptr_g,
                           const std::vector<int>* comp = nullptr, int G = 1) {
  const int Cg = B.C / G;  // CTAs per group (cluster)
  const int C = B.C;
  B.own_t.assign(D.nt, 0);
  if (!comp) {
    for (int t = 0; t < D.nt; ++t) B.own_t[t] = (int)((long)t * C / std::max(D.nt, 1));
  } else {
    // contiguous tet ranges within each component
    std::vector<int> n_k(G, 0), j_k(G, 0);
    for (int t = 0; t < D.nt; ++t) ++n_k[(*comp)[tets[4 * (size_t)t]]];
    for (int t = 0; t < D.nt; ++t) {
      const int k = (*comp)[tets[4 * (size_t)t]];
      B.own_t[t] = k * Cg + (int)((long)j_k[k]++ * Cg / std::max(n_k[k], 1));
    }
  }
  B.own_p.assign(D.P, -1);
  for (int t = 0; t < D.nt; ++t)
    for (int v = 0; v < 4; ++v) {
      const int p = tets[4 * (size_t)t + v];
      if (B.own_p[p] < 0) B.own_p[p] = B.own_t[t];
    }
  for (int p = 0; p < D.P; ++p)
    if (B.own_p[p] < 0)
      B.own_p[p] = comp ? (*comp)[p] * Cg : (int)((long)p * C / std::max(D.P, 1));
  B.own_b.assign(D.nb, -1);
  for (int a = 0; a < D.na; ++a)
    if (B.own_b[a_b[a]] < 0) B.own_b[a_b[a]] = B.own_p[a_p[a]];
  for (int pass = 0; pass < 2; ++pass)
    for (int h = 0; h < D.nh; ++h) {
      if (B.own_b[h_a[h]] < 0 && B.own_b[h_b[h]] >= 0) B.own_b[h_a[h]] = B.own_b[h_b[h]];
      if (B.own_b[h_b[h]] < 0 && B.own_b[h_a[h]] >= 0) B.own_b[h_b[h]] = B.own_b[h_a[h]];
    }
  for (int b = 0; b < D.nb; ++b)
    if (B.own_b[b] < 0) B.own_b[b] = comp ? (*comp)[D.P + b] * Cg : b % C;
  B.own_d.resize(D.nd);
  for (int d = 0; d < D.nd; ++d) B.own_d[d] = B.own_p[d_i[d]];
  B.own_a.resize(D.na);
  for (int a = 0; a < D.na; ++a) B.own_a[a] = B.own_p[a_p[a]];
  B.own_h.resize(D.nh);
  for (int h = 0; h < D.nh; ++h) B.own_h[h] = B.own_b[h_a[h]];
  B.own_s.resize(D.ns);
  for (int s = 0; s < D.ns; ++s)
    B.own_s[s] = s < D.nw ? B.own_b[w_body[s]] : B.own_p[slot_part[s - D.nw]];
  auto lists = [&](const std::vector<int>& own, std::vector<std::vector<int>>& Lx,
                   std::vector<int>& loc) {
    Lx.assign(C, {});
    loc.assign(own.size(), 0);
    for (size_t i = 0; i < own.size(); ++i) {
      loc[i] = (int)Lx[own[i]].size();
      Lx[own[i]].push_back((int)i);
    }
  };
  lists(B.own_t, B.Lt, B.loc_t);
  lists(B.own_d, B.Ld, B.loc_d);
  lists(B.own_a, B.La, B.loc_a);
  lists(B.own_h, B.Lh, B.loc_h);
  lists(B.own_s, B.Ls, B.loc_s);
  lists(B.own_p, B.Lp, B.loc_p);
  lists(B.own_b, B.Lb, B.loc_b);
  // halo nodes: foreign nodes touched by local elements (sorted, unique)
  B.halo.assign(C, {});
  auto own_of = [&](int gn) { return gn < D.P ? B.own_p[gn] : B.own_b[gn - D.P]; };
  for (int c = 0; c < C; ++c) {
    std::vector<int> h;
    auto need = [&](int gn) { if (own_of(gn) != c) h.push_back(gn); };
    for (int t : B.Lt[c])
      for (int v = 0; v < 4; ++v) need(tets[4 * (size_t)t + v]);
    for (int d : B.Ld[c]) { need(d_i[d]); need(d_j[d]); }
    for (int a : B.La[c]) { need(a_p[a]); need(D.P + a_b[a]); }
    for (int x : B.Lh[c]) { need(D.P + h_a[x]); need(D.P + h_b[x]); }
    for (int s : B.Ls[c]) {
      if (s < D.nw) need(D.P + w_body[s]);
      else {
        // the padded columns reference DOF 0 with zero values (contact.py:210-214):
        // read from its owner's shared memory at apply time (plan_upload), not
        // pushed to every CTA as a halo copy (the owner's gather would push it
        // to every other CTA of the cluster each PCR iteration)
        need(slot_part[s - D.nw]);
      }
    }
    std::sort(h.begin(), h.end());
    h.erase(std::unique(h.begin(), h.end()), h.end());
    B.halo[c] = h;
  }
  B.in_size.assign(C, 0);
  for (int c = 0; c < C; ++c) {
    int sz = 0;
    for (int p : B.Lp[c]) sz += 3 * (inc_ptr_g[p + 1] - inc_ptr_g[p]);
    for (int b : B.Lb[c]) sz += 6 * (inc_ptr_g[D.P + b + 1] - inc_ptr_g[D.P + b]);
    B.in_size[c] = sz;
  }
  auto mx = [&](const std::vector<std::vector<int>>& Lx) {
    size_t m = 1;
    for (auto& v : Lx) m = std::max(m, v.size());
    return (int)m;
  };
  ClPlan& P = B.P;
  P = ClPlan{};
  P.C = Cg;
  P.G = G;
  P.MT = mx(B.Lt); P.MD = mx(B.Ld); P.MA = mx(B.La); P.MH = mx(B.Lh); P.MS = mx(B.Ls);
  P.MP = mx(B.Lp); P.MB = mx(B.Lb);
  P.MW = 1;
  for (auto& v : B.Ls) {
    int w = 0;
    for (int s : v) w += s < D.nw ? 1 : 0;
    P.MW = std::max(P.MW, w);
  }
  P.NR = 6 * P.MT + P.MD + 3 * P.MA + 5 * P.MH + 3 * P.MS;
  P.ME = P.MT + P.MD + P.MA + P.MH + P.MS;
  P.MN = P.MP + P.MB;
  P.MDOFX = 1;
  for (int c = 0; c < C; ++c) {
    int n = 3 * (int)B.Lp[c].size() + 6 * (int)B.Lb[c].size();
    for (int gn : B.halo[c]) n += gn < D.P ? 3 : 6;
    P.MDOFX = std::max(P.MDOFX, n);
  }
  P.MIN = 2;
  for (int v : B.in_size) P.MIN = std::max(P.MIN, v);
  int off = 0;
  auto take = [&](int n) { const int o = off; off += (n + 1) & ~1; return o; };
  P.oZ = take(P.NR); P.oP = take(P.NR);
  P.oAP = take(P.NR); P.oAZ = take(P.NR); P.oD = take(P.NR);
  P.oJR = take(9 * P.MT); P.oJS = take(6 * P.MT); P.oJK = take(6 * P.MT);
  P.oRi = take(9 * P.MT); P.oE3 = take(3 * P.MT);
  P.oIn = take(P.MIN);
  P.oDir = take(3 * P.MD); P.oRw = take(3 * P.MA); P.oHJ = take(60 * P.MH);
  P.oWJ = take(18 * P.MW);
  P.oPres = take(P.MS); P.oGap = take(P.MS); P.oLc = take(3 * P.MS); P.oAct = take(P.MS);
  P.oDyn = take(P.MS); P.oBdn = take(P.MS); P.oBdf = take(2 * P.MS);
  P.oResD = take(P.MD); P.oResA = take(3 * P.MA); P.oResH = take(5 * P.MH);
  P.oU = take(P.MDOFX); P.oV = take(P.MDOFX); P.oAng = take(9 * P.MB);
  P.oRed = take(32 * Cg);  // [16 slots][C][value, tag]
  P.smem_doubles = off;
  B.smem_bytes = 8 * (size_t)off;
}

// device tables of a partition
static int plan_upload(ss_handle* H, PlanBuild& B, const Dims& D, const std::vector<int>& d_i,
                       const std::vector<int>& d_j, const std::vector<int>& tets,
                       const std::vector<int>& a_p, const std::vector<int>& a_b,
                       const std::vector<int>& h_a, const std::vector<int>& h_b,
                       const std::vector<int>& w_body, const std::vector<int>& slot_part,
                       const std::vector<int>& inc_ptr_g, const std::vector<int>& inc_g) {
  ClPlan& P = B.P;
  const int C = B.C;       // CTAs over all groups
  const int Cg = P.C;      // CTAs per group (cluster): DSMEM ranks
  auto own_of = [&](int gn) { return gn < D.P ? B.own_p[gn] : B.own_b[gn - D.P]; };
  // local U/V offset of a global node in CTA c (owned or halo)
  std::vector<std::vector<int>> halo_off(C);
  for (int c = 0; c < C; ++c) {
    int o = 3 * (int)B.Lp[c].size() + 6 * (int)B.Lb[c].size();
    for (int gn : B.halo[c]) {
      halo_off[c].push_back(o);
      o += gn < D.P ? 3 : 6;
    }
  }
  auto local_off = [&](int c, int gn) -> int {
    if (own_of(gn) == c) {
      if (gn < D.P) return 3 * B.loc_p[gn];
      return 3 * (int)B.Lp[c].size() + 6 * B.loc_b[gn - D.P];
    }
    const auto& h = B.halo[c];
    const size_t i = std::lower_bound(h.begin(), h.end(), gn) - h.begin();
    return halo_off[c][i];
  };
  // inbox destinations of every (family, element, vertex) incidence
  std::vector<int> dst_t(4 * (size_t)D.nt), dst_d(2 * (size_t)D.nd), dst_ap(D.na), dst_ab(D.na),
      dst_h(2 * (size_t)D.nh), dst_cn(D.ns), dst_cf(D.ns);
  std::vector<int> in_ptr((size_t)C * (P.MN + 1), 0), node((size_t)C * P.MN, 0);
  for (int c = 0; c < C; ++c) {
    int o = 0, n = 0;
    auto walk = [&](int gn) {
      in_ptr[(size_t)c * (P.MN + 1) + n] = o;
      node[(size_t)c * P.MN + n] = gn;
      const int w = gn < D.P ? 3 : 6;
      for (int k = inc_ptr_g[gn]; k < inc_ptr_g[gn + 1]; ++k) {
        const int code = inc_g[k];
        const int fam = (int)((unsigned)code >> 29), v = (code >> 25) & 15, e = code & 0x1FFFFFF;
        const int d = ((c % Cg) << 24) | o;
        switch (fam) {
          case F_DIST: dst_d[2 * (size_t)e + v] = d; break;
          case F_TET: dst_t[4 * (size_t)e + v] = d; break;
          case F_ATTP: dst_ap[e] = d; break;
          case F_ATTB: dst_ab[e] = d; break;
          case F_HINGE: dst_h[2 * (size_t)e + v] = d; break;
          case F_CN: dst_cn[e] = d; break;
          default: dst_cf[e] = d; break;
        }
        o += w;
      }
      ++n;
    };
    for (int p : B.Lp[c]) walk(p);
    for (int b : B.Lb[c]) walk(D.P + b);
    for (int k = n; k <= P.MN; ++k) in_ptr[(size_t)c * (P.MN + 1) + k] = o;
  }
  std::vector<int> cnt(8 * (size_t)C), elem((size_t)C * P.ME, 0), eref((size_t)C * P.ME * 4, 0),
      dest((size_t)C * P.ME * 4, 0);
  for (int c = 0; c < C; ++c) {
    int* k = &cnt[8 * (size_t)c];
    k[0] = (int)B.Lt[c].size(); k[1] = (int)B.Ld[c].size(); k[2] = (int)B.La[c].size();
    k[3] = (int)B.Lh[c].size(); k[4] = (int)B.Ls[c].size(); k[5] = (int)B.Lp[c].size();
    k[6] = (int)B.Lb[c].size(); k[7] = 0;
    int e = 0;
    auto put = [&](int g, std::initializer_list<int> nodes, std::initializer_list<int> dsts) {
      elem[(size_t)c * P.ME + e] = g;
      int q = 0;
      for (int gn : nodes) eref[((size_t)c * P.ME + e) * 4 + q++] = local_off(c, gn);
      q = 0;
      for (int d : dsts) dest[((size_t)c * P.ME + e) * 4 + q++] = d;
      ++e;
    };
    for (int t : B.Lt[c]) {
      const int* tv = &tets[4 * (size_t)t];
      put(t, {tv[0], tv[1], tv[2], tv[3]},
          {dst_t[4 * (size_t)t], dst_t[4 * (size_t)t + 1], dst_t[4 * (size_t)t + 2], dst_t[4 * (size_t)t + 3]});
    }
    for (int d : B.Ld[c]) put(d, {d_i[d], d_j[d]}, {dst_d[2 * (size_t)d], dst_d[2 * (size_t)d + 1]});
    for (int a : B.La[c]) put(a, {a_p[a], D.P + a_b[a]}, {dst_ap[a], dst_ab[a]});
    for (int x : B.Lh[c]) put(x, {D.P + h_a[x], D.P + h_b[x]}, {dst_h[2 * (size_t)x], dst_h[2 * (size_t)x + 1]});
    for (int s : B.Ls[c]) {
      if (s < D.nw) put(s, {D.P + w_body[s]}, {dst_cn[s], dst_cf[s]});
      else {
        // particle 0 of this cluster: local copy, or -1 - (owner rank << 24 | offset)
        // in the owner's U/V arrays (another group's particle 0 is replaced by the
        // slot's own particle)
        const int sp = slot_part[s - D.nw];
        put(s, {sp, sp}, {dst_cn[s], dst_cf[s]});
        if (own_of(0) / Cg == c / Cg) {
          const int o0 = own_of(0);
          eref[((size_t)c * P.ME + e - 1) * 4 + 1] =
              o0 == c ? local_off(c, 0) : -1 - (((o0 % Cg) << 24) | local_off(o0, 0));
        }
      }
    }
  }
  // halo pushes: owner -> every consumer holding a halo copy
  std::vector<std::vector<std::pair<int, int>>> consumers((size_t)D.P + D.nb);
  for (int c = 0; c < C; ++c)
    for (size_t i = 0; i < B.halo[c].size(); ++i)
      consumers[B.halo[c][i]].push_back({c, halo_off[c][i]});
  std::vector<int> hp_ptr((size_t)C * (P.MN + 1), 0), hpush;
  for (int c = 0; c < C; ++c) {
    int n = 0;
    auto emit = [&](int gn) {
      hp_ptr[(size_t)c * (P.MN + 1) + n] = (int)hpush.size();
      for (auto& pr : consumers[gn]) hpush.push_back(((pr.first % Cg) << 24) | pr.second);
      ++n;
    };
    for (int p : B.Lp[c]) emit(p);
    for (int b : B.Lb[c]) emit(D.P + b);
    for (int k = n; k <= P.MN; ++k) hp_ptr[(size_t)c * (P.MN + 1) + k] = (int)hpush.size();
  }
  const size_t bytes = 4 * (cnt.size() + elem.size() + eref.size() + dest.size() + node.size() +
                            in_ptr.size() + hp_ptr.size() + hpush.size()) + 9 * 256;
  CK(cudaMalloc(&H->plan_mem, bytes));
  char* base = (char*)H->plan_mem;
  size_t o = 0;
  auto up = [&](const std::vector<int>& v) -> const int* {
    int* d = (int*)(base + o);
    o += ((4 * v.size() + 255) / 256) * 256 + (v.empty() ? 256 : 0);
    if (!v.empty()) cudaMemcpy(d, v.data(), 4 * v.size(), cudaMemcpyHostToDevice);
    return d;
  };
  P.cnt = up(cnt);
  P.elem = up(elem);
  P.eref = up(eref);
  P.dest = up(dest);
  P.node = up(node);
  P.in_ptr = up(in_ptr);
  P.hp_ptr = up(hp_ptr);
  P.hpush = up(hpush);
  CK(cudaGetLastError());
  H->bytes += bytes;
  return SS_OK;
}

// reductions one k_newton_cluster launch performs at most (exact mode: two
// per PCR iteration, one per Newton tail)
static int c_max_reductions(const ss_handle* H) {
  return H->c.p.newton * (2 * std::max(H->c.p.pcr, 1) + 2) + 8;
}

// choose the smallest cluster whose shared-memory plan fits, or none
static int plan_cluster(ss_handle* H, const Dims& D, const std::vector<int>& d_i,
                        const std::vector<int>& d_j, const std::vector<int>& tets,
                        const std::vector<int>& a_p, const std::vector<int>& a_b,
                        const std::vector<int>& h_a, const std::vector<int>& h_b,
                        const std::vector<int>& w_body, const std::vector<int>& slot_part,
                        const std::vector<int>& inc_ptr_g, const std::vector<int>& inc_g,
                        int allow) {
  H->use_cluster = 0;
  if (!allow) return SS_OK;
  int dev = H->device, max_smem = 0;
  cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  const size_t budget = (size_t)max_smem - 2048;  // static reduction scratch
  // Multi-cluster plan (one env of G disconnected components, e.g. a coupled
  // n-snake scene, build_snake(n_snakes=n)): component k in cluster k, the
  // clusters combine their dot products through global memory.
  std::vector<int> comp;
  int G = 1;
  if (D.E == 1 && D.n_real == 1 && env_long("SS_MULTI_CLUSTER", 1)) {
    std::vector<int> par(D.P + D.nb);
    for (size_t i = 0; i < par.size(); ++i) par[i] = (int)i;
    auto root = [&](int x) {
      while (par[x] != x) x = par[x] = par[par[x]];
      return x;
    };
    auto join = [&](int x, int y) {
      x = root(x);
      y = root(y);
      if (x != y) par[std::max(x, y)] = std::min(x, y);
    };
    for (int t = 0; t < D.nt; ++t)
      for (int v = 1; v < 4; ++v) join(tets[4 * (size_t)t], tets[4 * (size_t)t + v]);
    for (int e = 0; e < D.nd; ++e) join(d_i[e], d_j[e]);
    for (int e = 0; e < D.na; ++e) join(a_p[e], D.P + a_b[e]);
    for (int e = 0; e < D.nh; ++e) join(D.P + h_a[e], D.P + h_b[e]);
    // components numbered in order of first appearance
    comp.assign(par.size(), 0);
    std::vector<int> seen(par.size(), -1);
    G = 0;
    for (size_t i = 0; i < par.size(); ++i) {
      const int r = root((int)i);
      if (seen[r] < 0) seen[r] = G++;
      comp[i] = seen[r];
    }
  }
  // rows of the largest cluster (16 CTAs x CL_RPT rows x CL_THREADS threads): a
  // larger scene (e.g. the 1M-tet snake) cannot fit one cluster
  const bool single_fits = (long)D.m <= 16L * CL_RPT * CL_THREADS;
  const bool multi = G >= 2 && G <= kClMaxGroups;  // co-residency decides below
  const bool dbg = env_long("SS_CLUSTER_DEBUG", 0) != 0;
  if (dbg) fprintf(stderr, "[plan_cluster] components %d single_fits %d\n", G, (int)single_fits);
  if (!single_fits && !multi) return SS_OK;
  // multi-cluster first (each component gets a whole cluster), else one cluster
  for (int Gp : {multi ? G : 0, single_fits ? 1 : 0})
  for (int C : {1, 2, 4, 8, 16}) {
    if (Gp == 0) break;
    PlanBuild B;
    B.C = C * Gp;
    plan_partition(B, D, d_i, d_j, tets, a_p, a_b, h_a, h_b, w_body, slot_part, inc_ptr_g,
                   Gp > 1 ? &comp : nullptr, Gp);
    if (dbg) fprintf(stderr, "[plan_cluster] G %d C %d smem %zu budget %zu\n", Gp, C, B.smem_bytes, budget);
    if (B.smem_bytes > budget) continue;
    // one element and one (node, axis) per thread; <= CL_RPT rows per thread
    {
      bool ok = B.P.NR <= CL_RPT * CL_THREADS;
      for (int c2 = 0; c2 < B.C; ++c2) {
        const size_t ne = B.Lt[c2].size() + B.Ld[c2].size() + B.La[c2].size() + B.Lh[c2].size() +
                          B.Ls[c2].size();
        if (ne > CL_THREADS || 3 * B.Lp[c2].size() + 6 * B.Lb[c2].size() > CL_THREADS) ok = false;
      }
      if (!ok) continue;
    }
    const void* fn = (const void*)(H->c.p.exact_j ? k_newton_cluster<true> : k_newton_cluster<false>);
    CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)B.smem_bytes));
    if (C > 8) CK(cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = C;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cfg.blockDim = dim3(CL_THREADS);
    cfg.gridDim = dim3(B.C);
    cfg.dynamicSmemBytes = B.smem_bytes;
    int nclus = 0;
    // every cluster of a multi-cluster env must be co-resident (they wait on each other)
    const cudaError_t oe = cudaOccupancyMaxActiveClusters(&nclus, fn, &cfg);
    if (dbg) fprintf(stderr, "[plan_cluster] G %d C %d max active clusters %d (%d)\n", Gp, C, nclus, (int)oe);
    if (oe != cudaSuccess || nclus < Gp) {
      cudaGetLastError();
      continue;
    }
    if (dbg) {
      for (int c2 = 0; c2 < B.C; ++c2) {
        int mx_inc = 0, n_inc = 0;
        for (int p : B.Lp[c2]) {
          mx_inc = std::max(mx_inc, inc_ptr_g[p + 1] - inc_ptr_g[p]);
          n_inc += inc_ptr_g[p + 1] - inc_ptr_g[p];
        }
        int mx_b = 0;
        for (int b : B.Lb[c2]) mx_b = std::max(mx_b, inc_ptr_g[D.P + b + 1] - inc_ptr_g[D.P + b]);
        fprintf(stderr,
                "[plan_cluster] cta %2d: tets %d dist %d att %d hinge %d slots %d | particles %d "
                "bodies %d halo %zu | inc %d max/particle %d max/body %d\n",
                c2, (int)B.Lt[c2].size(), (int)B.Ld[c2].size(), (int)B.La[c2].size(),
                (int)B.Lh[c2].size(), (int)B.Ls[c2].size(), (int)B.Lp[c2].size(),
                (int)B.Lb[c2].size(), B.halo[c2].size(), n_inc, mx_inc, mx_b);
      }
    }
    int rc = plan_upload(H, B, D, d_i, d_j, tets, a_p, a_b, h_a, h_b, w_body, slot_part,
                         inc_ptr_g, inc_g);
    if (rc) return rc;
    H->plan = B.P;
    H->plan.dbg = nullptr;
    if (getenv("SS_CLUSTER_STAMPS")) {
      CK(cudaMalloc(&H->plan.dbg, 256 * sizeof(long long)));  // [CTA < 16][16]
      CK(cudaMemset(H->plan.dbg, 0, 256 * sizeof(long long)));
    }
    if (Gp > 1) {
      // cross-cluster reduction buffers: per reduction of a launch, G partials
      // (4 doubles each) and an arrival counter (reset by a memset node per launch)
      const int xn = c_max_reductions(H);
      const size_t xb = (size_t)xn * Gp * kClXWords * 16;
      CK(cudaMalloc(&H->xmem, xb + 16));
      CK(cudaMemset(H->xmem, 0, xb + 16));
      H->plan.xbuf = (double*)H->xmem;
      H->plan.xcnt = (int*)((char*)H->xmem + xb);
      H->plan.xn = xn;
    } else {
      // the sticky fault flag alone (a bounded reduction wait that expired)
      CK(cudaMalloc(&H->xmem, 16));
      CK(cudaMemset(H->xmem, 0, 16));
      H->plan.xcnt = (int*)H->xmem;
    }
    H->use_cluster = 1;
    return SS_OK;
  }
  return SS_OK;
}

// ======================================================================
extern "C" {

int ss_abi_version(void) { return SS_ABI_VERSION; }
#ifndef SS_BUILD_ID
#define SS_BUILD_ID "unversioned"
#endif
// sha256 of the sources this library was compiled from (__graft_entry__.
// source_hash); the marker makes it findable in the file without loading it
extern "C" __attribute__((used)) const char ss_build_id_marker[] = "ss-build-id:" SS_BUILD_ID;
const char* ss_build_id(void) { return ss_build_id_marker + 12; }
const char* ss_last_error(void) { return g_err.c_str(); }

int ss_device_count(int* n) {
  CK(cudaGetDeviceCount(n));
  return SS_OK;
}

int ss_create(const ss_topology* t, const ss_params* p, int n_envs, int device,
              ss_handle** out) {
  if (!t || !p || !out) return fail(SS_EINVAL, "null argument");
  if (n_envs < 1) return fail(SS_EINVAL, "n_envs must be >= 1");
  if (t->num_particles < 1) return fail(SS_EINVAL, "scene has no particles");
  if (p->substeps < 1) return fail(SS_EINVAL, "substeps must be >= 1");
  if (p->newton_iters < 0 || p->pcr_iters < 0) return fail(SS_EINVAL, "negative iteration count");
  if (t->n_channels % 2) return fail(SS_EINVAL, "n_channels must be even (2 per link)");
  *out = nullptr;
  CK(cudaSetDevice(device));
  const GridCaps caps = grid_caps(device);
  struct GuardScope {  // SS_GUARD bands for this create only
    GuardScope() { g_guard = env_long("SS_GUARD", 0) ? 256 : 0; }
    ~GuardScope() {
      g_guard = 0;
      g_spans = nullptr;
    }
  } guard_scope;

  Dims D{};
  // lanes of one wave: ss_params.wave_envs, or by default at most
  // kAutoWave lanes. An [item][E] row is 8E bytes, so E <= 4096 keeps >= 64
  // item rows per 2 MB page and the per-env item walk inside the GPU's TLB
  // reach (65536 envs: 4756 steps/s at 4096 lanes, 3895 at 38912; bench
  // sweep in DESIGN.md). The memory cap is applied after the plan below.
  constexpr int kAutoWave = 4096;
  int wave_req = p->wave_envs > 0 ? std::min(p->wave_envs, n_envs) : std::min(kAutoWave, n_envs);
  // two concurrent lanes by default from 64 envs (1024 envs: 5,913 -> 6,127 snake-steps/s:
  // one wave's kernel tails overlap the other's; 2 sequential waves of 512: 5,756)
  const int lanes_req = (int)std::max(1L, std::min(4L, env_long("SS_LANES", 2)));
  if (lanes_req > 1 && p->wave_envs <= 0 && n_envs >= 32 * lanes_req)
    wave_req = std::min(wave_req, ((n_envs + lanes_req - 1) / lanes_req + 31) / 32 * 32);
  auto pad_lanes = [](int n) {
    int E = 1;
    if (n <= 32) {
      while (E < n) E <<= 1;
    } else {
      E = ((n + 31) / 32) * 32;
    }
    return E;
  };
  D.n_real = std::min(n_envs, wave_req);
  int E = pad_lanes(D.n_real);
  D.E = E;
  D.W = E < 32 ? E : 32;
  D.lgW = 0;
  while ((1 << D.lgW) < D.W) ++D.lgW;
  D.tiles = E / D.W;
  D.P = t->num_particles;
  D.nb = t->num_bodies;
  D.ndof = 3 * D.P + 6 * D.nb;
  D.bd0 = 3 * D.P;
  D.nd = t->n_dist;
  D.nt = t->n_tet;
  D.na = t->n_attach;
  D.nh = t->n_hinge;
  D.nw = p->ground_enabled ? t->n_wheel : 0;
  D.nq = p->ground_enabled ? (t->contact_particles ? t->n_contact_particles : D.P) : 0;
  D.ns = D.nw + D.nq;
  D.nch = t->n_channels;
  D.links = D.nch / 2;
  D.od = 0;
  D.ot = D.nd;
  D.oa = D.ot + 6 * D.nt;
  D.oh = D.oa + 3 * D.na;
  D.ms = D.oh + 5 * D.nh;
  D.on = D.ms;
  D.of = D.ms + D.ns;
  D.m = D.ms + 3 * D.ns;
  if ((long)D.nt >= (1L << 25) || (long)D.ns >= (1L << 25) || (long)D.nd >= (1L << 25))
    return fail(SS_EUNSUP, "more than 2^25 elements in one family");

  // validate indices
  for (int i = 0; i < 2 * D.nd; ++i)
    if (t->dist_pairs[i] < 0 || t->dist_pairs[i] >= D.P) return fail(SS_EINVAL, "dist_pairs out of range");
  for (int i = 0; i < 4 * D.nt; ++i)
    if (t->tets[i] < 0 || t->tets[i] >= D.P) return fail(SS_EINVAL, "tets out of range");
  for (int i = 0; i < D.na; ++i)
    if (t->attach_particle[i] < 0 || t->attach_particle[i] >= D.P || t->attach_body[i] < 0 ||
        t->attach_body[i] >= D.nb)
      return fail(SS_EINVAL, "attachment index out of range");
  for (int i = 0; i < D.nh; ++i)
    if (t->hinge_body_a[i] < 0 || t->hinge_body_a[i] >= D.nb || t->hinge_body_b[i] < 0 ||
        t->hinge_body_b[i] >= D.nb)
      return fail(SS_EINVAL, "hinge body out of range");
  for (int i = 0; i < D.nw; ++i)
    if (t->wheel_body[i] < 0 || t->wheel_body[i] >= D.nb) return fail(SS_EINVAL, "wheel body out of range");
  if (t->contact_particles)
    for (int i = 0; i < D.nq; ++i)
      if (t->contact_particles[i] < 0 || t->contact_particles[i] >= D.P)
        return fail(SS_EINVAL, "contact_particles out of range");
  for (int i = 0; i < D.nd; ++i)
    if (t->dist_channel && t->dist_channel[i] >= D.nch) return fail(SS_EINVAL, "dist_channel out of range");

  // ---- parameters (solver.py:195-232, 259)
  Par P{};
  const double h = p->dt / p->substeps;
  P.h = h;
  P.dt = p->dt;
  const double dmp = 0.0 > p->constraint_damping ? 0.0 : p->constraint_damping;
  P.gamma = 1.0 / (1.0 + dmp);
  for (int a = 0; a < 3; ++a) P.hg[a] = h * p->gravity[a];
  P.ground_h = p->ground_height;
  P.margin = p->contact_margin;
  P.mu = p->mu;
  P.fdyn = p->friction_compliance / (h * h);
  P.fb_delta = p->fb_delta;
  P.smin = p->fb_slope_min;
  P.smax = p->fb_slope_max;
  P.dmax = p->max_strain_rate * h;
  P.youngs = p->strain_youngs;
  P.ki = p->k_inflate;
  P.kd = p->k_deflate;
  P.cap = p->deflate_cap;
  P.supply = p->supply;
  P.half_h = 0.5 * h;
  P.newton = p->newton_iters;
  P.pcr = p->pcr_iters;
  P.substeps = p->substeps;
  P.exact_j = p->exact_jacobian ? 1 : 0;
  const double g = P.gamma;

  // actuated rows exist (solver.py:241-248)
  D.act_enabled = 0;
  if (D.nd && D.nch && t->has_strain && t->dist_channel)
    for (int i = 0; i < D.nd; ++i)
      if (t->dist_channel[i] >= 0) D.act_enabled = 1;

  // ---- host topology arrays
  std::vector<double> inv_mass(t->inv_mass, t->inv_mass + D.P);
  std::vector<double> body_im(D.nb), body_I(9 * (size_t)D.nb);
  for (int b = 0; b < D.nb; ++b) {
    body_im[b] = 1.0 / t->body_mass[b];
    for (int k = 0; k < 9; ++k) body_I[9 * b + k] = t->body_inertia[9 * b + k];
  }
  std::vector<int> d_i(D.nd), d_j(D.nd), d_chan(D.nd);
  std::vector<double> d_rest(D.nd), d_dyn(D.nd);
  for (int e = 0; e < D.nd; ++e) {
    d_i[e] = t->dist_pairs[2 * e];
    d_j[e] = t->dist_pairs[2 * e + 1];
    d_chan[e] = t->dist_channel ? t->dist_channel[e] : -1;
    d_rest[e] = t->dist_rest[e];
    d_dyn[e] = g * t->dist_compliance[e] / (h * h);
  }
  std::vector<int> t_idx(4 * (size_t)D.nt);
  std::vector<double> t_rinv(10 * (size_t)D.nt, 0.0), t_e3(3 * (size_t)D.nt);
  for (int e = 0; e < D.nt; ++e) {
    for (int v = 0; v < 4; ++v) t_idx[(size_t)v * D.nt + e] = t->tets[4 * (size_t)e + v];
    for (int k = 0; k < 9; ++k) t_rinv[10 * (size_t)e + k] = t->tet_rest_inv[9 * (size_t)e + k];
    // eh2 = gamma * compliance / (h*h) (solver.py:210); isotropic pattern
    // (constraints.py:26-40) stored as (diag, off-diagonal, shear)
    double eh[36];
    for (int k = 0; k < 36; ++k) eh[k] = g * t->tet_compliance[36 * (size_t)e + k] / (h * h);
    const double ed = eh[0], eo = eh[1], es = eh[21];
    bool ok = true;
    for (int i = 0; i < 6; ++i)
      for (int j = 0; j < 6; ++j) {
        double want;
        if (i < 3 && j < 3) want = i == j ? ed : eo;
        else if (i == j) want = es;
        else want = 0.0;
        if (memcmp(&eh[6 * i + j], &want, 8) != 0 && !(eh[6 * i + j] == 0.0 && want == 0.0)) ok = false;
      }
    if (!ok)
      return fail(SS_EUNSUP, "tet %d compliance is not the isotropic Voigt pattern of "
                             "constraints.py:26-40", e);
    t_e3[e] = ed;
    t_e3[(size_t)D.nt + e] = eo;
    t_e3[2 * (size_t)D.nt + e] = es;
  }
  std::vector<int> a_p(D.na), a_b(D.na);
  std::vector<double> a_anc(3 * (size_t)D.na), a_dyn(D.na);
  for (int e = 0; e < D.na; ++e) {
    a_p[e] = t->attach_particle[e];
    a_b[e] = t->attach_body[e];
    for (int k = 0; k < 3; ++k) a_anc[(size_t)k * D.na + e] = t->attach_anchor[3 * e + k];
    a_dyn[e] = g * t->attach_compliance[e] / (h * h);
  }
  std::vector<int> h_a(D.nh), h_b(D.nh);
  std::vector<double> h_v[5], h_dyn(D.nh);
  const double* hsrc[5] = {t->hinge_anchor_a, t->hinge_anchor_b, t->hinge_axis_a, t->hinge_tan1_b,
                           t->hinge_tan2_b};
  for (int q = 0; q < 5; ++q) h_v[q].assign(3 * (size_t)D.nh, 0.0);
  for (int e = 0; e < D.nh; ++e) {
    h_a[e] = t->hinge_body_a[e];
    h_b[e] = t->hinge_body_b[e];
    for (int q = 0; q < 5; ++q)
      for (int k = 0; k < 3; ++k) h_v[q][(size_t)k * D.nh + e] = hsrc[q][3 * e + k];
    h_dyn[e] = g * t->hinge_compliance[e] / (h * h);
  }
  std::vector<int> w_body(D.nw);
  std::vector<double> w_rad(D.nw), w_axis(3 * (size_t)D.nw);
  for (int e = 0; e < D.nw; ++e) {
    w_body[e] = t->wheel_body[e];
    w_rad[e] = t->wheel_radius[e];
    for (int k = 0; k < 3; ++k) w_axis[(size_t)k * D.nw + e] = t->wheel_axis[3 * e + k];
  }
  std::vector<int> slot_part(D.nq);
  for (int q = 0; q < D.nq; ++q) slot_part[q] = t->contact_particles ? t->contact_particles[q] : q;

  // ---- incidence lists in the reference accumulation order
  struct Inc { uint64_t key; int code; };
  std::vector<std::vector<Inc>> lists((size_t)D.P + D.nb);
  auto push = [&](int item, int rank, int fam, int v, int e) {
    uint64_t key = ((uint64_t)rank << 40) | ((uint64_t)e << 8) | (uint64_t)v;
    int code = (fam << 29) | (v << 25) | e;
    lists[item].push_back({key, code});
  };
  for (int e = 0; e < D.nd; ++e) {
    push(d_i[e], 0, F_DIST, 0, e);
    push(d_j[e], 0, F_DIST, 1, e);
  }
  for (int e = 0; e < D.nt; ++e)
    for (int v = 0; v < 4; ++v) push(t->tets[4 * (size_t)e + v], 1, F_TET, v, e);
  for (int e = 0; e < D.na; ++e) {
    push(a_p[e], 2, F_ATTP, 0, e);
    push(D.P + a_b[e], 2, F_ATTB, 1, e);
  }
  for (int e = 0; e < D.nh; ++e) {
    push(D.P + h_a[e], 3, F_HINGE, 0, e);
    push(D.P + h_b[e], 3, F_HINGE, 1, e);
  }
  for (int s = 0; s < D.ns; ++s) {
    const int item = s < D.nw ? D.P + w_body[s] : slot_part[s - D.nw];
    push(item, 4, F_CN, 0, s);
    push(item, 5, F_CF, 0, s);
  }
  std::vector<int> inc_ptr((size_t)D.P + D.nb + 1, 0), inc;
  std::vector<int2> inc_tet((size_t)D.P);
  std::vector<int> tdst(4 * (size_t)D.nt, 0);  // incidence of each tet vertex
  for (size_t i = 0; i < lists.size(); ++i) {
    std::stable_sort(lists[i].begin(), lists[i].end(),
                     [](const Inc& a, const Inc& b) { return a.key < b.key; });
    inc_ptr[i + 1] = inc_ptr[i] + (int)lists[i].size();
    int tb = -1, te = -1;
    for (size_t k = 0; k < lists[i].size(); ++k) {
      const int rank = (int)(lists[i][k].key >> 40);
      if (rank == 1 && tb < 0) tb = inc_ptr[i] + (int)k;
      if (rank == 1) te = inc_ptr[i] + (int)k + 1;
      const int code = lists[i][k].code;
      if ((int)((unsigned)code >> 29) == F_TET)
        tdst[4 * (size_t)(code & 0x1FFFFFF) + ((code >> 25) & 15)] = inc_ptr[i] + (int)k;
      inc.push_back(code);
    }
    if (i < (size_t)D.P) inc_tet[i] = make_int2(tb, te);
  }
  D.n_inc = (int)inc.size();
  // one large mesh: tet column sums in incidence order (ss_device.cuh tc_put;
  // SS_TC_INBOX=0 keeps the component-major [12][nt] layout)
  D.tc_inbox = tc_mode(D);

  // ---- allocations
  ss_handle* H = new ss_handle();
  H->caps = caps;
  g_spans = &H->guards;
  {
    // 0 = auto: the widest split up to 4 whose lanes still fit one resident
    // wave (coupled 2/10-snake scenes at E = 1: 7.8 -> 5.6 / 9.1 -> 7.1 ms per
    // frame at split 4, 5.3 / 6.9 at 8 — but 8 moved one ill-conditioned
    // parity case (test_gpu_params fb_slopes) past the 1e-10 per-step bound;
    // the 1M-tet snake fills the GPU already and stays at 1)
    const long gs = env_long("SS_GATHER_SPLIT", 0);
    H->gather_split = gs >= 8 ? 8 : gs >= 4 ? 4 : gs >= 2 ? 2 : gs == 1 ? 1 : 0;
  }
  H->device = device;
  H->c.D = D;
  H->c.p = P;
  CK(cudaStreamCreateWithFlags(&H->stream, cudaStreamNonBlocking));

  // topology
  Arena ta;
  auto plan_topo = [&](Arena& A) {
    Topo& T = H->c.T;
    T.inv_mass = A.take<double>(D.P);
    T.body_inv_mass = A.take<double>(D.nb);
    T.body_inertia = A.take<double>(9 * (size_t)D.nb);
    T.d_i = A.take<int>(D.nd);
    T.d_j = A.take<int>(D.nd);
    T.d_chan = A.take<int>(D.nd);
    T.d_rest = A.take<double>(D.nd);
    T.d_dyn = A.take<double>(D.nd);
    T.t_idx = A.take<int>(4 * (size_t)D.nt);
    T.t_rinv = A.take<double>(10 * (size_t)D.nt);
    T.t_e3 = A.take<double>(3 * (size_t)D.nt);
    T.a_p = A.take<int>(D.na);
    T.a_b = A.take<int>(D.na);
    T.a_anc = A.take<double>(3 * (size_t)D.na);
    T.a_dyn = A.take<double>(D.na);
    T.h_a = A.take<int>(D.nh);
    T.h_b = A.take<int>(D.nh);
    T.h_anca = A.take<double>(3 * (size_t)D.nh);
    T.h_ancb = A.take<double>(3 * (size_t)D.nh);
    T.h_axa = A.take<double>(3 * (size_t)D.nh);
    T.h_t1 = A.take<double>(3 * (size_t)D.nh);
    T.h_t2 = A.take<double>(3 * (size_t)D.nh);
    T.h_dyn = A.take<double>(D.nh);
    T.w_body = A.take<int>(D.nw);
    T.w_rad = A.take<double>(D.nw);
    T.w_axis = A.take<double>(3 * (size_t)D.nw);
    T.slot_part = A.take<int>(D.nq);
    T.inc_ptr = A.take<int>((size_t)D.P + D.nb + 1);
    T.inc = A.take<int>(inc.size());
    T.inc_tet = A.take<int2>((size_t)D.P);
    T.tdst = A.take<int>(4 * (size_t)D.nt);
  };
  plan_topo(ta);
  ta.cap = ta.off;
  ta.off = 0;
  {
    cudaError_t e = cudaMalloc(&H->topo_mem, ta.cap);
    if (e != cudaSuccess) {
      delete H;
      return fail(SS_ENOMEM, "cudaMalloc topology (%zu bytes): %s", ta.cap, cudaGetErrorString(e));
    }
  }
  ta.base = (char*)H->topo_mem;
  plan_topo(ta);
  H->bytes += ta.cap;
  auto up = [&](const void* dst, const void* src, size_t bytes) -> int {
    if (bytes) CK(cudaMemcpy((void*)dst, src, bytes, cudaMemcpyHostToDevice));
    return SS_OK;
  };
  const Topo& T = H->c.T;
  int rc = 0;
  rc |= up(T.inv_mass, inv_mass.data(), 8 * inv_mass.size());
  rc |= up(T.body_inv_mass, body_im.data(), 8 * body_im.size());
  rc |= up(T.body_inertia, body_I.data(), 8 * body_I.size());
  rc |= up(T.d_i, d_i.data(), 4 * d_i.size());
  rc |= up(T.d_j, d_j.data(), 4 * d_j.size());
  rc |= up(T.d_chan, d_chan.data(), 4 * d_chan.size());
  rc |= up(T.d_rest, d_rest.data(), 8 * d_rest.size());
  rc |= up(T.d_dyn, d_dyn.data(), 8 * d_dyn.size());
  rc |= up(T.t_idx, t_idx.data(), 4 * t_idx.size());
  rc |= up(T.t_rinv, t_rinv.data(), 8 * t_rinv.size());
  rc |= up(T.t_e3, t_e3.data(), 8 * t_e3.size());
  rc |= up(T.a_p, a_p.data(), 4 * a_p.size());
  rc |= up(T.a_b, a_b.data(), 4 * a_b.size());
  rc |= up(T.a_anc, a_anc.data(), 8 * a_anc.size());
  rc |= up(T.a_dyn, a_dyn.data(), 8 * a_dyn.size());
  rc |= up(T.h_a, h_a.data(), 4 * h_a.size());
  rc |= up(T.h_b, h_b.data(), 4 * h_b.size());
  rc |= up(T.h_anca, h_v[0].data(), 8 * h_v[0].size());
  rc |= up(T.h_ancb, h_v[1].data(), 8 * h_v[1].size());
  rc |= up(T.h_axa, h_v[2].data(), 8 * h_v[2].size());
  rc |= up(T.h_t1, h_v[3].data(), 8 * h_v[3].size());
  rc |= up(T.h_t2, h_v[4].data(), 8 * h_v[4].size());
  rc |= up(T.h_dyn, h_dyn.data(), 8 * h_dyn.size());
  rc |= up(T.w_body, w_body.data(), 4 * w_body.size());
  rc |= up(T.w_rad, w_rad.data(), 8 * w_rad.size());
  rc |= up(T.w_axis, w_axis.data(), 8 * w_axis.size());
  rc |= up(T.slot_part, slot_part.data(), 4 * slot_part.size());
  rc |= up(T.inc_ptr, inc_ptr.data(), 4 * inc_ptr.size());
  rc |= up(T.inc, inc.data(), 4 * inc.size());
  rc |= up(T.inc_tet, inc_tet.data(), sizeof(int2) * inc_tet.size());
  rc |= up(T.tdst, tdst.data(), 4 * tdst.size());
  if (rc) {
    ss_destroy(H);
    return SS_ECUDA;
  }

  // cluster-resident Newton solver plan (ss_params.solver_mode: 0 auto, 1 streaming,
  // 2 cluster). Auto picks the cluster solver for small batches, where the streaming
  // kernels are launch/latency-bound, and streaming above kAutoClusterMaxEnvs
  // (tools/solver_crossover.sh, v2.8 grids: 1 env 512 vs 129 steps/s, 16 envs 2862 vs
  // 1996, 32 envs 3537 vs 2877, 48 envs 2718 vs 2898, 64 envs 3622 vs 3862).
  {
    constexpr int kAutoClusterMaxEnvs = 32;
    H->keep = p->keep_matrix ? 1 : 0;
    if (H->keep && p->solver_mode == 2) {
      ss_destroy(H);
      return fail(SS_EUNSUP, "keep_matrix needs the streaming solver");
    }
    const bool want = p->solver_mode == 2 ||
                      (p->solver_mode == 0 && !H->keep && n_envs <= kAutoClusterMaxEnvs);
    std::vector<int> tets_v(t->tets, t->tets + 4 * (size_t)D.nt);
    int prc = plan_cluster(H, D, d_i, d_j, tets_v, a_p, a_b, h_a, h_b, w_body, slot_part,
                           inc_ptr, inc, want);
    if (prc) {
      ss_destroy(H);
      return prc;
    }
    if (p->solver_mode == 2 && !H->use_cluster) {
      ss_destroy(H);
      return fail(SS_EUNSUP, "scene does not fit the cluster-resident solver");
    }
  }

  // reduction grid (fixed: the partial-sum count per env)
  {
    const long n_el = (long)D.nd + D.nt + D.na + D.nh + D.ns;
    H->gy_red = (int)grid_items(D, n_el, H->caps.reduce).y;
    H->gy_dir = (int)grid_items(D, n_el, H->caps.dir).y;
    set_gy2(H, D);
  }

  // state + work (lane count read at call time: the wave cap may shrink it)
  auto plan_state = [&](Arena& A) {
    const size_t Es = H->c.D.E;
    State& S = H->c.S;
    S.pos = A.take<double>(3 * (size_t)D.P * Es);
    S.vel = A.take<double>(3 * (size_t)D.P * Es);
    S.bpos = A.take<double>(3 * (size_t)D.nb * Es);
    S.bquat = A.take<double>(4 * (size_t)D.nb * Es);
    S.blin = A.take<double>(3 * (size_t)D.nb * Es);
    S.bang = A.take<double>(3 * (size_t)D.nb * Es);
    S.lam = A.take<double>((size_t)D.ms * Es);
    S.quat = A.take<double>(4 * (size_t)D.nt * Es);
    S.dirs = A.take<double>(3 * (size_t)D.nd * Es);
    S.scale = A.take<double>((size_t)D.nd * Es);
    S.live = A.take<double>((size_t)D.nch * Es);
    S.target = A.take<double>((size_t)D.nch * Es);
    S.press = A.take<double>((size_t)D.nch * Es);
    S.warm = A.take<double>(3 * (size_t)D.nw * Es);
    S.warm_valid = A.take<int>((size_t)D.nw * Es);
    S.time = A.take<double>(Es);
    S.resid = A.take<double>(Es);
    S.nc_cnt = A.take<int>(Es);
    S.inv_cnt = A.take<int>(Es);
    S.nonfinite = A.take<int>(Es);
    S.gait = A.take<double>(6 * Es);
    S.gait_frame = A.take<int>(Es);
  };
  auto plan_work = [&](Arena& A) {
    const size_t Es = H->c.D.E;
    const int gy_max = std::max(std::max(H->gy_red, H->gy_dir), std::max(H->gy_red2, H->gy_dir2));
    Work& K = H->c.K;
    K.v = A.take<double>((size_t)D.ndof * Es);
    K.u = A.take<double>((size_t)D.ndof * Es);
    K.ang_inv = A.take<double>(9 * (size_t)D.nb * Es);
    K.res = A.take<double>((size_t)D.ms * Es);
    K.tS = A.take<double>(6 * (size_t)D.nt * Es);
    K.tC = D.tc_inbox == 1 ? A.take<double>(4 * (size_t)D.n_inc)
         : D.tc_inbox == 2 ? A.take<double>(3 * (size_t)D.n_inc * Es)
                           : A.take<double>(12 * (size_t)D.nt * Es);
    K.rw = A.take<double>(3 * (size_t)D.na * Es);
    K.hJ = A.take<double>(60 * (size_t)D.nh * Es);
    K.wJ = A.take<double>(18 * (size_t)D.nw * Es);
    K.present = A.take<int>((size_t)D.ns * Es);
    K.gap = A.take<double>((size_t)D.ns * Es);
    K.actf = A.take<double>((size_t)D.ns * Es);
    K.dynn = A.take<double>((size_t)D.ns * Es);
    K.lamc = A.take<double>(3 * (size_t)D.ns * Es);
    K.bdiag = A.take<double>((size_t)D.m * Es);
    K.x = A.take<double>((size_t)D.m * Es);
    K.r = A.take<double>((size_t)D.m * Es);
    K.z = A.take<double>((size_t)D.m * Es);
    K.p = A.take<double>((size_t)D.m * Es);
    K.ap = A.take<double>((size_t)D.m * Es);
    K.az = A.take<double>((size_t)D.m * Es);
    K.d = A.take<double>((size_t)D.m * Es);
    K.part = A.take<double>((size_t)gy_max * Es);
    K.cnt = A.take<int>(D.tiles);
    K.rho = A.take<double>(Es);
    K.alpha = A.take<double>(Es);
    K.beta = A.take<double>(Es);
    K.alpha_prev = A.take<double>(Es);
    K.last_step = A.take<int>(Es);
    K.broken = A.take<int>(Es);
    K.snap_rhs = p->keep_matrix ? A.take<double>((size_t)D.m * Es) : nullptr;
    // k_jtg ring (structured streaming path with E % 32 == 0; SS_JTG=0 off)
    const bool jtg = jtg_wanted(H, D);
    K.ring = jtg ? A.take<double>((size_t)jtg_ring_slots() * 12 * D.nt * 32) : nullptr;
    K.jctr = jtg ? A.take<int>(1 + 2 * (size_t)(Es / 32)) : nullptr;
  };
  Arena sa, wa;
  plan_state(sa);
  plan_work(wa);
  sa.cap = sa.off;
  wa.cap = wa.off;
  sa.off = wa.off = 0;
  // auto wave cap: shrink the wave until workspace + all state blocks fit
  if (p->wave_envs <= 0) {
    size_t free_b = 0, total_b = 0;
    cudaMemGetInfo(&free_b, &total_b);
    const double per_lane = (double)(sa.cap + wa.cap) / D.E;
    const double state_lane = (double)sa.cap / D.E;
    const double budget = 0.88 * (double)free_b;
    // work(E_w) + n_envs * state <= budget
    // lanes_req workspaces of E lanes each (concurrent lanes) + every env's state
    const double need =
        (double)n_envs * state_lane + (double)lanes_req * D.E * (per_lane - state_lane);
    if (need > budget && D.E > 32) {
      const double wl = (budget - n_envs * state_lane) / (lanes_req * (per_lane - state_lane));
      int ew = (int)(wl / 32) * 32;
      if (ew < 32) {
        ss_destroy(H);
        return fail(SS_ENOMEM, "%d envs do not fit in device memory even in waves", n_envs);
      }
      D.n_real = std::min(D.n_real, ew);  // only ever shrinks the wave
      D.E = pad_lanes(D.n_real);
      D.W = D.E < 32 ? D.E : 32;
      D.lgW = 0;
      while ((1 << D.lgW) < D.W) ++D.lgW;
      D.tiles = D.E / D.W;
      D.tc_inbox = tc_mode(D);
      H->c.D = D;
      H->gy_red = (int)grid_items(D, (long)D.nd + D.nt + D.na + D.nh + D.ns, H->caps.reduce).y;
      H->gy_dir = (int)grid_items(D, (long)D.nd + D.nt + D.na + D.nh + D.ns, H->caps.dir).y;
      set_gy2(H, D);
      sa = Arena();
      wa = Arena();
      plan_state(sa);
      plan_work(wa);
      sa.cap = sa.off;
      wa.cap = wa.off;
      sa.off = wa.off = 0;
    }
  }
  H->n_waves = (n_envs + D.E - 1) / D.E;
  const size_t sblock = sa.cap;
  {
    H->n_lanes = (lanes_req > 1 && H->n_waves > 1 && !H->use_cluster)
                     ? std::min(lanes_req, H->n_waves) : 1;
    // keep_matrix: the system snapshot (rhs, Jacobian blocks, M^-1) lives in
    // the workspace, so every wave gets its own workspace block — a wave
    // sharing a lane's block would overwrite an earlier wave's snapshot
    H->n_work = H->keep ? H->n_waves : H->n_lanes;
    cudaError_t e1 = cudaMalloc(&H->state_mem, sblock * H->n_waves);
    cudaError_t e2 = e1 == cudaSuccess ? cudaMalloc(&H->work_mem, wa.cap * H->n_work) : e1;
    if (e1 != cudaSuccess || e2 != cudaSuccess) {
      cudaGetLastError();
      ss_destroy(H);
      return fail(SS_ENOMEM, "cudaMalloc state/work (%zu x %d + %zu x %d bytes) for %d envs failed%s",
                  sblock, H->n_waves, wa.cap, H->n_work, n_envs,
                  H->keep ? " (keep_matrix needs one workspace per wave)" : "");
    }
  }
  std::vector<Work> blk_work(H->n_work);
  for (int l = 0; l < H->n_work; ++l) {
    Arena wl;
    wl.base = (char*)H->work_mem + wa.cap * l;
    plan_work(wl);
    blk_work[l] = H->c.K;
  }
  H->bytes += sblock * H->n_waves + wa.cap * H->n_work;
  CK(cudaMemsetAsync(H->state_mem, 0, sblock * H->n_waves, H->stream));
  // SS_POISON: workspace bytes 0xFF (doubles NaN, ints -1) instead of zeros
  CK(cudaMemsetAsync(H->work_mem, env_long("SS_POISON", 0) ? 0xFF : 0, wa.cap * H->n_work,
                     H->stream));
  // the reduction tickets start at zero by design (the last block resets them)
  for (int l = 0; l < H->n_work; ++l)
    CK(cudaMemsetAsync(blk_work[l].cnt, 0, sizeof(int) * D.tiles, H->stream));
  H->lane_stream[0] = H->stream;
  if (H->n_lanes > 1) {
    CK(cudaEventCreateWithFlags(&H->ev_fork, cudaEventDisableTiming));
    for (int l = 1; l < H->n_lanes; ++l) {
      CK(cudaStreamCreateWithFlags(&H->lane_stream[l], cudaStreamNonBlocking));
      CK(cudaEventCreateWithFlags(&H->ev_join[l], cudaEventDisableTiming));
    }
  }
  H->wave.assign(H->n_waves, H->c);
  H->wave_graphs.assign(H->n_waves, std::vector<cudaGraphExec_t>(6, nullptr));
  for (int w = 0; w < H->n_waves; ++w) {
    Arena a;
    a.base = (char*)H->state_mem + sblock * w;
    plan_state(a);  // writes H->c.S
    H->wave[w] = H->c;
    H->wave[w].K = blk_work[H->keep ? w : w % H->n_lanes];
    H->wave[w].D.n_real = std::min(D.E, n_envs - w * D.E);
    // reference constructor defaults
    const State& S = H->wave[w].S;
    auto fill = [&](double* ptr, size_t n, double val) {
      if (n) k_fill<<<256, 256, 0, H->stream>>>(ptr, n, val);
    };
    for (int b = 0; b < D.nb; ++b) fill(S.bquat + (size_t)(4 * b) * D.E, D.E, 1.0);
    fill(S.quat, (size_t)D.nt * D.E, 1.0);  // w component block [0][nt]
    fill(S.dirs, (size_t)D.nd * D.E, 1.0);  // x component block [0][nd]
    fill(S.scale, (size_t)D.nd * D.E, 1.0);
    fill(S.live, (size_t)D.nch * D.E, 1.0);
    fill(S.target, (size_t)D.nch * D.E, 1.0);
  }
  H->c = H->wave[0];
  H->c.D.n_real = n_envs;  // handle-level: total real envs
  {
    const size_t cmd_n = (size_t)H->n_waves * H->c.D.E * std::max(1, D.links);
    CK(cudaMalloc(&H->d_cmd, 8 * cmd_n));
    CK(cudaMemsetAsync(H->d_cmd, 0, 8 * cmd_n, H->stream));
  }
  for (const auto& g : H->guards) CK(cudaMemsetAsync(g.first, 0xA5, g.second, H->stream));
  // batched layouts, and one large mesh (E = 1 with >= 64k tets: 32 tets per
  // warp pair); small single scenes keep the one-thread kernels' reduction
  // order (test_gpu_params[fb_slopes] sits near its bound there)
  if (!H->c.p.exact_j && !H->use_cluster && D.nt > 0 &&
      (D.W == 32 || (D.W == 1 && D.nt >= env_long("SS_APPLY2_MIN_NT", 65536))) &&
      env_long("SS_APPLY2", 1))
    H->apply2 = 1;
  H->polar_split = (int)env_long("SS_POLAR_SPLIT", 1);
  H->polar_narrow = (D.W == 1 && D.nt <= 32 * 4096 && env_long("SS_POLAR_NARROW", 1)) ? 1 : 0;
  H->newton2 = (H->apply2 && env_long("SS_NEWTON2", 1)) ? 1 : 0;  // needs g_red2 (apply2 plan)
  // opt-in: bitwise equal but 60-68 ms/frame against 58.5 for k_pcr_step +
  // k_tet_jt (the separate kernels run at 0.95 / 0.91 of HBM; the fused one
  // loses the step's occupancy to the tet math)
  H->stepjt = (!H->c.p.exact_j && !H->use_cluster && D.nt > 0 && D.W == 32 &&
               env_long("SS_STEPJT", 0)) ? 1 : 0;
  // batched layouts only (W == 32): at few env lanes the element-owned kernel
  // keeps the v2.14 reduction order (an ill-conditioned parity case,
  // test_gpu_params[fb_slopes], sits at 1.4e-10 of its 1e-10 bound there)
  if (!H->c.p.exact_j && !H->use_cluster && D.W == 32 && env_long("SS_DIR2", 1)) H->dir2 = 1;
  // opt-in: no gain measured (coupled 2-snake frame 6.16 ms either way; 1024 envs and
  // the 1M-tet scene within noise, profiles/r2_summary.md)
  H->pdl = (int)env_long("SS_PDL", 0);
  // k_apply_rows3: the q / compact J / tet-row z tensor maps of every wave.
  // Opt-in (SS_APPLY3=1): bitwise k_apply_rows2, 32.5 vs 32.65 ms/frame on its
  // own at 1024 envs, but the whole two-lane step 7,058-7,070 vs 7,088-7,106
  // snake-steps/s (its 50 KB of shared memory per CTA); a 3-stage ring took
  // the u gather's L1 (6,315). The apply waits on the gathered u, not on q/S/z.
  if (H->apply2 && D.W == 32 && D.E % 32 == 0 && env_long("SS_APPLY3", 0)) {
    H->tm_apply.resize(H->n_waves);
    int bad = 0;
    for (int w = 0; w < H->n_waves; ++w) {
      const Ctx& cw = H->wave[w];
      bad |= make_tmap3(&H->tm_apply[w].q, cw.S.quat, D.E, D.nt, 4);
      bad |= make_tmap3(&H->tm_apply[w].s, cw.K.tS, D.E, D.nt, 6);
      bad |= make_tmap3(&H->tm_apply[w].z, cw.K.z + (size_t)D.ot * D.E, D.E, D.nt, 6);
    }
    H->apply3 = bad ? 0 : 1;
    if (bad) H->tm_apply.clear();
  }
  // one large mesh: the J^T x gather streams each warp's tet-run range of the
  // incidence-order column sums with bulk copies (bitwise the serial walk)
  if (D.tc_inbox && env_long("SS_GATHER_BULK", 1)) {
    CK(cudaFuncSetAttribute(k_gather_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)kGbSmem));
    int occ = 1, sms = 148;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_gather_bulk, SS_THREADS, kGbSmem);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, H->device);
    H->gbulk_grid = (int)env_long("SS_GB_GRID", (long)std::max(1, occ) * sms);
    H->gather_bulk = 1;
  }
  {
    int occ = 3, sms = 148;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_jtg, SS_THREADS, 0);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, H->device);
    H->jtg_grid = (int)env_long("SS_JTG_GRID", (long)std::max(1, occ) * sms);
    H->jplan = jtg_plan(H->c.D);
    H->jplan.ring = jtg_ring_slots();  // as allocated
    if (H->jplan.lag >= H->jplan.ring) H->jplan.lag = H->jplan.ring - 1;
  }
  // cp.async-staged k_apply_rows (structured streaming path; SS_APPLY_ASYNC=0 off)
  // opt-in (SS_APPLY_ASYNC=1): bitwise equal, 37.5 vs 37.9 ms/frame at 1024 envs
  // with 2 stages, slower with 3-4 (the staging buffers take the L1 the u gathers use)
  if (!H->c.p.exact_j && !H->use_cluster && D.nt > 0 && env_long("SS_APPLY_ASYNC", 0)) {
    H->apply_async_smem = SS_APPLYA_STAGES * 16 * SS_THREADS * sizeof(double);
    CK(cudaFuncSetAttribute(k_apply_rows_async, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)H->apply_async_smem));
    H->apply_async = 1;
  }
  {
    int frc = plan_fused(H, H->c.D, t->tets, d_i, d_j, a_p, slot_part);
    if (frc) {
      ss_destroy(H);
      return frc;
    }
  }
  CK(cudaStreamSynchronize(H->stream));
  *out = H;
  return SS_OK;
}

int ss_destroy(ss_handle* H) {
  if (!H) return SS_OK;
  cudaSetDevice(H->device);
  for (auto& gw : H->wave_graphs)
    for (auto& g : gw)
      if (g) cudaGraphExecDestroy(g);
  if (H->topo_mem) cudaFree(H->topo_mem);
  if (H->state_mem) cudaFree(H->state_mem);
  if (H->work_mem) cudaFree(H->work_mem);
  if (H->d_cmd) cudaFree(H->d_cmd);
  if (H->d_stage) cudaFree(H->d_stage);
  if (H->d_init) cudaFree(H->d_init);
  if (H->plan_mem) cudaFree(H->plan_mem);
  if (H->xmem) cudaFree(H->xmem);
  if (H->fplan_mem) cudaFree(H->fplan_mem);
  if (H->plan.dbg) cudaFree(H->plan.dbg);
  for (int l = 1; l < ss_handle::kMaxLanes; ++l) {
    if (H->lane_stream[l]) cudaStreamDestroy(H->lane_stream[l]);
    if (H->ev_join[l]) cudaEventDestroy(H->ev_join[l]);
  }
  if (H->ev_fork) cudaEventDestroy(H->ev_fork);
  if (H->stream) cudaStreamDestroy(H->stream);
  delete H;
  return SS_OK;
}

int ss_num_envs(const ss_handle* H) { return H ? H->c.D.n_real : 0; }

static int ensure_stage(ss_handle* H, size_t bytes) {
  if (bytes <= H->stage_bytes) return SS_OK;
  if (H->d_stage) CK(cudaFree(H->d_stage));
  H->d_stage = nullptr;
  CK(cudaMalloc(&H->d_stage, bytes));
  H->stage_bytes = bytes;
  return SS_OK;
}

// split a global env range into (wave, first lane, count, offset in the range)
struct WaveChunk {
  int w, lane0, cnt, off;
};
static std::vector<WaveChunk> wave_chunks(const ss_handle* H, int env0, int n) {
  std::vector<WaveChunk> out;
  const int E = H->c.D.E;
  int g = env0;
  while (g < env0 + n) {
    const int w = g / E, lane = g % E;
    const int cnt = std::min(env0 + n - g, E - lane);
    out.push_back({w, lane, cnt, g - env0});
    g += cnt;
  }
  return out;
}

// state I/O of envs [env0, env0+n): host (staged) or device (direct) pointers,
// env-major [n][A*B] on the caller's side, [item][E] per wave on the device
static int state_io(ss_handle* H, int env0, int n, const ss_state_view* v, bool set, bool dev) {
  if (!H || !v) return fail(SS_EINVAL, "null argument");
  const Dims& D = H->c.D;
  if (env0 < 0 || n < 0 || env0 + n > D.n_real) return fail(SS_EINVAL, "env range out of bounds");
  if (n == 0) return SS_OK;
  CK(cudaSetDevice(H->device));
  for (const WaveChunk& ch : wave_chunks(H, env0, n)) {
    Field f[32];
    int nf = 0;
    state_fields(H, ch.w, v, f, &nf);
    const int n_real_w = H->wave[ch.w].D.n_real;
    for (int i = 0; i < nf; ++i) {
      if (!f[i].host || f[i].A * f[i].B == 0) continue;
      const size_t elem = f[i].is_int ? 4 : 8;
      const size_t K = (size_t)f[i].A * f[i].B;
      const size_t bytes = elem * K * ch.cnt;
      char* user = (char*)f[i].host + elem * K * ch.off;
      char* buf = user;
      if (!dev) {
        int rc = ensure_stage(H, bytes);
        if (rc) return rc;
        buf = (char*)H->d_stage;
        if (set) CK(cudaMemcpyAsync(buf, user, bytes, cudaMemcpyHostToDevice, H->stream));
      }
      if (set) {
        if (f[i].is_int)
          k_scatter<int><<<512, 256, 0, H->stream>>>((int*)f[i].dev, (const int*)buf, ch.cnt, f[i].A,
                                                     f[i].B, f[i].swap, D.E, ch.lane0, n_real_w);
        else
          k_scatter<double><<<512, 256, 0, H->stream>>>((double*)f[i].dev, (const double*)buf,
                                                        ch.cnt, f[i].A, f[i].B, f[i].swap, D.E,
                                                        ch.lane0, n_real_w);
      } else {
        if (f[i].is_int)
          k_gather_state<int><<<512, 256, 0, H->stream>>>((int*)buf, (const int*)f[i].dev, ch.cnt,
                                                          f[i].A, f[i].B, f[i].swap, D.E, ch.lane0);
        else
          k_gather_state<double><<<512, 256, 0, H->stream>>>((double*)buf, (const double*)f[i].dev,
                                                             ch.cnt, f[i].A, f[i].B, f[i].swap,
                                                             D.E, ch.lane0);
      }
      CK(cudaGetLastError());
      if (!dev) {
        if (!set) CK(cudaMemcpyAsync(user, buf, bytes, cudaMemcpyDeviceToHost, H->stream));
        CK(cudaStreamSynchronize(H->stream));  // the staging buffer is reused per field
      }
    }
  }
  if (dev) CK(cudaStreamSynchronize(H->stream));
  return SS_OK;
}

int ss_set_state(ss_handle* H, int env0, int n, const ss_state_view* v) {
  return state_io(H, env0, n, v, true, false);
}
int ss_get_state(ss_handle* H, int env0, int n, ss_state_view* v) {
  return state_io(H, env0, n, v, false, false);
}
int ss_set_state_device(ss_handle* H, int env0, int n, const ss_state_view* v) {
  return state_io(H, env0, n, v, true, true);
}
int ss_get_state_device(ss_handle* H, int env0, int n, ss_state_view* v) {
  return state_io(H, env0, n, v, false, true);
}

// on_device: 0 host commands, 1 device commands, 2 on-device gait (cmd unused)
static int step_impl(ss_handle* H, const double* cmd, int on_device, int latency, int n_frames) {
  if (!H) return fail(SS_EINVAL, "null handle");
  NvtxRange nv_step("ss_step");
  if (n_frames < 0) return fail(SS_EINVAL, "n_frames must be >= 0");
  CK(cudaSetDevice(H->device));
  const Dims& D = H->c.D;
  const int has_cmd = D.nch == 0 ? 0 : (on_device == 2 ? 2 : (cmd != nullptr ? 1 : 0));
  const int key = 2 * has_cmd + (latency ? 1 : 0);
  for (int w = 0; w < H->n_waves; ++w) {
    cudaGraphExec_t g;
    int rc = get_graph(H, w, has_cmd, latency ? 1 : 0, &g);
    if (rc) return rc;
  }
  for (int f = 0; f < n_frames; ++f) {
    // every env of the frame, wave after wave (envs are independent); with two
    // lanes the odd waves run on the second stream, joined once per frame (the
    // command buffer is rewritten by the next frame)
    if (has_cmd == 1)
      CK(cudaMemcpyAsync(H->d_cmd, cmd + (size_t)f * D.n_real * D.links,
                         8 * (size_t)D.n_real * D.links,
                         on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, H->stream));
    if (H->n_lanes > 1) {
      CK(cudaEventRecord(H->ev_fork, H->stream));
      for (int l = 1; l < H->n_lanes; ++l) CK(cudaStreamWaitEvent(H->lane_stream[l], H->ev_fork, 0));
    }
    for (int w = 0; w < H->n_waves; ++w)
      CK(cudaGraphLaunch(H->wave_graphs[w][key], H->lane_stream[w % H->n_lanes]));
    for (int l = 1; l < H->n_lanes; ++l) {
      CK(cudaEventRecord(H->ev_join[l], H->lane_stream[l]));
      CK(cudaStreamWaitEvent(H->stream, H->ev_join[l], 0));
    }
  }
  return SS_OK;
}

int ss_step(ss_handle* H, const double* commands, int latency, int n_frames) {
  return step_impl(H, commands, 0, latency, n_frames);
}
int ss_step_device(ss_handle* H, const double* d_commands, int latency, int n_frames) {
  return step_impl(H, d_commands, 1, latency, n_frames);
}
int ss_step_gait(ss_handle* H, int latency, int n_frames) {
  return step_impl(H, nullptr, 2, latency, n_frames);
}

int ss_set_channel_targets(ss_handle* H, const double* commands, int latency) {
  if (!H) return fail(SS_EINVAL, "null handle");
  const Dims& D = H->c.D;
  if (D.nch == 0 || D.links == 0) return SS_OK;  // no channels: nothing to tick
  if (!commands) return fail(SS_EINVAL, "null commands");
  CK(cudaSetDevice(H->device));
  CK(cudaMemcpyAsync(H->d_cmd, commands, 8 * (size_t)D.n_real * D.links, cudaMemcpyHostToDevice,
                     H->stream));
  for (int w = 0; w < H->n_waves; ++w) {
    const Ctx& c = H->wave[w];
    const double* d_cmd = H->d_cmd + (size_t)w * D.E * D.links;
    k_tick<<<grid_items(c.D, D.links, H->caps.eval), SS_THREADS, 0, H->stream>>>(c, d_cmd,
                                                                                 latency ? 1 : 0);
  }
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(H->stream));  // the caller's host buffer may go away
  return SS_OK;
}

int ss_set_gait(ss_handle* H, int env0, int n, const double* params, const int* frame0) {
  if (!H || (!params && n > 0)) return fail(SS_EINVAL, "null argument");
  const Dims& D = H->c.D;
  if (env0 < 0 || n < 0 || env0 + n > D.n_real) return fail(SS_EINVAL, "env range out of bounds");
  for (int i = 0; i < n; ++i) {
    const double* g = params + 6 * (size_t)i;
    for (int k = 0; k < 6; ++k)
      if (!std::isfinite(g[k])) return fail(SS_EINVAL, "gait parameter %d of env %d not finite", k, env0 + i);
    if (g[5] < 1.0 || g[5] != std::floor(g[5]))
      return fail(SS_EINVAL, "links_per_snake of env %d must be a positive integer", env0 + i);
  }
  if (frame0)
    for (int i = 0; i < n; ++i)
      if (frame0[i] < 0) return fail(SS_EINVAL, "negative gait frame for env %d", env0 + i);
  CK(cudaSetDevice(H->device));
  for (const WaveChunk& ch : wave_chunks(H, env0, n)) {
    const State& S = H->wave[ch.w].S;
    // [6][E] items: copy item-major rows for this chunk
    std::vector<double> rows(6 * (size_t)ch.cnt);
    for (int k = 0; k < 6; ++k)
      for (int i = 0; i < ch.cnt; ++i) rows[(size_t)k * ch.cnt + i] = params[6 * (size_t)(ch.off + i) + k];
    for (int k = 0; k < 6; ++k)
      CK(cudaMemcpyAsync(S.gait + (size_t)k * D.E + ch.lane0, rows.data() + (size_t)k * ch.cnt,
                         8 * (size_t)ch.cnt, cudaMemcpyHostToDevice, H->stream));
    std::vector<int> fr(ch.cnt, 0);
    if (frame0)
      for (int i = 0; i < ch.cnt; ++i) fr[i] = frame0[ch.off + i];
    CK(cudaMemcpyAsync(S.gait_frame + ch.lane0, fr.data(), 4 * (size_t)ch.cnt,
                       cudaMemcpyHostToDevice, H->stream));
    CK(cudaStreamSynchronize(H->stream));  // host staging vectors go out of scope
  }
  return SS_OK;
}

int ss_get_gait(ss_handle* H, int env0, int n, double* params, int* frame) {
  if (!H || (n > 0 && (!params || !frame))) return fail(SS_EINVAL, "null argument");
  const Dims& D = H->c.D;
  if (env0 < 0 || n < 0 || env0 + n > D.n_real) return fail(SS_EINVAL, "env range out of bounds");
  CK(cudaSetDevice(H->device));
  CK(cudaStreamSynchronize(H->stream));
  for (const WaveChunk& ch : wave_chunks(H, env0, n)) {
    const State& S = H->wave[ch.w].S;
    std::vector<double> rows(6 * (size_t)ch.cnt);
    for (int k = 0; k < 6; ++k)
      CK(cudaMemcpy(rows.data() + (size_t)k * ch.cnt, S.gait + (size_t)k * D.E + ch.lane0,
                    8 * (size_t)ch.cnt, cudaMemcpyDeviceToHost));
    for (int k = 0; k < 6; ++k)
      for (int i = 0; i < ch.cnt; ++i) params[6 * (size_t)(ch.off + i) + k] = rows[(size_t)k * ch.cnt + i];
    CK(cudaMemcpy(frame + ch.off, S.gait_frame + ch.lane0, 4 * (size_t)ch.cnt,
                  cudaMemcpyDeviceToHost));
  }
  return SS_OK;
}

int ss_get_stats(ss_handle* H, int env0, int n, ss_env_stats* out) {
  if (!H || !out) return fail(SS_EINVAL, "null argument");
  const Dims& D = H->c.D;
  if (env0 < 0 || n < 0 || env0 + n > D.n_real) return fail(SS_EINVAL, "env range out of bounds");
  CK(cudaSetDevice(H->device));
  std::vector<int> nc(n), inv(n), nf(n);
  std::vector<double> res(n);
  for (const WaveChunk& ch : wave_chunks(H, env0, n)) {
    const State& S = H->wave[ch.w].S;
    const size_t c4 = 4 * (size_t)ch.cnt;
    CK(cudaMemcpyAsync(nc.data() + ch.off, S.nc_cnt + ch.lane0, c4, cudaMemcpyDeviceToHost, H->stream));
    CK(cudaMemcpyAsync(inv.data() + ch.off, S.inv_cnt + ch.lane0, c4, cudaMemcpyDeviceToHost, H->stream));
    CK(cudaMemcpyAsync(nf.data() + ch.off, S.nonfinite + ch.lane0, c4, cudaMemcpyDeviceToHost, H->stream));
    CK(cudaMemcpyAsync(res.data() + ch.off, S.resid + ch.lane0, 2 * c4, cudaMemcpyDeviceToHost, H->stream));
  }
  CK(cudaStreamSynchronize(H->stream));
  const Par& P = H->c.p;
  for (int i = 0; i < n; ++i) {
    out[i].newton_iterations = P.substeps * P.newton;
    out[i].pcr_iterations = P.substeps * P.newton * P.pcr;
    out[i].contact_count = nc[i];
    out[i].inverted_tets = inv[i];
    out[i].residual = res[i];
    out[i].finite = nf[i] ? 0 : 1;
    out[i]._pad = 0;
  }
  return SS_OK;
}

int ss_get_com(ss_handle* H, int env0, int n, double* out) {
  if (!H || !out) return fail(SS_EINVAL, "null argument");
  const Dims& D = H->c.D;
  if (env0 < 0 || n < 0 || env0 + n > D.n_real) return fail(SS_EINVAL, "env range out of bounds");
  if (n == 0) return SS_OK;
  CK(cudaSetDevice(H->device));
  int rc = ensure_stage(H, 24 * (size_t)n);
  if (rc) return rc;
  for (const WaveChunk& ch : wave_chunks(H, env0, n)) {
    const int L = H->c.D.W;
    k_com<<<(ch.cnt + L - 1) / L, 256, 0, H->stream>>>(H->wave[ch.w], ch.lane0, ch.cnt,
                                                       H->d_stage + 3 * (size_t)ch.off);
    CK(cudaGetLastError());
  }
  CK(cudaMemcpyAsync(out, H->d_stage, 24 * (size_t)n, cudaMemcpyDeviceToHost, H->stream));
  CK(cudaStreamSynchronize(H->stream));
  return SS_OK;
}

int ss_observe(ss_handle* H, int env0, int n, double* out) {
  if (!H || !out) return fail(SS_EINVAL, "null argument");
  const Dims& D = H->c.D;
  if (env0 < 0 || n < 0 || env0 + n > D.n_real) return fail(SS_EINVAL, "env range out of bounds");
  if (n == 0) return SS_OK;
  CK(cudaSetDevice(H->device));
  const size_t per = 4 + (size_t)D.nb;
  int rc = ensure_stage(H, 8 * per * n);
  if (rc) return rc;
  for (const WaveChunk& ch : wave_chunks(H, env0, n)) {
    const int L = D.W;
    k_observe<<<(ch.cnt + L - 1) / L, 256, 0, H->stream>>>(H->wave[ch.w], ch.lane0, ch.cnt,
                                                           H->d_stage + per * ch.off);
    CK(cudaGetLastError());
  }
  CK(cudaMemcpyAsync(out, H->d_stage, 8 * per * n, cudaMemcpyDeviceToHost, H->stream));
  CK(cudaStreamSynchronize(H->stream));
  return SS_OK;
}

int ss_export_system(ss_handle* H, int env, ss_system_view* v) {
  if (!H || !v) return fail(SS_EINVAL, "null argument");
  if (!H->keep) return fail(SS_EINVAL, "no system snapshot; create with keep_matrix and step");
  const Dims& D = H->c.D;
  if (env < 0 || env >= D.n_real) return fail(SS_EINVAL, "env out of range");
  CK(cudaSetDevice(H->device));
  const int w = env / D.E, lane = env % D.E;
  // staging layout: doubles then ints
  const size_t nD[] = {6 * (size_t)D.nd, 72 * (size_t)D.nt, 27 * (size_t)D.na, 60 * (size_t)D.nh,
                       18 * (size_t)D.ns, (size_t)D.ms, (size_t)D.ms, 3 * (size_t)D.ns,
                       3 * (size_t)D.ns, (size_t)D.ndof, 9 * (size_t)D.nb};
  const size_t nI[] = {6 * (size_t)D.nd, 12 * (size_t)D.nt, 9 * (size_t)D.na, 12 * (size_t)D.nh,
                       6 * (size_t)D.ns, (size_t)D.ns};
  size_t td = 0, ti = 0;
  for (size_t x : nD) td += x;
  for (size_t x : nI) ti += x;
  int rc = ensure_stage(H, 8 * td + 4 * ti);
  if (rc) return rc;
  double* dp[11];
  int* ip[6];
  {
    double* q = H->d_stage;
    for (int k = 0; k < 11; ++k) {
      dp[k] = q;
      q += nD[k];
    }
    int* r = reinterpret_cast<int*>(q);
    for (int k = 0; k < 6; ++k) {
      ip[k] = r;
      r += nI[k];
    }
  }
  SysOut o{dp[0], dp[1], dp[2], dp[3], dp[4], ip[0], ip[1], ip[2], ip[3], ip[4], ip[5],
           dp[5], dp[6], dp[7], dp[8], dp[9], dp[10]};
  const long items = (long)D.nd + D.nt + D.na + D.nh + D.ns + D.P + D.nb;
  k_export_system<<<(unsigned)((items + 255) / 256), 256, 0, H->stream>>>(H->wave[w], lane, o);
  CK(cudaGetLastError());
  double* hd[] = {v->dist_vals, v->tet_vals, v->att_vals, v->hinge_vals, v->slot_vals,
                  v->rhs_static, v->dyn_static, v->rhs_slot, v->dyn_slot, v->minv_diag, v->ang_inv};
  int32_t* hi[] = {v->dist_idx, v->tet_idx, v->att_idx, v->hinge_idx, v->slot_idx, v->slot_present};
  for (int k = 0; k < 11; ++k)
    if (nD[k] && hd[k]) CK(cudaMemcpyAsync(hd[k], dp[k], 8 * nD[k], cudaMemcpyDeviceToHost, H->stream));
  for (int k = 0; k < 6; ++k)
    if (nI[k] && hi[k]) CK(cudaMemcpyAsync(hi[k], ip[k], 4 * nI[k], cudaMemcpyDeviceToHost, H->stream));
  CK(cudaStreamSynchronize(H->stream));
  return SS_OK;
}

// packed byte offsets of the fields of one env (state_fields order)
static size_t init_layout(ss_handle* H, Field* f, int nf, size_t* off) {
  size_t o = 0;
  for (int i = 0; i < nf; ++i) {
    off[i] = o;
    o += (f[i].is_int ? 4 : 8) * (size_t)f[i].A * f[i].B;
    o = (o + 7) & ~(size_t)7;
  }
  return o;
}

int ss_capture_init(ss_handle* H, int env) {
  if (!H) return fail(SS_EINVAL, "null handle");
  const Dims& D = H->c.D;
  if (env < 0 || env >= D.n_real) return fail(SS_EINVAL, "env out of range");
  CK(cudaSetDevice(H->device));
  ss_state_view none{};
  Field f[32];
  int nf = 0;
  const int w = env / D.E, lane = env % D.E;
  state_fields(H, w, &none, f, &nf);
  size_t off[32];
  const size_t bytes = init_layout(H, f, nf, off);
  if (!H->d_init) CK(cudaMalloc(&H->d_init, bytes));
  for (int i = 0; i < nf; ++i) {
    if (f[i].A * f[i].B == 0) continue;
    if (f[i].is_int)
      k_gather_state<int><<<64, 256, 0, H->stream>>>((int*)(H->d_init + off[i]), (const int*)f[i].dev,
                                                     1, f[i].A, f[i].B, f[i].swap, D.E, lane);
    else
      k_gather_state<double><<<64, 256, 0, H->stream>>>((double*)(H->d_init + off[i]),
                                                        (const double*)f[i].dev, 1, f[i].A, f[i].B,
                                                        f[i].swap, D.E, lane);
    CK(cudaGetLastError());
  }
  CK(cudaStreamSynchronize(H->stream));
  return SS_OK;
}

int ss_reset_envs(ss_handle* H, const int* env_ids, int n, uint64_t seed, double pos_sigma,
                  double vel_sigma) {
  if (!H || (n > 0 && !env_ids)) return fail(SS_EINVAL, "null argument");
  if (!H->d_init) return fail(SS_EINVAL, "no reset template (ss_capture_init)");
  if (pos_sigma < 0.0 || vel_sigma < 0.0 || !std::isfinite(pos_sigma) || !std::isfinite(vel_sigma))
    return fail(SS_EINVAL, "perturbation sigmas must be finite and >= 0");
  const Dims& D = H->c.D;
  for (int i = 0; i < n; ++i)
    if (env_ids[i] < 0 || env_ids[i] >= D.n_real) return fail(SS_EINVAL, "env %d out of range", env_ids[i]);
  if (n == 0) return SS_OK;
  CK(cudaSetDevice(H->device));
  int rc = ensure_stage(H, 8 * (size_t)n + 8);
  if (rc) return rc;
  ss_state_view none{};
  for (int w = 0; w < H->n_waves; ++w) {
    std::vector<int> lanes, envs;
    for (int i = 0; i < n; ++i)
      if (env_ids[i] / D.E == w) {
        lanes.push_back(env_ids[i] % D.E);
        envs.push_back(env_ids[i]);
      }
    const int nl = (int)lanes.size();
    if (!nl) continue;
    int* d_l = reinterpret_cast<int*>(H->d_stage);
    int* d_e = d_l + n;
    CK(cudaMemcpyAsync(d_l, lanes.data(), 4 * (size_t)nl, cudaMemcpyHostToDevice, H->stream));
    CK(cudaMemcpyAsync(d_e, envs.data(), 4 * (size_t)nl, cudaMemcpyHostToDevice, H->stream));
    Field f[32];
    int nf = 0;
    state_fields(H, w, &none, f, &nf);
    size_t off[32];
    init_layout(H, f, nf, off);
    for (int i = 0; i < nf; ++i) {
      if (f[i].A * f[i].B == 0) continue;
      // fields 0/1 are particle positions / velocities (state_fields order)
      const double sig = i == 0 ? pos_sigma : (i == 1 ? vel_sigma : 0.0);
      if (f[i].is_int)
        k_reset_field<int><<<64, 256, 0, H->stream>>>((int*)f[i].dev, (const int*)(H->d_init + off[i]),
                                                      d_l, d_e, nl, f[i].A, f[i].B, f[i].swap, D.E,
                                                      0.0, seed, i, nullptr);
      else
        k_reset_field<double><<<64, 256, 0, H->stream>>>(
            (double*)f[i].dev, (const double*)(H->d_init + off[i]), d_l, d_e, nl, f[i].A, f[i].B,
            f[i].swap, D.E, sig, seed, i, i < 2 ? H->c.T.inv_mass : nullptr);
      CK(cudaGetLastError());
    }
    // the gait clock restarts with the episode
    std::vector<int> zeros(nl, 0);
    for (int j = 0; j < nl; ++j)
      CK(cudaMemcpyAsync(H->wave[w].S.gait_frame + lanes[j], zeros.data(), 4, cudaMemcpyHostToDevice,
                         H->stream));
    CK(cudaStreamSynchronize(H->stream));
  }
  return SS_OK;
}

int ss_synchronize(ss_handle* H) {
  if (!H) return fail(SS_EINVAL, "null handle");
  CK(cudaSetDevice(H->device));
  CK(cudaStreamSynchronize(H->stream));
  return SS_OK;
}

void* ss_stream(ss_handle* H) { return H ? (void*)H->stream : nullptr; }

int ss_launches_per_frame(ss_handle* H) {
  if (!H) return 0;
  if (!H->launches) {
    cudaGraphExec_t g;
    if (get_graph(H, 0, 1, 1, &g)) return -1;
  }
  return H->launches * H->n_waves;
}

int64_t ss_device_bytes(ss_handle* H) { return H ? (int64_t)H->bytes : 0; }

int ss_cluster_stamps(ss_handle* H, long long* out) {
  if (!H || !out) return fail(SS_EINVAL, "null argument");
  if (!H->plan.dbg) return fail(SS_EINVAL, "stamps off (set SS_CLUSTER_STAMPS)");
  const long n = std::max(1L, std::min(16L, env_long("SS_CLUSTER_STAMPS", 1)));
  CK(cudaMemcpy(out, H->plan.dbg, 16 * n * sizeof(long long), cudaMemcpyDeviceToHost));
  return SS_OK;
}

int ss_check_guards(ss_handle* H, int64_t* bad_bytes) {
  if (!H || !bad_bytes) return fail(SS_EINVAL, "null argument");
  CK(cudaSetDevice(H->device));
  CK(cudaDeviceSynchronize());
  int64_t bad = 0;
  std::vector<unsigned char> buf;
  for (const auto& g : H->guards) {
    buf.resize(g.second);
    CK(cudaMemcpy(buf.data(), g.first, g.second, cudaMemcpyDeviceToHost));
    for (unsigned char b : buf) bad += b != 0xA5;
  }
  *bad_bytes = H->guards.empty() ? -1 : bad;
  return SS_OK;
}

int ss_solver_info(ss_handle* H, int* info) {
  if (!H || !info) return fail(SS_EINVAL, "null argument");
  info[0] = H->use_cluster;
  info[1] = H->use_cluster ? H->plan.C : 0;
  info[2] = H->use_cluster ? 8 * H->plan.smem_doubles : 0;
  info[3] = H->c.D.E;
  info[4] = H->n_waves;
  info[5] = H->fused;
  info[6] = H->fused ? H->fplan.n_blocks : 0;
  info[7] = H->fused ? H->fused_chunks : 0;
  info[8] = H->use_cluster ? H->plan.G : 0;
  info[9] = 0;
  if (H->use_cluster && H->plan.xcnt) {
    CK(cudaStreamSynchronize(H->stream));
    CK(cudaMemcpy(&info[9], H->plan.xcnt, sizeof(int), cudaMemcpyDeviceToHost));
  }
  return SS_OK;
}

int ss_kernel_names(const char** names, int cap) {
  for (int i = 0; i < kNumKernels && i < cap; ++i) names[i] = kKernelNames[i];
  return kNumKernels;
}

int ss_profile_frames(ss_handle* H, const double* commands, int latency, int n_frames,
                      double* ms_total, int* launches) {
  if (!H || !ms_total || !launches) return fail(SS_EINVAL, "null argument");
  CK(cudaSetDevice(H->device));
  const Dims& D = H->c.D;
  const int has_cmd = commands != nullptr && D.nch > 0;
  for (int i = 0; i < kNumKernels; ++i) {
    ms_total[i] = 0.0;
    launches[i] = 0;
  }
  const size_t frame_bytes = 8 * (size_t)D.n_real * D.links;
  for (int f = 0; f < n_frames; ++f) {
    if (has_cmd)
      CK(cudaMemcpyAsync(H->d_cmd, commands + (size_t)f * D.n_real * D.links, frame_bytes,
                         cudaMemcpyHostToDevice, H->stream));
    Prof prof;
    for (int w = 0; w < H->n_waves; ++w) {
      int nl = 0;
      int rc = enqueue_frame(H, w, has_cmd, latency, &nl, &prof);
      if (rc) return rc;
    }
    CK(cudaStreamSynchronize(H->stream));
    for (auto& e : prof.ev) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, e.second.first, e.second.second);
      if (e.first >= 0) {
        ms_total[e.first] += ms;
        launches[e.first] += 1;
      }
      cudaEventDestroy(e.second.first);
      cudaEventDestroy(e.second.second);
    }
  }
  return SS_OK;
}

// ------------------------------------------------ device scene builder
static int link_counts(const ss_link_mesh_params* p, int32_t* c) {
  const int S = p->sections, W = p->width_nodes, H = p->height_nodes;
  if (W < 5 || H < 2 || S < 2) return fail(SS_EINVAL, "link grid needs at least 5x2 nodes and 2 sections");
  if (p->n_links < 0) return fail(SS_EINVAL, "n_links must be >= 0");
  const int n_ring = S - S / 3 - (S % 3 >= 2 ? 1 : 0);
  c[0] = S * W * H;
  c[1] = 5 * (S - 1) * (W - 1) * (H - 1);
  c[2] = 2 * H + H * (S - 1) + n_ring * (2 * (W - 1) + 2 * (H - 1)) + 4 * S;
  c[3] = 6;
  return SS_OK;
}

int ss_link_mesh_counts(const ss_link_mesh_params* p, int32_t* counts) {
  if (!p || !counts) return fail(SS_EINVAL, "null argument");
  return link_counts(p, counts);
}

int ss_build_link_meshes(const ss_link_mesh_params* p, int device, ss_link_mesh_out* o) {
  if (!p || !o) return fail(SS_EINVAL, "null argument");
  int32_t cnt[4];
  int rc = link_counts(p, cnt);
  if (rc) return rc;
  const long L = p->n_links;
  if (L == 0) return SS_OK;
  if (!p->origins || !p->channels) return fail(SS_EINVAL, "null origins / channels");
  CK(cudaSetDevice(device));
  const size_t nP = (size_t)L * cnt[0], nT = (size_t)L * cnt[1], nC = (size_t)L * cnt[2];
  // one device block: doubles, then ints
  const size_t nd = 3 * L + 3 * nP + nP + 9 * nT + nT + 36 * nT + 2 * nC;
  const size_t ni = 2 * L + 4 * nT + 2 * nC + 2 * nC + 12 * L + 1;
  char* mem = nullptr;
  CK(cudaMalloc(&mem, 8 * nd + 4 * ni));
  double* dd = (double*)mem;
  double* d_orig = dd; dd += 3 * L;
  double* d_pos = dd; dd += 3 * nP;
  double* d_mass = dd; dd += nP;
  double* d_rinv = dd; dd += 9 * nT;
  double* d_vol = dd; dd += nT;
  double* d_comp = dd; dd += 36 * nT;
  double* d_rest = dd; dd += nC;
  double* d_ccomp = dd; dd += nC;
  int* di = (int*)dd;
  int* d_chan = di; di += 2 * L;
  int* d_tets = di; di += 4 * nT;
  int* d_pairs = di; di += 2 * nC;
  int* d_kind = di; di += nC;
  int* d_cch = di; di += nC;
  int* d_mounts = di; di += 12 * L;
  int* d_bad = di;
  cudaError_t e = cudaSuccess;
  auto ok = [&](cudaError_t x) { if (e == cudaSuccess) e = x; };
  ok(cudaMemcpy(d_orig, p->origins, 24 * L, cudaMemcpyHostToDevice));
  ok(cudaMemcpy(d_chan, p->channels, 8 * L, cudaMemcpyHostToDevice));
  ok(cudaMemset(d_bad, 0, 4));
  SsbLink g;
  g.S = p->sections; g.W = p->width_nodes; g.H = p->height_nodes; g.L = (int)L;
  g.dx = p->dx; g.dy = p->dy; g.dz = p->dz; g.hw = p->half_width;
  g.E = p->youngs_modulus; g.nu = p->poisson; g.rho = p->density;
  g.c_act = p->actuation_compliance; g.c_inext = p->inextensible_compliance;
  g.c_struct = p->structural_compliance;
  g.origin = d_orig; g.chan = d_chan;
  g.NP = cnt[0]; g.NT = cnt[1]; g.NC = cnt[2];
  auto blocks = [](size_t n) { return (unsigned)std::min<size_t>((n + 255) / 256, 148 * 16); };
  if (e == cudaSuccess) {
    ssb_k_particles<<<blocks(nP), 256>>>(g, d_pos);
    ssb_k_tets<<<blocks(nT), 256>>>(g, d_tets, d_rinv, d_vol, d_comp, d_bad);
    ssb_k_masses<<<blocks(nP), 256>>>(g, d_vol, d_mass);
    ssb_k_cables<<<blocks(nC), 256>>>(g, d_pairs, d_rest, d_ccomp, d_kind, d_cch, d_mounts);
    e = cudaGetLastError();
  }
  int bad = 0;
  ok(cudaMemcpy(&bad, d_bad, 4, cudaMemcpyDeviceToHost));
  auto down = [&](void* h, const void* d, size_t bytes) { if (h && bytes) ok(cudaMemcpy(h, d, bytes, cudaMemcpyDeviceToHost)); };
  down(o->positions, d_pos, 24 * nP);
  down(o->masses, d_mass, 8 * nP);
  down(o->tets, d_tets, 16 * nT);
  down(o->rest_inv, d_rinv, 72 * nT);
  down(o->rest_volume, d_vol, 8 * nT);
  down(o->compliance, d_comp, 288 * nT);
  down(o->pairs, d_pairs, 8 * nC);
  down(o->rest, d_rest, 8 * nC);
  down(o->cable_compliance, d_ccomp, 8 * nC);
  down(o->kind, d_kind, 4 * nC);
  down(o->channel, d_cch, 4 * nC);
  down(o->mounts, d_mounts, 48 * L);
  cudaFree(mem);
  if (e != cudaSuccess) return fail(SS_ECUDA, "scene builder: %s", cudaGetErrorString(e));
  if (bad) return fail(SS_EINVAL, "degenerate rest tetrahedron (%d tets)", bad);
  return SS_OK;
}

// ------------------------------------------------------- kernel-level ABI
#define KSTREAM ((cudaStream_t)stream)
#define KBLK(n) (unsigned)(((long)(n) + 255) / 256), 256, 0, KSTREAM

int ssk_block_forward(const int32_t* dof_idx, const double* vals, int n, int r, int k,
                      const double* u, double* out_rows, void* stream) {
  if (n * r > 0) kk_block_forward<<<KBLK((long)n * r)>>>(dof_idx, vals, n, r, k, u, out_rows);
  CK(cudaGetLastError());
  return SS_OK;
}
int ssk_block_transpose(const int32_t* dof_idx, const double* vals, int n, int r, int k,
                        const double* x_rows, double* y, int ndof, void* stream) {
  const long nk = (long)n * k;
  if (ndof <= 0) return SS_OK;
  if (nk <= 0) return SS_OK;  // y += 0
  if (nk > 0x7fffffffL) return fail(SS_EINVAL, "block_transpose: n*k exceeds int32");
  // CSR transpose: stable radix sort of (dof, e*k+j) pairs by dof
  int *keys_out = nullptr, *vals_in = nullptr, *vals_out = nullptr;
  void* tmp = nullptr;
  size_t tmp_bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, dof_idx, keys_out, vals_in, vals_out, (int)nk,
                                  0, 32, KSTREAM);
  CK(cudaMalloc(&keys_out, 4 * nk));
  CK(cudaMalloc(&vals_in, 4 * nk));
  CK(cudaMalloc(&vals_out, 4 * nk));
  CK(cudaMalloc(&tmp, tmp_bytes));
  kk_iota<<<256, 256, 0, KSTREAM>>>(vals_in, nk);
  cudaError_t e = cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, dof_idx, keys_out, vals_in,
                                                  vals_out, (int)nk, 0, 32, KSTREAM);
  if (e == cudaSuccess) {
    kk_block_transpose<<<KBLK(ndof)>>>(keys_out, vals_out, nk, vals, r, k, x_rows, y, ndof);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(KSTREAM);
  cudaFree(keys_out);
  cudaFree(vals_in);
  cudaFree(vals_out);
  cudaFree(tmp);
  if (e != cudaSuccess) return fail(SS_ECUDA, "block_transpose: %s", cudaGetErrorString(e));
  return SS_OK;
}
int ssk_block_rowdiag(const int32_t* dof_idx, const double* vals, int n, int r, int k,
                      const double* minv_diag, double* out_rows, void* stream) {
  if (n * r > 0) kk_block_rowdiag<<<KBLK((long)n * r)>>>(dof_idx, vals, n, r, k, minv_diag, out_rows);
  CK(cudaGetLastError());
  return SS_OK;
}
int ssk_minv_apply(const double* minv_diag, const double* ang_inv, int nb, int body_dof0,
                   const double* u, double* out, int ndof, void* stream) {
  if (ndof > 0) kk_minv_apply<<<KBLK(ndof)>>>(minv_diag, ang_inv, nb, body_dof0, u, out, ndof);
  CK(cudaGetLastError());
  return SS_OK;
}
int ssk_ereg_apply(const double* vals6, const double* x_rows, double* out_rows, int n,
                   void* stream) {
  if (n > 0) kk_ereg_apply<<<KBLK((long)n * 6)>>>(vals6, x_rows, out_rows, n);
  CK(cudaGetLastError());
  return SS_OK;
}
int ssk_dot(const double* a, const double* b, int n, double* out_host, void* stream) {
  double* d = nullptr;
  CK(cudaMalloc(&d, 8));
  kk_dot<<<1, 256, 0, KSTREAM>>>(a, b, n, d);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaMemcpyAsync(out_host, d, 8, cudaMemcpyDeviceToHost, KSTREAM);
  if (e == cudaSuccess) e = cudaStreamSynchronize(KSTREAM);
  cudaFree(d);
  if (e != cudaSuccess) return fail(SS_ECUDA, "ssk_dot: %s", cudaGetErrorString(e));
  return SS_OK;
}
int ssk_eval_distance(const double* pos, const int32_t* pairs, const double* rest,
                      const double* scale, double* dirs, double* out_res, int n, void* stream) {
  if (n > 0) kk_eval_distance<<<KBLK(n)>>>(pos, pairs, rest, scale, dirs, out_res, n);
  CK(cudaGetLastError());
  return SS_OK;
}
int ssk_eval_tetra(const double* pos, const int32_t* tets, const double* rest_inv, double* quats,
                   double tol, int maxiter, double* out_res, double* out_vals, int n,
                   int* n_inverted, void* stream) {
  int* d = nullptr;
  CK(cudaMalloc(&d, 4));
  cudaError_t e = cudaMemsetAsync(d, 0, 4, KSTREAM);
  if (e == cudaSuccess && n > 0)
    kk_eval_tetra<<<KBLK(n)>>>(pos, tets, rest_inv, quats, tol, maxiter, out_res, out_vals, n, d);
  if (e == cudaSuccess) e = cudaGetLastError();
  int h = 0;
  if (e == cudaSuccess) e = cudaMemcpyAsync(&h, d, 4, cudaMemcpyDeviceToHost, KSTREAM);
  if (e == cudaSuccess) e = cudaStreamSynchronize(KSTREAM);
  cudaFree(d);
  if (e != cudaSuccess) return fail(SS_ECUDA, "ssk_eval_tetra: %s", cudaGetErrorString(e));
  if (n_inverted) *n_inverted = h;
  return SS_OK;
}

int ssk_malloc(void** ptr, int64_t bytes, int device) {
  if (!ptr) return fail(SS_EINVAL, "null argument");
  CK(cudaSetDevice(device));
  CK(cudaMalloc(ptr, bytes > 0 ? (size_t)bytes : 8));
  return SS_OK;
}
int ssk_free(void* ptr) {
  CK(cudaFree(ptr));
  return SS_OK;
}
int ssk_memcpy(void* dst, const void* src, int64_t bytes, int kind) {
  const cudaMemcpyKind k = kind == 1 ? cudaMemcpyHostToDevice
                           : kind == 2 ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
  if (bytes > 0) CK(cudaMemcpy(dst, src, (size_t)bytes, k));
  return SS_OK;
}

}  // extern "C"
