/*
 * softsnake_b200.h — C ABI of the B200-native implicit compliant-constraint
 * time step (arXiv:1904.02833 soft-snake simulator hot path).
 *
 * The reference has no native boundary: its hot path is
 *   Simulator.step(commands, latency)          softsnake/solver.py:296-314
 * driving the kernel-backend plugin interface
 *   kernels/__init__.py:24-41 (block_forward, block_transpose, block_rowdiag,
 *   minv_apply, ereg_apply, dot, eval_distance, eval_tetra).
 * This header replaces both:
 *   - ss_* : a Simulator-level ABI. One handle = a batch of independent
 *            environments (copies of one scene) resident on one GPU.
 *   - ssk_*: a kernel-level ABI with the exact argument meaning of the
 *            reference backend functions, on DEVICE pointers (test/parity use).
 *
 * Conventions (mirroring the reference):
 *   - all floating point is IEEE binary64, all indices int32, arrays
 *     C-contiguous in the reference's shapes;
 *   - caller owns host buffers, the handle owns device memory;
 *   - every call returns 0 on success or a negative SS_E* code, with a
 *     thread-local message in ss_last_error();
 *   - non-finite states are not errors: they are flagged per environment
 *     (ss_env_stats.finite), like the reference which never raises inside
 *     step() (solver.py:296; harness.py:196-207 checks COM afterwards).
 *   - one CUDA stream per device; calls on one handle must be serialised by
 *     the caller; handles on different devices may run concurrently.
 */
#ifndef SOFTSNAKE_B200_H
#define SOFTSNAKE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SS_ABI_VERSION 1

#define SS_OK 0
#define SS_EINVAL (-1)   /* bad argument -> Python ValueError   */
#define SS_ECUDA (-2)    /* CUDA failure   -> Python RuntimeError */
#define SS_ENOMEM (-3)   /* device allocation failed             */
#define SS_EUNSUP (-4)   /* topology outside what the kernels support */

/* Scene topology: every array verbatim from the reference containers.
 * Shapes in brackets; NULL allowed when the count is 0. */
typedef struct ss_topology {
  int32_t num_particles;            /* P   state.py:129-131               */
  int32_t num_bodies;               /* nb  state.py:133-135               */
  const double* inv_mass;           /* [P]     ParticleSet.inv_mass       */
  const double* body_mass;          /* [nb]    SystemState.body_mass      */
  const double* body_inertia;       /* [nb,3,3] body frame                */
  /* DistanceSet  constraints.py:62-100 */
  int32_t n_dist;
  const int32_t* dist_pairs;        /* [nd,2] */
  const double* dist_rest;          /* [nd]   */
  const double* dist_compliance;    /* [nd]   */
  const int32_t* dist_channel;      /* [nd]   -1 = not actuated */
  /* TetraSet  constraints.py:140-177 */
  int32_t n_tet;
  const int32_t* tets;              /* [nt,4]   */
  const double* tet_rest_inv;       /* [nt,3,3] */
  const double* tet_compliance;     /* [nt,6,6] (isotropic pattern, constraints.py:26-40) */
  /* AttachmentSet  constraints.py:201-245 */
  int32_t n_attach;
  const int32_t* attach_particle;   /* [na]   */
  const int32_t* attach_body;       /* [na]   */
  const double* attach_anchor;      /* [na,3] */
  const double* attach_compliance;  /* [na]   */
  /* HingeSet  constraints.py:282-356 */
  int32_t n_hinge;
  const int32_t* hinge_body_a;      /* [nh] */
  const int32_t* hinge_body_b;      /* [nh] */
  const double* hinge_anchor_a;     /* [nh,3] */
  const double* hinge_anchor_b;     /* [nh,3] */
  const double* hinge_axis_a;       /* [nh,3] */
  const double* hinge_tan1_b;       /* [nh,3] */
  const double* hinge_tan2_b;       /* [nh,3] */
  const double* hinge_compliance;   /* [nh]   */
  /* WheelCollider list  contact.py:35-41 */
  int32_t n_wheel;
  const int32_t* wheel_body;        /* [nw]   */
  const double* wheel_radius;       /* [nw]   */
  const double* wheel_axis;         /* [nw,3] axis_local */
  /* Simulator.contact_particles (solver.py:165); NULL => all particles */
  int32_t n_contact_particles;
  const int32_t* contact_particles;
  /* ChannelBank.pressures length (2 * links), 0 = no pneumatics */
  int32_t n_channels;
  int32_t has_strain;               /* Simulator(strain=StrainLaw) given */
} ss_topology;

/* SolverConfig (solver.py:95-117) + StrainLaw + ChannelBank constants. */
typedef struct ss_params {
  double dt;
  int32_t substeps, newton_iters, pcr_iters;
  double gravity[3];
  double ground_height;
  int32_t ground_enabled;
  double contact_margin;
  double mu;
  double friction_compliance;
  double fb_delta, fb_slope_min, fb_slope_max;
  double max_strain_rate;
  double constraint_damping;
  double strain_youngs;             /* StrainLaw.youngs_modulus_pa  pneumatics.py:32-43 */
  double k_inflate, k_deflate, deflate_cap, supply;   /* pneumatics.py:88-96 */
  /* 1: apply each tet Jacobian through its materialised 6x12 columns, so
   * every J^T x / J u sum is bitwise numba's; 0 (default): structured
   * chain-rule application of the same operator, ~5x fewer FP64 ops,
   * rounding-level (1e-16) differences. */
  int32_t exact_jacobian;
  /* Newton-loop solver: 0 auto (cluster-resident up to 32 envs when the
   * scene fits, else streaming), 1 streaming batched kernels, 2
   * cluster-resident: one env per <=16-CTA cluster, PCR state in shared
   * memory (error if the scene does not fit). */
  int32_t solver_mode;
  /* envs per wave (0 = auto: min(n_envs, 4096), split over two concurrent
   * lanes from 64 envs, lowered further if the workspaces plus all env state
   * would not fit in device memory). Persistent state is kept for every env;
   * waves alternate between the lanes' workspaces and streams. */
  int32_t wave_envs;
  /* SolverConfig.keep_matrix (solver.py:113, 511-518): keep the last
   * substep's Newton system readable through ss_export_system (forces the
   * streaming solver; one extra rhs copy per frame). */
  int32_t keep_matrix;
} ss_params;

/* Full per-environment state. Host pointers;
 * every array is [n_envs, <reference shape>] C-contiguous. NULL = skip. */
typedef struct ss_state_view {
  double* positions;      /* [n,P,3]  state.py:59-72  */
  double* velocities;     /* [n,P,3]  */
  double* body_pos;       /* [n,nb,3] state.py:98-109 */
  double* body_quat;      /* [n,nb,4] [w,x,y,z] */
  double* body_lin_vel;   /* [n,nb,3] */
  double* body_ang_vel;   /* [n,nb,3] world frame */
  double* lam_dist;       /* [n,nd]    solver.py:251-254 */
  double* lam_tetra;      /* [n,nt,6]  */
  double* lam_attach;     /* [n,na,3]  */
  double* lam_hinge;      /* [n,nh,5]  */
  double* tet_quats;      /* [n,nt,4]  constraints.py:146 */
  double* dist_dirs;      /* [n,nd,3]  constraints.py:70 */
  double* dist_scale;     /* [n,nd]    constraints.py:69 */
  double* strain_live;    /* [n,nch]   solver.py:247 */
  double* strain_target;  /* [n,nch]   solver.py:248 */
  double* pressures;      /* [n,nch]   pneumatics.py:92 */
  double* warm;           /* [n,nw,3]  solver.py:255,522 (lambda_n, lambda_f0, lambda_f1) */
  int32_t* warm_valid;    /* [n,nw]    1 = key ('wheel', body) present */
  double* time;           /* [n]       state.py:109 */
} ss_state_view;

/* StepStats (solver.py:142-151) for the last frame, per environment. */
typedef struct ss_env_stats {
  int32_t newton_iterations;
  int32_t pcr_iterations;
  int32_t contact_count;
  int32_t inverted_tets;
  double residual;
  int32_t finite;         /* 1 if positions finite after the frame */
  int32_t _pad;
} ss_env_stats;

typedef struct ss_handle ss_handle;

int ss_abi_version(void);
/* sha256 (hex) of the CUDA sources and this header the library was built
 * from; __graft_entry__.build() rebuilds when it differs from the tree. */
const char* ss_build_id(void);
const char* ss_last_error(void);
int ss_device_count(int* n);

/* ---- device-side scene construction ----
 * The link meshes of build_snake (snake.py:97-189): particle grid,
 * five-tet cells with TetraElement.from_positions (constraints.py:128-137)
 * and tetra_compliance (constraints.py:26-40), lumped masses, the cable
 * network and the frame mounts, for every link of every snake, built on the
 * device and copied into caller-owned host arrays (links concatenated in
 * the reference order; particle base = link * particles_per_link). Every
 * value is bitwise the reference's numpy result (ss_build.cuh). The rigid
 * bodies, hinges, wheels and attachment anchors (O(links)) stay on the host.
 */
typedef struct ss_link_mesh_params {
  int32_t sections, width_nodes, height_nodes;  /* S, W, H (scene.py:20-22) */
  int32_t n_links;                              /* all snakes' links       */
  double dx, dy, dz;          /* link_length/(S-1), link_width/(W-1), link_height/(H-1) */
  double half_width;          /* 0.5 * link_width                          */
  double youngs_modulus, poisson, density;
  double actuation_compliance, inextensible_compliance, structural_compliance;
  const double* origins;      /* [n_links, 3] (snake.py:314-316)          */
  const int32_t* channels;    /* [n_links, 2] left, right channel         */
} ss_link_mesh_params;
/* per-link counts: counts[0] particles, [1] tets, [2] cables, [3] mounts per face */
int ss_link_mesh_counts(const ss_link_mesh_params* p, int32_t* counts);
typedef struct ss_link_mesh_out {  /* host arrays, n_links x the per-link counts */
  double* positions;        /* [P, 3]   */
  double* masses;           /* [P]      */
  int32_t* tets;            /* [T, 4]   */
  double* rest_inv;         /* [T, 3, 3] */
  double* rest_volume;      /* [T]      */
  double* compliance;       /* [T, 6, 6] */
  int32_t* pairs;           /* [C, 2]   */
  double* rest;             /* [C]      */
  double* cable_compliance; /* [C]      */
  int32_t* kind;            /* [C]      */
  int32_t* channel;         /* [C]      */
  int32_t* mounts;          /* [n_links, 2, 6] start face, end face */
} ss_link_mesh_out;
int ss_build_link_meshes(const ss_link_mesh_params* p, int device, ss_link_mesh_out* out);

/* Simulator.__init__ (solver.py:157-265) for n_envs independent copies:
 * upload topology, allocate state for n_envs copies on `device`. The
 * initial state of every env is zero except quaternions (identity), dirs
 * (1,0,0), scale 1, strains 1 — the reference constructor defaults
 * (constraints.py:80-82,156-158; solver.py:247-255). Call ss_set_state. */
int ss_create(const ss_topology* topo, const ss_params* params, int n_envs,
              int device, ss_handle** out);
int ss_destroy(ss_handle* h);
int ss_num_envs(const ss_handle* h);

/* Write / read the persistent state of envs [env0, env0+n) — what the
 * reference keeps in sim.state, the lam_* arrays, tetras.quats,
 * distances.dirs/scale, the strain trackers, channels.pressures and _warm
 * (state.py:59-109, solver.py:247-255, constraints.py:69-70,146,
 * pneumatics.py:92). Host pointers, env-major; NULL fields are skipped. */
int ss_set_state(ss_handle* h, int env0, int n, const ss_state_view* s);
int ss_get_state(ss_handle* h, int env0, int n, ss_state_view* s);
/* Same with DEVICE pointers in the view (same env-major [n][...] layouts,
 * e.g. torch CUDA tensors): scattered / gathered on the device without a
 * host round trip; returns once the copies are complete. */
int ss_set_state_device(ss_handle* h, int env0, int n, const ss_state_view* view);
int ss_get_state_device(ss_handle* h, int env0, int n, ss_state_view* view);

/* Advance every env by n_frames frames of dt (Simulator.step, solver.py:296).
 * commands: host [n_frames, n_envs, n_channels/2] psi, or NULL (no tick,
 * like step(commands=None)). latency: ChannelBank.tick latency flag. */
int ss_step(ss_handle* h, const double* commands, int latency, int n_frames);

/* Same, commands already on the device ([n_frames, n_envs, links]). */
int ss_step_device(ss_handle* h, const double* d_commands, int latency, int n_frames);

/* On-device gait generator (snake.py:235-241): per env params[n][6] =
 * {amplitude psi, angular rate rad/s, phase offset, turn bias, time offset
 * t0 s, links per snake}; frame0[n] (nullable = 0) is the frame index the
 * env's gait clock starts at. ss_step_gait then advances every env with
 * a_i = clamp(sin(w (t0 + f dt) + alpha (i mod lps)) + bias, -1, 1) * A
 * computed inside the frame graph (no host commands), f += 1 per frame. */
int ss_set_gait(ss_handle* h, int env0, int n, const double* params, const int* frame0);
int ss_step_gait(ss_handle* h, int latency, int n_frames);
/* Simulator.set_channel_targets (solver.py:274-277): one pneumatic tick of
 * every env toward commands[n_envs][links] psi (ChannelBank.tick,
 * pneumatics.py:102-116) without stepping; the strain target follows at the
 * next ss_step (solver.py:299-301). */
int ss_set_channel_targets(ss_handle* h, const double* commands, int latency);
/* Read back the gait parameters (same layout as ss_set_gait) and each env's
 * current gait frame counter (frames stepped since its clock started). */
int ss_get_gait(ss_handle* h, int env0, int n, double* params, int* frame);

int ss_get_stats(ss_handle* h, int env0, int n, ss_env_stats* out);

/* Episode resets on the device: ss_capture_init
 * stores env `env`'s full state (every ss_state_view field) as the reset
 * template; ss_reset_envs writes it into envs env_ids[0..n) and restarts
 * their gait clocks. pos_sigma / vel_sigma > 0 add deterministic N(0,
 * sigma^2) perturbations to the live particles' positions / velocities,
 * drawn per (seed, env id, element) so an env's draw does not depend on
 * which other envs reset with it. */
int ss_capture_init(ss_handle* h, int env);
int ss_reset_envs(ss_handle* h, const int* env_ids, int n, uint64_t seed, double pos_sigma,
                  double vel_sigma);

/* The last substep's Newton system of one env (keep_matrix handles only),
 * in the reference's snapshot layout (solver.py:511-518) for
 * Simulator.last_system / export_system (solver.py:548-581): per-family
 * Jacobian blocks and DOF indices, static rows in reference row order,
 * contact slots uncompacted (present flags; present slots in slot order are
 * the reference's contacts), the mass inverse. Host pointers, caller-owned. */
typedef struct {
  double* dist_vals;   /* [nd][1][6] */
  int32_t* dist_idx;   /* [nd][6] */
  double* tet_vals;    /* [nt][6][12] */
  int32_t* tet_idx;    /* [nt][12] */
  double* att_vals;    /* [na][3][9] */
  int32_t* att_idx;    /* [na][9] */
  double* hinge_vals;  /* [nh][5][12] */
  int32_t* hinge_idx;  /* [nh][12] */
  double* slot_vals;   /* [ns][3][6] normal, friction t1, friction t2 */
  int32_t* slot_idx;   /* [ns][6] */
  int32_t* slot_present; /* [ns] */
  double* rhs_static;  /* [m_static] */
  double* dyn_static;  /* [m_static] (0 on tet rows: E_tet enters as blocks) */
  double* rhs_slot;    /* [ns][3] */
  double* dyn_slot;    /* [ns][3] */
  double* minv_diag;   /* [ndof] (angular entries 0) */
  double* ang_inv;     /* [nb][3][3] */
} ss_system_view;
int ss_export_system(ss_handle* h, int env, ss_system_view* out);
/* center_of_mass (state.py:285-292) per env -> host [n,3]. */
int ss_get_com(ss_handle* h, int env0, int n, double* out);
/* Rollout observables of envs [env0, env0+n) into host out[n][4 + nb]:
 * centre of mass (3, state.py:285-292), kinetic energy (state.py:271-282)
 * and the heading yaw of every body (snake.py:185-188; link curvature and
 * head yaw follow from the frame bodies' yaws, snake.py:212-232).
 * Replaces the per-frame host readbacks of harness.py:183-205. */
int ss_observe(ss_handle* h, int env0, int n, double* out);
int ss_synchronize(ss_handle* h);
/* cudaStream_t of the handle, as void* (for timing with CUDA events). */
void* ss_stream(ss_handle* h);
/* Number of kernel launches one frame issues (for bench accounting). */
int ss_launches_per_frame(ss_handle* h);
/* Bytes of device memory held by the handle. */
int64_t ss_device_bytes(ss_handle* h);
/* info[0] 1 if the cluster-resident solver is used, info[1] CTAs per
 * cluster, info[2] shared bytes per CTA, info[3] env lanes per wave,
 * info[4] number of waves, info[5] 1 if the PCR loop's J^T z gather is
 * fused (k_gather_fused), info[6] its particle blocks, info[7] its chunks
 * over all blocks, info[8] clusters per environment (> 1: a multi-component
 * scene with one cluster per component, dot products combined through
 * global memory), info[9] nonzero if a cross-cluster reduction faulted
 * (a cluster never arrived or the plan's reduction count was exceeded).
 * info must hold 10 ints. */
int ss_solver_info(ss_handle* h, int* info);
/* Debug: with SS_GUARD=1 set at ss_create every device array is followed by
 * a 0xA5 guard band; *bad_bytes = guard bytes changed since (an out-of-
 * bounds write), or -1 when the handle has no guards. */
int ss_check_guards(ss_handle* h, int64_t* bad_bytes);
/* Debug: clock64 phase stamps of one PCR iteration of the cluster solver
 * (handle created with SS_CLUSTER_STAMPS=n set): out[16 n], 16 per CTA for
 * the first n (<= 16) CTAs. */
int ss_cluster_stamps(ss_handle* h, long long* out);
/* Kernel names (static strings) of the step, in profiler slot order;
 * returns the number of kernels. */
int ss_kernel_names(const char** names, int cap);
/* Run n_frames like ss_step but un-graphed, every launch bracketed by CUDA
 * events on the handle's stream; accumulates per-kernel milliseconds and
 * launch counts into slot order of ss_kernel_names. */
int ss_profile_frames(ss_handle* h, const double* commands, int latency, int n_frames,
                      double* ms_total, int* launches);

/* ---------------------------------------------------------------------
 * Kernel-level ABI: one call per reference backend function, on device
 * pointers, same shapes and semantics (kernels/numba_backend.py). Block
 * kernels are bitwise equal to the numba kernels (no FMA contraction,
 * reference accumulation order). stream may be NULL (default stream).
 * ------------------------------------------------------------------- */
/* numba_backend.py:31-40 */
int ssk_block_forward(const int32_t* dof_idx, const double* vals, int n, int r,
                      int k, const double* u, double* out_rows, void* stream);
/* numba_backend.py:43-52 (accumulates into y; reference scatter order) */
int ssk_block_transpose(const int32_t* dof_idx, const double* vals, int n,
                        int r, int k, const double* x_rows, double* y,
                        int ndof, void* stream);
/* numba_backend.py:55-65 */
int ssk_block_rowdiag(const int32_t* dof_idx, const double* vals, int n, int r,
                      int k, const double* minv_diag, double* out_rows,
                      void* stream);
/* numba_backend.py:68-82 */
int ssk_minv_apply(const double* minv_diag, const double* ang_inv, int nb,
                   int body_dof0, const double* u, double* out, int ndof,
                   void* stream);
/* numba_backend.py:85-94 */
int ssk_ereg_apply(const double* vals6, const double* x_rows, double* out_rows,
                   int n, void* stream);
/* numba_backend.py:97-102 (deterministic tree order, not sequential) */
int ssk_dot(const double* a, const double* b, int n, double* out_host,
            void* stream);
/* numba_backend.py:105-120 */
int ssk_eval_distance(const double* pos, const int32_t* pairs, const double* rest,
                      const double* scale, double* dirs, double* out_res, int n,
                      void* stream);
/* numba_backend.py:137-312; returns inverted count in *n_inverted */
int ssk_eval_tetra(const double* pos, const int32_t* tets, const double* rest_inv,
                   double* quats, double tol, int maxiter, double* out_res,
                   double* out_vals, int n, int* n_inverted, void* stream);

/* Device memory helpers for FFI callers without a CUDA runtime of their own
 * (the kernel-level ABI above takes device pointers). */
int ssk_malloc(void** ptr, int64_t bytes, int device);
int ssk_free(void* ptr);
int ssk_memcpy(void* dst, const void* src, int64_t bytes, int kind); /* 1 H2D, 2 D2H, 3 D2D */

#ifdef __cplusplus
}
#endif
#endif /* SOFTSNAKE_B200_H */
