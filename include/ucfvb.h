/*
 * ucfvb.h -- C ABI of the B200-native hybrid NAD stage pass (arXiv 2510.25906).
 *
 * Drop-in boundary for `class ucfv::Solver` (/root/reference/proj/include/ucfv/solver.hpp:52-100).
 * Every entry point below names the reference interface it replaces. The ABI
 * is plain C: opaque handles, plain pointers and sizes, int status codes.
 *
 * Status codes (ucfvb_status): 0 ok; 1 non-physical state (the reference's
 * NonPhysicalError, euler.hpp:18-20); 2 invalid argument (std::invalid_argument
 * / MeshError); 3 CUDA runtime failure; 4 unsupported feature (e.g. a boundary
 * condition that is an arbitrary std::function and cannot run on the device).
 * ucfvb_last_error() returns the message of the last failing call on a handle
 * (or the thread's last global message for calls without a handle).
 *
 * Memory/threading contract: host arrays are owned by the caller and copied
 * in/out; device state lives in the handle between calls; every call is
 * blocking at return (kernels are stream-ordered internally); a handle is not
 * reentrant (same as ucfv::Solver).
 */
#ifndef UCFVB_H
#define UCFVB_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define UCFVB_ABI_VERSION 1

enum ucfvb_status {
  UCFVB_OK = 0,
  UCFVB_NONPHYSICAL = 1,
  UCFVB_INVALID = 2,
  UCFVB_CUDA = 3,
  UCFVB_UNSUPPORTED = 4
};

/* SchemeMode (solver.hpp:18) */
enum ucfvb_mode { UCFVB_LINEAR = 0, UCFVB_MUSCL = 1, UCFVB_CWENOZ = 2, UCFVB_HYBRID = 3, UCFVB_FIRST = 4 };
/* LimiterKind (solver.hpp:19) */
enum ucfvb_limiter { UCFVB_BARTH_JESPERSEN = 0, UCFVB_VENKATAKRISHNAN = 1 };
/* RiemannKind (solver.hpp:20) */
enum ucfvb_riemann { UCFVB_HLLC = 0, UCFVB_HLL = 1 };
/* SiExponent (stencil.hpp:12) */
enum ucfvb_si_exponent { UCFVB_SI_PAPER = 0, UCFVB_SI_LEGACY = 1 };
/* time integrators: SSPRK(5,4) = Solver::advance (time_integrator.cpp:42-74);
 * SSPRK3 (Shu-Osher) is the BASELINE.json integrator the reference lacks. */
enum ucfvb_rk { UCFVB_RK54 = 0, UCFVB_RK3 = 1 };
/* Scheme labels (detector.hpp:13): 0 Linear, 1 CWENOZ, 2 MUSCL, 3 FirstOrder */
enum ucfvb_scheme { UCFVB_SCHEME_LINEAR = 0, UCFVB_SCHEME_CWENOZ = 1, UCFVB_SCHEME_MUSCL = 2, UCFVB_SCHEME_FIRST = 3 };
/* boundary conditions the device can evaluate: bc_outflow / bc_wall / bc_fixed
 * (solver.cpp:22-34). Arbitrary BoundaryFn lambdas are rejected (UNSUPPORTED). */
enum ucfvb_bc_kind { UCFVB_BC_NONE = 0, UCFVB_BC_OUTFLOW = 1, UCFVB_BC_WALL = 2, UCFVB_BC_FIXED = 3 };

/* NadMargins (detector.hpp:24-31) */
typedef struct ucfvb_margins {
  double alpha_m, beta_m, alpha_w, beta_w, kappa, deact_n;
} ucfvb_margins;

/* SolverOptions (solver.hpp:29-43); ucfvb_options_default() gives the reference defaults. */
typedef struct ucfvb_options {
  int32_t order;
  int32_t mode;
  int32_t limiter;
  int32_t riemann;
  ucfvb_margins margins;
  double lambda1p;
  double weno_eps;
  double weno_b;
  double cfl;
  double venkat_kappa;
  int32_t si_exponent;
  int32_t detect_every_stage;
  double gamma;
  /* B200 extras (no reference counterpart) */
  int32_t keep_taps;   /* 1: keep final per-cell dofs for ucfvb_get_dofs (debug tap) */
  int32_t use_graphs;  /* 1: capture RK steps in CUDA graphs */
} ucfvb_options;

/* One boundary patch binding: patch name -> kind (+ state for FIXED). */
typedef struct ucfvb_bc {
  const char* patch;
  int32_t kind;
  double state[4];
} ucfvb_bc;

/*
 * Flattened `ucfv::Mesh` (mesh.hpp:17-111). Cell i owns faces
 * cell_faces[cell_face_ptr[i] .. cell_face_ptr[i+1]) in the reference's
 * cell order; cell vertices likewise. Per-face arrays follow `Face`.
 */
typedef struct ucfvb_mesh_view {
  int32_t n_vertices, n_cells, n_faces, n_qp, n_patches;
  double period_x, period_y;
  const double* vertices;        /* [n_vertices][2] */
  const int32_t* cell_vtx_ptr;   /* [n_cells+1] */
  const int32_t* cell_vtx;
  const int32_t* cell_face_ptr;  /* [n_cells+1] */
  const int32_t* cell_faces;
  const double* cell_centroid;   /* [n_cells][2] */
  const double* cell_area;       /* [n_cells] */
  const double* cell_h;          /* [n_cells] h_c = sqrt(area) */
  const int32_t* face_vtx;       /* [n_faces][2] */
  const int32_t* face_left;      /* [n_faces] */
  const int32_t* face_right;     /* [n_faces] -1 on boundary */
  const double* face_normal;     /* [n_faces][2] */
  const double* face_length;     /* [n_faces] */
  const double* face_midpoint;   /* [n_faces][2] */
  const double* face_qp;         /* [n_faces][n_qp][2] */
  const double* face_qw;         /* [n_faces][n_qp] */
  const int32_t* face_patch;     /* [n_faces] -1 interior */
  const int32_t* face_partner;   /* [n_faces] periodic partner or -1 */
  const int32_t* face_shift;     /* [n_faces][2] shift_ix, shift_iy */
  const int32_t* face_partner_qp;/* [n_faces][n_qp] (-1 when not periodic) */
  const char* const* patch_names;/* [n_patches] */
} ucfvb_mesh_view;

/*
 * Flattened `ucfv::StencilSet` (stencil.hpp:36-50), cell c:
 *   central entries   central[3*j..3*j+2] = (cell, px, py), j in [central_ptr[c], central_ptr[c+1])  (self first, M+1 entries)
 *   pinv              K x M row-major at pinv[pinv_off[c] ..]
 *   pinv_linear       2 x M row-major at pinv_lin[pinv_lin_off[c] ..]
 *   directional       stencils s in [dir_ptr[c], dir_ptr[c+1]); members of s are
 *                     dir_members[dir_member_ptr[s] .. dir_member_ptr[s+1]) (indices into central, self 0 first);
 *                     pinv_dir 2 x (len-1) at pinv_dir[pinv_dir_off[s] ..]
 *   oi                K x K at oi[c*K*K ..]
 *   cell_phi          Q_c x K at phi[phi_off[c] ..], Q_c = qp_ptr[c+1]-qp_ptr[c]
 *   cell_qp_slot      qp_slot[qp_ptr[c] .. qp_ptr[c+1])  slot = (face*n_qp+q)*2+side
 */
typedef struct ucfvb_stencil_view {
  int32_t order, K, n_qp, si_exponent, n_cells, n_dir_stencils;
  const int64_t* central_ptr;
  const int32_t* central;
  const int64_t* pinv_off;
  const double* pinv;
  const int64_t* pinv_lin_off;
  const double* pinv_lin;
  const int64_t* dir_ptr;
  const int64_t* dir_member_ptr;
  const int32_t* dir_members;
  const int64_t* pinv_dir_off;
  const double* pinv_dir;
  const double* oi;
  const int64_t* qp_ptr;
  const int64_t* phi_off;
  const double* phi;
  const int32_t* qp_slot;
} ucfvb_stencil_view;

typedef struct ucfvb_solver ucfvb_solver;
typedef struct ucfvb_mesh ucfvb_mesh;
typedef struct ucfvb_stencils ucfvb_stencils;

/* ---- version / errors --------------------------------------------------- */
int32_t ucfvb_abi_version(void);
/* message of the last failing call on `h` (h may be NULL: thread-global message) */
const char* ucfvb_last_error(const ucfvb_solver* h);

/* ---- options ------------------------------------------------------------ */
/* SolverOptions{} defaults (solver.hpp:29-43, detector.hpp:24-31) */
void ucfvb_options_default(ucfvb_options* opt);

/* ---- host setup (the callers on either side of the path) */
/* generate_structured_tri (mesh.cpp:137-157) + interior-vertex jitter of
 * +-jitter*h per coordinate from `seed` (splitmix64) + tag_rect_patches
 * (mesh.cpp:119-135) + pair_periodic (mesh.cpp:368-446) on `periodic_axis`
 * (0 none, 1 x, 2 y, 3 both) with tolerance `tol`. diagonal: 0 uniform, 1 alternating. */
int32_t ucfvb_mesh_structured_tri(int32_t nx, int32_t ny, double x0, double y0, double x1, double y1,
                                  int32_t diagonal, double jitter, uint64_t seed, int32_t periodic_axis,
                                  double tol, int32_t n_qp, ucfvb_mesh** out);
/* generate_structured_quad (mesh.cpp:160-170) + pairing */
int32_t ucfvb_mesh_structured_quad(int32_t nx, int32_t ny, double x0, double y0, double x1, double y1,
                                   int32_t periodic_axis, double tol, int32_t n_qp, ucfvb_mesh** out);
int32_t ucfvb_mesh_get_view(const ucfvb_mesh* m, ucfvb_mesh_view* out);
void ucfvb_mesh_free(ucfvb_mesh* m);

/* build_stencils (stencil.cpp:192-284), multithreaded; n_threads <= 0: all cores */
int32_t ucfvb_build_stencils(const ucfvb_mesh_view* mesh, int32_t order, int32_t si_exponent,
                             int32_t n_threads, ucfvb_stencils** out);
int32_t ucfvb_stencils_get_view(const ucfvb_stencils* s, ucfvb_stencil_view* out);
void ucfvb_stencils_free(ucfvb_stencils* s);

/* project_initial (cases.cpp:62-76) of a built-in initial condition at the
 * quadrature degree `degree`; u_out is [n_cells][4].
 * ic: 0 = isentropic vortex ic_vortex(scale*x, scale*y) (cases.cpp:14-27),
 *         params[0] = scale;
 *     1 = shock into a sine wave (BASELINE config 2): params = {x_shock,
 *         rho_L, u_L, v_L, p_L, amp, wavenumber};
 *     2 = random four-quadrant Riemann data (BASELINE config 3): params =
 *         {x_split, y_split, noise}, quadrant states drawn from `seed`;
 *         after projection every conserved value is scaled by
 *         (1 + noise*(2U-1)) with U from splitmix64(seed, 4*cell+var). */
int32_t ucfvb_project_initial(const ucfvb_mesh_view* mesh, int32_t ic, const double* params,
                              int32_t n_params, uint64_t seed, int32_t degree, double gamma,
                              int32_t n_threads, double* u_out);

/* ---- solver: Solver(mesh, opt, bcs) (solver.cpp:36-74) ------------------ */
int32_t ucfvb_create(const ucfvb_mesh_view* mesh, const ucfvb_stencil_view* stencils,
                     const ucfvb_options* opt, const ucfvb_bc* bcs, int32_t n_bcs, int32_t device,
                     ucfvb_solver** out);
void ucfvb_destroy(ucfvb_solver* h);

/* Solver::state() write / read (solver.hpp:56-57): u is [n_cells][4] AoS */
int32_t ucfvb_set_state(ucfvb_solver* h, const double* u);
int32_t ucfvb_get_state(ucfvb_solver* h, double* u);

/* Solver::max_stable_dt (solver.cpp:103-111) */
int32_t ucfvb_max_stable_dt(ucfvb_solver* h, double* dt);

/* Solver::advance (solver.cpp:381-387): one step of `rk` from t, in place */
int32_t ucfvb_advance(ucfvb_solver* h, double dt, double t, int32_t rk);

/* Solver::compute_residual (solver.cpp:316-379): out = dU/dt of host field u */
int32_t ucfvb_compute_residual(ucfvb_solver* h, const double* u, double t, double* out);

/* run_simulation's stepping loop (run.cpp:97-132) kept on the device: n_steps
 * of dt = min(max_stable_dt, t_end - t) then advance; t is device-resident.
 * Writes the final t; census_out (nullable) receives [n_steps][4] int64
 * first-stage label counts per step (run.cpp:110-116). */
int32_t ucfvb_run_steps(ucfvb_solver* h, int32_t n_steps, int32_t rk, double t0, double t_end,
                        double* t_out, int64_t* census_out);

/* Host state in, host state out: u_in -> n_steps steps of ucfvb_run_steps
 * (dt = max_stable_dt() each step) -> u_out, with a single synchronisation
 * (state() + the advance loop of run_simulation, run.cpp:96-132, for callers
 * that keep the state on the host). u_in / u_out ([n_cells][4]) should be
 * pinned for asynchronous PCIe transfers; u_out may alias u_in. On failure the
 * device state is the failing step's input (as ucfvb_run_steps). */
int32_t ucfvb_advance_host(ucfvb_solver* h, const double* u_in, double* u_out, int32_t n_steps, int32_t rk,
                           double t0, double* t_out);
/* ucfvb_advance_host over n_batch independent states of the same mesh (an
 * ensemble of run_simulation loops, run.cpp:87-132, one per initial state):
 * entry i is u_in[i] -> n_steps steps -> u_out[i], t_out[i] (nullable) its
 * final time. The entries are pipelined: the upload of entry i+1 and the
 * download of entry i-1 run on copy streams while entry i is stepped, so the
 * PCIe transfers leave the critical path; results are bit-identical to
 * n_batch ucfvb_advance_host calls. Buffers should be pinned; u_out[i] may
 * alias u_in[i] but no other entry's input. One synchronisation, at the end.
 * On failure (the message names the entry) later entries are not computed. */
int32_t ucfvb_advance_host_batch(ucfvb_solver* h, int32_t n_batch, const double* const* u_in,
                                 double* const* u_out, int32_t n_steps, int32_t rk, double t0, double* t_out);
/* ucfvb_run_steps plus each step's dt (run.cpp:99-112 CensusRow::dt): dt_out
 * (nullable) receives [n_steps] doubles; step k's end time is t0 + dt_0 + ...
 * + dt_k summed in step order, exactly as run_simulation's `t += dt`. */
int32_t ucfvb_run_steps_log(ucfvb_solver* h, int32_t n_steps, int32_t rk, double t0, double t_end,
                            double* t_out, int64_t* census_out, double* dt_out);

/* run_simulation's loop with its own termination (run.cpp:96-132): steps
 * `dt = min(max_stable_dt, t_end - t); advance` while t < t_end - 1e-14 t_end,
 * at most max_steps, device-resident (batches of graph launches, the loop
 * condition is evaluated on the device). n_steps_out receives the steps taken;
 * census_out [max_steps][4] / dt_out [max_steps] (nullable) their rows. */
int32_t ucfvb_run_until(ucfvb_solver* h, int32_t max_steps, int32_t rk, double t0, double t_end, double* t_out,
                        int32_t* n_steps_out, int64_t* census_out, double* dt_out);

/* CensusRow / TimingRow (run.hpp:15-25) */
typedef struct ucfvb_census_row {
  int32_t step;
  double t, dt;
  int64_t counts[4]; /* Linear, CWENOZ, MUSCL, FirstOrder */
} ucfvb_census_row;
typedef struct ucfvb_timing_row {
  int32_t step;
  double wall;
  double reconstruct, detect, weights, flux; /* per-step PhaseTimes deltas, seconds */
} ucfvb_timing_row;

/* Run outputs, byte-identical to the reference writers (every double "%.17g"):
 * write_field_snapshot (run.cpp:160-190; legacy-VTK ASCII with density,
 * pressure, velocity and the scheme label; state [n_cells][4], labels from
 * ucfvb_get_step_labels), write_census_csv (run.cpp:192-202),
 * write_timing_csv (run.cpp:204-213). Host-only: no device needed. */
int32_t ucfvb_write_field_snapshot(const ucfvb_mesh_view* mesh, const double* state, const uint8_t* labels,
                                   double gamma, const char* path);
int32_t ucfvb_write_census_csv(const ucfvb_census_row* rows, int32_t n_rows, int64_t n_cells, const char* path);
int32_t ucfvb_write_timing_csv(const ucfvb_timing_row* rows, int32_t n_rows, const char* path);

/* Solver::step_labels (solver.hpp:66) and the current-stage labels */
int32_t ucfvb_get_step_labels(ucfvb_solver* h, uint8_t* labels);
int32_t ucfvb_get_labels(ucfvb_solver* h, uint8_t* labels);
/* label counts of step_labels: Linear, CWENOZ, MUSCL, FirstOrder */
int32_t ucfvb_get_census(ucfvb_solver* h, int64_t counts[4]);
/* Troubled-cell class lists (an implementation choice; results are identical):
 * policy 0 = 32-cell chunk lists (k_troubled_split), 1 = dense per-cell lists
 * (k_troubled_cells), 2 = adaptive (default): after every synchronising call
 * the lists of the next ones follow the last stage's chunk fill -- chunks when
 * the troubled cells fill >= 3/4 of the chunks that hold them, else per-cell
 * lists (the first call of a solver uses chunks). Stats of
 * the last synchronised stage's lists: CWENOZ cells, MUSCL cells, CWENOZ
 * chunks, MUSCL chunks, 1 if per-cell lists are in use (cells whose
 * reconstruction fell back to first order stay counted in their list).
 * No reference counterpart. */
int32_t ucfvb_set_list_policy(ucfvb_solver* h, int32_t policy);
int32_t ucfvb_get_list_stats(ucfvb_solver* h, int64_t stats[5]);
/* NAD threshold ties (north_star tie band): cells whose detector value lies
 * within 1e-12 (relative) of a threshold, summed over every detecting stage
 * of the last advance / compute_residual / run call (a cell counts once per
 * stage it ties in) */
int32_t ucfvb_get_nad_ties(ucfvb_solver* h, int64_t* ties);

/* parity taps: val_left_/val_right_ in [face*n_qp+q][4] order (solver.hpp:91),
 * dofs_ in [cell][k][4] order (requires keep_taps) */
int32_t ucfvb_get_face_values(ucfvb_solver* h, double* left, double* right);
int32_t ucfvb_get_dofs(ucfvb_solver* h, double* dofs);

/* PhaseTimes (solver.hpp:45-50) in seconds: reconstruct, detect, weights, flux.
 * Accumulated with CUDA events when timing is enabled (off by default). */
int32_t ucfvb_set_phase_timing(ucfvb_solver* h, int32_t enabled);
int32_t ucfvb_get_phase_times(ucfvb_solver* h, double times[4]);

/* sizes */
int32_t ucfvb_n_cells(const ucfvb_solver* h);
int32_t ucfvb_n_faces(const ucfvb_solver* h);
int32_t ucfvb_n_qp(const ucfvb_solver* h);

/* ---- domain decomposition (multi-GPU) --------------------
 * A subdomain is rank r's part of a partitioned mesh: its owned cells plus
 * the stencil-depth halo every owned residual depends on (face neighbours to
 * depth 2 for spread + NAD, then central stencils and face neighbours of those),
 * as a self-contained local mesh + stencil set. Local cells are ordered
 * [owned interior | owned cells some peer holds | halo grouped by owner rank],
 * each group in global order: each peer's halo block is one contiguous receive
 * range, and the owned cells that are sent come last, so a stage updates them
 * first and exchanges the halo while it updates the interior. Halo cells beyond the
 * classification layers carry inert (zero-weight) stencils; faces leaving the
 * local set belong to the local patch "__halo__" and are never integrated. */
/* recursive coordinate bisection of cell centroids into n_parts balanced parts */
int32_t ucfvb_partition_rcb(const ucfvb_mesh_view* mesh, int32_t n_parts, int32_t* part);
typedef struct ucfvb_subdomain ucfvb_subdomain;
int32_t ucfvb_subdomain_build(const ucfvb_mesh_view* mesh, const ucfvb_stencil_view* stencils,
                              const int32_t* part, int32_t n_parts, int32_t rank, ucfvb_subdomain** out);
int32_t ucfvb_subdomain_views(const ucfvb_subdomain* s, ucfvb_mesh_view* mesh, ucfvb_stencil_view* stencils);
/* n_owned, n_local, n_peers */
int32_t ucfvb_subdomain_info(const ucfvb_subdomain* s, int32_t* n_owned, int32_t* n_local, int32_t* n_peers);
/* owned cells [0, n_interior) that no peer holds (never sent) */
int32_t ucfvb_subdomain_interior(const ucfvb_subdomain* s, int32_t* n_interior);
/* global cell id of every local cell [n_local] */
int32_t ucfvb_subdomain_global_ids(const ucfvb_subdomain* s, int32_t* gid);
/* peer i: its rank, how many owned cells go to it, and the local range
 * [recv_begin, recv_begin + n_recv) its owned cells fill */
int32_t ucfvb_subdomain_peer(const ucfvb_subdomain* s, int32_t i, int32_t* rank, int32_t* n_send,
                             int32_t* n_recv, int32_t* recv_begin);
/* local ids (owned cells) sent to peer i, in the peer's receive order */
int32_t ucfvb_subdomain_send_list(const ucfvb_subdomain* s, int32_t i, int32_t* local_ids);
void ucfvb_subdomain_free(ucfvb_subdomain* s);

/* Solver on a subdomain (ucfvb_create on the subdomain views + the owned
 * count): residuals, RK updates, dt and census cover owned cells only. */
int32_t ucfvb_create_sub(const ucfvb_subdomain* sub, const ucfvb_options* opt, const ucfvb_bc* bcs,
                         int32_t n_bcs, int32_t device, ucfvb_solver** out);
/* Attach an NCCL communicator (unique id from ucfvb_nccl_unique_id on rank 0,
 * broadcast by the caller): every RK stage then ends with a grouped
 * ncclSend/ncclRecv of the stage state's halo, max_stable_dt/run_steps use a
 * min all-reduce, and run_steps' census a sum all-reduce. */
int32_t ucfvb_nccl_unique_id(uint8_t id[128]);
int32_t ucfvb_attach_nccl(ucfvb_solver* h, const uint8_t id[128], int32_t rank, int32_t world);

/* In-process loopback group: the n subdomain solvers of one n-part partition
 * (parts[i] created with ucfvb_create_sub on rank i's subdomain, all on one
 * device), stepped together with the same schedule a rank runs -- sent cells
 * first, the halo exchange forked onto an exchange stream while the interior
 * is updated -- with device-to-device copies (one cudaMemcpyAsync per peer
 * block) as the transport and the dt min / error word reduced by kernels
 * across the group; one CUDA graph captures a step of all parts. For testing
 * the multi-GPU exchange schedule on a single device. The parts must outlive
 * the group and are not stepped on their own while it exists. */
typedef struct ucfvb_group ucfvb_group;
int32_t ucfvb_group_create(ucfvb_solver* const* parts, int32_t n, ucfvb_group** out);
/* n_steps RK steps of every part with device dt (run_steps); on a failure
 * every part keeps the failing step's input and the call returns its status */
int32_t ucfvb_group_run_steps(ucfvb_group* g, int32_t n_steps, int32_t rk, double t0, double* t_out);
int64_t ucfvb_group_launch_count(const ucfvb_group* g);
void ucfvb_group_free(ucfvb_group* g);

/* ---- device-resident entry points (benchmark "value" leg) ---------------- */
/* device pointer to the [n_cells][4] state; valid until the next call */
int32_t ucfvb_state_device_ptr(ucfvb_solver* h, double** dptr);
/* CUDA stream the handle launches on (as void* = cudaStream_t) */
int32_t ucfvb_stream(ucfvb_solver* h, void** stream);
/* number of kernel launches issued by the last ucfvb_run_steps / advance call */
int64_t ucfvb_launch_count(const ucfvb_solver* h);

#ifdef __cplusplus
}
#endif

#endif /* UCFVB_H */
