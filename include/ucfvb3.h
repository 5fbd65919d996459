/*
 * ucfvb3.h -- C ABI of the 3D stage pass (BASELINE configs 4-5).
 *
 * The reference solver is 2D only (`Vec2`, `kNumVars = 4`,
 * /root/reference/proj/include/ucfv/euler.hpp:14-16); its `count_dofs` already
 * admits d = 3 (src/basis.cpp:25-31). This header generalises the same
 * drop-in boundary -- `class ucfv::Solver` (include/ucfv/solver.hpp:52-100) --
 * to three dimensions and five conserved variables (rho, rho u, rho v, rho w, E):
 *
 *   ucfvb3_create            <-> Solver(mesh, opt, bcs)             (solver.cpp:36-74)
 *   ucfvb3_set/get_state     <-> Solver::state()                    (solver.hpp:61)
 *   ucfvb3_max_stable_dt     <-> Solver::max_stable_dt()            (solver.cpp:103-111)
 *   ucfvb3_advance           <-> Solver::advance()                  (solver.cpp:381-387)
 *   ucfvb3_compute_residual  <-> Solver::compute_residual()         (solver.cpp:316-379)
 *   ucfvb3_get_labels        <-> Solver::step_labels()              (solver.cpp:371-374)
 *
 * The 3D discretisation (mesh, face rules, basis, directional cones, 3D HLLC)
 * is defined by this builder; see DESIGN.md §11. There is no reference to pin
 * it against ("parity unpinned" for 3D): the oracle is oracle/ucfv3_port.c,
 * a plain-C restatement of the reference's 2D stage functions in 3D.
 *
 * Meshes are fully periodic boxes (what configs 4-5 need), so every face is
 * interior: face f separates face_left[f] and face_right[f]; its quadrature
 * points are stored in the left cell's frame. Status codes and options are
 * those of ucfvb.h.
 */
#ifndef UCFVB3_H
#define UCFVB3_H

#include <stdint.h>

#include "ucfvb.h"

#ifdef __cplusplus
extern "C" {
#endif

#define UCFVB3_NV 5

enum ucfvb3_cell_kind { UCFVB3_HEX = 0, UCFVB3_TET = 1 };
/* built-in initial conditions for ucfvb3_project_initial */
enum ucfvb3_ic {
  UCFVB3_IC_TGV = 0,          /* Taylor-Green vortex at Mach params[0] (config 4) */
  UCFVB3_IC_RANDOM_PHASE = 1, /* solenoidal random-phase field, E(k) ~ k^4 exp(-2 (k/k0)^2) (config 5):
                                 params = {rms Mach, k0, kmax}; point value at the centroid */
  UCFVB3_IC_UNIFORM = 2,      /* uniform state params = {rho, u, v, w, p} */
  UCFVB3_IC_BLAST = 3         /* params = {x, y, z, radius, rho_in, p_in, rho_out, p_out} at rest */
};

typedef struct ucfvb3_mesh ucfvb3_mesh;
typedef struct ucfvb3_stencils ucfvb3_stencils;
typedef struct ucfvb3_solver ucfvb3_solver;

/*
 * Flattened periodic 3D mesh. Each lattice cube ((k*ny + j)*nx + i) holds
 * n_types cells (hex: 1; tet: the 6 Freudenthal tetrahedra), numbered as
 * cell_order says. Faces per cell nf (hex 6, tet 4),
 * quadrature points per face nq.
 */
typedef struct ucfvb3_mesh_view {
  int32_t kind, nx, ny, nz, n_types;
  int32_t n_cells, n_faces, nf, nq, nvc;
  /* 0: cell = cube * n_types + type; 1 (tetrahedra, nx*ny*nz % 32 == 0): cubes in
   * blocks of 32, type-major inside a block: cell = ((cube/32)*6 + type)*32 + cube%32,
   * so every 32-cell chunk holds a single type */
  int32_t cell_order;
  double period[3];
  const double* cell_vtx;       /* [n_cells][nvc][3] vertex coordinates, unwrapped around the cell */
  const double* cell_centroid;  /* [n_cells][3] */
  const double* cell_volume;    /* [n_cells] */
  const double* cell_h;         /* [n_cells] h_c = volume^(1/3) */
  const int32_t* cell_faces;    /* [n_cells][nf] */
  const int32_t* cell_nbr;      /* [n_cells][nf] cell across each local face */
  const int32_t* cell_nbr_shift;/* [n_cells][nf][3] periods to add to the neighbour's coordinates */
  const int8_t* cell_side;      /* [n_cells][nf] 0: the cell is the face's left cell, 1: right */
  const int32_t* face_left;     /* [n_faces] */
  const int32_t* face_right;    /* [n_faces] */
  const double* face_qp;        /* [n_faces][nq][3] points in the left cell's frame */
  const double* face_normal;    /* [n_faces][nq][3] unit normal, outward of the left cell */
  const double* face_wa;        /* [n_faces][nq] rule weight x area element */
  const double* face_vtx;       /* [n_faces][4][3] face vertices in the left cell's frame (tri: 3 used), outward CCW */
} ucfvb3_mesh_view;

/*
 * Operator data, uniform sizes. Operator rows: op_index[c] selects the row of
 * pinv / pinv_lin / dir_members / pinv_dir / oi / phi used by cell c (the
 * cell itself, or its lattice class when built with lattice_classes = 1 on an
 * unjittered mesh: translated cells share identical operators).
 *   central     [n_cells][M+1] cell ids, self first (BFS rings, stencil.cpp:31-71)
 *   pinv        [n_ops][K][M]   (stencil.cpp:152-166)
 *   pinv_lin    [n_ops][3][M]   QR of the first three columns (stencil.cpp:218-224)
 *   dir_members [n_ops][nf][MD] indices 1..M into central (stencil.cpp:73-117, cones instead of sectors)
 *   pinv_dir    [n_ops][nf][3][MD]
 *   oi          [n_ops][K][K]   (stencil.cpp:168-190)
 *   phi         [n_ops][Q][K]   Q = nf*nq, cell-local face order, qp order (stencil.cpp:262-281)
 *   qp_slot     [n_cells][Q]    (face*nq + q)*2 + side
 */
typedef struct ucfvb3_stencil_view {
  int32_t order, K, M, MD, nf, nq, Q, n_cells, n_ops, si_exponent;
  const int32_t* central;
  const int32_t* op_index;
  const double* pinv;
  const double* pinv_lin;
  const int32_t* dir_members;
  const double* pinv_dir;
  const double* oi;
  const double* phi;
  const int32_t* qp_slot;
} ucfvb3_stencil_view;

const char* ucfvb3_last_error(const ucfvb3_solver* h);

/* periodic box [0,lx]x[0,ly]x[0,lz] of nx*ny*nz cubes (hex, or 6 tets each),
 * every vertex jittered by U(-jitter, jitter)*h per coordinate from `seed`;
 * face rules for polynomial order `order` (quads: Gauss n x n with
 * n = ceil((order+1)/2); triangles: 3-point degree 2 (order 1) or 6-point
 * degree 4 (order >= 2)). */
int32_t ucfvb3_mesh_periodic_box(int32_t nx, int32_t ny, int32_t nz, double lx, double ly, double lz,
                                 int32_t kind, double jitter, uint64_t seed, int32_t order, int32_t n_threads,
                                 ucfvb3_mesh** out);
int32_t ucfvb3_mesh_get_view(const ucfvb3_mesh* m, ucfvb3_mesh_view* out);
void ucfvb3_mesh_free(ucfvb3_mesh* m);

/* build_stencils in 3D; lattice_classes = 1 shares operator rows between
 * translated cells (only valid on an unjittered mesh; required for config 5's
 * 12.6 M cells). */
int32_t ucfvb3_build_stencils(const ucfvb3_mesh_view* mesh, int32_t order, int32_t si_exponent,
                              int32_t lattice_classes, int32_t n_threads, ucfvb3_stencils** out);
int32_t ucfvb3_stencils_get_view(const ucfvb3_stencils* s, ucfvb3_stencil_view* out);
void ucfvb3_stencils_free(ucfvb3_stencils* s);

/* cell averages [n_cells][5] of a built-in initial condition (ucfvb3_ic);
 * degree = volume quadrature degree (project_initial, cases.cpp:62-76). */
int32_t ucfvb3_project_initial(const ucfvb3_mesh_view* mesh, int32_t ic, const double* params, int32_t n_params,
                               uint64_t seed, int32_t degree, double gamma, int32_t n_threads, double* u_out);

/* ---- solver ------------------------------------------------------------- */
int32_t ucfvb3_create(const ucfvb3_mesh_view* mesh, const ucfvb3_stencil_view* stencils, const ucfvb_options* opt,
                      int32_t device, ucfvb3_solver** out);
void ucfvb3_destroy(ucfvb3_solver* h);
int32_t ucfvb3_set_state(ucfvb3_solver* h, const double* u);  /* [n_cells][5] */
int32_t ucfvb3_get_state(ucfvb3_solver* h, double* u);
int32_t ucfvb3_max_stable_dt(ucfvb3_solver* h, double* dt);
/* one step, in place; rk = UCFVB_RK3 or UCFVB_RK54 */
int32_t ucfvb3_advance(ucfvb3_solver* h, double dt, double t, int32_t rk);
/* n_steps steps with dt = max_stable_dt() computed on the device each step
 * (run_simulation's loop, run.cpp:92-139, without a host round trip); the
 * final time is returned in *t_out. */
int32_t ucfvb3_run_steps(ucfvb3_solver* h, int32_t n_steps, double t0, int32_t rk, double* t_out);
/* host state in ([n_cells][5], pinned for async copies) -> n_steps steps
 * -> host state out, one synchronisation (as ucfvb_advance_host) */
int32_t ucfvb3_advance_host(ucfvb3_solver* h, const double* u_in, double* u_out, int32_t n_steps, int32_t rk,
                            double t0, double* t_out);
/* ucfvb3_advance_host over n_batch independent states of the mesh, pipelined
 * as ucfvb_advance_host_batch (include/ucfvb.h): the upload of entry i+1 and
 * the download of entry i-1 overlap the stepping of entry i; every entry's
 * bits equal its own ucfvb3_advance_host call. t_out (nullable): [n_batch].
 * Every entry starts from reset error counters; the first failing entry is
 * reported (its u_out is its failing step's input), the others are unaffected. */
int32_t ucfvb3_advance_host_batch(ucfvb3_solver* h, int32_t n_batch, const double* const* u_in,
                                  double* const* u_out, int32_t n_steps, int32_t rk, double t0, double* t_out);
int32_t ucfvb3_compute_residual(ucfvb3_solver* h, const double* u, double t, double* out);
/* which = 0: labels of the last stage; 1: step labels (first stage of the last step) */
int32_t ucfvb3_get_labels(ucfvb3_solver* h, int32_t which, uint8_t* out);
/* face values [n_faces][nq][2][5] (side 0 = left cell's value) of the last stage */
int32_t ucfvb3_get_face_values(ucfvb3_solver* h, double* out);
/* census of the step labels: {linear, cwenoz, muscl, first} */
int32_t ucfvb3_get_census(ucfvb3_solver* h, int64_t out[4]);
/* NAD threshold near-ties of the last detection stage */
int32_t ucfvb3_get_nad_ties(ucfvb3_solver* h, int64_t* out);
/* PhaseTimes (solver.hpp:45-50) of the device pass: events between kernel
 * groups of un-graphed stages while enabled; seconds accumulated per group
 * {reconstruct (central), detect (spread), weights (CWENOZ+MUSCL), flux, gather+RK} */
int32_t ucfvb3_set_phase_timing(ucfvb3_solver* h, int32_t on);
int32_t ucfvb3_get_phase_times(ucfvb3_solver* h, double out[5]);
int64_t ucfvb3_launch_count(const ucfvb3_solver* h);
/* stream the solver launches on (cudaStream_t as void*) */
void* ucfvb3_stream(const ucfvb3_solver* h);

/* ---- domain decomposition (1/2/4/8 GPUs; decompose3.cpp) ------------------ */
/* recursive coordinate bisection of the cell centroids into n_parts parts */
int32_t ucfvb3_partition_rcb(const ucfvb3_mesh_view* mesh, int32_t n_parts, int32_t* part);
typedef struct ucfvb3_subdomain ucfvb3_subdomain;
/* rank `rank`'s owned cells + stencil-depth halo as a self-contained local
 * mesh/stencil pair; local order [owned | halo grouped by owner] */
int32_t ucfvb3_subdomain_build(const ucfvb3_mesh_view* mesh, const ucfvb3_stencil_view* stencils,
                               const int32_t* part, int32_t n_parts, int32_t rank, ucfvb3_subdomain** out);
int32_t ucfvb3_subdomain_views(const ucfvb3_subdomain* s, ucfvb3_mesh_view* mesh, ucfvb3_stencil_view* stencils);
int32_t ucfvb3_subdomain_info(const ucfvb3_subdomain* s, int32_t* n_owned, int32_t* n_local, int32_t* n_peers);
int32_t ucfvb3_subdomain_global_ids(const ucfvb3_subdomain* s, int32_t* gid);
int32_t ucfvb3_subdomain_peer(const ucfvb3_subdomain* s, int32_t i, int32_t* rank, int32_t* n_send,
                              int32_t* n_recv, int32_t* recv_begin);
int32_t ucfvb3_subdomain_send_list(const ucfvb3_subdomain* s, int32_t i, int32_t* local_ids);
void ucfvb3_subdomain_free(ucfvb3_subdomain* s);
const char* ucfvb3_decomp_last_error(void);
/* solver over a subdomain (borrowed; must outlive the solver): RK updates
 * and census cover the owned cells, errors only owned faces; after
 * ucfvb3_attach_nccl every stage ends with an NCCL halo exchange and dt is a
 * min all-reduce, all inside the captured step graph */
int32_t ucfvb3_create_sub(const ucfvb3_subdomain* sub, const ucfvb_options* opt, int32_t device,
                          ucfvb3_solver** out);
int32_t ucfvb3_attach_nccl(ucfvb3_solver* h, const uint8_t unique_id[128], int32_t rank, int32_t world);

#ifdef __cplusplus
}
#endif

#endif /* UCFVB3_H */
