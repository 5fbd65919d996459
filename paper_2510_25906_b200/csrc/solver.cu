// GpuSolver: the device-resident replacement of ucfv::Solver
// (/root/reference/proj/include/ucfv/solver.hpp:52-100) behind the C ABI of
// include/ucfvb.h. One CUDA stream per handle; one RK step is captured as a
// CUDA graph (per integrator, buffer parity and dt source) and replayed.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include <dlfcn.h>
#include <nccl.h>

#include "kernels.cuh"
#include "kernels_tma.cuh"
#include "kernels_cells.cuh"
#include "layout.hpp"
#include "decompose.hpp"
#include "solver.hpp"
#include "nccl_dl.hpp"

namespace ucfvb {

#define CK(x)                                                                                        \
  do {                                                                                               \
    cudaError_t e_ = (x);                                                                            \
    if (e_ != cudaSuccess)                                                                           \
      throw ApiError(UCFVB_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_));                   \
  } while (0)

void nccl_unique_id(uint8_t id[128]) {
  ncclUniqueId u;
  NK(nccl().GetUniqueId(&u));
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  std::memcpy(id, &u, 128);
}

// Stage kernels are launched with programmatic stream serialization (PDL):
// the next kernel's blocks start while the previous one drains and wait in
// griddepcontrol.wait before touching its outputs. UCFVB_PDL=0 disables it.
static bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("UCFVB_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

template <typename... KArgs, typename... Args>
static void launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                     Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  CK(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...));
}

// ---- kernel dispatch over (K, NQ, NF) ----------------------------------------
struct KernelSet {
  void (*central)(dim3, cudaStream_t, const Layout&, const Physics&, const Scratch&, const double4*, int);
  void (*spread)(dim3, cudaStream_t, const Layout&, const Scratch&, const double4*, int, int);
  void (*cwenoz)(dim3, cudaStream_t, const Layout&, const Physics&, const Scratch&, const double4*, int);
  void (*muscl)(dim3, cudaStream_t, const Layout&, const Physics&, const Scratch&, const double4*, int);
  void (*constant)(dim3, cudaStream_t, const Layout&, const Scratch&, const double4*);
  void (*face_flux)(dim3, cudaStream_t, const Layout&, const Physics&, const Scratch&);
  void (*gather)(dim3, cudaStream_t, const Layout&, const Scratch&, const RkEpilogue&, int, DtState*, double);
  int faces_per_flux_block;
  // TMA-staged persistent central kernel (fast path); grid filled in at create
  bool central_tma = false;
  using Launch = void (*)(dim3, cudaStream_t, const Layout&, const Physics&, const Scratch&, const double4*, int);
  void (*central_tma_setup)(int n_sm, int* grid, Launch* launch) = nullptr;
  int central_tma_grid = 0;
  // TMA-staged persistent CWENOZ+MUSCL kernel over chunk lists (fast path)
  Launch troubled = nullptr;
  void (*troubled_setup)(int n_sm, int* grid, Launch* launch) = nullptr;
  int troubled_grid = 0;
  // per-cell-record CWENOZ+MUSCL kernel over dense cell lists (fast path)
  Launch cells = nullptr;
  void (*cells_setup)(int n_sm, int* grid, Launch* launch) = nullptr;
  int cells_grid = 0;
  void (*pack_records)(cudaStream_t, const Layout&, unsigned char*, unsigned char*, unsigned char*,
                       unsigned char*) = nullptr;
  uint32_t rec_bytes[4] = {0, 0, 0, 0};  // CA, CB, MA, MB per cell
};

using StageLaunch = void (*)(dim3, cudaStream_t, const Layout&, const Physics&, const Scratch&, const double4*, int);

template <int K, int NQ, int NF, int MM>
void central_tma_launcher(dim3 g, cudaStream_t st, const Layout& L, const Physics& p, const Scratch& S,
                          const double4* U, int f) {
  launch_k(k_central_tma<K, NQ, NF, MM, 1>, g, dim3(kBlock), CentralStage<K, NQ, NF, MM>::BYTES + 16, st, L, p, S,
           U, f);
}

template <int K, int NQ, int NF, int MM, int MD>
void troubled_split_launcher(dim3 g, cudaStream_t st, const Layout& L, const Physics& p, const Scratch& S,
                             const double4* U, int f) {
  launch_k(k_troubled_split<K, NQ, NF, MM, MD>, g, dim3(kBlock),
           TroubledStage<K, NQ, NF, MM, MD>::SPLIT_BYTES + 16, st, L, p, S, U, f);
}

template <int K, int NQ, int NF, int MM, int MD>
void troubled_cells_launcher(dim3 g, cudaStream_t st, const Layout& L, const Physics& p, const Scratch& S,
                             const double4* U, int f) {
  launch_k(k_troubled_cells<K, NQ, NF, MM, MD>, g, dim3(kBlock), CellRec<K, NQ, NF, MM, MD>::BYTES + 16, st, L, p,
           S, U, f);
}

// raise the dynamic smem limit and size the persistent grid (resident blocks x SMs)
template <typename Kfn>
int persistent_grid(Kfn k, uint32_t smem, int n_sm) {
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  int per_sm = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, kBlock, smem));
  return std::max(1, per_sm) * n_sm;
}

template <int K, int NQ, int NF, int MMT, int MDT, bool UNI>
KernelSet make_set() {
  KernelSet s;
  s.central = [](dim3 g, cudaStream_t st, const Layout& L, const Physics& p, const Scratch& S, const double4* U,
                 int f) { launch_k(k_central<K, NQ, NF, MMT, MDT, UNI>, g, kBlock, 0, st, L, p, S, U, f); };
  s.spread = [](dim3 g, cudaStream_t st, const Layout& L, const Scratch& S, const double4* U, int f, int d) {
    launch_k(k_spread<K, NQ, NF, MMT, MDT, UNI>, g, kBlock, 0, st, L, S, U, f, d);
  };
  s.cwenoz = [](dim3 g, cudaStream_t st, const Layout& L, const Physics& p, const Scratch& S, const double4* U,
                int f) { launch_k(k_cwenoz<K, NQ, NF, MMT, MDT, UNI>, g, kBlock, 0, st, L, p, S, U, f); };
  s.muscl = [](dim3 g, cudaStream_t st, const Layout& L, const Physics& p, const Scratch& S, const double4* U,
               int f) { launch_k(k_muscl<K, NQ, NF, MMT, MDT, UNI>, g, kBlock, 0, st, L, p, S, U, f); };
  s.constant = [](dim3 g, cudaStream_t st, const Layout& L, const Scratch& S, const double4* U) {
    launch_k(k_constant<NQ, NF, UNI>, g, kBlock, 0, st, L, S, U);
  };
  s.face_flux = [](dim3 g, cudaStream_t st, const Layout& L, const Physics& p, const Scratch& S) {
    launch_k(k_face_flux<NQ>, g, kBlock, 0, st, L, p, S);
  };
  s.gather = [](dim3 g, cudaStream_t st, const Layout& L, const Scratch& S, const RkEpilogue& rk, int f, DtState* ds,
                 double gamma) {
    if (rk.nterms <= 3)
      launch_k(k_gather_rk<NF, UNI, 3>, g, kBlock, 0, st, L, S, rk, f, ds, gamma);
    else
      launch_k(k_gather_rk<NF, UNI, 5>, g, kBlock, 0, st, L, S, rk, f, ds, gamma);
  };
  s.faces_per_flux_block = (kBlock / 32) * (32 / NQ);
  if constexpr (MMT > 0 && UNI) {
    s.central_tma = true;
    s.central_tma_setup = [](int n_sm, int* grid, KernelSet::Launch* launch) {
      *grid = persistent_grid(k_central_tma<K, NQ, NF, MMT, 1>, CentralStage<K, NQ, NF, MMT>::BYTES + 16, n_sm);
      *launch = central_tma_launcher<K, NQ, NF, MMT>;
    };
    s.troubled_setup = [](int n_sm, int* grid, KernelSet::Launch* launch) {
      *grid = persistent_grid(k_troubled_split<K, NQ, NF, MMT, MDT>,
                              TroubledStage<K, NQ, NF, MMT, MDT>::SPLIT_BYTES + 16, n_sm);
      *launch = troubled_split_launcher<K, NQ, NF, MMT, MDT>;
    };
    using R = CellRec<K, NQ, NF, MMT, MDT>;
    s.cells_setup = [](int n_sm, int* grid, KernelSet::Launch* launch) {
      *grid = persistent_grid(k_troubled_cells<K, NQ, NF, MMT, MDT>, R::BYTES + 16, n_sm);
      *launch = troubled_cells_launcher<K, NQ, NF, MMT, MDT>;
    };
    s.pack_records = [](cudaStream_t st, const Layout& L, unsigned char* ca, unsigned char* cb, unsigned char* ma,
                        unsigned char* mb) {
      k_pack_records<K, NQ, NF, MMT, MDT><<<(L.n + 255) / 256, 256, 0, st>>>(L, ca, cb, ma, mb);
    };
    s.rec_bytes[0] = R::CA;
    s.rec_bytes[1] = R::CB;
    s.rec_bytes[2] = R::MA;
    s.rec_bytes[3] = R::MB;
  }
  return s;
}

// Fast path: uniform face count and the nominal stencil sizes (M = 2K,
// M_dir = 4; every BASELINE mesh) with fully unrolled gathers; anything else
// (mixed tri/quad meshes, rank-retry stencils) runs the generic instantiation.
static KernelSet pick_kernels(int K, int NQ, int NF, int MM, int MD, bool uniform) {
  const char* force = std::getenv("UCFVB_FORCE_GENERIC");
  const bool fast = uniform && MM == 2 * K && MD == 4 && !(force && force[0] == '1');
#define UCFVB_CASE(k, q, f)                               \
  if (K == k && NQ == q && NF == f) {                     \
    if (fast) return make_set<k, q, f, 2 * k, 4, true>(); \
    return make_set<k, q, f, 0, 0, false>();              \
  }
  UCFVB_CASE(2, 1, 3) UCFVB_CASE(2, 1, 4)
  UCFVB_CASE(5, 2, 3) UCFVB_CASE(5, 2, 4)
  UCFVB_CASE(9, 2, 3) UCFVB_CASE(9, 2, 4)
  UCFVB_CASE(14, 3, 3) UCFVB_CASE(14, 3, 4)
#undef UCFVB_CASE
  throw ApiError(UCFVB_UNSUPPORTED, "solver: reconstruction order with K=" + std::to_string(K) + ", n_qp=" +
                                        std::to_string(NQ) + " is not instantiated (orders 1-4 are)");
}

template <typename T>
static T* dalloc(size_t n, std::vector<void*>& owned) {
  void* p = nullptr;
  if (n == 0) n = 1;
  CK(cudaMalloc(&p, n * sizeof(T)));
  owned.push_back(p);
  return static_cast<T*>(p);
}

template <typename T>
static T* dupload(const std::vector<T>& h, std::vector<void*>& owned) {
  T* d = dalloc<T>(h.size(), owned);
  if (!h.empty()) CK(cudaMemcpy(d, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice));
  return d;
}

// Spiteri & Ruuth SSPRK(5,4) coefficients (time_integrator.cpp:11-29)
namespace rk54 {
constexpr double a10 = 0.391752226571890;
constexpr double b20 = 0.444370493651235, b21 = 0.555629506348765, a21 = 0.368410593050371;
constexpr double b30 = 0.620101851488403, b32 = 0.379898148511597, a32 = 0.251891774271694;
constexpr double b40 = 0.178079954393132, b43 = 0.821920045606868, a43 = 0.544974750228521;
constexpr double c52 = 0.517231671970585, c53 = 0.096059710526147, a53 = 0.063692468666290;
constexpr double c54 = 0.386708617503269, a54 = 0.226007483236906;
}  // namespace rk54

struct GpuSolver::Impl {
  HostLayout host;
  Layout L{};
  Physics ph{};
  Scratch S{};
  ucfvb_options opt{};
  KernelSet ks{};
  cudaStream_t stream = nullptr;
  int device = 0;
  int n_sm = 148;
  std::vector<void*> owned;
  double4* ubuf[2] = {nullptr, nullptr};
  int cur = 0;
  double4* work[6] = {};  // RK3: u1,u2 ; RK54: ua,ub,uc,ud,rhs3 ; [5] = compute_residual input
  double4* rhs = nullptr;
  DtState* ds = nullptr;
  unsigned long long* census_dev = nullptr;
  size_t census_cap = 0;
  double* dtlog_dev = nullptr;
  size_t dtlog_cap = 0;
  int* step_zero = nullptr;  // device int 0 (census row for advance())
  bool stage_is_first = true;
  bool timing = false;
  double phase[4] = {0, 0, 0, 0};
  cudaEvent_t ev[5] = {};
  int64_t launches = 0;
  // graphs: [rk][with_dt][parity]
  cudaGraphExec_t graph[2][2][2] = {};
  int64_t graph_launches[2][2][2] = {};
  std::string last_error;
  // decomposition / NCCL (halo exchange after every stage)
  struct DevPeer {
    int rank = 0, n_send = 0, recv_begin = 0, n_recv = 0;
    int* send_idx = nullptr;
    size_t send_off = 0;
  };
  std::vector<DevPeer> peers;
  double4* sendbuf = nullptr;
  ncclComm_t comm = nullptr;
  int world = 1, rank = 0;

  size_t l2_window_bytes = 0, l2_persist_bytes = 0;
  // Class lists for the troubled cells: 32-cell chunk lists (TMA-staged
  // k_troubled_split, the default) or dense per-cell lists (k_cwenoz /
  // k_muscl; UCFVB_TROUBLED=lists or set_list_policy). Chunks measured faster
  // on configs 1-3, including config 3's half-full chunks (profiles/round1.md).
  bool per_cell_lists = false;
  int* hcounts = nullptr;  // pinned copy of S.counts after the last synchronising call
  void fetch_counts() { CK(cudaMemcpyAsync(hcounts, S.counts, 4 * sizeof(int), cudaMemcpyDeviceToHost, stream)); }
  void drop_graphs() {
    for (auto& a : graph)
      for (auto& b : a)
        for (auto& g : b)
          if (g) {
            CK(cudaGraphExecDestroy(g));
            g = nullptr;
          }
  }
  dim3 grid_owned() const { return dim3((L.n_owned + kBlock - 1) / kBlock); }

  // halo exchange of a stage state: pack per peer, then one grouped send/recv
  int64_t exchange(double4* buf) {
    if (!comm || peers.empty()) return 0;
    int64_t nl = 0;
    for (const DevPeer& p : peers)
      if (p.n_send) {
        launch_k(k_halo_pack, dim3((p.n_send + 255) / 256), 256, 0, stream, buf, p.send_idx, p.n_send, sendbuf + p.send_off);
        ++nl;
      }
    NK(nccl().GroupStart());
    for (const DevPeer& p : peers) {
      if (p.n_send) NK(nccl().Send(sendbuf + p.send_off, 4 * static_cast<size_t>(p.n_send), ncclDouble, p.rank, comm,
                                   stream));
      if (p.n_recv) NK(nccl().Recv(buf + p.recv_begin, 4 * static_cast<size_t>(p.n_recv), ncclDouble, p.rank, comm,
                                   stream));
    }
    NK(nccl().GroupEnd());
    return nl;
  }

  // min(h/speed) over the owned cells of `src` into ds->dmin_bits
  int64_t launch_dt_reduce(const double4* src) {
    launch_k(k_dt, dim3((L.n_owned + kBlock - 1) / kBlock), kBlock, 0, stream, L, src, opt.gamma, ds, S.err);
    return 1;
  }
  // turn the reduced min into this step's dt (on subdomains after a min all-reduce)
  int64_t launch_dt_finalize() {
    if (!comm) {
      launch_k(k_dt_finalize, 1, 1, 0, stream, ds, S.err, 1);
      return 1;
    }
    launch_k(k_dt_collect, 1, 1, 0, stream, ds);
    NK(nccl().AllReduce(&ds->dmin, &ds->dmin, 1, ncclDouble, ncclMin, comm, stream));
    launch_k(k_dt_finalize, 1, 1, 0, stream, ds, S.err, 0);
    return 2;
  }

  dim3 grid_cells() const { return dim3((L.n + kBlock - 1) / kBlock); }
  // four lanes per cell (reconstruction kernels)
  dim3 grid_cells4() const { return dim3((4 * L.n + kBlock - 1) / kBlock); }
  dim3 grid_central() const {
    if (ks.central_tma) return dim3(std::min(ks.central_tma_grid, (L.n + 31) / 32));
    return grid_cells4();
  }
  dim3 grid_list() const {
    const int want = (4 * L.n + kBlock - 1) / kBlock;
    return dim3(std::max(1, std::min(want, n_sm * 16)));
  }

  void record(int i) {
    if (timing) CK(cudaEventRecord(ev[i], stream));
  }

  // one compute_residual stage on the stream (solver.cpp:316-379)
  // dt_next: this stage's output starts the next step; reduce its max_stable_dt term
  int64_t launch_stage(const double4* U, bool first, const RkEpilogue& rk, bool census, bool dt_next = false) {
    int64_t nl = 0;
    const int taps = opt.keep_taps ? FL_TAPS : 0;
    const int mode = opt.mode;
    record(0);
    if (mode == UCFVB_HYBRID) {
      const bool detect = first || opt.detect_every_stage;
      ks.central(grid_central(), stream, L, ph, S, U, FL_EVAL | FL_DOFS | (detect ? FL_NAD : FL_PRECHECK));
      record(1);
      if (ks.troubled && !per_cell_lists) {
        ks.spread(grid_cells(), stream, L, S, U, taps | FL_CHUNKS, detect ? 1 : 0);
        record(2);
        ks.troubled(dim3(std::min(ks.troubled_grid, (L.n + 31) / 32)), stream, L, ph, S, U,
                    FL_NAD | FL_FALLBACK | taps);
        nl += 3;
      } else if (ks.cells) {
        ks.spread(grid_cells(), stream, L, S, U, taps, detect ? 1 : 0);
        record(2);
        ks.cells(dim3(std::min(ks.cells_grid, (L.n + 31) / 32 + 2)), stream, L, ph, S, U, FL_NAD | FL_FALLBACK | taps);
        nl += 3;
      } else {
        ks.spread(grid_cells(), stream, L, S, U, taps, detect ? 1 : 0);
        record(2);
        ks.cwenoz(grid_list(), stream, L, ph, S, U, FL_NAD | FL_FALLBACK | taps);
        ks.muscl(grid_list(), stream, L, ph, S, U, FL_NAD | FL_FALLBACK | taps);
        nl += 4;
      }
    } else if (mode == UCFVB_LINEAR) {
      ks.central(grid_central(), stream, L, ph, S, U, FL_EVAL | (taps ? FL_DOFS : 0));
      record(1);
      record(2);
      nl += 1;
    } else if (mode == UCFVB_CWENOZ) {
      ks.central(grid_central(), stream, L, ph, S, U, FL_DOFS);
      record(1);
      record(2);
      ks.cwenoz(grid_cells4(), stream, L, ph, S, U, taps);
      nl += 2;
    } else if (mode == UCFVB_MUSCL) {
      record(1);
      record(2);
      ks.muscl(grid_cells4(), stream, L, ph, S, U, taps);
      nl += 1;
    } else {
      record(1);
      record(2);
      ks.constant(grid_cells(), stream, L, S, U);
      nl += 1;
    }
    record(3);
    int ff = 0;
    if (first) ff |= FL_STEP_LABELS | (census ? FL_CENSUS : 0);
    ks.face_flux(dim3((L.n_faces + ks.faces_per_flux_block - 1) / ks.faces_per_flux_block), stream, L, ph, S);
    ks.gather(grid_owned(), stream, L, S, rk, ff | (dt_next ? FL_DT : 0), ds, opt.gamma);
    ++nl;
    record(4);
    CK(cudaGetLastError());
    accumulate_phases();
    return nl + 1;
  }

  void accumulate_phases() {
    if (!timing) return;
    CK(cudaEventSynchronize(ev[4]));
    float ms[4];
    for (int i = 0; i < 4; ++i) CK(cudaEventElapsedTime(&ms[i], ev[i], ev[i + 1]));
    for (int i = 0; i < 4; ++i) phase[i] += 1e-3 * ms[i];
  }

  static void add_term(RkEpilogue& e, const double4* t, double coef, bool dt_scaled) {
    e.term[e.nterms] = t;
    e.coef[e.nterms] = coef;
    e.dt_scaled[e.nterms] = dt_scaled ? 1 : 0;
    ++e.nterms;
  }

  // All launches of one time step (the body a graph captures). `src` is the
  // state at t, `dst` receives the state at t+dt. With `with_dt` the step
  // starts with k_dt (device dt, run_steps); otherwise ds->dt was set by the host.
  int64_t launch_step(int rk, bool with_dt, const double4* src, double4* dst, bool census) {
    int64_t nl = 0;
    const double* dt = &ds->dt;
    if (with_dt) nl += launch_dt_finalize();  // dmin of src: k_dt (first step) or the previous final gather
    if (rk == UCFVB_RK3) {
      double4 *u1 = work[0], *u2 = work[1];
      RkEpilogue e1{};
      e1.dt = dt;
      e1.out = u1;
      add_term(e1, src, 1.0, false);
      add_term(e1, src, 0.0, false);
      add_term(e1, nullptr, 1.0, true);
      nl += launch_stage(src, true, e1, census);
      nl += exchange(u1);
      RkEpilogue e2{};
      e2.dt = dt;
      e2.out = u2;
      add_term(e2, src, 0.75, false);
      add_term(e2, u1, 0.25, false);
      add_term(e2, nullptr, 0.25, true);
      nl += launch_stage(u1, false, e2, census);
      nl += exchange(u2);
      RkEpilogue e3{};
      e3.dt = dt;
      e3.out = dst;
      add_term(e3, src, 1.0 / 3.0, false);
      add_term(e3, u2, 2.0 / 3.0, false);
      add_term(e3, nullptr, 2.0 / 3.0, true);
      nl += launch_stage(u2, false, e3, census, with_dt);
      nl += exchange(dst);
    } else {
      using namespace rk54;
      double4 *ua = work[0], *ub = work[1], *uc = work[2], *ud = work[3], *r3 = work[4];
      RkEpilogue e{};
      e.dt = dt;
      e.out = ua;
      add_term(e, src, 1.0, false);
      add_term(e, src, 0.0, false);
      add_term(e, nullptr, a10, true);
      nl += launch_stage(src, true, e, census);
      nl += exchange(ua);
      e = RkEpilogue{};
      e.dt = dt;
      e.out = ub;
      add_term(e, src, b20, false);
      add_term(e, ua, b21, false);
      add_term(e, nullptr, a21, true);
      nl += launch_stage(ua, false, e, census);
      nl += exchange(ub);
      e = RkEpilogue{};
      e.dt = dt;
      e.out = uc;
      add_term(e, src, b30, false);
      add_term(e, ub, b32, false);
      add_term(e, nullptr, a32, true);
      nl += launch_stage(ub, false, e, census);
      nl += exchange(uc);
      e = RkEpilogue{};
      e.dt = dt;
      e.out = ud;
      e.rhs_out = r3;
      add_term(e, src, b40, false);
      add_term(e, uc, b43, false);
      add_term(e, nullptr, a43, true);
      nl += launch_stage(uc, false, e, census);
      nl += exchange(ud);
      e = RkEpilogue{};
      e.dt = dt;
      e.out = dst;
      add_term(e, ub, c52, false);
      add_term(e, uc, c53, false);
      add_term(e, r3, a53, true);
      add_term(e, ud, c54, false);
      add_term(e, nullptr, a54, true);
      nl += launch_stage(ud, false, e, census, with_dt);
      nl += exchange(dst);
    }
    // inside the step (graph): a failure on any rank stops every rank's later
    // kernels (they exit on a set error word), so no rank writes past the
    // failing step and all can return to its input state
    nl += allreduce_error();
    return nl;
  }

  cudaGraphExec_t get_graph(int rk, bool with_dt, int parity) {
    cudaGraphExec_t& g = graph[rk][with_dt][parity];
    if (g) return g;
    cudaGraph_t gr;
    CK(cudaStreamBeginCapture(stream, cudaStreamCaptureModeThreadLocal));
    const int64_t nl = launch_step(rk, with_dt, ubuf[parity], ubuf[parity ^ 1], /*census=*/false);
    CK(cudaStreamEndCapture(stream, &gr));
    CK(cudaGraphInstantiate(&g, gr, 0));
    CK(cudaGraphDestroy(gr));
    graph_launches[rk][with_dt][parity] = nl;
    return g;
  }

  int err_step = 0;
  char* host_stage = nullptr;  // pinned DtState + error word for advance_host
  int read_error(int* kind, int* face, int* cell) {
    int e[4];
    CK(cudaMemcpyAsync(e, S.err, sizeof e, cudaMemcpyDeviceToHost, stream));
    CK(cudaStreamSynchronize(stream));
    *kind = e[0];
    *face = e[1];
    *cell = e[2];
    err_step = e[3];
    return e[0];
  }

  // the tie count covers one public call (include/ucfvb.h: ucfvb_get_nad_ties)
  void reset_ties() { CK(cudaMemsetAsync(S.ties, 0, sizeof(unsigned long long), stream)); }

  void reset_error() {
    const int e[4] = {0, INT_MAX, INT_MAX, INT_MAX};
    CK(cudaMemcpyAsync(S.err, e, sizeof e, cudaMemcpyHostToDevice, stream));
  }

  // translate the device error word into the reference's exceptions
  void raise_device_error(int kind, int face, int cell) {
    reset_error();
    CK(cudaStreamSynchronize(stream));
    if (kind & 4) throw ApiError(UCFVB_INVALID, "cwenoz: central linear weight lambda1' must exceed 1");
    if (kind & 2)
      throw ApiError(UCFVB_NONPHYSICAL, "non-physical state in max_stable_dt at cell " + std::to_string(cell));
    if (kind & 1) {
      std::string where = " at face " + std::to_string(face);
      throw ApiError(UCFVB_NONPHYSICAL, "non-physical state" + where);
    }
  }

  // every rank learns the job's error word: the kind by max (the kind bits of
  // one step are exclusive), the failing step / face / cell by min, so every
  // rank rolls back to the same step (run_impl, advance_host)
  int64_t allreduce_error() {
    if (!comm) return 0;
    NK(nccl().GroupStart());
    NK(nccl().AllReduce(S.err, S.err, 1, ncclInt32, ncclMax, comm, stream));
    NK(nccl().AllReduce(S.err + 1, S.err + 1, 3, ncclInt32, ncclMin, comm, stream));
    NK(nccl().GroupEnd());
    return 0;
  }

  void check_after() {
    int k, f, c;
    if (read_error(&k, &f, &c)) raise_device_error(k, f, c);
  }

  // Owns every resource, so a constructor that throws half-way (unsupported
  // order, out of memory) releases what it had acquired through unique_ptr.
  size_t l2_limit_before = 0;
  bool l2_limit_set = false;
  ~Impl() {
    if (stream) cudaStreamSynchronize(stream);
    for (auto& a : graph)
      for (auto& b : a)
        for (auto& g : b)
          if (g) cudaGraphExecDestroy(g);
    if (comm) nccl().CommDestroy(comm);
    for (void* p : owned) cudaFree(p);
    if (census_dev) cudaFree(census_dev);
    if (dtlog_dev) cudaFree(dtlog_dev);
    if (host_stage) cudaFreeHost(host_stage);
    if (hcounts) cudaFreeHost(hcounts);
    for (auto& e : ev)
      if (e) cudaEventDestroy(e);
    if (stream) cudaStreamDestroy(stream);
    // the persisting-L2 carve-out is device-wide: give back what we raised
    if (l2_limit_set) cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, l2_limit_before);
  }
};

GpuSolver::GpuSolver(const ucfvb_mesh_view& m, const ucfvb_stencil_view& s, const ucfvb_options& o,
                     const ucfvb_bc* bcs, int n_bcs, int device, int n_owned)
    : p_(new Impl) {
  Impl& I = *p_;
  I.opt = o;
  I.device = device;
  // validate_margins (detector.cpp:9-16)
  const ucfvb_margins& mg = o.margins;
  if (mg.alpha_m < 0.0 || mg.beta_m < 0.0)
    throw ApiError(UCFVB_INVALID, "NAD margins: alpha_m and beta_m must be non-negative");
  if (mg.beta_w > 0.0 && (mg.beta_w > mg.beta_m || mg.alpha_w > mg.alpha_m))
    throw ApiError(UCFVB_INVALID,
                   "NAD margins: delta_w <= delta_m requires beta_w <= beta_m and alpha_w <= alpha_m");
  if (mg.kappa < 0.0) throw ApiError(UCFVB_INVALID, "NAD margins: kappa must be >= 0");
  if (o.mode < 0 || o.mode > 4) throw ApiError(UCFVB_INVALID, "solver: unknown scheme mode");

  // boundary conditions by patch name (solver.cpp:46-60)
  Physics& ph = I.ph;
  if (m.n_patches > kMaxPatches) throw ApiError(UCFVB_UNSUPPORTED, "solver: more than 16 boundary patches");
  for (int i = 0; i < n_bcs; ++i) {
    int pid = -1;
    for (int p = 0; p < m.n_patches; ++p)
      if (bcs[i].patch && std::strcmp(m.patch_names[p], bcs[i].patch) == 0) pid = p;
    if (pid < 0)
      throw ApiError(UCFVB_INVALID,
                     std::string("solver: unknown boundary patch '") + (bcs[i].patch ? bcs[i].patch : "") + "'");
    if (bcs[i].kind < UCFVB_BC_NONE || bcs[i].kind > UCFVB_BC_FIXED)
      throw ApiError(UCFVB_UNSUPPORTED, "solver: boundary condition kind not available on the device");
    ph.bc[pid].kind = bcs[i].kind;
    for (int v = 0; v < 4; ++v) ph.bc[pid].state[v] = bcs[i].state[v];
  }
  // faces leaving a subdomain's local cell set (ucfvb_subdomain_build) need no BC: never integrated
  int halo_patch = -1;
  for (int p = 0; p < m.n_patches; ++p)
    if (std::strcmp(m.patch_names[p], "__halo__") == 0) halo_patch = p;
  for (int f = 0; f < m.n_faces; ++f)
    if (m.face_right[f] < 0 && m.face_partner[f] < 0) {
      const int p = m.face_patch[f];
      if (p == halo_patch && p >= 0) continue;
      if (p < 0 || ph.bc[p].kind == UCFVB_BC_NONE)
        throw ApiError(UCFVB_INVALID, "solver: boundary face " + std::to_string(f) +
                                          " has no boundary condition (patch " +
                                          (p >= 0 ? std::string(m.patch_names[p]) : std::string("<none>")) + ")");
    }

  CK(cudaSetDevice(device));
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, device));
  I.n_sm = prop.multiProcessorCount;
  CK(cudaStreamCreateWithFlags(&I.stream, cudaStreamNonBlocking));
  for (auto& e : I.ev) CK(cudaEventCreate(&e));

  I.host = build_layout(m, s, o, 0, n_owned < 0 ? m.n_cells : n_owned, halo_patch);
  const HostLayout& H = I.host;
  bool uniform = true;
  for (int c = 0; c < H.n; ++c) uniform &= H.nfc[c] == H.NF;
  I.ks = pick_kernels(H.K, H.NQ, H.NF, H.MM, H.MD, uniform);
  if (const char* tl = std::getenv("UCFVB_TROUBLED")) I.per_cell_lists = std::strcmp(tl, "lists") == 0;
  CK(cudaMallocHost(&I.hcounts, 4 * sizeof(int)));
  std::memset(I.hcounts, 0, 4 * sizeof(int));
  if (I.ks.central_tma) {
    I.ks.central_tma_setup(I.n_sm, &I.ks.central_tma_grid, &I.ks.central);
    I.ks.troubled_setup(I.n_sm, &I.ks.troubled_grid, &I.ks.troubled);
    I.ks.cells_setup(I.n_sm, &I.ks.cells_grid, &I.ks.cells);
  }
  auto& own = I.owned;
  Layout& L = I.L;
  L.n = H.n;
  L.n_owned = H.n_owned;
  L.MM = H.MM;
  L.MD = H.MD;
  L.st_idx = dupload(H.st_idx, own);
  L.pinv = dupload(H.pinv, own);
  L.phi = dupload(H.phi, own);
  L.phi01 = dupload(H.phi01, own);
  L.pinv_lin = dupload(H.pinv_lin, own);
  L.dir_idx = dupload(H.dir_idx, own);
  L.pinv_dir = dupload(H.pinv_dir, own);
  L.oi = dupload(H.oi, own);
  L.nbr = dupload(H.nbr, own);
  L.dest = dupload(H.dest, own);
  L.cface = dupload(H.cface, own);
  L.n_faces = H.n_faces;
  L.fnx = dupload(H.fnx, own);
  L.fny = dupload(H.fny, own);
  L.flen = dupload(H.flen, own);
  L.fkind = dupload(H.fkind, own);
  L.fpatch = dupload(H.fpatch, own);
  L.fslot = dupload(H.fslot, own);
  L.nfc = dupload(H.nfc, own);
  L.deact_thr = dupload(H.deact_thr, own);
  L.eps2 = dupload(H.eps2, own);
  L.h = dupload(H.h, own);
  L.inv_vol = dupload(H.inv_vol, own);
  if (I.ks.pack_records) {  // per-cell records of the troubled-cell rows (kernels_cells.cuh)
    unsigned char* rec[4];
    for (int i = 0; i < 4; ++i) rec[i] = dalloc<unsigned char>(static_cast<size_t>(H.n) * I.ks.rec_bytes[i], own);
    L.rec_ca = rec[0];
    L.rec_cb = rec[1];
    L.rec_ma = rec[2];
    L.rec_mb = rec[3];
    I.ks.pack_records(I.stream, L, rec[0], rec[1], rec[2], rec[3]);
    CK(cudaGetLastError());
  }

  // the operator data now lives on the device: keep only what the taps need
  {
    HostLayout& Hm = I.host;
    auto drop = [](auto& v) { std::remove_reference_t<decltype(v)>().swap(v); };
    drop(Hm.st_idx); drop(Hm.pinv); drop(Hm.phi); drop(Hm.phi01); drop(Hm.pinv_lin); drop(Hm.dir_idx);
    drop(Hm.pinv_dir); drop(Hm.oi); drop(Hm.nbr); drop(Hm.cface); drop(Hm.fnx); drop(Hm.fny); drop(Hm.flen);
    drop(Hm.fkind); drop(Hm.fpatch); drop(Hm.fslot); drop(Hm.deact_thr); drop(Hm.eps2); drop(Hm.h); drop(Hm.inv_vol);
  }
  ph.mp = MarginParams{mg.alpha_m, mg.beta_m, mg.alpha_w, mg.beta_w, mg.kappa, mg.deact_n};
  ph.gamma = o.gamma;
  ph.lambda1p = o.lambda1p;
  ph.lam0 = 1.0 - 1.0 / o.lambda1p;
  ph.inv_lam0 = 1.0 / ph.lam0;
  for (int nd = 1; nd <= 4; ++nd) {
    ph.nd_d[nd] = static_cast<double>(nd);
    ph.lams[nd] = (1.0 - ph.lam0) / nd;
    ph.inv_nd[nd] = 1.0 / nd;
  }
  ph.weno_eps = o.weno_eps;
  ph.weno_b = o.weno_b;
  ph.limiter = o.limiter;
  ph.hll = o.riemann == UCFVB_HLL ? 1 : 0;
  for (int q = 0; q < 4; ++q) ph.qw[q] = H.qw[q];

  const size_t nch = static_cast<size_t>(H.n_pad / 32);
  Scratch& S = I.S;
  const size_t n_fp = 2 * static_cast<size_t>(H.n_faces) * H.NQ + 1;  // + scratch slot for padded qps
  // face points, face fluxes and dofs are produced and consumed within one
  // stage: one allocation, so one L2 access-policy window can keep them resident
  const size_t n_ff = nch * H.NF * 32, n_dofs = nch * H.K * 32;
  double4* stage_buf = dalloc<double4>(n_fp + n_ff + n_dofs, own);
  S.fp = stage_buf;
  S.rs = stage_buf + n_fp;
  S.dofs = stage_buf + n_fp + n_ff;
  {
    const char* e = std::getenv("UCFVB_L2_PERSIST");
    const bool want = !(e && e[0] == '0');
    int max_persist = 0, max_window = 0;
    CK(cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, device));
    CK(cudaDeviceGetAttribute(&max_window, cudaDevAttrMaxAccessPolicyWindowSize, device));
    const size_t bytes = (n_fp + n_ff + n_dofs) * sizeof(double4);
    if (want && max_persist > 0 && max_window > 0) {
      size_t limit = 0;
      CK(cudaDeviceGetLimit(&limit, cudaLimitPersistingL2CacheSize));
      const size_t persist = std::min<size_t>(max_persist, std::max(limit, bytes));
      I.l2_limit_before = limit;
      I.l2_limit_set = true;
      CK(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, persist));
      cudaStreamAttrValue attr{};
      attr.accessPolicyWindow.base_ptr = stage_buf;
      attr.accessPolicyWindow.num_bytes = std::min<size_t>(bytes, max_window);
      attr.accessPolicyWindow.hitRatio =
          static_cast<float>(std::min(1.0, static_cast<double>(persist) / attr.accessPolicyWindow.num_bytes));
      attr.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
      attr.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
      CK(cudaStreamSetAttribute(I.stream, cudaStreamAttributeAccessPolicyWindow, &attr));
      I.l2_window_bytes = attr.accessPolicyWindow.num_bytes;
      I.l2_persist_bytes = persist;
    }
  }
  S.raw = dalloc<uint8_t>(H.n_pad, own);
  S.labels = dalloc<uint8_t>(H.n_pad, own);
  S.step_labels = dalloc<uint8_t>(H.n_pad, own);
  S.list_c = dalloc<int>(H.n, own);
  S.list_m = dalloc<int>(H.n, own);
  S.counts = dalloc<int>(4, own);
  S.chunks_c = dalloc<int2>(nch, own);
  S.chunks_m = dalloc<int2>(nch, own);
  S.ties = dalloc<unsigned long long>(1, own);
  S.err = dalloc<int>(4, own);
  I.step_zero = dalloc<int>(1, own);
  CK(cudaMemset(I.step_zero, 0, sizeof(int)));
  CK(cudaMemset(S.fp, 0, n_fp * sizeof(double4)));
  CK(cudaMemset(S.rs, 0, n_ff * sizeof(double4)));
  CK(cudaMemset(S.dofs, 0, nch * H.K * 32 * sizeof(double4)));
  CK(cudaMemset(S.ties, 0, sizeof(unsigned long long)));
  CK(cudaMemset(S.raw, 0, H.n_pad));
  // labels_ start Linear (solver.cpp:72-73); forced modes label every cell once
  const int init_label = o.mode == UCFVB_CWENOZ ? 1 : o.mode == UCFVB_MUSCL ? 2 : o.mode == UCFVB_FIRST ? 3 : 0;
  CK(cudaMemset(S.labels, init_label, H.n_pad));
  CK(cudaMemset(S.step_labels, 0, H.n_pad));
  S.step = I.step_zero;
  S.census = nullptr;
  for (auto& b : I.ubuf) {
    b = dalloc<double4>(H.n_pad, own);
    CK(cudaMemset(b, 0, H.n_pad * sizeof(double4)));
  }
  for (auto& w : I.work) {
    w = dalloc<double4>(H.n_pad, own);
    CK(cudaMemset(w, 0, H.n_pad * sizeof(double4)));
  }
  I.rhs = dalloc<double4>(H.n_pad, own);
  I.ds = dalloc<DtState>(1, own);
  I.reset_error();
  CK(cudaStreamSynchronize(I.stream));
}

GpuSolver::~GpuSolver() = default;  // Impl::~Impl releases everything

int GpuSolver::n_cells() const { return p_->L.n; }
int GpuSolver::n_faces() const { return p_->host.n_faces; }
int GpuSolver::n_qp() const { return p_->host.NQ; }
int GpuSolver::K() const { return p_->host.K; }
int64_t GpuSolver::launch_count() const { return p_->launches; }
void* GpuSolver::stream() const { return p_->stream; }
double* GpuSolver::state_device_ptr() { return reinterpret_cast<double*>(p_->ubuf[p_->cur]); }

void GpuSolver::set_state(const double* u) {
  Impl& I = *p_;
  CK(cudaMemcpyAsync(I.ubuf[I.cur], u, sizeof(double4) * I.L.n, cudaMemcpyHostToDevice, I.stream));
  CK(cudaStreamSynchronize(I.stream));
}

void GpuSolver::get_state(double* u) {
  Impl& I = *p_;
  CK(cudaMemcpyAsync(u, I.ubuf[I.cur], sizeof(double4) * I.L.n, cudaMemcpyDeviceToHost, I.stream));
  CK(cudaStreamSynchronize(I.stream));
}

double GpuSolver::max_stable_dt() {
  Impl& I = *p_;
  DtState h{};
  h.dmin_bits = static_cast<unsigned long long>(0x7e37e43c8800759cULL);  // bits of 1e300
  h.t = 0.0;
  h.dt = 0.0;
  h.step = -1;
  h.t_end = INFINITY;
  h.cfl = I.opt.cfl;
  CK(cudaMemcpyAsync(I.ds, &h, sizeof h, cudaMemcpyHostToDevice, I.stream));
  I.launches = I.launch_dt_reduce(I.ubuf[I.cur]) + I.launch_dt_finalize();
  CK(cudaGetLastError());
  I.allreduce_error();
  CK(cudaMemcpyAsync(&h, I.ds, sizeof h, cudaMemcpyDeviceToHost, I.stream));
  I.check_after();
  return h.dt;
}

void GpuSolver::advance(double dt, double t, int rk) {
  Impl& I = *p_;
  if (rk != UCFVB_RK3 && rk != UCFVB_RK54) throw ApiError(UCFVB_INVALID, "advance: unknown integrator");
  DtState h{};
  h.dmin_bits = static_cast<unsigned long long>(0x7e37e43c8800759cULL);
  h.t = t;
  h.dt = dt;
  h.step = 0;
  h.t_end = INFINITY;
  h.cfl = I.opt.cfl;
  CK(cudaMemcpyAsync(I.ds, &h, sizeof h, cudaMemcpyHostToDevice, I.stream));
  I.reset_ties();
  I.S.step = I.step_zero;
  I.stage_is_first = true;  // Solver::advance (solver.cpp:382)
  if (I.opt.use_graphs && !I.timing) {
    cudaGraphExec_t g = I.get_graph(rk, false, I.cur);
    CK(cudaGraphLaunch(g, I.stream));
    I.launches = I.graph_launches[rk][0][I.cur];
  } else {
    I.launches = I.launch_step(rk, false, I.ubuf[I.cur], I.ubuf[I.cur ^ 1], false);
  }
  I.allreduce_error();
  I.fetch_counts();
  int k, f, c;
  if (I.read_error(&k, &f, &c)) I.raise_device_error(k, f, c);  // state stays at t (reference semantics)
  I.cur ^= 1;
  I.stage_is_first = false;
}

void GpuSolver::compute_residual(const double* u, double t, double* out) {
  Impl& I = *p_;
  (void)t;
  double4* in = I.work[5];
  CK(cudaMemcpyAsync(in, u, sizeof(double4) * I.L.n, cudaMemcpyHostToDevice, I.stream));
  RkEpilogue e{};
  e.rhs_out = I.rhs;
  e.dt = &I.ds->dt;
  I.reset_ties();
  I.launches = I.launch_stage(in, I.stage_is_first, e, false);
  I.stage_is_first = false;
  int k, f, c;
  if (I.read_error(&k, &f, &c)) I.raise_device_error(k, f, c);
  CK(cudaMemcpyAsync(out, I.rhs, sizeof(double4) * I.L.n, cudaMemcpyDeviceToHost, I.stream));
  CK(cudaStreamSynchronize(I.stream));
}

double GpuSolver::run_steps(int n_steps, int rk, double t0, double t_end, int64_t* census_out, double* dt_out) {
  int done = 0;
  return run_impl(n_steps, rk, t0, t_end, false, census_out, dt_out, &done);
}

double GpuSolver::run_until(int max_steps, int rk, double t0, double t_end, int64_t* census_out, double* dt_out,
                            int* n_done) {
  return run_impl(max_steps, rk, t0, t_end, true, census_out, dt_out, n_done);
}

// run_simulation's stepping loop (run.cpp:96-132) on the device. Fixed count:
// n_steps steps. `until`: steps while t < t_end - 1e-14 t_end, at most
// n_steps; launched in batches, the device raises kErrDone at the loop end.
double GpuSolver::run_impl(int n_steps, int rk, double t0, double t_end, bool until, int64_t* census_out,
                           double* dt_out, int* n_done) {
  Impl& I = *p_;
  if (rk != UCFVB_RK3 && rk != UCFVB_RK54) throw ApiError(UCFVB_INVALID, "run_steps: unknown integrator");
  *n_done = 0;
  if (n_steps <= 0) return t0;
  const bool census = census_out != nullptr;
  if (census && I.census_cap < static_cast<size_t>(n_steps)) {
    if (I.census_dev) CK(cudaFree(I.census_dev));
    CK(cudaMalloc(&I.census_dev, sizeof(unsigned long long) * 4 * n_steps));
    I.census_cap = n_steps;
  }
  if (census) CK(cudaMemsetAsync(I.census_dev, 0, sizeof(unsigned long long) * 4 * n_steps, I.stream));
  if (dt_out && I.dtlog_cap < static_cast<size_t>(n_steps)) {
    if (I.dtlog_dev) CK(cudaFree(I.dtlog_dev));
    CK(cudaMalloc(&I.dtlog_dev, sizeof(double) * n_steps));
    I.dtlog_cap = n_steps;
  }
  DtState h{};
  h.dmin_bits = static_cast<unsigned long long>(0x7e37e43c8800759cULL);
  h.t = t0;
  h.dt = 0.0;
  h.step = -1;
  h.t_end = t_end;
  h.cfl = I.opt.cfl;
  h.dt_log = dt_out ? I.dtlog_dev : nullptr;
  h.until = until ? 1 : 0;
  CK(cudaMemcpyAsync(I.ds, &h, sizeof h, cudaMemcpyHostToDevice, I.stream));
  I.reset_ties();
  // census rows are indexed by the device step counter
  I.S.census = census ? I.census_dev : nullptr;
  I.S.step = &I.ds->step;
  const bool graphs = I.opt.use_graphs && !I.timing;
  const int cur0 = I.cur;
  // the first step's max_stable_dt term; each step's final gather reduces the next one
  int64_t nl = I.launch_dt_reduce(I.ubuf[I.cur]);
  const int batch = until ? 32 : n_steps;
  int launched = 0;
  int k = 0, f = 0, c = 0;
  while (launched < n_steps) {
    const int nb = std::min(batch, n_steps - launched);
    for (int s = 0; s < nb; ++s) {
      if (graphs) {
        // graphs capture the census flag; keep separate graphs only for census runs
        if (census) {
          nl += I.launch_step(rk, true, I.ubuf[I.cur], I.ubuf[I.cur ^ 1], true);
        } else {
          cudaGraphExec_t g = I.get_graph(rk, true, I.cur);
          CK(cudaGraphLaunch(g, I.stream));
          nl += I.graph_launches[rk][1][I.cur];
        }
      } else {
        nl += I.launch_step(rk, true, I.ubuf[I.cur], I.ubuf[I.cur ^ 1], census);
      }
      I.cur ^= 1;
    }
    launched += nb;
    if (!until) break;
    I.allreduce_error();
    if (I.read_error(&k, &f, &c)) break;  // t_end reached (kErrDone) or a failure
  }
  I.launches = nl;
  I.S.step = I.step_zero;
  I.S.census = nullptr;
  if (census && I.comm)
    NK(nccl().AllReduce(I.census_dev, I.census_dev, 4 * static_cast<size_t>(n_steps), ncclUint64, ncclSum, I.comm,
                        I.stream));
  if (!until) I.allreduce_error();
  CK(cudaMemcpyAsync(&h, I.ds, sizeof h, cudaMemcpyDeviceToHost, I.stream));
  I.fetch_counts();
  I.read_error(&k, &f, &c);
  // steps that ran to completion: the device counter holds the last started step
  int ran = launched;
  if (until && (k & kErrDone)) ran = h.step + 1;
  if (k & ~kErrDone) {
    // step s reads ubuf[(cur0 + s) & 1] and never overwrites it: the failing
    // step's input is the last good state (the reference throws out of
    // advance()/max_stable_dt() before touching state_)
    const int failed = std::min(std::max(0, I.err_step), n_steps - 1);
    I.cur = (cur0 + failed) & 1;
    *n_done = failed;
    try {
      I.raise_device_error(k & ~kErrDone, f, c);
    } catch (ApiError& e) {
      throw ApiError(e.code, "run failed at step " + std::to_string(failed) + ": " + e.what());
    }
  }
  if (k & kErrDone) {
    I.reset_error();
    I.cur = (cur0 + ran) & 1;
  }
  *n_done = ran;
  if (census && ran > 0) {
    std::vector<unsigned long long> tmp(4 * static_cast<size_t>(ran));
    CK(cudaMemcpy(tmp.data(), I.census_dev, tmp.size() * sizeof(tmp[0]), cudaMemcpyDeviceToHost));
    for (size_t i = 0; i < tmp.size(); ++i) census_out[i] = static_cast<int64_t>(tmp[i]);
  }
  if (dt_out && ran > 0) CK(cudaMemcpy(dt_out, I.dtlog_dev, sizeof(double) * ran, cudaMemcpyDeviceToHost));
  I.stage_is_first = false;
  CK(cudaStreamSynchronize(I.stream));
  return h.t + h.dt;
}

// Everything is enqueued before the single synchronisation: H2D of the state,
// the dt-state reset (from pinned staging), the step graphs, the error word
// and dt-state read-back (pinned) and the D2H of the result. u_in / u_out
// should be pinned host memory for truly asynchronous PCIe transfers.
double GpuSolver::advance_host(const double* u_in, double* u_out, int n_steps, int rk, double t0) {
  Impl& I = *p_;
  if (rk != UCFVB_RK3 && rk != UCFVB_RK54) throw ApiError(UCFVB_INVALID, "advance_host: unknown integrator");
  if (n_steps <= 0) throw ApiError(UCFVB_INVALID, "advance_host: n_steps must be >= 1");
  if (!I.host_stage) CK(cudaMallocHost(&I.host_stage, sizeof(DtState) + 4 * sizeof(int)));
  auto* hs = reinterpret_cast<DtState*>(I.host_stage);
  int* he = reinterpret_cast<int*>(I.host_stage + sizeof(DtState));
  const size_t bytes = sizeof(double4) * I.L.n;
  CK(cudaMemcpyAsync(I.ubuf[I.cur], u_in, bytes, cudaMemcpyHostToDevice, I.stream));
  *hs = DtState{};
  hs->dmin_bits = static_cast<unsigned long long>(0x7e37e43c8800759cULL);  // bits of 1e300
  hs->t = t0;
  hs->step = -1;
  hs->t_end = INFINITY;
  hs->cfl = I.opt.cfl;
  CK(cudaMemcpyAsync(I.ds, hs, sizeof(DtState), cudaMemcpyHostToDevice, I.stream));
  I.reset_ties();
  I.S.step = &I.ds->step;
  const int cur0 = I.cur;
  int64_t nl = I.launch_dt_reduce(I.ubuf[I.cur]);
  for (int s = 0; s < n_steps; ++s) {
    if (I.opt.use_graphs && !I.timing) {
      cudaGraphExec_t g = I.get_graph(rk, true, I.cur);
      CK(cudaGraphLaunch(g, I.stream));
      nl += I.graph_launches[rk][1][I.cur];
    } else {
      nl += I.launch_step(rk, true, I.ubuf[I.cur], I.ubuf[I.cur ^ 1], false);
    }
    I.cur ^= 1;
  }
  I.launches = nl;
  I.S.step = I.step_zero;
  I.allreduce_error();
  CK(cudaMemcpyAsync(he, I.S.err, 4 * sizeof(int), cudaMemcpyDeviceToHost, I.stream));
  CK(cudaMemcpyAsync(hs, I.ds, sizeof(DtState), cudaMemcpyDeviceToHost, I.stream));
  CK(cudaMemcpyAsync(u_out, I.ubuf[I.cur], bytes, cudaMemcpyDeviceToHost, I.stream));
  I.fetch_counts();
  CK(cudaStreamSynchronize(I.stream));
  CK(cudaGetLastError());
  I.stage_is_first = false;
  if (he[0]) {
    const int failed = std::min(std::max(0, he[3]), n_steps - 1);
    I.cur = (cur0 + failed) & 1;
    I.raise_device_error(he[0], he[1], he[2]);
  }
  return hs->t + hs->dt;
}

void GpuSolver::get_labels(uint8_t* out, bool step) {
  Impl& I = *p_;
  CK(cudaMemcpyAsync(out, step ? I.S.step_labels : I.S.labels, I.L.n, cudaMemcpyDeviceToHost, I.stream));
  CK(cudaStreamSynchronize(I.stream));
}

void GpuSolver::get_census(int64_t counts[4]) {
  std::vector<uint8_t> lab(n_cells());
  get_labels(lab.data(), true);
  counts[0] = counts[1] = counts[2] = counts[3] = 0;
  for (int c = 0; c < p_->L.n_owned; ++c) ++counts[lab[c] & 3];  // owned cells (subdomains: not the halo)
}

int64_t GpuSolver::nad_ties() {
  Impl& I = *p_;
  unsigned long long t = 0;
  CK(cudaMemcpy(&t, I.S.ties, sizeof t, cudaMemcpyDeviceToHost));
  return static_cast<int64_t>(t);
}

void GpuSolver::get_face_values(double* left, double* right) {
  Impl& I = *p_;
  const HostLayout& H = I.host;
  const int NQ = H.NQ;
  std::vector<double4> fp(2 * static_cast<size_t>(H.n_faces) * NQ);
  CK(cudaMemcpyAsync(fp.data(), I.S.fp, fp.size() * sizeof(double4), cudaMemcpyDeviceToHost, I.stream));
  CK(cudaStreamSynchronize(I.stream));
  // every cell-local qp knows both its reference slot (qp_slot) and where the
  // device stored it (dest): invert through the cells
  for (int c = 0; c < H.n; ++c)
    for (int64_t q = H.qp_ptr[c]; q < H.qp_ptr[c + 1]; ++q) {
      const int slot = H.qp_slot[q];
      const int lq = static_cast<int>(q - H.qp_ptr[c]);
      const double4 v = fp[H.dest[aos_index(c, lq, H.Q)]];
      double* dst = ((slot & 1) ? right : left) + 4 * static_cast<int64_t>(slot >> 1);
      dst[0] = v.x;
      dst[1] = v.y;
      dst[2] = v.z;
      dst[3] = v.w;
    }
}

void GpuSolver::get_dofs(double* dofs) {
  Impl& I = *p_;
  const HostLayout& H = I.host;
  if (!I.opt.keep_taps && I.opt.mode != UCFVB_HYBRID)
    throw ApiError(UCFVB_INVALID, "get_dofs: create the solver with keep_taps = 1");
  const size_t nch = static_cast<size_t>(H.n_pad / 32);
  std::vector<double4> d(nch * H.K * 32);
  CK(cudaMemcpyAsync(d.data(), I.S.dofs, d.size() * sizeof(double4), cudaMemcpyDeviceToHost, I.stream));
  CK(cudaStreamSynchronize(I.stream));
  for (int c = 0; c < H.n; ++c)
    for (int k = 0; k < H.K; ++k) {
      const double4 v = d[aos_index(c, k, H.K)];
      double* dst = dofs + (static_cast<int64_t>(c) * H.K + k) * 4;
      dst[0] = v.x;
      dst[1] = v.y;
      dst[2] = v.z;
      dst[3] = v.w;
    }
}

void GpuSolver::set_phase_timing(bool on) { p_->timing = on; }
void GpuSolver::get_phase_times(double t[4]) {
  for (int i = 0; i < 4; ++i) t[i] = p_->phase[i];
}

void GpuSolver::attach_nccl(const uint8_t id[128], int rank, int world, const ucfvb_subdomain* sub) {
  Impl& I = *p_;
  if (!sub) throw ApiError(UCFVB_INVALID, "attach_nccl: the solver was not created on a subdomain");
  if (I.comm) throw ApiError(UCFVB_INVALID, "attach_nccl: a communicator is already attached");
  ncclUniqueId u;
  std::memcpy(&u, id, 128);
  CK(cudaSetDevice(I.device));
  NK(nccl().CommInitRank(&I.comm, world, u, rank));
  I.world = world;
  I.rank = rank;
  size_t off = 0;
  for (const auto& p : sub->peers) {
    Impl::DevPeer d;
    d.rank = p.rank;
    d.n_send = static_cast<int>(p.send.size());
    d.recv_begin = p.recv_begin;
    d.n_recv = p.n_recv;
    d.send_off = off;
    off += p.send.size();
    if (d.n_send) {
      d.send_idx = dalloc<int>(p.send.size(), I.owned);
      CK(cudaMemcpy(d.send_idx, p.send.data(), p.send.size() * sizeof(int), cudaMemcpyHostToDevice));
    }
    I.peers.push_back(d);
  }
  I.sendbuf = dalloc<double4>(std::max<size_t>(1, off), I.owned);
  // graphs captured before the exchange existed are stale
  I.drop_graphs();
}

void GpuSolver::set_list_policy(int policy) {
  Impl& I = *p_;
  if (policy < 0 || policy > 1) throw ApiError(UCFVB_INVALID, "set_list_policy: policy must be 0 or 1");
  if ((policy == 1) != I.per_cell_lists) {
    I.per_cell_lists = policy == 1;
    I.drop_graphs();
  }
}

void GpuSolver::get_list_stats(int64_t out[5]) {
  Impl& I = *p_;
  for (int i = 0; i < 4; ++i) out[i] = I.hcounts[i];
  out[4] = I.per_cell_lists ? 1 : 0;
}

}  // namespace ucfvb
