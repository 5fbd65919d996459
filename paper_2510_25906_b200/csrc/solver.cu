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

// meshes from this size run k_spread with 8 cells per thread (kernels.cuh)
constexpr int kSpreadWideCells = 1 << 20;

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
  // UCFVB_CELLS_SPLIT: the CWENOZ tiles and the MUSCL tiles in two launches
  Launch cells_c = nullptr, cells_m = nullptr;
  void (*cells_split_setup)(int n_sm, int* grid_c, Launch* launch_c, int* grid_m, Launch* launch_m) = nullptr;
  int cells_c_grid = 0, cells_m_grid = 0;
  void (*pack_records)(cudaStream_t, const Layout&, unsigned char*, unsigned char*) = nullptr;
  // per cell: CWENOZ record stride, group A bytes (= group B's offset), MUSCL record stride, group A bytes
  uint32_t rec_bytes[4] = {0, 0, 0, 0};
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

template <int K, int NQ, int NF, int MM, int MD, int WHICH = 0>
void troubled_cells_launcher(dim3 g, cudaStream_t st, const Layout& L, const Physics& p, const Scratch& S,
                             const double4* U, int f) {
  launch_k(k_troubled_cells<K, NQ, NF, MM, MD, WHICH>, g, dim3(4 * kCellTile),
           CellTile<K, NQ, NF, MM, MD, kCellTile, WHICH>::BYTES + 16, st, L, p, S, U, f);
}

// raise the dynamic smem limit and size the persistent grid (resident blocks x SMs)
template <typename Kfn>
int persistent_grid(Kfn k, uint32_t smem, int n_sm, int threads = kBlock) {
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  int per_sm = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, threads, smem));
  return std::max(1, per_sm) * n_sm;
}

template <int K, int NQ, int NF, int MMT, int MDT, bool UNI>
KernelSet make_set() {
  KernelSet s;
  s.central = [](dim3 g, cudaStream_t st, const Layout& L, const Physics& p, const Scratch& S, const double4* U,
                 int f) { launch_k(k_central<K, NQ, NF, MMT, MDT, UNI>, g, kBlock, 0, st, L, p, S, U, f); };
  s.spread = [](dim3 g, cudaStream_t st, const Layout& L, const Scratch& S, const double4* U, int f, int d) {
    // g.x = blocks of the one-cell-per-thread form; large meshes run 8 cells per thread
    if (L.n >= kSpreadWideCells)
      launch_k(k_spread<K, NQ, NF, MMT, MDT, UNI, 8>, dim3((g.x + 7) / 8), kBlock, 0, st, L, S, U, f, d);
    else
      launch_k(k_spread<K, NQ, NF, MMT, MDT, UNI, 1>, g, kBlock, 0, st, L, S, U, f, d);
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
      *grid = persistent_grid(k_troubled_cells<K, NQ, NF, MMT, MDT>,
                              CellRec<K, NQ, NF, MMT, MDT, kCellTile>::BYTES + 16, n_sm, 4 * kCellTile);
      *launch = troubled_cells_launcher<K, NQ, NF, MMT, MDT>;
    };
    s.cells_split_setup = [](int n_sm, int* gc, KernelSet::Launch* lc, int* gm, KernelSet::Launch* lm) {
      *gc = persistent_grid(k_troubled_cells<K, NQ, NF, MMT, MDT, 1>,
                            CellTile<K, NQ, NF, MMT, MDT, kCellTile, 1>::BYTES + 16, n_sm, 4 * kCellTile);
      *lc = troubled_cells_launcher<K, NQ, NF, MMT, MDT, 1>;
      *gm = persistent_grid(k_troubled_cells<K, NQ, NF, MMT, MDT, 2>,
                            CellTile<K, NQ, NF, MMT, MDT, kCellTile, 2>::BYTES + 16, n_sm, 4 * kCellTile);
      *lm = troubled_cells_launcher<K, NQ, NF, MMT, MDT, 2>;
    };
    s.pack_records = [](cudaStream_t st, const Layout& L, unsigned char* rc, unsigned char* rm) {
      k_pack_records<K, NQ, NF, MMT, MDT><<<(L.n + 255) / 256, 256, 0, st>>>(L, rc, rm);
    };
    s.rec_bytes[0] = R::GC;
    s.rec_bytes[1] = R::CA;
    s.rec_bytes[2] = R::GM;
    s.rec_bytes[3] = R::MA;
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
  // k_troubled_split) or dense per-cell lists (k_troubled_cells over per-cell
  // records; generic k_cwenoz / k_muscl off the fast path). Adaptive by
  // default: chunks stage whole 32-cell chunks of rows, so they win only when
  // the troubled cells fill the chunks they occupy (config 2: 84 %, chunks
  // 62.6 vs 74 us/stage; config 3: 50 %, per-cell lists 4.0 vs 6.0 ms/stage;
  // profiles/round2.md). UCFVB_TROUBLED=chunks|lists or set_list_policy pins it.
  bool per_cell_lists = false;
  bool lists_auto = true;
  int* hcounts = nullptr;  // pinned copy of S.counts after the last synchronising call
  // after a synchronising call: the adaptive policy follows the last stage's chunk fill
  void adapt_lists() {
    if (!lists_auto || !ks.troubled || !ks.cells) return;
    const int64_t cells = int64_t(hcounts[0]) + hcounts[1], chunks = int64_t(hcounts[2]) + hcounts[3];
    if (chunks <= 0) return;
    const bool want = 4 * cells < 3 * 32 * chunks;
    if (want != per_cell_lists) {
      per_cell_lists = want;
      drop_graphs();
    }
  }
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

  // ---- halo exchange of a stage state (subdomains) ------------------------
  // Owned cells are ordered [interior | sent] (ucfvb_subdomain_build): the
  // stage's gather updates the sent cells [n_int, n_owned) first, the exchange
  // (pack per peer + transport) then runs on comm_stream -- forked from and
  // joined back into the solver stream with events, inside the step graph --
  // while the gather updates the interior [0, n_int). Transports: NCCL
  // (attach_nccl: grouped ncclSend/ncclRecv) or an in-process loopback group
  // (ucfvb_group_*: one cudaMemcpyAsync per peer block, single device).
  int n_int = -1;  // < 0: no exchange attached
  cudaStream_t comm_stream = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  bool in_group = false;
  double4* pending_xout = nullptr;  // loopback: this stage's output, awaiting the group's copies
  bool exchanging() const { return n_int >= 0 && !peers.empty(); }

  void ensure_comm_stream() {
    if (comm_stream) return;
    CK(cudaStreamCreateWithFlags(&comm_stream, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming));
  }

  // on comm_stream: pack the owned cells each peer needs, then (NCCL) one
  // grouped send/recv into buf's halo blocks
  int64_t exchange_start(double4* buf) {
    int64_t nl = 0;
    for (const DevPeer& p : peers)
      if (p.n_send) {
        launch_k(k_halo_pack, dim3((p.n_send + 255) / 256), 256, 0, comm_stream, buf, p.send_idx, p.n_send,
                 sendbuf + p.send_off);
        ++nl;
      }
    if (comm) {
      NK(nccl().GroupStart());
      for (const DevPeer& p : peers) {
        if (p.n_send)
          NK(nccl().Send(sendbuf + p.send_off, 4 * static_cast<size_t>(p.n_send), ncclDouble, p.rank, comm,
                         comm_stream));
        if (p.n_recv)
          NK(nccl().Recv(buf + p.recv_begin, 4 * static_cast<size_t>(p.n_recv), ncclDouble, p.rank, comm,
                         comm_stream));
      }
      NK(nccl().GroupEnd());
    }
    return nl;
  }
  // the next kernel on the solver stream waits for the exchange
  void exchange_join() {
    CK(cudaEventRecord(ev_join, comm_stream));
    CK(cudaStreamWaitEvent(stream, ev_join, 0));
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
  // xout: this stage's output state, whose halo is exchanged (subdomains)
  int64_t launch_stage(const double4* U, bool first, const RkEpilogue& rk, bool census, bool dt_next = false,
                       double4* xout = nullptr) {
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
        if (UCFVB_CELLS_SPLIT && L.n >= kSpreadWideCells) {  // small meshes: one launch (config 1: +3.5 us/stage split)
          ks.cells_c(dim3(std::min(ks.cells_c_grid, (L.n + kCellTile - 1) / kCellTile + 1)), stream, L, ph, S, U,
                     FL_NAD | FL_FALLBACK | taps);
          ks.cells_m(dim3(std::min(ks.cells_m_grid, (L.n + kCellTile - 1) / kCellTile + 1)), stream, L, ph, S, U,
                     FL_NAD | FL_FALLBACK | taps);
          nl += 4;
        } else {
          ks.cells(dim3(std::min(ks.cells_grid, (L.n + kCellTile - 1) / kCellTile + 2)), stream, L, ph, S, U,
                   FL_NAD | FL_FALLBACK | taps);
          nl += 3;
        }
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
    ff |= dt_next ? FL_DT : 0;
    if (xout && exchanging()) {
      RkEpilogue sent = rk, interior = rk;
      sent.c_begin = n_int;
      sent.c_end = L.n_owned;
      interior.c_begin = 0;
      interior.c_end = n_int;
      nl += launch_gather(sent, ff);
      CK(cudaEventRecord(ev_fork, stream));
      CK(cudaStreamWaitEvent(comm_stream, ev_fork, 0));
      nl += exchange_start(xout);
      nl += launch_gather(interior, ff);
      if (in_group)
        pending_xout = xout;  // the group pushes the peer blocks, then joins
      else
        exchange_join();
    } else {
      nl += launch_gather(rk, ff);
    }
    record(4);
    CK(cudaGetLastError());
    accumulate_phases();
    return nl + 1;
  }

  // the gather + RK update of owned cells [rk.c_begin, rk.c_end) (all owned when c_end == 0)
  int64_t launch_gather(const RkEpilogue& rk, int flags) {
    const int n = (rk.c_end ? rk.c_end : L.n_owned) - rk.c_begin;
    if (n <= 0) return 0;
    ks.gather(dim3((n + kBlock - 1) / kBlock), stream, L, S, rk, flags, ds, opt.gamma);
    return 1;
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

  struct StagePlan {
    const double4* U;
    bool first;
    RkEpilogue rk;
    bool dt_next;
  };

  // The stages of one time step: `src` is the state at t, `dst` receives the
  // state at t+dt (combine2 orders, time_integrator.cpp:31-38, 42-74; SSP-RK3
  // Shu-Osher). Each stage's output (rk.out) is what its halo exchange sends.
  std::vector<StagePlan> step_plan(int rk, bool with_dt, const double4* src, double4* dst) {
    const double* dt = &ds->dt;
    std::vector<StagePlan> plan;
    auto stage = [&](const double4* U, bool first, double4* out, std::initializer_list<std::pair<const double4*, double>> t,
                     std::initializer_list<int> scaled, double4* rhs_out, bool dt_next) {
      RkEpilogue e{};
      e.dt = dt;
      e.out = out;
      e.rhs_out = rhs_out;
      auto sc = scaled.begin();
      for (const auto& [term, coef] : t) add_term(e, term, coef, *sc++ != 0);
      plan.push_back(StagePlan{U, first, e, dt_next});
    };
    if (rk == UCFVB_RK3) {
      double4 *u1 = work[0], *u2 = work[1];
      stage(src, true, u1, {{src, 1.0}, {src, 0.0}, {nullptr, 1.0}}, {0, 0, 1}, nullptr, false);
      stage(u1, false, u2, {{src, 0.75}, {u1, 0.25}, {nullptr, 0.25}}, {0, 0, 1}, nullptr, false);
      stage(u2, false, dst, {{src, 1.0 / 3.0}, {u2, 2.0 / 3.0}, {nullptr, 2.0 / 3.0}}, {0, 0, 1}, nullptr, with_dt);
    } else {
      using namespace rk54;
      double4 *ua = work[0], *ub = work[1], *uc = work[2], *ud = work[3], *r3 = work[4];
      stage(src, true, ua, {{src, 1.0}, {src, 0.0}, {nullptr, a10}}, {0, 0, 1}, nullptr, false);
      stage(ua, false, ub, {{src, b20}, {ua, b21}, {nullptr, a21}}, {0, 0, 1}, nullptr, false);
      stage(ub, false, uc, {{src, b30}, {ub, b32}, {nullptr, a32}}, {0, 0, 1}, nullptr, false);
      stage(uc, false, ud, {{src, b40}, {uc, b43}, {nullptr, a43}}, {0, 0, 1}, r3, false);
      stage(ud, false, dst, {{ub, c52}, {uc, c53}, {r3, a53}, {ud, c54}, {nullptr, a54}}, {0, 0, 1, 0, 1}, nullptr,
            with_dt);
    }
    return plan;
  }

  // All launches of one time step (the body a graph captures). With `with_dt`
  // the step starts from the reduced max_stable_dt of `src` (k_dt for a run's
  // first step, else the previous step's final gather); otherwise ds->dt was
  // set by the host.
  int64_t launch_step(int rk, bool with_dt, const double4* src, double4* dst, bool census) {
    int64_t nl = 0;
    if (with_dt) nl += launch_dt_finalize();
    for (const StagePlan& sp : step_plan(rk, with_dt, src, dst))
      nl += launch_stage(sp.U, sp.first, sp.rk, census, sp.dt_next, sp.rk.out);
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
  // advance_host_batch: device staging per direction, copy streams, events, pinned per-entry slots
  double4* pipe_up[2] = {nullptr, nullptr};
  double4* pipe_down[2] = {nullptr, nullptr};
  cudaStream_t up_stream = nullptr, down_stream = nullptr;
  cudaEvent_t pipe_ev[8] = {};
  char* pipe_host = nullptr;
  int pipe_slots = 0;
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
    if (pipe_host) cudaFreeHost(pipe_host);
    for (auto& e : pipe_ev)
      if (e) cudaEventDestroy(e);
    if (up_stream) cudaStreamDestroy(up_stream);
    if (down_stream) cudaStreamDestroy(down_stream);
    if (hcounts) cudaFreeHost(hcounts);
    for (auto& e : ev)
      if (e) cudaEventDestroy(e);
    if (stream) cudaStreamDestroy(stream);
    if (comm_stream) cudaStreamDestroy(comm_stream);
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_join) cudaEventDestroy(ev_join);
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
  if (const char* tl = std::getenv("UCFVB_TROUBLED")) {  // diagnostics: pin the list policy
    I.per_cell_lists = std::strcmp(tl, "lists") == 0;
    I.lists_auto = false;
  }
  CK(cudaMallocHost(&I.hcounts, 4 * sizeof(int)));
  std::memset(I.hcounts, 0, 4 * sizeof(int));
  if (I.ks.central_tma) {
    I.ks.central_tma_setup(I.n_sm, &I.ks.central_tma_grid, &I.ks.central);
    I.ks.troubled_setup(I.n_sm, &I.ks.troubled_grid, &I.ks.troubled);
    I.ks.cells_setup(I.n_sm, &I.ks.cells_grid, &I.ks.cells);
    if (UCFVB_CELLS_SPLIT)
      I.ks.cells_split_setup(I.n_sm, &I.ks.cells_c_grid, &I.ks.cells_c, &I.ks.cells_m_grid, &I.ks.cells_m);
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
    // one CWENOZ and one MUSCL record per cell (64-byte-line multiples), group B behind group A
    unsigned char* rc = dalloc<unsigned char>(static_cast<size_t>(H.n) * I.ks.rec_bytes[0], own);
    unsigned char* rm = dalloc<unsigned char>(static_cast<size_t>(H.n) * I.ks.rec_bytes[2], own);
    L.rec_ca = rc;
    L.rec_cb = rc + I.ks.rec_bytes[1];
    L.rec_ma = rm;
    L.rec_mb = rm + I.ks.rec_bytes[3];
    I.ks.pack_records(I.stream, L, rc, rm);
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
    // the persisting carve-out pays only while the stage buffers are L2-sized
    // (config 2: 117 MB, +21 %); for config 3 (4.8 GB) it evicts the stencil
    // gathers' lines and costs 17 % (measured, profiles/round2.md)
    const bool want = !(e && e[0] == '0') && (n_fp + n_ff + n_dofs) * sizeof(double4) <= (size_t(256) << 20);
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
  I.adapt_lists();
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
  I.adapt_lists();
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
  I.adapt_lists();
  if (he[0]) {
    const int failed = std::min(std::max(0, he[3]), n_steps - 1);
    I.cur = (cur0 + failed) & 1;
    I.raise_device_error(he[0], he[1], he[2]);
  }
  return hs->t + hs->dt;
}

// The pipelined form of advance_host over independent states of one mesh (an
// ensemble): the upload of state i+1 and the download of result i-1 run on two
// copy streams (both PCIe directions) while state i is stepped. Two device
// staging buffers per direction; the compute stream copies staging -> state
// buffer and state buffer -> staging device-to-device (2 x 32 B/cell at HBM
// rate), so the captured step graphs and their buffers are untouched.
void GpuSolver::advance_host_batch(int n_batch, const double* const* u_in, double* const* u_out, int n_steps, int rk,
                                   double t0, double* t_out) {
  Impl& I = *p_;
  if (rk != UCFVB_RK3 && rk != UCFVB_RK54) throw ApiError(UCFVB_INVALID, "advance_host_batch: unknown integrator");
  if (n_steps <= 0) throw ApiError(UCFVB_INVALID, "advance_host_batch: n_steps must be >= 1");
  if (n_batch <= 0) throw ApiError(UCFVB_INVALID, "advance_host_batch: n_batch must be >= 1");
  for (int i = 0; i < n_batch; ++i)
    if (!u_in[i] || !u_out[i]) throw ApiError(UCFVB_INVALID, "advance_host_batch: null state pointer");
  const size_t bytes = sizeof(double4) * I.L.n;
  if (!I.pipe_up[0]) {
    for (int i = 0; i < 2; ++i) {
      I.pipe_up[i] = dalloc<double4>(I.L.n, I.owned);
      I.pipe_down[i] = dalloc<double4>(I.L.n, I.owned);
    }
    CK(cudaStreamCreateWithFlags(&I.up_stream, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&I.down_stream, cudaStreamNonBlocking));
    for (auto& e : I.pipe_ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  // pinned per-entry slots: the dt-state each entry starts from, and what it ended with
  const size_t slot = 2 * sizeof(DtState) + 4 * sizeof(int);
  if (I.pipe_slots < n_batch) {
    if (I.pipe_host) CK(cudaFreeHost(I.pipe_host));
    I.pipe_host = nullptr;
    CK(cudaMallocHost(&I.pipe_host, slot * n_batch));
    I.pipe_slots = n_batch;
  }
  auto hs_in = [&](int i) { return reinterpret_cast<DtState*>(I.pipe_host + slot * i); };
  auto hs_out = [&](int i) { return reinterpret_cast<DtState*>(I.pipe_host + slot * i + sizeof(DtState)); };
  auto he = [&](int i) { return reinterpret_cast<int*>(I.pipe_host + slot * i + 2 * sizeof(DtState)); };
  // events: [0..1] upload landed, [2..3] upload buffer consumed, [4..5] result staged, [6..7] download done
  cudaEvent_t* ev = I.pipe_ev;
  I.reset_ties();
  I.S.step = &I.ds->step;
  const int cur0 = I.cur;
  int64_t nl = 0;
  for (int i = 0; i < n_batch; ++i) {
    const int b = i & 1;
    if (i >= 2) CK(cudaStreamWaitEvent(I.up_stream, ev[2 + b], 0));
    CK(cudaMemcpyAsync(I.pipe_up[b], u_in[i], bytes, cudaMemcpyHostToDevice, I.up_stream));
    CK(cudaEventRecord(ev[b], I.up_stream));
    CK(cudaStreamWaitEvent(I.stream, ev[b], 0));
    I.cur = cur0;
    CK(cudaMemcpyAsync(I.ubuf[I.cur], I.pipe_up[b], bytes, cudaMemcpyDeviceToDevice, I.stream));
    CK(cudaEventRecord(ev[2 + b], I.stream));
    DtState* hs = hs_in(i);
    *hs = DtState{};
    hs->dmin_bits = static_cast<unsigned long long>(0x7e37e43c8800759cULL);  // bits of 1e300
    hs->t = t0;
    hs->step = -1;
    hs->t_end = INFINITY;
    hs->cfl = I.opt.cfl;
    CK(cudaMemcpyAsync(I.ds, hs, sizeof(DtState), cudaMemcpyHostToDevice, I.stream));
    nl += I.launch_dt_reduce(I.ubuf[I.cur]);
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
    I.allreduce_error();
    CK(cudaMemcpyAsync(he(i), I.S.err, 4 * sizeof(int), cudaMemcpyDeviceToHost, I.stream));
    CK(cudaMemcpyAsync(hs_out(i), I.ds, sizeof(DtState), cudaMemcpyDeviceToHost, I.stream));
    if (i >= 2) CK(cudaStreamWaitEvent(I.stream, ev[6 + b], 0));
    CK(cudaMemcpyAsync(I.pipe_down[b], I.ubuf[I.cur], bytes, cudaMemcpyDeviceToDevice, I.stream));
    CK(cudaEventRecord(ev[4 + b], I.stream));
    CK(cudaStreamWaitEvent(I.down_stream, ev[4 + b], 0));
    CK(cudaMemcpyAsync(u_out[i], I.pipe_down[b], bytes, cudaMemcpyDeviceToHost, I.down_stream));
    CK(cudaEventRecord(ev[6 + b], I.down_stream));
  }
  I.launches = nl;
  I.S.step = I.step_zero;
  I.fetch_counts();
  CK(cudaStreamSynchronize(I.stream));
  CK(cudaStreamSynchronize(I.down_stream));
  CK(cudaGetLastError());
  I.stage_is_first = false;
  I.adapt_lists();
  for (int i = 0; i < n_batch; ++i) {
    if (he(i)[0]) {
      // the error word is sticky: entry i failed and the later entries did not run
      I.cur = cur0;
      const int k = he(i)[0], f = he(i)[1], c = he(i)[2];
      try {
        I.raise_device_error(k, f, c);
      } catch (ApiError& e) {
        throw ApiError(e.code, std::string(e.what()) + " (batch entry " + std::to_string(i) + ")");
      }
    }
    if (t_out) t_out[i] = hs_out(i)->t + hs_out(i)->dt;
  }
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

// the subdomain's exchange plan on the device: send lists per peer, one
// contiguous send buffer, the interior / sent split and the exchange stream
static void setup_exchange(GpuSolver::Impl& I, const ucfvb_subdomain* sub) {
  if (!I.peers.empty()) throw ApiError(UCFVB_INVALID, "solver: an exchange is already attached");
  size_t off = 0;
  for (const auto& p : sub->peers) {
    GpuSolver::Impl::DevPeer d;
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
  I.n_int = sub->n_interior;
  I.ensure_comm_stream();
  // graphs captured before the exchange existed are stale
  I.drop_graphs();
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
  setup_exchange(I, sub);
}

// ---- in-process loopback group ---------------------------------------------
// min of the parts' collected dt terms, written back to every part
__global__ void k_group_dt_min(DtState* const* ds, int n) {
  double m = ds[0]->dmin;
  for (int i = 1; i < n; ++i) m = smin(m, ds[i]->dmin);
  for (int i = 0; i < n; ++i) ds[i]->dmin = m;
}
// the job's error word (as allreduce_error): kind by max, step / face / cell by min
__global__ void k_group_err(int* const* err, int n) {
  int e[4] = {err[0][0], err[0][1], err[0][2], err[0][3]};
  for (int i = 1; i < n; ++i) {
    e[0] = max(e[0], err[i][0]);
    for (int j = 1; j < 4; ++j) e[j] = min(e[j], err[i][j]);
  }
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < 4; ++j) err[i][j] = e[j];
}

struct GpuGroup::Impl {
  std::vector<GpuSolver::Impl*> P;
  std::vector<cudaEvent_t> ev_part, ev_sent;
  cudaEvent_t ev_lead = nullptr;
  DtState** d_ds = nullptr;
  int** d_err = nullptr;
  // push plan: part p sends its peer block e to part `to`, into `to`'s receive range
  struct Push {
    int to;
    size_t src_off;
    int dst_begin, n;
  };
  std::vector<std::vector<Push>> push;
  std::vector<std::vector<int>> senders;  // parts whose copies part q waits for
  cudaGraphExec_t graph[2][2] = {};
  int64_t graph_launches[2][2] = {};
  int64_t launches = 0;
  cudaStream_t lead() const { return P[0]->stream; }

  void all_to_lead() {
    for (size_t p = 1; p < P.size(); ++p) {
      CK(cudaEventRecord(ev_part[p], P[p]->stream));
      CK(cudaStreamWaitEvent(lead(), ev_part[p], 0));
    }
  }
  void lead_to_all() {
    CK(cudaEventRecord(ev_lead, lead()));
    for (size_t p = 1; p < P.size(); ++p) CK(cudaStreamWaitEvent(P[p]->stream, ev_lead, 0));
  }

  // one RK step of every part (device dt): the same kernels and exchange
  // schedule as a rank's step, with the group's copies as the transport
  int64_t launch_step(int rk, int parity) {
    int64_t nl = 0;
    const int n = static_cast<int>(P.size());
    for (auto* q : P) {
      launch_k(k_dt_collect, 1, 1, 0, q->stream, q->ds);
      ++nl;
    }
    all_to_lead();
    k_group_dt_min<<<1, 1, 0, lead()>>>(d_ds, n);
    ++nl;
    lead_to_all();
    std::vector<std::vector<GpuSolver::Impl::StagePlan>> plan(n);
    for (int p = 0; p < n; ++p) {
      GpuSolver::Impl* q = P[p];
      launch_k(k_dt_finalize, 1, 1, 0, q->stream, q->ds, q->S.err, 0);
      ++nl;
      plan[p] = q->step_plan(rk, true, q->ubuf[parity], q->ubuf[parity ^ 1]);
    }
    for (size_t i = 0; i < plan[0].size(); ++i) {
      for (int p = 0; p < n; ++p) {
        const auto& sp = plan[p][i];
        nl += P[p]->launch_stage(sp.U, sp.first, sp.rk, false, sp.dt_next, sp.rk.out);
      }
      // every part pushes its packed peer blocks into the receivers' halo ranges
      for (int p = 0; p < n; ++p) {
        GpuSolver::Impl* q = P[p];
        for (const Push& x : push[p])
          CK(cudaMemcpyAsync(P[x.to]->pending_xout + x.dst_begin, q->sendbuf + x.src_off,
                             sizeof(double4) * static_cast<size_t>(x.n), cudaMemcpyDeviceToDevice, q->comm_stream));
        CK(cudaEventRecord(ev_sent[p], q->comm_stream));
      }
      for (int p = 0; p < n; ++p)
        for (int from : senders[p]) CK(cudaStreamWaitEvent(P[p]->stream, ev_sent[from], 0));
    }
    for (int p = 0; p < n; ++p) CK(cudaStreamWaitEvent(P[p]->stream, ev_sent[p], 0));  // own exchange stream joined
    all_to_lead();
    k_group_err<<<1, 1, 0, lead()>>>(d_err, n);
    ++nl;
    lead_to_all();
    return nl;
  }

  cudaGraphExec_t get_graph(int rk, int parity) {
    cudaGraphExec_t& g = graph[rk][parity];
    if (g) return g;
    cudaGraph_t gr;
    CK(cudaStreamBeginCapture(lead(), cudaStreamCaptureModeThreadLocal));
    lead_to_all();
    const int64_t nl = launch_step(rk, parity);
    all_to_lead();
    CK(cudaStreamEndCapture(lead(), &gr));
    CK(cudaGraphInstantiate(&g, gr, 0));
    CK(cudaGraphDestroy(gr));
    graph_launches[rk][parity] = nl;
    return g;
  }

  ~Impl() {
    for (auto& a : graph)
      for (auto& g : a)
        if (g) cudaGraphExecDestroy(g);
    for (auto e : ev_part)
      if (e) cudaEventDestroy(e);
    for (auto e : ev_sent)
      if (e) cudaEventDestroy(e);
    if (ev_lead) cudaEventDestroy(ev_lead);
    if (d_ds) cudaFree(d_ds);
    if (d_err) cudaFree(d_err);
  }
};

GpuGroup::GpuGroup(GpuSolver* const* parts, const ucfvb_subdomain* const* subs, int n) : p_(new Impl) {
  Impl& G = *p_;
  if (n < 1) throw ApiError(UCFVB_INVALID, "group: needs at least one part");
  for (int p = 0; p < n; ++p) {
    if (!subs[p]) throw ApiError(UCFVB_INVALID, "group: every part must be created on a subdomain");
    if (subs[p]->rank != p || subs[p]->n_parts != n)
      throw ApiError(UCFVB_INVALID, "group: part i must be rank i of an n-part partition");
    GpuSolver::Impl& I = *parts[p]->p_;
    if (I.comm || I.in_group) throw ApiError(UCFVB_INVALID, "group: a part already has an exchange attached");
    if (I.device != parts[0]->p_->device) throw ApiError(UCFVB_INVALID, "group: all parts must share one device");
    G.P.push_back(&I);
  }
  CK(cudaSetDevice(G.P[0]->device));
  for (int p = 0; p < n; ++p) {
    setup_exchange(*G.P[p], subs[p]);
    G.P[p]->in_group = true;
  }
  G.push.resize(n);
  G.senders.resize(n);
  for (int p = 0; p < n; ++p)
    for (const auto& d : G.P[p]->peers) {
      if (!d.n_send) continue;
      const GpuSolver::Impl::DevPeer* back = nullptr;
      for (const auto& e : G.P[d.rank]->peers)
        if (e.rank == p) back = &e;
      if (!back || back->n_recv != d.n_send) throw ApiError(UCFVB_INVALID, "group: inconsistent exchange plans");
      G.push[p].push_back(Impl::Push{d.rank, d.send_off, back->recv_begin, d.n_send});
      G.senders[d.rank].push_back(p);
    }
  G.ev_part.resize(n);
  G.ev_sent.resize(n);
  for (int p = 0; p < n; ++p) {
    CK(cudaEventCreateWithFlags(&G.ev_part[p], cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&G.ev_sent[p], cudaEventDisableTiming));
  }
  CK(cudaEventCreateWithFlags(&G.ev_lead, cudaEventDisableTiming));
  std::vector<DtState*> hds(n);
  std::vector<int*> herr(n);
  for (int p = 0; p < n; ++p) {
    hds[p] = G.P[p]->ds;
    herr[p] = G.P[p]->S.err;
  }
  CK(cudaMalloc(&G.d_ds, n * sizeof(DtState*)));
  CK(cudaMalloc(&G.d_err, n * sizeof(int*)));
  CK(cudaMemcpy(G.d_ds, hds.data(), n * sizeof(DtState*), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(G.d_err, herr.data(), n * sizeof(int*), cudaMemcpyHostToDevice));
}

GpuGroup::~GpuGroup() = default;

// run_steps over the group (device dt, graph-replayed): every part advances
// n_steps; on a failure every part returns to the failing step's input
double GpuGroup::run_steps(int n_steps, int rk, double t0) {
  Impl& G = *p_;
  if (rk != UCFVB_RK3 && rk != UCFVB_RK54) throw ApiError(UCFVB_INVALID, "group: unknown integrator");
  if (n_steps <= 0) return t0;
  CK(cudaSetDevice(G.P[0]->device));
  const int cur0 = G.P[0]->cur;
  for (auto* q : G.P) {
    if (q->cur != cur0) throw ApiError(UCFVB_INVALID, "group: parts out of step");
    DtState h{};
    h.dmin_bits = static_cast<unsigned long long>(0x7e37e43c8800759cULL);  // bits of 1e300
    h.t = t0;
    h.step = -1;
    h.t_end = INFINITY;
    h.cfl = q->opt.cfl;
    CK(cudaMemcpyAsync(q->ds, &h, sizeof h, cudaMemcpyHostToDevice, q->stream));
    q->reset_ties();
    q->S.step = &q->ds->step;
    G.launches += q->launch_dt_reduce(q->ubuf[q->cur]);
    CK(cudaStreamSynchronize(q->stream));
  }
  for (int s = 0; s < n_steps; ++s) {
    const int par = (cur0 + s) & 1;
    if (G.P[0]->opt.use_graphs) {
      CK(cudaGraphLaunch(G.get_graph(rk, par), G.lead()));
      G.launches += G.graph_launches[rk][par];
    } else {
      G.lead_to_all();
      G.launches += G.launch_step(rk, par);
      G.all_to_lead();
    }
  }
  CK(cudaStreamSynchronize(G.lead()));
  CK(cudaGetLastError());
  DtState h{};
  CK(cudaMemcpy(&h, G.P[0]->ds, sizeof h, cudaMemcpyDeviceToHost));
  int e[4];
  CK(cudaMemcpy(e, G.P[0]->S.err, sizeof e, cudaMemcpyDeviceToHost));
  for (auto* q : G.P) {
    q->S.step = q->step_zero;
    q->fetch_counts();
    q->stage_is_first = false;
    q->cur = (cur0 + n_steps) & 1;
  }
  if (e[0]) {
    const int failed = std::min(std::max(0, e[3]), n_steps - 1);
    for (auto* q : G.P) q->cur = (cur0 + failed) & 1;
    try {
      G.P[0]->raise_device_error(e[0], e[1], e[2]);
    } catch (ApiError& err) {
      for (auto* q : G.P) q->reset_error();
      for (auto* q : G.P) CK(cudaStreamSynchronize(q->stream));
      throw ApiError(err.code, "group run failed at step " + std::to_string(failed) + ": " + err.what());
    }
  }
  return h.t + h.dt;
}

int64_t GpuGroup::launch_count() const { return p_->launches; }

void GpuSolver::set_list_policy(int policy) {
  Impl& I = *p_;
  if (policy < 0 || policy > 2) throw ApiError(UCFVB_INVALID, "set_list_policy: policy must be 0, 1 or 2");
  I.lists_auto = policy == 2;
  if (policy != 2 && (policy == 1) != I.per_cell_lists) {
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
