// Host-side conversion of the flat reference views (include/ucfvb.h) into
// the device layout consumed by kernels.cuh (32-cell AoSoA chunks).
#pragma once

#include <cstdint>
#include <functional>
#include <stdexcept>
#include <string>
#include <vector>

#include "ucfvb.h"

namespace ucfvb {

struct ApiError : std::runtime_error {
  int code;
  ApiError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

struct HostLayout {
  int n = 0, n_owned = 0, n_pad = 0, K = 0, NQ = 0, NF = 0, Q = 0, MM = 0, MD = 0;
  std::vector<int32_t> st_idx, dir_idx, nbr, dest, cface;
  std::vector<double> pinv, phi, phi01, pinv_lin, pinv_dir, oi;
  std::vector<uint8_t> nfc;
  // face arrays (canonical orientation) and the face-major face-point slots
  std::vector<double> fnx, fny, flen;
  std::vector<int8_t> fkind, fpatch;
  std::vector<int32_t> fslot;  // [n_faces][2] residual slots of the face's owners
  std::vector<double> deact_thr, eps2, h, inv_vol;
  double qw[4] = {0, 0, 0, 0};
  // reference slot of each cell-local qp, for the val_left_/val_right_ tap
  std::vector<int64_t> qp_ptr;
  std::vector<int32_t> qp_slot;
  int n_faces = 0;
};

// Builds the layout; throws ApiError(UCFVB_INVALID / UCFVB_UNSUPPORTED).
HostLayout build_layout(const ucfvb_mesh_view& m, const ucfvb_stencil_view& s, const ucfvb_options& o,
                        int n_threads, int n_owned, int halo_patch);

// parallel_for over [0, n) in contiguous ranges (std::thread; no OpenMP runtime needed)
void parallel_for(int64_t n, int n_threads, const std::function<void(int64_t, int64_t)>& body);

inline size_t aos_index(int c, int e, int E) {
  return ((static_cast<size_t>(c >> 5) * E) + e) * 32 + (c & 31);
}

}  // namespace ucfvb
