// 3D subdomain (see decompose3.cpp).
#pragma once

#include <cstdint>
#include <vector>

#include "ucfvb3.h"

struct ucfvb3_subdomain {
  int rank = 0, n_parts = 1, n_owned = 0, n_local = 0, n_faces = 0;
  std::vector<int32_t> gid;
  // local mesh
  std::vector<double> cell_vtx, centroid, volume, h, face_qp, face_n, face_wa, face_vtx;
  std::vector<int32_t> cell_faces, cell_nbr, cell_nbr_shift, face_left, face_right;
  std::vector<int8_t> cell_side;
  // local stencils (per-cell operator rows copied; lattice-class rows borrowed from the global set)
  std::vector<int32_t> central, op_index, dir_members, qp_slot;
  std::vector<double> pinv, pinv_lin, pinv_dir, oi, phi;
  struct Peer {
    int rank = 0;
    std::vector<int32_t> send;  // local ids of owned cells the peer holds as halo, in its order
    int recv_begin = 0, n_recv = 0;
  };
  std::vector<Peer> peers;
  ucfvb3_mesh_view mv{};
  ucfvb3_stencil_view sv{};
};
