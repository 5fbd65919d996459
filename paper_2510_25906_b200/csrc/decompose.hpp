// Domain decomposition (see decompose.cpp).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "ucfvb.h"

struct ucfvb_subdomain {
  int rank = 0, n_parts = 1, n_owned = 0, n_local = 0;
  int n_interior = 0;  // owned cells [0, n_interior) that no peer holds (never sent)
  std::vector<int32_t> gid, part_of_local;
  // local mesh (vertices borrowed from the global view)
  std::vector<int32_t> cvp, cv, cfp, cf, fvtx, fl, fr, patch, partner, shift, pqp;
  std::vector<double> centroid, area, h, normal, length, midpoint, qp, qw;
  std::vector<std::string> patch_names;
  std::vector<const char*> pnames;
  // local stencils
  std::vector<int64_t> central_ptr, pinv_off, pinv_lin_off, dir_ptr, dir_member_ptr, pinv_dir_off, qp_ptr, phi_off;
  std::vector<int32_t> central, dir_members, qp_slot;
  std::vector<double> pinv, pinv_lin, pinv_dir, oi, phi;
  struct Peer {
    int rank = 0;
    std::vector<int32_t> send;
    int recv_begin = 0, n_recv = 0;
  };
  std::vector<Peer> peers;
  ucfvb_mesh_view mv{};
  ucfvb_stencil_view sv{};
};

namespace ucfvb {
void partition_rcb(const ucfvb_mesh_view& m, int n_parts, int32_t* part);
ucfvb_subdomain* build_subdomain(const ucfvb_mesh_view& m, const ucfvb_stencil_view& s, const int32_t* part,
                                 int n_parts, int r);
}  // namespace ucfvb
