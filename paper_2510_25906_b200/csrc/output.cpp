// Run outputs: the reference's legacy-VTK field snapshot
// and census / timing CSVs (run.cpp:157-213), byte-identical to its writers
// (every double as "%.17g", run.cpp:17-21). The VTK body is formatted by
// several host threads into per-range buffers and written in cell order, so a
// config-3 snapshot (8.4 M cells) does not serialise on snprintf.
#include <algorithm>
#include <cstdio>
#include <fstream>
#include <string>
#include <vector>

#include "layout.hpp"
#include "setup.hpp"
#include "ucfvb.h"

namespace ucfvb {

namespace {

inline void put(std::string& s, double x) {
  char buf[32];
  const int n = std::snprintf(buf, sizeof buf, "%.17g", x);
  s.append(buf, n);
}

inline void put(std::string& s, long long x) {
  char buf[24];
  const int n = std::snprintf(buf, sizeof buf, "%lld", x);
  s.append(buf, n);
}

// pressure (euler.hpp:30-32), host compiled with -ffp-contract=off
inline double pressure(const double* s, double g) { return (g - 1.0) * (s[3] - 0.5 * (s[1] * s[1] + s[2] * s[2]) / s[0]); }

// format rows [0, n) by `row` on several threads and append them in order
template <typename F>
void emit(std::ofstream& out, int64_t n, F&& row) {
  constexpr int64_t kRange = 1 << 15;
  const int64_t nr = (n + kRange - 1) / kRange;
  std::vector<std::string> part(static_cast<size_t>(nr));
  parallel_for(nr, 0, [&](int64_t a, int64_t b) {
    for (int64_t r = a; r < b; ++r) {
      std::string& s = part[static_cast<size_t>(r)];
      const int64_t i1 = std::min(n, (r + 1) * kRange);
      for (int64_t i = r * kRange; i < i1; ++i) row(s, i);
    }
  });
  for (const std::string& s : part) out.write(s.data(), static_cast<std::streamsize>(s.size()));
}

std::ofstream open_out(const char* path) {
  if (!path) throw ApiError(UCFVB_INVALID, "output: null path");
  std::ofstream out(path, std::ios::binary);
  if (!out) throw ApiError(UCFVB_INVALID, std::string("cannot open output file: ") + path);
  return out;
}

}  // namespace

// write_field_snapshot (run.cpp:160-190)
void write_field_snapshot(const ucfvb_mesh_view& m, const double* state, const uint8_t* labels, double gamma,
                          const char* path) {
  if (!state || !labels) throw ApiError(UCFVB_INVALID, "write_field_snapshot: null state/labels");
  std::ofstream out = open_out(path);
  out << "# vtk DataFile Version 3.0\n";
  out << "ucfv fields\n";
  out << "ASCII\n";
  out << "DATASET UNSTRUCTURED_GRID\n";
  out << "POINTS " << m.n_vertices << " double\n";
  emit(out, m.n_vertices, [&](std::string& s, int64_t i) {
    put(s, m.vertices[2 * i]);
    s += ' ';
    put(s, m.vertices[2 * i + 1]);
    s += " 0\n";
  });
  const int64_t list_len = static_cast<int64_t>(m.cell_vtx_ptr[m.n_cells]) + m.n_cells;
  out << "CELLS " << m.n_cells << " " << list_len << "\n";
  emit(out, m.n_cells, [&](std::string& s, int64_t c) {
    const int a = m.cell_vtx_ptr[c], b = m.cell_vtx_ptr[c + 1];
    put(s, static_cast<long long>(b - a));
    for (int i = a; i < b; ++i) {
      s += ' ';
      put(s, static_cast<long long>(m.cell_vtx[i]));
    }
    s += '\n';
  });
  out << "CELL_TYPES " << m.n_cells << "\n";
  emit(out, m.n_cells, [&](std::string& s, int64_t c) {
    const int nv = m.cell_vtx_ptr[c + 1] - m.cell_vtx_ptr[c];
    s += nv == 3 ? "5\n" : (nv == 4 ? "9\n" : "7\n");
  });
  out << "CELL_DATA " << m.n_cells << "\n";
  out << "SCALARS density double 1\nLOOKUP_TABLE default\n";
  emit(out, m.n_cells, [&](std::string& s, int64_t c) {
    put(s, state[4 * c]);
    s += '\n';
  });
  out << "SCALARS pressure double 1\nLOOKUP_TABLE default\n";
  emit(out, m.n_cells, [&](std::string& s, int64_t c) {
    put(s, pressure(state + 4 * c, gamma));
    s += '\n';
  });
  out << "VECTORS velocity double\n";
  emit(out, m.n_cells, [&](std::string& s, int64_t c) {
    const double* u = state + 4 * c;
    put(s, u[1] / u[0]);
    s += ' ';
    put(s, u[2] / u[0]);
    s += " 0\n";
  });
  out << "SCALARS scheme int 1\nLOOKUP_TABLE default\n";
  emit(out, m.n_cells, [&](std::string& s, int64_t c) {
    put(s, static_cast<long long>(labels[c]));
    s += '\n';
  });
  if (!out) throw ApiError(UCFVB_INVALID, std::string("write failed: ") + path);
}

// write_census_csv (run.cpp:192-202)
void write_census_csv(const ucfvb_census_row* rows, int n_rows, int64_t n_cells, const char* path) {
  if (n_rows > 0 && !rows) throw ApiError(UCFVB_INVALID, "write_census_csv: null rows");
  std::ofstream out = open_out(path);
  std::string s = "step,t,dt,linear,cwenoz,muscl,first,frac_linear,frac_cwenoz,frac_muscl,frac_first\n";
  for (int i = 0; i < n_rows; ++i) {
    const ucfvb_census_row& r = rows[i];
    put(s, static_cast<long long>(r.step));
    s += ',';
    put(s, r.t);
    s += ',';
    put(s, r.dt);
    for (int k = 0; k < 4; ++k) {
      s += ',';
      put(s, static_cast<long long>(r.counts[k]));
    }
    for (int k = 0; k < 4; ++k) {
      s += ',';
      // static_cast<double>(long) / int (run.cpp:200): the int converts to double
      put(s, static_cast<double>(r.counts[k]) / static_cast<double>(static_cast<int>(n_cells)));
    }
    s += '\n';
  }
  out << s;
  if (!out) throw ApiError(UCFVB_INVALID, std::string("write failed: ") + path);
}

// write_timing_csv (run.cpp:204-213)
void write_timing_csv(const ucfvb_timing_row* rows, int n_rows, const char* path) {
  if (n_rows > 0 && !rows) throw ApiError(UCFVB_INVALID, "write_timing_csv: null rows");
  std::ofstream out = open_out(path);
  std::string s = "step,wall,reconstruct,detect,weights,flux\n";
  for (int i = 0; i < n_rows; ++i) {
    const ucfvb_timing_row& r = rows[i];
    put(s, static_cast<long long>(r.step));
    for (double x : {r.wall, r.reconstruct, r.detect, r.weights, r.flux}) {
      s += ',';
      put(s, x);
    }
    s += '\n';
  }
  out << s;
  if (!out) throw ApiError(UCFVB_INVALID, std::string("write failed: ") + path);
}

}  // namespace ucfvb
