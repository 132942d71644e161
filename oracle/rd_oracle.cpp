// rd_oracle.cpp -- TEST INFRASTRUCTURE ONLY: the CPU parity oracle.
//
// A line-by-line CPU restatement (no Eigen, which is absent from this image)
// of the reference rdsolve solve path.  Citations are relative to
// /root/reference/proj.  Parity status: the reference cannot be compiled here
// (Eigen/doctest/CLI11 missing), so this oracle is pinned
// against the reference's own known-answer tests (tests/test_*.cpp hand cases,
// re-expressed in tests/test_oracle_kats.py) and Appendix A of SURVEY.md;
// the Eigen-internal orders it restates (dot product, LLT) are marked
// "restated, unverifiable here".
//
// Built with -O3 -ffp-contract=off and no -march, mirroring the reference's
// Release flags (CMakeLists.txt:6-7,31): no FMA contraction anywhere.
//
// Nothing in the product path (paper_2102_03515_b200/) links or loads this.

#include "rd_oracle.h"

#include <algorithm>
#include <array>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

namespace {

constexpr double kPi = 3.14159265358979323846;  // std::numbers::pi (target.cpp:9)

thread_local std::string g_err;

// ---------------------------------------------------------------------------
// parallel.cpp:12-73 -- fixed chunk grid (min(n,128) chunks, boundaries c*n/chunks),
// work distributed over g_threads workers; reduce sums partials in chunk order.
int g_threads = 1;

int64_t chunk_count(int64_t n) { return std::min<int64_t>(n, 128); }

void for_each_chunk(int64_t n, const std::function<void(int64_t, int64_t, int64_t)>& body) {
  if (n <= 0) return;
  const int64_t chunks = chunk_count(n);
  auto run_chunk = [&](int64_t c) { body(c, c * n / chunks, (c + 1) * n / chunks); };
  const int workers = static_cast<int>(std::min<int64_t>(g_threads, chunks));
  if (workers <= 1) {
    for (int64_t c = 0; c < chunks; ++c) run_chunk(c);
    return;
  }
  std::atomic<int64_t> next(0);
  auto work = [&]() {
    for (;;) {
      const int64_t c = next.fetch_add(1);
      if (c >= chunks) return;
      run_chunk(c);
    }
  };
  std::vector<std::thread> pool;
  for (int t = 0; t < workers - 1; ++t) pool.emplace_back(work);
  work();
  for (auto& th : pool) th.join();
}

void parallel_for(int64_t n, const std::function<void(int64_t, int64_t)>& body) {
  for_each_chunk(n, [&](int64_t, int64_t b, int64_t e) { body(b, e); });
}

double parallel_reduce(int64_t n, const std::function<double(int64_t, int64_t)>& partial) {
  if (n <= 0) return 0.0;
  std::vector<double> parts(static_cast<size_t>(chunk_count(n)), 0.0);
  for_each_chunk(n, [&](int64_t c, int64_t b, int64_t e) { parts[static_cast<size_t>(c)] = partial(b, e); });
  double sum = 0.0;
  for (double v : parts) sum += v;
  return sum;
}

// ---------------------------------------------------------------------------
// Containers (types.hpp:8-15): CSR with int32 indices, fp64 values.
struct V3 {
  double c[3];
};

struct Csr {
  int rows = 0, cols = 0;
  std::vector<int> rp{0};
  std::vector<int> ci;
  std::vector<double> v;
  int64_t nnz() const { return static_cast<int64_t>(ci.size()); }
};

using Vec = std::vector<double>;

// ---------------------------------------------------------------------------
// mesh.cpp
struct Mesh {
  std::vector<V3> vertices;
  std::vector<std::array<int, 4>> tets;
  std::vector<uint8_t> boundary;
  std::vector<uint8_t> refinement_edge;
  std::vector<int> generation;
  int nv() const { return static_cast<int>(vertices.size()); }
  int nt() const { return static_cast<int>(tets.size()); }
};

// mesh.cpp:14-18
bool on_unit_boundary(const V3& x) {
  for (int c = 0; c < 3; ++c)
    if (std::abs(x.c[c]) <= 1e-14 || std::abs(x.c[c] - 1.0) <= 1e-14) return true;
  return false;
}

// mesh.cpp:29-65 (vertex id (k*nv+j)*nv+i, 6 Kuhn chains per cell in perms order, tag 3, gen 0)
Mesh build_structured_cube(int n) {
  if (n < 1) throw std::invalid_argument("build_structured_cube: n must be >= 1");
  Mesh m;
  const int nv = n + 1;
  auto vid = [nv](int i, int j, int k) { return (k * nv + j) * nv + i; };
  m.vertices.reserve(static_cast<size_t>(nv) * nv * nv);
  for (int k = 0; k < nv; ++k)
    for (int j = 0; j < nv; ++j)
      for (int i = 0; i < nv; ++i) {
        V3 x{{static_cast<double>(i) / n, static_cast<double>(j) / n, static_cast<double>(k) / n}};
        m.vertices.push_back(x);
        m.boundary.push_back(on_unit_boundary(x) ? 1 : 0);
      }
  constexpr int perms[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
  m.tets.reserve(static_cast<size_t>(n) * n * n * 6);
  for (int k = 0; k < n; ++k)
    for (int j = 0; j < n; ++j)
      for (int i = 0; i < n; ++i)
        for (const auto& perm : perms) {
          std::array<int, 4> t;
          int c[3] = {i, j, k};
          t[0] = vid(c[0], c[1], c[2]);
          for (int s = 0; s < 3; ++s) {
            c[perm[s]] += 1;
            t[static_cast<size_t>(s) + 1] = vid(c[0], c[1], c[2]);
          }
          m.tets.push_back(t);
          m.refinement_edge.push_back(3);
          m.generation.push_back(0);
        }
  return m;
}

std::array<V3, 4> tet_vertices(const Mesh& m, int t) {
  const auto& tt = m.tets[static_cast<size_t>(t)];
  return {m.vertices[static_cast<size_t>(tt[0])], m.vertices[static_cast<size_t>(tt[1])],
          m.vertices[static_cast<size_t>(tt[2])], m.vertices[static_cast<size_t>(tt[3])]};
}

// mesh.cpp:188-191: |(v1-v0) x (v2-v0) . (v3-v0)| / 6  (Eigen cross; 3-dot = (a0b0+a1b1)+a2b2)
double tet_volume(const Mesh& m, int t) {
  const auto v = tet_vertices(m, t);
  double a[3], b[3], d[3];
  for (int c = 0; c < 3; ++c) {
    a[c] = v[1].c[c] - v[0].c[c];
    b[c] = v[2].c[c] - v[0].c[c];
    d[c] = v[3].c[c] - v[0].c[c];
  }
  const double x0 = a[1] * b[2] - a[2] * b[1];
  const double x1 = a[2] * b[0] - a[0] * b[2];
  const double x2 = a[0] * b[1] - a[1] * b[0];
  const double dot = (x0 * d[0] + x1 * d[1]) + x2 * d[2];
  return std::abs(dot) / 6.0;
}

// ---------------------------------------------------------------------------
// quadrature.cpp
struct Rule {
  std::vector<std::array<double, 4>> pts;
  std::vector<double> w;
  int size() const { return static_cast<int>(w.size()); }
};

Rule make_centroid() {  // quadrature.cpp:14-19
  Rule r;
  r.pts.push_back({0.25, 0.25, 0.25, 0.25});
  r.w.push_back(1.0);
  return r;
}

Rule make_degree2() {  // quadrature.cpp:21-30
  const double a = 0.1381966011250105;
  const double b = 0.5854101966249685;
  Rule r;
  for (int i = 0; i < 4; ++i) {
    std::array<double, 4> p{a, a, a, a};
    p[static_cast<size_t>(i)] = b;
    r.pts.push_back(p);
    r.w.push_back(0.25);
  }
  return r;
}

Rule make_degree5() {  // quadrature.cpp:24-55 (14-point Keast, literal constants :27-32)
  const double wa = 0.1126879257180162;
  const double a = 0.3108859192633005;
  const double wb = 0.0734930431163619;
  const double b = 0.0927352503108912;
  const double wc = 0.0425460207770812;
  const double c = 0.0455037041256497;
  Rule r;
  for (int i = 0; i < 4; ++i) {
    std::array<double, 4> p{a, a, a, a};
    p[static_cast<size_t>(i)] = 1.0 - 3.0 * a;
    r.pts.push_back(p);
    r.w.push_back(wa);
  }
  for (int i = 0; i < 4; ++i) {
    std::array<double, 4> p{b, b, b, b};
    p[static_cast<size_t>(i)] = 1.0 - 3.0 * b;
    r.pts.push_back(p);
    r.w.push_back(wb);
  }
  for (int i = 0; i < 4; ++i)
    for (int j = i + 1; j < 4; ++j) {
      const double m = 0.5 - c;
      std::array<double, 4> p{m, m, m, m};
      p[static_cast<size_t>(i)] = c;
      p[static_cast<size_t>(j)] = c;
      r.pts.push_back(p);
      r.w.push_back(wc);
    }
  return r;
}

// quadrature.cpp:57-82: three levels of centroid subdivision; every value is a
// dyadic rational (denominators <= 256), so the column means are exact in any order.
Rule make_subdivision64() {
  using Cell = std::array<std::array<double, 4>, 4>;  // cell[row][col], row = vertex
  std::vector<Cell> cells(1);
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < 4; ++j) cells[0][static_cast<size_t>(i)][static_cast<size_t>(j)] = i == j ? 1.0 : 0.0;
  auto colmean = [](const Cell& c) {
    std::array<double, 4> g{};
    for (int j = 0; j < 4; ++j) {
      double s = 0.0;
      for (int i = 0; i < 4; ++i) s += c[static_cast<size_t>(i)][static_cast<size_t>(j)];
      g[static_cast<size_t>(j)] = s / 4.0;
    }
    return g;
  };
  for (int level = 0; level < 3; ++level) {
    std::vector<Cell> next;
    for (const Cell& cell : cells) {
      const auto g = colmean(cell);
      for (int i = 0; i < 4; ++i) {
        Cell child = cell;
        child[static_cast<size_t>(i)] = g;
        next.push_back(child);
      }
    }
    cells.swap(next);
  }
  Rule r;
  for (const Cell& cell : cells) {
    r.pts.push_back(colmean(cell));
    r.w.push_back(1.0 / static_cast<double>(cells.size()));
  }
  return r;
}

const Rule& rule_by_id(int id) {
  static const Rule r0 = make_centroid(), r1 = make_degree2(), r2 = make_degree5(),
                    r3 = make_subdivision64();
  switch (id) {
    case 0: return r0;
    case 1: return r1;
    case 2: return r2;
    case 3: return r3;
  }
  throw std::invalid_argument("unknown rule");
}

// quadrature.cpp:106-114: p = Zero; p += lambda_k * v_k, k = 0..3
V3 physical_point(const std::array<double, 4>& lam, const std::array<V3, 4>& v) {
  V3 p{{0.0, 0.0, 0.0}};
  for (int k = 0; k < 4; ++k)
    for (int c = 0; c < 3; ++c) p.c[c] = p.c[c] + lam[static_cast<size_t>(k)] * v[static_cast<size_t>(k)].c[c];
  return p;
}

// ---------------------------------------------------------------------------
// target.cpp (+ ball, sine+random: BASELINE configs 2/3)
enum Smoothness { smooth_h2, discontinuous, smooth_nonzero_bc };

double sin3(const V3& x) {  // target.cpp:12-15
  return std::sin(kPi * x.c[0]) * std::sin(kPi * x.c[1]) * std::sin(kPi * x.c[2]);
}

// tests/oracles.hpp:97-108 splitmix64 on [-1,1)
void pseudo_random(int n, uint64_t seed, double* out) {
  uint64_t s = seed + 0x9e3779b97f4a7c15ULL;
  for (int i = 0; i < n; ++i) {
    uint64_t z = (s += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    z = z ^ (z >> 31);
    out[i] = 2.0 * (static_cast<double>(z >> 11) * 0x1.0p-53) - 1.0;
  }
}

struct Target {
  int kind = OR_TARGET_SMOOTH;
  Smoothness tag = smooth_h2;
  int n = 0;                 // lattice resolution (sine+random only)
  std::vector<double> nodal;  // (n+1)^3 random nodal values, zero on the boundary

  // P1 interpolant on the Kuhn lattice: cell = floor(n x) clamped, local
  // coordinates sorted descending pick the chain (ties -> first in mesh.cpp:46 perms order).
  double interp(const V3& x) const {
    const int nv = n + 1;
    int cell[3];
    double xi[3];
    for (int d = 0; d < 3; ++d) {
      const double s = x.c[d] * static_cast<double>(n);
      int ci = static_cast<int>(std::floor(s));
      ci = std::min(std::max(ci, 0), n - 1);
      cell[d] = ci;
      xi[d] = s - static_cast<double>(ci);
    }
    constexpr int perms[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
    int p = 0;
    for (; p < 5; ++p)
      if (xi[perms[p][0]] >= xi[perms[p][1]] && xi[perms[p][1]] >= xi[perms[p][2]]) break;
    const int* pm = perms[p];
    const double lam[4] = {1.0 - xi[pm[0]], xi[pm[0]] - xi[pm[1]], xi[pm[1]] - xi[pm[2]], xi[pm[2]]};
    int c[3] = {cell[0], cell[1], cell[2]};
    double val = 0.0;
    val = val + lam[0] * nodal[static_cast<size_t>((c[2] * nv + c[1]) * nv + c[0])];
    for (int s = 0; s < 3; ++s) {
      c[pm[s]] += 1;
      val = val + lam[s + 1] * nodal[static_cast<size_t>((c[2] * nv + c[1]) * nv + c[0])];
    }
    return val;
  }

  // gradient of the P1 interpolant at x, on the tet the point location of interp() picks:
  // I_h r = r0 (1 - xi_a) + r1 (xi_a - xi_b) + r2 (xi_b - xi_c) + r3 xi_c with xi = n x - cell
  // and (a, b, c) the chain, so d/dx_a = n (r1 - r0), d/dx_b = n (r2 - r1), d/dx_c = n (r3 - r2)
  void interp_grad(const V3& x, double* g) const {
    const int nv = n + 1;
    int cell[3];
    double xi[3];
    for (int d = 0; d < 3; ++d) {
      const double s = x.c[d] * static_cast<double>(n);
      int ci = static_cast<int>(std::floor(s));
      ci = std::min(std::max(ci, 0), n - 1);
      cell[d] = ci;
      xi[d] = s - static_cast<double>(ci);
    }
    constexpr int perms[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
    int p = 0;
    for (; p < 5; ++p)
      if (xi[perms[p][0]] >= xi[perms[p][1]] && xi[perms[p][1]] >= xi[perms[p][2]]) break;
    const int* pm = perms[p];
    int c[3] = {cell[0], cell[1], cell[2]};
    double r[4];
    r[0] = nodal[static_cast<size_t>((c[2] * nv + c[1]) * nv + c[0])];
    for (int s = 0; s < 3; ++s) {
      c[pm[s]] += 1;
      r[s + 1] = nodal[static_cast<size_t>((c[2] * nv + c[1]) * nv + c[0])];
    }
    const double dn = static_cast<double>(n);
    for (int s = 0; s < 3; ++s) g[pm[s]] = dn * (r[s + 1] - r[s]);
  }

  // the exact gradient of the target field (h1_semi_error's exact_grad for the error gate
  // ||grad(u_h - u_bar)||): sin3 as manufactured_exact(0).grad_u (target.cpp:45-58), the
  // random part piecewise constant (interp_grad), indicators zero almost everywhere
  void grad(const V3& x, double* g) const {
    g[0] = g[1] = g[2] = 0.0;
    switch (kind) {
      case OR_TARGET_SMOOTH:
      case OR_TARGET_NONZERO_BC:
      case OR_TARGET_SINE_RANDOM: {
        const double sx = std::sin(kPi * x.c[0]), cx = std::cos(kPi * x.c[0]);
        const double sy = std::sin(kPi * x.c[1]), cy = std::cos(kPi * x.c[1]);
        const double sz = std::sin(kPi * x.c[2]), cz = std::cos(kPi * x.c[2]);
        const double cp = 1.0 * kPi;
        g[0] = cp * cx * sy * sz;
        g[1] = cp * sx * cy * sz;
        g[2] = cp * sx * sy * cz;
        if (kind == OR_TARGET_SINE_RANDOM) {
          double gr[3];
          interp_grad(x, gr);
          for (int d = 0; d < 3; ++d) g[d] = g[d] + 0.1 * gr[d];
        }
        return;
      }
      case OR_TARGET_QUADRATIC:  // x y + 2 z
        g[0] = x.c[1];
        g[1] = x.c[0];
        g[2] = 2.0;
        return;
      default: return;  // box, ball, zero, one
    }
  }

  double operator()(const V3& x) const {
    switch (kind) {
      case OR_TARGET_SMOOTH: return sin3(x);  // target.cpp:17-23
      case OR_TARGET_BOX: {                  // target.cpp:25-35 (open box)
        const bool inside = x.c[0] > 0.25 && x.c[0] < 0.75 && x.c[1] > 0.25 && x.c[1] < 0.75 &&
                            x.c[2] > 0.25 && x.c[2] < 0.75;
        return inside ? 1.0 : 0.0;
      }
      case OR_TARGET_NONZERO_BC: return 1.0 + sin3(x);  // target.cpp:37-43
      case OR_TARGET_BALL: {  // open ball r=0.25 at (1/2,1/2,1/2), squared-distance test
        const double dx = x.c[0] - 0.5, dy = x.c[1] - 0.5, dz = x.c[2] - 0.5;
        return (dx * dx + dy * dy) + dz * dz < 0.0625 ? 1.0 : 0.0;
      }
      case OR_TARGET_SINE_RANDOM: return sin3(x) + 0.1 * interp(x);
      case OR_TARGET_ZERO: return 0.0;                                // test_assembly.cpp:102-106
      case OR_TARGET_ONE: return 1.0;                                 // test_assembly.cpp:108-124
      case OR_TARGET_QUADRATIC: return x.c[0] * x.c[1] + 2.0 * x.c[2];  // test_assembly.cpp:37
    }
    throw std::invalid_argument("unknown target");
  }
};

Target make_target(int kind, int n, uint64_t seed) {
  Target t;
  t.kind = kind;
  switch (kind) {
    case OR_TARGET_SMOOTH: t.tag = smooth_h2; break;
    case OR_TARGET_BOX: t.tag = discontinuous; break;
    case OR_TARGET_NONZERO_BC: t.tag = smooth_nonzero_bc; break;
    case OR_TARGET_BALL: t.tag = discontinuous; break;
    case OR_TARGET_SINE_RANDOM: {
      if (n < 1) throw std::invalid_argument("sine+random target needs n >= 1");
      t.tag = smooth_h2;
      t.n = n;
      const int nv = n + 1;
      const int total = nv * nv * nv;
      t.nodal.resize(static_cast<size_t>(total));
      pseudo_random(total, seed, t.nodal.data());
      for (int k = 0; k < nv; ++k)
        for (int j = 0; j < nv; ++j)
          for (int i = 0; i < nv; ++i)
            if (i == 0 || j == 0 || k == 0 || i == n || j == n || k == n)
              t.nodal[static_cast<size_t>((k * nv + j) * nv + i)] = 0.0;
      break;
    }
    case OR_TARGET_ZERO:
    case OR_TARGET_ONE:
    case OR_TARGET_QUADRATIC: t.tag = smooth_h2; break;
    default: throw std::invalid_argument("unknown target kind");
  }
  return t;
}

// ---------------------------------------------------------------------------
// assembly.cpp
struct VertexTets {
  std::vector<int> offset, tet;
};

VertexTets build_vertex_tets(const Mesh& m) {  // assembly.cpp:14-31 (counting sort, ascending tets)
  VertexTets a;
  a.offset.assign(static_cast<size_t>(m.nv()) + 1, 0);
  for (const auto& t : m.tets)
    for (int v : t) ++a.offset[static_cast<size_t>(v) + 1];
  for (size_t v = 1; v < a.offset.size(); ++v) a.offset[v] += a.offset[v - 1];
  a.tet.resize(static_cast<size_t>(4) * m.nt());
  std::vector<int> cur(a.offset.begin(), a.offset.end() - 1);
  for (int t = 0; t < m.nt(); ++t)
    for (int v : m.tets[static_cast<size_t>(t)]) a.tet[static_cast<size_t>(cur[static_cast<size_t>(v)]++)] = t;
  return a;
}

struct LocalGeom {
  double volume;
  double grad[4][3];
};

// assembly.cpp:33-51 with Eigen's 3x3 determinant (bruteforce_det3_helper) and
// cofactor inverse (compute_inverse_size3_helper) -- exact for n = 2^k lattices.
LocalGeom local_geom(const std::array<V3, 4>& v) {
  double J[3][3];
  for (int r = 0; r < 3; ++r) {
    J[r][0] = v[1].c[r] - v[0].c[r];
    J[r][1] = v[2].c[r] - v[0].c[r];
    J[r][2] = v[3].c[r] - v[0].c[r];
  }
  auto det3 = [&](int a, int b, int c) { return J[0][a] * (J[1][b] * J[2][c] - J[1][c] * J[2][b]); };
  const double det = det3(0, 1, 2) - det3(1, 0, 2) + det3(2, 0, 1);
  LocalGeom g;
  g.volume = std::abs(det) / 6.0;
  if (!(g.volume > 0.0)) throw std::runtime_error("assembly: degenerate tet");
  auto cof = [&](int i, int j) {
    const int i1 = (i + 1) % 3, i2 = (i + 2) % 3, j1 = (j + 1) % 3, j2 = (j + 2) % 3;
    return J[i1][j1] * J[i2][j2] - J[i1][j2] * J[i2][j1];
  };
  const double c0[3] = {cof(0, 0), cof(1, 0), cof(2, 0)};
  const double d2 = (c0[0] * J[0][0] + c0[1] * J[1][0]) + c0[2] * J[2][0];
  const double invdet = 1.0 / d2;
  double inv[3][3];
  inv[0][0] = c0[0] * invdet;
  inv[0][1] = c0[1] * invdet;
  inv[0][2] = c0[2] * invdet;
  inv[1][0] = cof(0, 1) * invdet;
  inv[1][1] = cof(1, 1) * invdet;
  inv[1][2] = cof(2, 1) * invdet;
  inv[2][0] = cof(0, 2) * invdet;
  inv[2][1] = cof(1, 2) * invdet;
  inv[2][2] = cof(2, 2) * invdet;
  for (int i = 0; i < 3; ++i)
    for (int c = 0; c < 3; ++c) g.grad[i + 1][c] = inv[i][c];
  for (int c = 0; c < 3; ++c) g.grad[0][c] = -((g.grad[1][c] + g.grad[2][c]) + g.grad[3][c]);
  return g;
}

double dot3(const double* a, const double* b) { return (a[0] * b[0] + a[1] * b[1]) + a[2] * b[2]; }

// assembly.cpp:53-132: row-gather assembly of cK*K + cM*M; columns = sorted unique
// dofs of incident-tet vertices; per slot accumulate over incident tets ascending,
// jv = 0..3; then prune exact zeros.
Csr assemble_matrix(const Mesh& m, const std::vector<int>& row_of_vert,
                    const std::vector<int>& vert_of_row, double cK, double cM,
                    const std::vector<uint8_t>* tet_mask = nullptr) {
  const VertexTets adj = build_vertex_tets(m);
  const int n = static_cast<int>(vert_of_row.size());
  std::vector<std::vector<int>> cols(static_cast<size_t>(n));
  parallel_for(n, [&](int64_t rb, int64_t re) {
    std::vector<int> cand;
    for (int64_t r = rb; r < re; ++r) {
      const int v = vert_of_row[static_cast<size_t>(r)];
      cand.clear();
      for (int k = adj.offset[static_cast<size_t>(v)]; k < adj.offset[static_cast<size_t>(v) + 1]; ++k) {
        const int t = adj.tet[static_cast<size_t>(k)];
        if (tet_mask && !(*tet_mask)[static_cast<size_t>(t)]) continue;
        for (int w : m.tets[static_cast<size_t>(t)]) {
          const int c = row_of_vert[static_cast<size_t>(w)];
          if (c >= 0) cand.push_back(c);
        }
      }
      std::sort(cand.begin(), cand.end());
      cand.erase(std::unique(cand.begin(), cand.end()), cand.end());
      cols[static_cast<size_t>(r)] = cand;
    }
  });
  std::vector<int> rp(static_cast<size_t>(n) + 1, 0);
  for (int r = 0; r < n; ++r)
    rp[static_cast<size_t>(r) + 1] = rp[static_cast<size_t>(r)] + static_cast<int>(cols[static_cast<size_t>(r)].size());
  std::vector<double> vals(static_cast<size_t>(rp[static_cast<size_t>(n)]), 0.0);
  parallel_for(n, [&](int64_t rb, int64_t re) {
    for (int64_t r = rb; r < re; ++r) {
      const auto& rc = cols[static_cast<size_t>(r)];
      double* va = vals.data() + rp[static_cast<size_t>(r)];
      const int v = vert_of_row[static_cast<size_t>(r)];
      for (int k = adj.offset[static_cast<size_t>(v)]; k < adj.offset[static_cast<size_t>(v) + 1]; ++k) {
        const int t = adj.tet[static_cast<size_t>(k)];
        if (tet_mask && !(*tet_mask)[static_cast<size_t>(t)]) continue;
        const auto& tet = m.tets[static_cast<size_t>(t)];
        const LocalGeom g = local_geom(tet_vertices(m, t));
        int iv = 0;
        while (tet[static_cast<size_t>(iv)] != v) ++iv;
        for (int jv = 0; jv < 4; ++jv) {
          const int c = row_of_vert[static_cast<size_t>(tet[static_cast<size_t>(jv)])];
          if (c < 0) continue;
          double val = 0.0;
          if (cK != 0.0) val += cK * g.volume * dot3(g.grad[iv], g.grad[jv]);
          if (cM != 0.0) val += cM * g.volume * (iv == jv ? 0.1 : 0.05);
          const auto pos = std::lower_bound(rc.begin(), rc.end(), c) - rc.begin();
          va[pos] += val;
        }
      }
    }
  });
  // prune (v != 0.0) and compress (assembly.cpp:129-130)
  Csr A;
  A.rows = n;
  A.cols = n;
  A.rp.assign(static_cast<size_t>(n) + 1, 0);
  for (int r = 0; r < n; ++r) {
    const auto& rc = cols[static_cast<size_t>(r)];
    for (size_t q = 0; q < rc.size(); ++q) {
      const double x = vals[static_cast<size_t>(rp[static_cast<size_t>(r)]) + q];
      if (x != 0.0) {
        A.ci.push_back(rc[q]);
        A.v.push_back(x);
      }
    }
    A.rp[static_cast<size_t>(r) + 1] = static_cast<int>(A.ci.size());
  }
  return A;
}

struct DofMap {
  std::vector<int> vertex_to_dof, dof_to_vertex;
  int n_dofs() const { return static_cast<int>(dof_to_vertex.size()); }
};

DofMap interior_dof_map(const Mesh& m) {  // assembly.cpp:187-197
  DofMap d;
  d.vertex_to_dof.assign(static_cast<size_t>(m.nv()), -1);
  for (int v = 0; v < m.nv(); ++v)
    if (!m.boundary[static_cast<size_t>(v)]) {
      d.vertex_to_dof[static_cast<size_t>(v)] = d.n_dofs();
      d.dof_to_vertex.push_back(v);
    }
  return d;
}

const Rule& rule_for(const Target& t) {  // assembly.cpp:140-144
  return t.tag == discontinuous ? rule_by_id(3) : rule_by_id(2);
}

// assembly.cpp:146-174: f_r = sum_{t ascending} vol_t * sum_q (w_q u(x_q)) lambda_q,iv
Vec load_vector(const Mesh& m, const DofMap& dm, const Target& target) {
  const VertexTets adj = build_vertex_tets(m);
  const Rule& rule = rule_for(target);
  Vec f(static_cast<size_t>(dm.n_dofs()));
  parallel_for(dm.n_dofs(), [&](int64_t rb, int64_t re) {
    for (int64_t r = rb; r < re; ++r) {
      const int v = dm.dof_to_vertex[static_cast<size_t>(r)];
      double s = 0.0;
      for (int k = adj.offset[static_cast<size_t>(v)]; k < adj.offset[static_cast<size_t>(v) + 1]; ++k) {
        const int t = adj.tet[static_cast<size_t>(k)];
        const auto& tet = m.tets[static_cast<size_t>(t)];
        int iv = 0;
        while (tet[static_cast<size_t>(iv)] != v) ++iv;
        const auto verts = tet_vertices(m, t);
        const double vol = tet_volume(m, t);
        double acc = 0.0;
        for (int q = 0; q < rule.size(); ++q) {
          const V3 x = physical_point(rule.pts[static_cast<size_t>(q)], verts);
          acc += rule.w[static_cast<size_t>(q)] * target(x) * rule.pts[static_cast<size_t>(q)][static_cast<size_t>(iv)];
        }
        s += vol * acc;
      }
      f[static_cast<size_t>(r)] = s;
    }
  });
  return f;
}

struct System {
  double rho = 1.0;
  Csr K, M, A;
  Vec f;
  DofMap dm;
};

// Eigen sparse union add (CwiseBinaryOp<scalar_sum_op>): both -> l + r, one side -> x + 0 / 0 + x.
Csr scaled_sum(double rho, const Csr& K, const Csr& M) {
  Csr A;
  A.rows = K.rows;
  A.cols = K.cols;
  A.rp.assign(static_cast<size_t>(K.rows) + 1, 0);
  for (int r = 0; r < K.rows; ++r) {
    int a = K.rp[static_cast<size_t>(r)], ae = K.rp[static_cast<size_t>(r) + 1];
    int b = M.rp[static_cast<size_t>(r)], be = M.rp[static_cast<size_t>(r) + 1];
    while (a < ae || b < be) {
      if (a < ae && b < be && K.ci[static_cast<size_t>(a)] == M.ci[static_cast<size_t>(b)]) {
        A.ci.push_back(K.ci[static_cast<size_t>(a)]);
        A.v.push_back(rho * K.v[static_cast<size_t>(a)] + M.v[static_cast<size_t>(b)]);
        ++a;
        ++b;
      } else if (a < ae && (b >= be || K.ci[static_cast<size_t>(a)] < M.ci[static_cast<size_t>(b)])) {
        A.ci.push_back(K.ci[static_cast<size_t>(a)]);
        A.v.push_back(rho * K.v[static_cast<size_t>(a)] + 0.0);
        ++a;
      } else {
        A.ci.push_back(M.ci[static_cast<size_t>(b)]);
        A.v.push_back(0.0 + M.v[static_cast<size_t>(b)]);
        ++b;
      }
    }
    A.rp[static_cast<size_t>(r) + 1] = static_cast<int>(A.ci.size());
  }
  return A;
}

System build_system(const Mesh& m, double rho, const Target& target) {  // assembly.cpp:225-238
  if (!(rho > 0.0)) throw std::invalid_argument("build_system: rho must be > 0");
  System s;
  s.rho = rho;
  s.dm = interior_dof_map(m);
  s.K = assemble_matrix(m, s.dm.vertex_to_dof, s.dm.dof_to_vertex, 1.0, 0.0);
  s.M = assemble_matrix(m, s.dm.vertex_to_dof, s.dm.dof_to_vertex, 0.0, 1.0);
  s.A = scaled_sum(rho, s.K, s.M);
  s.f = load_vector(m, s.dm, target);
  return s;
}

// ---------------------------------------------------------------------------
// linalg.cpp
Csr from_triplets(int rows, int cols, const std::vector<int>& ti, const std::vector<int>& tj,
                  const std::vector<double>& tv) {  // linalg.cpp:11-17 (setFromTriplets: dups summed in insertion order; prune)
  const size_t n = ti.size();
  std::vector<size_t> order(n);
  for (size_t k = 0; k < n; ++k) order[k] = k;
  for (size_t k = 0; k < n; ++k)
    if (ti[k] < 0 || ti[k] >= rows || tj[k] < 0 || tj[k] >= cols)
      throw std::invalid_argument("from_triplets: index out of range");
  std::stable_sort(order.begin(), order.end(), [&](size_t a, size_t b) {
    return ti[a] != ti[b] ? ti[a] < ti[b] : tj[a] < tj[b];
  });
  Csr A;
  A.rows = rows;
  A.cols = cols;
  A.rp.assign(static_cast<size_t>(rows) + 1, 0);
  size_t k = 0;
  for (int r = 0; r < rows; ++r) {
    while (k < n && ti[order[k]] == r) {
      const int c = tj[order[k]];
      double s = tv[order[k]];
      ++k;
      while (k < n && ti[order[k]] == r && tj[order[k]] == c) s += tv[order[k++]];
      if (s != 0.0) {
        A.ci.push_back(c);
        A.v.push_back(s);
      }
    }
    A.rp[static_cast<size_t>(r) + 1] = static_cast<int>(A.ci.size());
  }
  return A;
}

// linalg.cpp:19-33: y_i = ((0 + v0 x0) + v1 x1) + ... in column order
Vec spmv(const Csr& A, const Vec& x) {
  if (A.cols != static_cast<int>(x.size())) throw std::invalid_argument("spmv: dimension mismatch");
  Vec y(static_cast<size_t>(A.rows));
  parallel_for(A.rows, [&](int64_t b, int64_t e) {
    for (int64_t i = b; i < e; ++i) {
      double s = 0.0;
      for (int k = A.rp[static_cast<size_t>(i)]; k < A.rp[static_cast<size_t>(i) + 1]; ++k)
        s += A.v[static_cast<size_t>(k)] * x[static_cast<size_t>(A.ci[static_cast<size_t>(k)])];
      y[static_cast<size_t>(i)] = s;
    }
  });
  return y;
}

// Eigen 3.4 VectorXd::dot with SSE2 (packet of 2, two packet accumulators,
// Redux.h LinearVectorizedTraversal) -- restated, unverifiable here (no Eigen).
double eigen_dot(const double* a, const double* b, int64_t n) {
  if (n <= 0) return 0.0;
  const int64_t aligned2 = (n / 4) * 4, aligned = (n / 2) * 2;
  double res;
  if (aligned) {
    double p0a = a[0] * b[0], p0b = a[1] * b[1];
    if (aligned > 2) {
      double p1a = a[2] * b[2], p1b = a[3] * b[3];
      for (int64_t i = 4; i < aligned2; i += 4) {
        p0a = p0a + a[i] * b[i];
        p0b = p0b + a[i + 1] * b[i + 1];
        p1a = p1a + a[i + 2] * b[i + 2];
        p1b = p1b + a[i + 3] * b[i + 3];
      }
      p0a = p0a + p1a;
      p0b = p0b + p1b;
      if (aligned > aligned2) {
        p0a = p0a + a[aligned2] * b[aligned2];
        p0b = p0b + a[aligned2 + 1] * b[aligned2 + 1];
      }
    }
    res = p0a + p0b;
    for (int64_t i = aligned; i < n; ++i) res = res + a[i] * b[i];
  } else {
    res = a[0] * b[0];
  }
  return res;
}

double dot(const Vec& a, const Vec& b) { return eigen_dot(a.data(), b.data(), static_cast<int64_t>(a.size())); }

// Dense Cholesky (Eigen LLT<MatrixXd>, linalg.cpp:46-51, amg.cpp:111-115).  Eigen's
// blocked kernel order is unverifiable here; this is the left-looking order the
// device's one-CTA factorization uses (so oracle and device agree bit-for-bit).
struct Llt {
  int n = 0;
  std::vector<double> L;  // row-major lower factor
  bool ok = true;
};

Llt llt_compute(int n, const std::vector<double>& A) {
  Llt f;
  f.n = n;
  f.L.assign(static_cast<size_t>(n) * n, 0.0);
  for (int j = 0; j < n; ++j) {
    double s = A[static_cast<size_t>(j) * n + j];
    for (int k = 0; k < j; ++k) s -= f.L[static_cast<size_t>(j) * n + k] * f.L[static_cast<size_t>(j) * n + k];
    if (!(s > 0.0)) {
      f.ok = false;
      return f;
    }
    const double d = std::sqrt(s);
    f.L[static_cast<size_t>(j) * n + j] = d;
    for (int i = j + 1; i < n; ++i) {
      double t = A[static_cast<size_t>(i) * n + j];
      for (int k = 0; k < j; ++k) t -= f.L[static_cast<size_t>(i) * n + k] * f.L[static_cast<size_t>(j) * n + k];
      f.L[static_cast<size_t>(i) * n + j] = t / d;
    }
  }
  return f;
}

Vec llt_solve(const Llt& f, const Vec& b) {
  const int n = f.n;
  Vec y(static_cast<size_t>(n)), x(static_cast<size_t>(n));
  for (int i = 0; i < n; ++i) {
    double s = b[static_cast<size_t>(i)];
    for (int k = 0; k < i; ++k) s -= f.L[static_cast<size_t>(i) * n + k] * y[static_cast<size_t>(k)];
    y[static_cast<size_t>(i)] = s / f.L[static_cast<size_t>(i) * n + i];
  }
  for (int i = n - 1; i >= 0; --i) {  // back substitution, sums in descending k
    double s = y[static_cast<size_t>(i)];
    for (int k = n - 1; k > i; --k) s -= f.L[static_cast<size_t>(k) * n + i] * x[static_cast<size_t>(k)];
    x[static_cast<size_t>(i)] = s / f.L[static_cast<size_t>(i) * n + i];
  }
  return x;
}

std::vector<double> to_dense(const Csr& A) {
  std::vector<double> D(static_cast<size_t>(A.rows) * A.cols, 0.0);
  for (int r = 0; r < A.rows; ++r)
    for (int k = A.rp[static_cast<size_t>(r)]; k < A.rp[static_cast<size_t>(r) + 1]; ++k)
      D[static_cast<size_t>(r) * A.cols + A.ci[static_cast<size_t>(k)]] = A.v[static_cast<size_t>(k)];
  return D;
}

// ---------------------------------------------------------------------------
// amg.cpp
std::pair<std::vector<uint8_t>, Csr> coarsen_redblack(const Csr& A) {  // amg.cpp:7-56
  const int n = A.rows;
  enum : uint8_t { unmarked = 0, coarse = 1, fine = 2 };
  std::vector<uint8_t> state(static_cast<size_t>(n), unmarked);
  for (int i = 0; i < n; ++i) {
    if (state[static_cast<size_t>(i)] != unmarked) continue;
    state[static_cast<size_t>(i)] = coarse;
    for (int k = A.rp[static_cast<size_t>(i)]; k < A.rp[static_cast<size_t>(i) + 1]; ++k) {
      const int j = A.ci[static_cast<size_t>(k)];
      if (j != i && state[static_cast<size_t>(j)] == unmarked) state[static_cast<size_t>(j)] = fine;
    }
  }
  for (int i = 0; i < n; ++i) {  // guard :22-29
    if (state[static_cast<size_t>(i)] != fine) continue;
    bool has_coarse = false;
    for (int k = A.rp[static_cast<size_t>(i)]; k < A.rp[static_cast<size_t>(i) + 1] && !has_coarse; ++k)
      has_coarse = A.ci[static_cast<size_t>(k)] != i && state[static_cast<size_t>(A.ci[static_cast<size_t>(k)])] == coarse;
    if (!has_coarse) state[static_cast<size_t>(i)] = coarse;
  }
  std::vector<int> cidx(static_cast<size_t>(n), -1);
  int nc = 0;
  for (int i = 0; i < n; ++i)
    if (state[static_cast<size_t>(i)] == coarse) cidx[static_cast<size_t>(i)] = nc++;
  std::vector<int> ti, tj;
  std::vector<double> tv;
  for (int i = 0; i < n; ++i) {
    if (state[static_cast<size_t>(i)] == coarse) {
      ti.push_back(i);
      tj.push_back(cidx[static_cast<size_t>(i)]);
      tv.push_back(1.0);
      continue;
    }
    int count = 0;
    for (int k = A.rp[static_cast<size_t>(i)]; k < A.rp[static_cast<size_t>(i) + 1]; ++k)
      if (A.ci[static_cast<size_t>(k)] != i && state[static_cast<size_t>(A.ci[static_cast<size_t>(k)])] == coarse) ++count;
    const double w = 1.0 / count;
    for (int k = A.rp[static_cast<size_t>(i)]; k < A.rp[static_cast<size_t>(i) + 1]; ++k)
      if (A.ci[static_cast<size_t>(k)] != i && state[static_cast<size_t>(A.ci[static_cast<size_t>(k)])] == coarse) {
        ti.push_back(i);
        tj.push_back(cidx[static_cast<size_t>(A.ci[static_cast<size_t>(k)])]);
        tv.push_back(w);
      }
  }
  Csr P = from_triplets(n, nc, ti, tj, tv);
  std::vector<uint8_t> flags(static_cast<size_t>(n));
  for (int i = 0; i < n; ++i) flags[static_cast<size_t>(i)] = state[static_cast<size_t>(i)] == coarse ? 1 : 0;
  return {std::move(flags), std::move(P)};
}

Csr transpose(const Csr& A) {  // SpMat(P.transpose()): rows of the result ascending in column
  Csr T;
  T.rows = A.cols;
  T.cols = A.rows;
  T.rp.assign(static_cast<size_t>(A.cols) + 1, 0);
  for (int c : A.ci) ++T.rp[static_cast<size_t>(c) + 1];
  for (size_t c = 1; c < T.rp.size(); ++c) T.rp[c] += T.rp[c - 1];
  T.ci.resize(A.ci.size());
  T.v.resize(A.v.size());
  std::vector<int> cur(T.rp.begin(), T.rp.end() - 1);
  for (int r = 0; r < A.rows; ++r)
    for (int k = A.rp[static_cast<size_t>(r)]; k < A.rp[static_cast<size_t>(r) + 1]; ++k) {
      const int c = A.ci[static_cast<size_t>(k)];
      const int pos = cur[static_cast<size_t>(c)]++;
      T.ci[static_cast<size_t>(pos)] = r;
      T.v[static_cast<size_t>(pos)] = A.v[static_cast<size_t>(k)];
    }
  return T;
}

// Eigen conservative_sparse_sparse_product for RowMajor x RowMajor: output row j
// accumulates, in order over A's row j entries (k, a_jk) and then B's row k
// entries (i, b_ki), values[i] = b_ki * a_jk on first touch, += afterwards;
// columns sorted; no pruning.
Csr spgemm(const Csr& A, const Csr& B) {
  Csr C;
  C.rows = A.rows;
  C.cols = B.cols;
  C.rp.assign(static_cast<size_t>(A.rows) + 1, 0);
  std::vector<double> values(static_cast<size_t>(B.cols), 0.0);
  std::vector<char> mask(static_cast<size_t>(B.cols), 0);
  std::vector<int> idx;
  for (int j = 0; j < A.rows; ++j) {
    idx.clear();
    for (int ka = A.rp[static_cast<size_t>(j)]; ka < A.rp[static_cast<size_t>(j) + 1]; ++ka) {
      const double y = A.v[static_cast<size_t>(ka)];
      const int k = A.ci[static_cast<size_t>(ka)];
      for (int kb = B.rp[static_cast<size_t>(k)]; kb < B.rp[static_cast<size_t>(k) + 1]; ++kb) {
        const int i = B.ci[static_cast<size_t>(kb)];
        const double x = B.v[static_cast<size_t>(kb)];
        if (!mask[static_cast<size_t>(i)]) {
          mask[static_cast<size_t>(i)] = 1;
          values[static_cast<size_t>(i)] = x * y;
          idx.push_back(i);
        } else {
          values[static_cast<size_t>(i)] += x * y;
        }
      }
    }
    std::sort(idx.begin(), idx.end());
    for (int i : idx) {
      C.ci.push_back(i);
      C.v.push_back(values[static_cast<size_t>(i)]);
      mask[static_cast<size_t>(i)] = 0;
    }
    C.rp[static_cast<size_t>(j) + 1] = static_cast<int>(C.ci.size());
  }
  return C;
}

Csr prune(const Csr& A) {
  Csr B;
  B.rows = A.rows;
  B.cols = A.cols;
  B.rp.assign(static_cast<size_t>(A.rows) + 1, 0);
  for (int r = 0; r < A.rows; ++r) {
    for (int k = A.rp[static_cast<size_t>(r)]; k < A.rp[static_cast<size_t>(r) + 1]; ++k)
      if (A.v[static_cast<size_t>(k)] != 0.0) {
        B.ci.push_back(A.ci[static_cast<size_t>(k)]);
        B.v.push_back(A.v[static_cast<size_t>(k)]);
      }
    B.rp[static_cast<size_t>(r) + 1] = static_cast<int>(B.ci.size());
  }
  return B;
}

Csr galerkin_coarse(const Csr& A, const Csr& P) {  // amg.cpp:58-65
  if (A.cols != P.rows) throw std::invalid_argument("galerkin_coarse: dims");
  const Csr AP = spgemm(A, P);
  const Csr Pt = transpose(P);
  return prune(spgemm(Pt, AP));
}

// amg.cpp:67-88: forward i = 0..n-1 then backward; s = f_i; s -= v x_col (col != i); x_i = s/d
Vec sgs_sweep(const Csr& A, const Vec& f, const Vec& u) {
  const int n = A.rows;
  Vec x = u;
  auto relax = [&](int i) {
    double s = f[static_cast<size_t>(i)];
    double d = 0.0;
    for (int k = A.rp[static_cast<size_t>(i)]; k < A.rp[static_cast<size_t>(i) + 1]; ++k) {
      if (A.ci[static_cast<size_t>(k)] == i)
        d = A.v[static_cast<size_t>(k)];
      else
        s -= A.v[static_cast<size_t>(k)] * x[static_cast<size_t>(A.ci[static_cast<size_t>(k)])];
    }
    if (d == 0.0) throw std::runtime_error("sgs_sweep: zero diagonal");
    x[static_cast<size_t>(i)] = s / d;
  };
  for (int i = 0; i < n; ++i) relax(i);
  for (int i = n - 1; i >= 0; --i) relax(i);
  return x;
}

struct Level {
  Csr A, P, Pt;
  std::vector<uint8_t> flags;
  bool has_p = false;
};

struct Amg {
  std::vector<Level> levels;
  Llt coarsest;
  int smoothing_steps = 1;
};

Amg build_amg(const Csr& A, int threshold, int m) {  // amg.cpp:90-117
  Amg h;
  h.smoothing_steps = m;
  Csr current = A;
  while (current.rows > threshold) {
    Level lv;
    lv.A = current;
    auto fp = coarsen_redblack(lv.A);
    if (fp.second.cols >= fp.second.rows) break;
    lv.flags = std::move(fp.first);
    lv.P = std::move(fp.second);
    lv.Pt = transpose(lv.P);
    lv.has_p = true;
    current = galerkin_coarse(lv.A, lv.P);
    h.levels.push_back(std::move(lv));
  }
  Level last;
  last.A = current;
  h.levels.push_back(std::move(last));
  if (current.rows > 0) {
    h.coarsest = llt_compute(current.rows, to_dense(current));
    if (!h.coarsest.ok) throw std::runtime_error("build_amg: coarsest level not positive definite");
  }
  return h;
}

Vec vcycle(const Amg& h, size_t level, const Vec& r) {  // amg.cpp:119-132
  const Level& lv = h.levels[level];
  if (level + 1 == h.levels.size()) return llt_solve(h.coarsest, r);
  Vec z(r.size(), 0.0);
  for (int s = 0; s < h.smoothing_steps; ++s) z = sgs_sweep(lv.A, r, z);
  const Vec Az = spmv(lv.A, z);
  Vec res(r.size());
  for (size_t i = 0; i < r.size(); ++i) res[i] = r[i] - Az[i];
  const Vec rc = spmv(lv.Pt, res);
  const Vec zc = vcycle(h, level + 1, rc);
  const Vec Pz = spmv(lv.P, zc);
  for (size_t i = 0; i < z.size(); ++i) z[i] = z[i] + Pz[i];
  for (int s = 0; s < h.smoothing_steps; ++s) z = sgs_sweep(lv.A, r, z);
  return z;
}

Vec amg_apply(const Amg& h, const Vec& r) {  // amg.cpp:136-141
  if (h.levels.empty() || static_cast<int>(r.size()) != h.levels.front().A.rows)
    throw std::invalid_argument("amg_apply: dimension mismatch");
  if (r.empty()) return r;
  return vcycle(h, 0, r);
}

struct PcgOut {
  Vec x;
  int iterations = 0;
  bool converged = false;
  std::vector<double> history;
};

// linalg.cpp:64-102
PcgOut pcg(const std::function<Vec(const Vec&)>& apply_A, const std::function<Vec(const Vec&)>& apply_P,
           const Vec& f, double tol, int max_iter) {
  PcgOut out;
  const size_t n = f.size();
  out.x.assign(n, 0.0);
  Vec r = f;
  Vec z = apply_P(r);
  double rz = dot(r, z);
  if (rz < 0.0) throw std::runtime_error("pcg: preconditioner not positive definite");
  const double rz0 = rz;
  if (rz0 == 0.0) {
    out.converged = true;
    return out;
  }
  Vec p = z;
  for (int it = 1; it <= max_iter; ++it) {
    const Vec Ap = apply_A(p);
    const double pAp = dot(p, Ap);
    if (pAp <= 0.0) throw std::runtime_error("pcg: operator not positive definite (p'Ap <= 0)");
    const double alpha = rz / pAp;
    for (size_t i = 0; i < n; ++i) out.x[i] = out.x[i] + alpha * p[i];
    for (size_t i = 0; i < n; ++i) r[i] = r[i] - alpha * Ap[i];
    z = apply_P(r);
    const double rz_next = dot(r, z);
    if (rz_next < 0.0) throw std::runtime_error("pcg: preconditioner not positive definite");
    const double rel = std::sqrt(rz_next / rz0);
    out.iterations = it;
    out.history.push_back(rel);
    if (rel <= tol) {
      out.converged = true;
      return out;
    }
    const double beta = rz_next / rz;
    rz = rz_next;
    for (size_t i = 0; i < n; ++i) p[i] = z[i] + beta * p[i];
  }
  return out;
}

std::vector<double> nodal_field(const Mesh& m, const DofMap& dm, const double* c) {  // assembly.cpp:358-363
  std::vector<double> nodal(static_cast<size_t>(m.nv()), 0.0);
  for (int d = 0; d < dm.n_dofs(); ++d) nodal[static_cast<size_t>(dm.dof_to_vertex[static_cast<size_t>(d)])] = c[d];
  return nodal;
}

struct Exact {  // target.cpp:45-58
  double c;
  double u(const V3& x) const { return c * sin3(x); }
  void grad(const V3& x, double* g) const {
    const double sx = std::sin(kPi * x.c[0]), cx = std::cos(kPi * x.c[0]);
    const double sy = std::sin(kPi * x.c[1]), cy = std::cos(kPi * x.c[1]);
    const double sz = std::sin(kPi * x.c[2]), cz = std::cos(kPi * x.c[2]);
    g[0] = c * kPi * cx * sy * sz;
    g[1] = c * kPi * sx * cy * sz;
    g[2] = c * kPi * sx * sy * cz;
  }
};

Exact manufactured_exact(double rho) {
  if (rho < 0.0) throw std::invalid_argument("manufactured_exact: rho must be >= 0");
  return Exact{1.0 / (3.0 * rho * kPi * kPi + 1.0)};
}

// a target field as the exact function of l2_error / h1_semi_error (std::function callbacks
// in the reference: exact = target.evaluator, exact_grad = its gradient)
struct TargetExact {
  const Target& t;
  double u(const V3& x) const { return t(x); }
  void grad(const V3& x, double* g) const { t.grad(x, g); }
};

// assembly.cpp:265-285
template <class Ex>
double l2_error(const Mesh& m, const DofMap& dm, const double* coeffs, const Ex& ex) {
  const auto nodal = nodal_field(m, dm, coeffs);
  const Rule& rule = rule_by_id(2);
  const double err2 = parallel_reduce(m.nt(), [&](int64_t b, int64_t e) {
    double s = 0.0;
    for (int64_t t = b; t < e; ++t) {
      const auto verts = tet_vertices(m, static_cast<int>(t));
      const auto& tet = m.tets[static_cast<size_t>(t)];
      double acc = 0.0;
      for (int q = 0; q < rule.size(); ++q) {
        const auto& lam = rule.pts[static_cast<size_t>(q)];
        const V3 x = physical_point(lam, verts);
        double u = 0.0;
        for (int i = 0; i < 4; ++i) u += lam[static_cast<size_t>(i)] * nodal[static_cast<size_t>(tet[static_cast<size_t>(i)])];
        const double d = u - ex.u(x);
        acc += rule.w[static_cast<size_t>(q)] * d * d;
      }
      s += tet_volume(m, static_cast<int>(t)) * acc;
    }
    return s;
  });
  return std::sqrt(err2);
}

// assembly.cpp:287-310
template <class Ex>
double h1_semi_error(const Mesh& m, const DofMap& dm, const double* coeffs, const Ex& ex) {
  const auto nodal = nodal_field(m, dm, coeffs);
  const Rule& rule = rule_by_id(2);
  const double err2 = parallel_reduce(m.nt(), [&](int64_t b, int64_t e) {
    double s = 0.0;
    for (int64_t t = b; t < e; ++t) {
      const auto verts = tet_vertices(m, static_cast<int>(t));
      const LocalGeom g = local_geom(verts);
      const auto& tet = m.tets[static_cast<size_t>(t)];
      double gu[3] = {0.0, 0.0, 0.0};
      for (int i = 0; i < 4; ++i)
        for (int c = 0; c < 3; ++c) gu[c] = gu[c] + nodal[static_cast<size_t>(tet[static_cast<size_t>(i)])] * g.grad[i][c];
      double acc = 0.0;
      for (int q = 0; q < rule.size(); ++q) {
        const V3 x = physical_point(rule.pts[static_cast<size_t>(q)], verts);
        double ge[3];
        ex.grad(x, ge);
        const double d0 = gu[0] - ge[0], d1 = gu[1] - ge[1], d2 = gu[2] - ge[2];
        acc += rule.w[static_cast<size_t>(q)] * ((d0 * d0 + d1 * d1) + d2 * d2);
      }
      s += g.volume * acc;
    }
    return s;
  });
  return std::sqrt(err2);
}

// assembly.cpp:312-331: the squared L2 distance to the TARGET field with the target's
// own rule (rule_for, assembly.cpp:140-144), target minus fe_value
double l2_error_target_squared(const Mesh& m, const DofMap& dm, const double* coeffs, const Target& tg) {
  const auto nodal = nodal_field(m, dm, coeffs);
  const Rule& rule = rule_for(tg);
  return parallel_reduce(m.nt(), [&](int64_t b, int64_t e) {
    double s = 0.0;
    for (int64_t t = b; t < e; ++t) {
      const auto verts = tet_vertices(m, static_cast<int>(t));
      const auto& tet = m.tets[static_cast<size_t>(t)];
      double acc = 0.0;
      for (int q = 0; q < rule.size(); ++q) {
        const auto& lam = rule.pts[static_cast<size_t>(q)];
        const V3 x = physical_point(lam, verts);
        double u = 0.0;
        for (int i = 0; i < 4; ++i) u += lam[static_cast<size_t>(i)] * nodal[static_cast<size_t>(tet[static_cast<size_t>(i)])];
        const double d = tg(x) - u;
        acc += rule.w[static_cast<size_t>(q)] * d * d;
      }
      s += tet_volume(m, static_cast<int>(t)) * acc;
    }
    return s;
  });
}

// bench.cpp:55-63 target_dual_norm with target_residual (assembly.cpp:354-356) and
// hminus1_norm[_with] (assembly.cpp:333-352): r = f - M u, w = K^-1 r, sqrt(r . w)
double target_dual_norm(const System& s, const double* coeffs) {
  const int n = s.dm.n_dofs();
  const Vec u(coeffs, coeffs + n);
  const Vec Mu = spmv(s.M, u);
  Vec r(static_cast<size_t>(n));
  for (int i = 0; i < n; ++i) r[static_cast<size_t>(i)] = s.f[static_cast<size_t>(i)] - Mu[static_cast<size_t>(i)];
  Vec w;
  if (n <= 2000) {
    const Llt f = llt_compute(n, to_dense(s.K));
    if (!f.ok) throw std::runtime_error("dense_cholesky_solve: matrix not positive definite");
    w = llt_solve(f, r);
  } else {
    const Amg hk = build_amg(s.K, 64, 1);
    w = pcg([&](const Vec& x) { return spmv(s.K, x); }, [&](const Vec& x) { return amg_apply(hk, x); }, r, 1e-11, 500)
            .x;
  }
  const double rw = dot(r, w);
  if (rw < 0.0) throw std::runtime_error("hminus1_norm: negative dual pairing");
  return std::sqrt(rw);
}

// ---------------------------------------------------------------------------
// adapt.cpp / mesh.cpp:67-156 (§8(f)3: the adaptive loop)

// Eigen VectorXd::sum with SSE2: the same Redux.h LinearVectorizedTraversal as eigen_dot
double eigen_sum(const double* a, int64_t n) {
  if (n <= 0) return 0.0;
  const int64_t aligned2 = (n / 4) * 4, aligned = (n / 2) * 2;
  double res;
  if (aligned) {
    double p0a = a[0], p0b = a[1];
    if (aligned > 2) {
      double p1a = a[2], p1b = a[3];
      for (int64_t i = 4; i < aligned2; i += 4) {
        p0a = p0a + a[i];
        p0b = p0b + a[i + 1];
        p1a = p1a + a[i + 2];
        p1b = p1b + a[i + 3];
      }
      p0a = p0a + p1a;
      p0b = p0b + p1b;
      if (aligned > aligned2) {
        p0a = p0a + a[aligned2];
        p0b = p0b + a[aligned2 + 1];
      }
    }
    res = p0a + p0b;
    for (int64_t i = aligned; i < n; ++i) res = res + a[i];
  } else {
    res = a[0];
  }
  return res;
}

double norm3(const double* d) { return std::sqrt((d[0] * d[0] + d[1] * d[1]) + d[2] * d[2]); }
double dist3(const V3& a, const V3& b) {
  const double d[3] = {a.c[0] - b.c[0], a.c[1] - b.c[1], a.c[2] - b.c[2]};
  return norm3(d);
}

struct Estimate {
  Vec per_tet;
  double global = 0.0;
};

// adapt.cpp:35-124: eta_tau^2 = a_tau^2 vol ||target - u_h||^2_tau (the estimator's own rule:
// subdivision64 for discontinuous targets, degree 5 otherwise) + for every interior face, in
// ascending (sorted vertex key, tet) order, 1/2 rho^-1/2 a_F area [rho grad u_h . n]^2 on both sides
Estimate estimate(const Mesh& m, const DofMap& dm, const double* coeffs, double rho, const Target& tg) {
  const double inv_sqrt_rho = 1.0 / std::sqrt(rho);
  const auto nodal = nodal_field(m, dm, coeffs);
  const int nt = m.nt();
  const Rule& rule = tg.tag == discontinuous ? rule_by_id(3) : rule_by_id(2);
  Vec eta_sq(static_cast<size_t>(nt));
  std::vector<std::array<double, 3>> grad(static_cast<size_t>(nt));
  parallel_for(nt, [&](int64_t b, int64_t e) {
    for (int64_t t = b; t < e; ++t) {
      const auto verts = tet_vertices(m, static_cast<int>(t));
      const auto& tet = m.tets[static_cast<size_t>(t)];
      const LocalGeom lg = local_geom(verts);  // |J.determinant()| / 6 and J.inverse() rows
      double g[3] = {0.0, 0.0, 0.0}, g0[3] = {0.0, 0.0, 0.0};
      for (int i = 0; i < 3; ++i) {
        const double s = nodal[static_cast<size_t>(tet[static_cast<size_t>(i + 1)])];
        for (int c = 0; c < 3; ++c) {
          g[c] = g[c] + s * lg.grad[i + 1][c];
          g0[c] = g0[c] - lg.grad[i + 1][c];
        }
      }
      const double s0 = nodal[static_cast<size_t>(tet[0])];
      for (int c = 0; c < 3; ++c) g[c] = g[c] + s0 * g0[c];
      grad[static_cast<size_t>(t)] = {g[0], g[1], g[2]};
      double acc = 0.0;
      for (int q = 0; q < rule.size(); ++q) {
        const auto& lam = rule.pts[static_cast<size_t>(q)];
        const V3 x = physical_point(lam, verts);
        double uh = 0.0;
        for (int i = 0; i < 4; ++i) uh += lam[static_cast<size_t>(i)] * nodal[static_cast<size_t>(tet[static_cast<size_t>(i)])];
        const double d = tg(x) - uh;
        acc += rule.w[static_cast<size_t>(q)] * d * d;
      }
      double h = 0.0;
      for (int a = 0; a < 4; ++a)
        for (int c = a + 1; c < 4; ++c) h = std::max(h, dist3(verts[static_cast<size_t>(a)], verts[static_cast<size_t>(c)]));
      const double a_tau = std::min(h * inv_sqrt_rho, 1.0);
      eta_sq[static_cast<size_t>(t)] = a_tau * a_tau * lg.volume * acc;
    }
  });
  struct FaceRef {
    std::array<int, 3> key;
    int tet;
  };
  constexpr int kOpp[4][3] = {{1, 2, 3}, {0, 2, 3}, {0, 1, 3}, {0, 1, 2}};
  std::vector<FaceRef> faces;
  faces.reserve(static_cast<size_t>(nt) * 4);
  for (int t = 0; t < nt; ++t) {
    const auto& tet = m.tets[static_cast<size_t>(t)];
    for (int l = 0; l < 4; ++l) {
      std::array<int, 3> key = {tet[static_cast<size_t>(kOpp[l][0])], tet[static_cast<size_t>(kOpp[l][1])],
                                tet[static_cast<size_t>(kOpp[l][2])]};
      std::sort(key.begin(), key.end());
      faces.push_back({key, t});
    }
  }
  std::sort(faces.begin(), faces.end(), [](const FaceRef& a, const FaceRef& b) {
    if (a.key != b.key) return a.key < b.key;
    return a.tet < b.tet;
  });
  for (size_t i = 0; i + 1 < faces.size(); ++i) {
    if (faces[i].key != faces[i + 1].key) continue;
    const FaceRef& fa = faces[i];
    const FaceRef& fb = faces[i + 1];
    const V3& v0 = m.vertices[static_cast<size_t>(fa.key[0])];
    const V3& v1 = m.vertices[static_cast<size_t>(fa.key[1])];
    const V3& v2 = m.vertices[static_cast<size_t>(fa.key[2])];
    double a[3], b[3];
    for (int c = 0; c < 3; ++c) {
      a[c] = v1.c[c] - v0.c[c];
      b[c] = v2.c[c] - v0.c[c];
    }
    const double cr[3] = {a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0]};
    const double cn = norm3(cr);
    const double area = 0.5 * cn;
    const double sq = (cr[0] * cr[0] + cr[1] * cr[1]) + cr[2] * cr[2];  // normalized(): v / sqrt(|v|^2)
    const double nr = std::sqrt(sq);
    const double nn[3] = {sq > 0.0 ? cr[0] / nr : cr[0], sq > 0.0 ? cr[1] / nr : cr[1], sq > 0.0 ? cr[2] / nr : cr[2]};
    const auto& ga = grad[static_cast<size_t>(fa.tet)];
    const auto& gb = grad[static_cast<size_t>(fb.tet)];
    const double dg[3] = {ga[0] - gb[0], ga[1] - gb[1], ga[2] - gb[2]};
    const double jump = rho * ((dg[0] * nn[0] + dg[1] * nn[1]) + dg[2] * nn[2]);
    const double h_f = std::max({dist3(v0, v1), dist3(v1, v2), dist3(v0, v2)});
    const double a_f = std::min(h_f * inv_sqrt_rho, 1.0);
    const double term = 0.5 * inv_sqrt_rho * a_f * area * jump * jump;
    eta_sq[static_cast<size_t>(fa.tet)] += term;
    eta_sq[static_cast<size_t>(fb.tet)] += term;
    ++i;
  }
  Estimate est;
  est.per_tet.resize(static_cast<size_t>(nt));
  for (int t = 0; t < nt; ++t) est.per_tet[static_cast<size_t>(t)] = std::sqrt(eta_sq[static_cast<size_t>(t)]);
  est.global = std::sqrt(eigen_sum(eta_sq.data(), nt));
  return est;
}

// adapt.cpp:126-150
std::vector<int> mark_dorfler(const Vec& eta, double theta) {
  if (!(theta > 0.0 && theta <= 1.0)) throw std::invalid_argument("mark_dorfler: theta must be in (0, 1]");
  const int nt = static_cast<int>(eta.size());
  std::vector<int> order(static_cast<size_t>(nt));
  for (int t = 0; t < nt; ++t) order[static_cast<size_t>(t)] = t;
  std::sort(order.begin(), order.end(), [&](int a, int b) {
    const double ea = eta[static_cast<size_t>(a)], eb = eta[static_cast<size_t>(b)];
    if (ea != eb) return ea > eb;
    return a < b;
  });
  double total = 0.0;
  for (int t : order) total += eta[static_cast<size_t>(t)] * eta[static_cast<size_t>(t)];
  const double goal = theta * theta * total;
  std::vector<int> marked;
  double acc = 0.0;
  for (int t : order) {
    const double e = eta[static_cast<size_t>(t)];
    if (acc >= goal || e == 0.0) break;
    marked.push_back(t);
    acc += e * e;
  }
  return marked;
}

int64_t edge_key(int a, int b) {  // mesh.cpp:20-23
  if (a > b) std::swap(a, b);
  return (static_cast<int64_t>(a) << 32) | static_cast<uint32_t>(b);
}

// mesh.cpp:67-145: bisect the marked tets at edge (0, d), then every tet still carrying a split
// edge, round by round; midpoints numbered in order of first split (tets ascending)
Mesh bisect_marked(const Mesh& mesh, const std::vector<int>& marked) {
  Mesh m = mesh;
  std::vector<uint8_t> flag(m.tets.size(), 0);
  for (int t : marked) {
    if (t < 0 || t >= m.nt()) throw std::out_of_range("bisect_marked: tet index out of range");
    flag[static_cast<size_t>(t)] = 1;
  }
  std::unordered_map<int64_t, int> midpoint;
  auto mid_vertex = [&](int a, int b) {
    const int64_t key = edge_key(a, b);
    const auto it = midpoint.find(key);
    if (it != midpoint.end()) return it->second;
    const int z = m.nv();
    const V3& va = m.vertices[static_cast<size_t>(a)];
    const V3& vb = m.vertices[static_cast<size_t>(b)];
    const V3 x{{0.5 * (va.c[0] + vb.c[0]), 0.5 * (va.c[1] + vb.c[1]), 0.5 * (va.c[2] + vb.c[2])}};
    m.vertices.push_back(x);
    m.boundary.push_back(on_unit_boundary(x) ? 1 : 0);
    midpoint.emplace(key, z);
    return z;
  };
  constexpr int kLocalEdges[6][2] = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}};
  int round = 0;
  while (std::find(flag.begin(), flag.end(), uint8_t{1}) != flag.end()) {
    if (++round > 1000) throw std::logic_error("bisect_marked: conforming closure did not terminate");
    std::vector<std::array<int, 4>> tets;
    std::vector<uint8_t> tags;
    std::vector<int> gens;
    tets.reserve(m.tets.size() * 2);
    for (size_t t = 0; t < m.tets.size(); ++t) {
      if (!flag[t]) {
        tets.push_back(m.tets[t]);
        tags.push_back(m.refinement_edge[t]);
        gens.push_back(m.generation[t]);
        continue;
      }
      const auto p = m.tets[t];
      const int d = m.refinement_edge[t];
      const int z = mid_vertex(p[0], p[static_cast<size_t>(d)]);
      std::array<int, 4> c1 = p;
      c1[static_cast<size_t>(d)] = z;
      std::array<int, 4> c2;
      for (int q = 0; q < d; ++q) c2[static_cast<size_t>(q)] = p[static_cast<size_t>(q + 1)];
      c2[static_cast<size_t>(d)] = z;
      for (int q = d + 1; q < 4; ++q) c2[static_cast<size_t>(q)] = p[static_cast<size_t>(q)];
      const uint8_t nd = static_cast<uint8_t>(d == 1 ? 3 : d - 1);
      const int g = m.generation[t] + 1;
      tets.push_back(c1);
      tags.push_back(nd);
      gens.push_back(g);
      tets.push_back(c2);
      tags.push_back(nd);
      gens.push_back(g);
    }
    m.tets = std::move(tets);
    m.refinement_edge = std::move(tags);
    m.generation = std::move(gens);
    flag.assign(m.tets.size(), 0);
    for (size_t t = 0; t < m.tets.size(); ++t) {
      const auto& v = m.tets[t];
      for (const auto& e : kLocalEdges)
        if (midpoint.count(edge_key(v[static_cast<size_t>(e[0])], v[static_cast<size_t>(e[1])]))) {
          flag[t] = 1;
          break;
        }
    }
  }
  return m;
}

Mesh uniform_refine(const Mesh& mesh) {  // mesh.cpp:147-156: three full sweeps
  Mesh m = mesh;
  for (int sweep = 0; sweep < 3; ++sweep) {
    std::vector<int> all(m.tets.size());
    for (size_t t = 0; t < all.size(); ++t) all[t] = static_cast<int>(t);
    m = bisect_marked(m, all);
  }
  return m;
}

int n_interior(const Mesh& m) {  // mesh_stats(...).n_interior_dofs
  int k = 0;
  for (uint8_t b : m.boundary) k += b ? 0 : 1;
  return k;
}

struct AdaptLevel {
  int level = 0, dofs = 0;
  double eta = 0.0, err_l2_sq = 0.0, err_hm1_sq = 0.0;
  int iterations = 0;
  double seconds = 0.0;
};

// adapt.cpp:152-205 with the AMG solver of bench.cpp:65-74 / test_adapt.cpp:36-41:
// build_amg(A) then pcg(A, amg_precond, f, tol, 500)
std::vector<AdaptLevel> adaptive_solve(const Mesh& initial, const Target& tg, double rho, int dof_budget,
                                       double tol, double theta, Mesh* final_mesh, Vec* final_coeffs) {
  std::vector<AdaptLevel> hist;
  Mesh mesh = initial;
  int level = 0;
  for (;;) {
    const auto t0 = std::chrono::steady_clock::now();
    const System sys = build_system(mesh, rho, tg);
    PcgOut res;
    if (!sys.f.empty()) {
      const Amg h = build_amg(sys.A, 64, 1);
      const Csr& A = sys.A;
      res = pcg([&A](const Vec& v) { return spmv(A, v); }, [&h](const Vec& r) { return amg_apply(h, r); }, sys.f,
                tol, 500);
    }
    const Estimate est = estimate(mesh, sys.dm, res.x.data(), rho, tg);
    const double l2_sq = l2_error_target_squared(mesh, sys.dm, res.x.data(), tg);
    const double hm1 = target_dual_norm(sys, res.x.data());
    AdaptLevel row;
    row.level = level;
    row.dofs = sys.dm.n_dofs();
    row.eta = est.global;
    row.err_l2_sq = l2_sq;
    row.err_hm1_sq = hm1 * hm1;
    row.iterations = res.iterations;
    row.seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    hist.push_back(row);
    if (row.dofs >= dof_budget) {
      if (final_mesh) *final_mesh = std::move(mesh);
      if (final_coeffs) *final_coeffs = std::move(res.x);
      return hist;
    }
    if (++level > 200) throw std::runtime_error("adaptive_solve: level cap reached before the dof budget");
    const std::vector<int> marked = mark_dorfler(est.per_tet, theta);
    Mesh refined = bisect_marked(mesh, marked);
    if (n_interior(refined) == row.dofs)
      throw std::runtime_error("adaptive_solve: refinement stagnated at level " + std::to_string(level - 1) +
                               " (" + std::to_string(row.dofs) + " dofs)");
    mesh = std::move(refined);
  }
}

// ---------------------------------------------------------------------------
// bddc.cpp (§8(f)4): RCB partition, interface / corner / face-class constraints, subdomain
// Schur complements, the constrained coarse basis, and the BDDC preconditioner.  Dense linear
// algebra replaces Eigen's SimplicialLLT (AMD-ordered) / PartialPivLU / GEMM kernels, whose
// orders are unverifiable here: parity on this row is to rounding (the reference's own
// test_bddc.cpp bars are 1e-10 .. 1e-7), not bit for bit.
struct Partition {
  int p = 0;
  std::vector<int> owner;
  std::vector<std::vector<int>> dof_subdomains;
  std::vector<uint8_t> is_interface;
};

// bddc.cpp:45-111
Partition partition_geometric(const Mesh& mesh, const DofMap& dm, int p) {
  if (p < 2) throw std::invalid_argument("partition_geometric: p must be >= 2");
  if (p > mesh.nt()) throw std::invalid_argument("partition_geometric: more subdomains than tets");
  const int nt = mesh.nt();
  std::vector<V3> centroid(static_cast<size_t>(nt));
  for (int t = 0; t < nt; ++t) {
    const auto v = tet_vertices(mesh, t);
    for (int c = 0; c < 3; ++c)
      centroid[static_cast<size_t>(t)].c[c] = 0.25 * (((v[0].c[c] + v[1].c[c]) + v[2].c[c]) + v[3].c[c]);
  }
  Partition part;
  part.p = p;
  part.owner.assign(static_cast<size_t>(nt), -1);
  std::function<void(std::vector<int>&, int, int)> rcb = [&](std::vector<int>& ids, int parts, int label) {
    if (parts == 1) {
      for (int t : ids) part.owner[static_cast<size_t>(t)] = label;
      return;
    }
    V3 lo = centroid[static_cast<size_t>(ids.front())], hi = lo;
    for (int t : ids)
      for (int c = 0; c < 3; ++c) {
        lo.c[c] = std::min(lo.c[c], centroid[static_cast<size_t>(t)].c[c]);
        hi.c[c] = std::max(hi.c[c], centroid[static_cast<size_t>(t)].c[c]);
      }
    int axis = 0;
    double ext = hi.c[0] - lo.c[0];
    for (int a = 1; a < 3; ++a)
      if (hi.c[a] - lo.c[a] > ext) {
        ext = hi.c[a] - lo.c[a];
        axis = a;
      }
    std::sort(ids.begin(), ids.end(), [&](int a, int b) {
      const double ca = centroid[static_cast<size_t>(a)].c[axis], cb = centroid[static_cast<size_t>(b)].c[axis];
      if (ca != cb) return ca < cb;
      return a < b;
    });
    const int p1 = parts / 2;
    const auto n1 = static_cast<int64_t>(ids.size()) * p1 / parts;
    std::vector<int> left(ids.begin(), ids.begin() + n1), right(ids.begin() + n1, ids.end());
    rcb(left, p1, label);
    rcb(right, parts - p1, label + p1);
  };
  std::vector<int> all(static_cast<size_t>(nt));
  for (int t = 0; t < nt; ++t) all[static_cast<size_t>(t)] = t;
  rcb(all, p, 0);
  part.dof_subdomains.assign(static_cast<size_t>(dm.n_dofs()), {});
  for (int t = 0; t < nt; ++t)
    for (int v : mesh.tets[static_cast<size_t>(t)]) {
      const int d = dm.vertex_to_dof[static_cast<size_t>(v)];
      if (d >= 0) part.dof_subdomains[static_cast<size_t>(d)].push_back(part.owner[static_cast<size_t>(t)]);
    }
  part.is_interface.assign(static_cast<size_t>(dm.n_dofs()), 0);
  for (int d = 0; d < dm.n_dofs(); ++d) {
    auto& ss = part.dof_subdomains[static_cast<size_t>(d)];
    std::sort(ss.begin(), ss.end());
    ss.erase(std::unique(ss.begin(), ss.end()), ss.end());
    part.is_interface[static_cast<size_t>(d)] = ss.size() >= 2 ? 1 : 0;
  }
  return part;
}

// dense row-major helpers
using Dense = std::vector<double>;
// Eigen PartialPivLU restated unblocked: row pivot = first largest |a_ik|, rank-1 updates
struct Lu {
  int n = 0;
  Dense a;
  std::vector<int> piv;
};
Lu lu_compute(int n, Dense a) {
  Lu f;
  f.n = n;
  f.piv.resize(static_cast<size_t>(n));
  for (int k = 0; k < n; ++k) {
    int pr = k;
    double best = std::abs(a[static_cast<size_t>(k) * n + k]);
    for (int i = k + 1; i < n; ++i)
      if (std::abs(a[static_cast<size_t>(i) * n + k]) > best) {
        best = std::abs(a[static_cast<size_t>(i) * n + k]);
        pr = i;
      }
    f.piv[static_cast<size_t>(k)] = pr;
    if (pr != k)
      for (int j = 0; j < n; ++j) std::swap(a[static_cast<size_t>(k) * n + j], a[static_cast<size_t>(pr) * n + j]);
    const double d = a[static_cast<size_t>(k) * n + k];
    if (d == 0.0) continue;
    for (int i = k + 1; i < n; ++i) {
      const double l = a[static_cast<size_t>(i) * n + k] / d;
      a[static_cast<size_t>(i) * n + k] = l;
      for (int j = k + 1; j < n; ++j) a[static_cast<size_t>(i) * n + j] -= l * a[static_cast<size_t>(k) * n + j];
    }
  }
  f.a = std::move(a);
  return f;
}
Vec lu_solve(const Lu& f, Vec b) {
  const int n = f.n;
  for (int k = 0; k < n; ++k) std::swap(b[static_cast<size_t>(k)], b[static_cast<size_t>(f.piv[static_cast<size_t>(k)])]);
  for (int i = 0; i < n; ++i)
    for (int k = 0; k < i; ++k) b[static_cast<size_t>(i)] -= f.a[static_cast<size_t>(i) * n + k] * b[static_cast<size_t>(k)];
  for (int i = n - 1; i >= 0; --i) {
    for (int k = i + 1; k < n; ++k) b[static_cast<size_t>(i)] -= f.a[static_cast<size_t>(i) * n + k] * b[static_cast<size_t>(k)];
    b[static_cast<size_t>(i)] /= f.a[static_cast<size_t>(i) * n + i];
  }
  return b;
}

struct BddcSub {
  std::vector<int> tets, interior, boundary, boundary_index, primal_index;
  Csr A_IB, A_BI;
  Llt llt;  // dense A_II factor
  Dense S, C, Phi;  // nB x nB, n_con x nB, nB x n_con
  Lu saddle;
  Vec scaling;
  int nI = 0, nB = 0, ncon = 0;
};
struct Bddc {
  Partition part;
  std::vector<int> interface_dofs, interface_index;
  Csr A_CC;
  std::vector<BddcSub> subs;
  int n_primal = 0;
  Dense coarse;
  Llt coarse_llt;
};

Csr extract_submatrix(const Csr& A, const std::vector<int>& rows, const std::vector<int>& col_index, int ncols) {
  Csr B;  // bddc.cpp:16-30: rows in order, kept columns mapped (ascending stays ascending)
  B.rows = static_cast<int>(rows.size());
  B.cols = ncols;
  B.rp.assign(rows.size() + 1, 0);
  for (size_t r = 0; r < rows.size(); ++r) {
    const int i = rows[r];
    std::vector<std::pair<int, double>> e;
    for (int k = A.rp[static_cast<size_t>(i)]; k < A.rp[static_cast<size_t>(i) + 1]; ++k) {
      const int c = col_index[static_cast<size_t>(A.ci[static_cast<size_t>(k)])];
      if (c >= 0 && A.v[static_cast<size_t>(k)] != 0.0) e.push_back({c, A.v[static_cast<size_t>(k)]});
    }
    std::sort(e.begin(), e.end());
    for (auto& q : e) {
      B.ci.push_back(q.first);
      B.v.push_back(q.second);
    }
    B.rp[r + 1] = static_cast<int>(B.ci.size());
  }
  return B;
}

Vec llt_solve_vec(const Llt& f, const Vec& b) { return llt_solve(f, b); }

// bddc.cpp:113-301
Bddc build_bddc(const Mesh& mesh, const System& sys, const Partition& part) {
  Bddc op;
  op.part = part;
  const DofMap& dm = sys.dm;
  const int nd = dm.n_dofs(), p = part.p;
  op.interface_index.assign(static_cast<size_t>(nd), -1);
  for (int d = 0; d < nd; ++d)
    if (part.is_interface[static_cast<size_t>(d)]) {
      op.interface_index[static_cast<size_t>(d)] = static_cast<int>(op.interface_dofs.size());
      op.interface_dofs.push_back(d);
    }
  const int nC = static_cast<int>(op.interface_dofs.size());
  op.A_CC = extract_submatrix(sys.A, op.interface_dofs, op.interface_index, nC);
  std::vector<uint8_t> near_boundary(static_cast<size_t>(nd), 0);
  constexpr int edges[6][2] = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}};
  for (const auto& tet : mesh.tets)
    for (const auto& e : edges) {
      const int a = tet[static_cast<size_t>(e[0])], b = tet[static_cast<size_t>(e[1])];
      if (mesh.boundary[static_cast<size_t>(a)] != mesh.boundary[static_cast<size_t>(b)]) {
        const int iv = mesh.boundary[static_cast<size_t>(a)] ? b : a;
        near_boundary[static_cast<size_t>(dm.vertex_to_dof[static_cast<size_t>(iv)])] = 1;
      }
    }
  std::vector<uint8_t> is_corner(static_cast<size_t>(nd), 0);
  for (int d : op.interface_dofs) {
    const size_t mult = part.dof_subdomains[static_cast<size_t>(d)].size();
    is_corner[static_cast<size_t>(d)] = (mult >= 3 || (mult >= 2 && near_boundary[static_cast<size_t>(d)])) ? 1 : 0;
  }
  std::map<std::vector<int>, int> class_of_key;
  std::vector<std::vector<int>> class_dofs, class_key;
  for (int d : op.interface_dofs) {
    if (is_corner[static_cast<size_t>(d)]) continue;
    const auto& key = part.dof_subdomains[static_cast<size_t>(d)];
    auto it = class_of_key.find(key);
    if (it == class_of_key.end()) {
      it = class_of_key.emplace(key, static_cast<int>(class_dofs.size())).first;
      class_dofs.emplace_back();
      class_key.push_back(key);
    }
    class_dofs[static_cast<size_t>(it->second)].push_back(d);
  }
  std::vector<int> corner_primal(static_cast<size_t>(nd), -1);
  int np = 0;
  for (int d : op.interface_dofs)
    if (is_corner[static_cast<size_t>(d)]) corner_primal[static_cast<size_t>(d)] = np++;
  const int first_class = np;
  np += static_cast<int>(class_dofs.size());
  op.n_primal = np;
  std::vector<std::vector<int>> sub_classes(static_cast<size_t>(p));
  for (size_t c = 0; c < class_key.size(); ++c)
    for (int sdx : class_key[c]) sub_classes[static_cast<size_t>(sdx)].push_back(static_cast<int>(c));
  op.subs.resize(static_cast<size_t>(p));
  for (int t = 0; t < mesh.nt(); ++t) op.subs[static_cast<size_t>(part.owner[static_cast<size_t>(t)])].tets.push_back(t);
  for (int d = 0; d < nd; ++d) {
    const auto& ss = part.dof_subdomains[static_cast<size_t>(d)];
    if (ss.size() == 1)
      op.subs[static_cast<size_t>(ss[0])].interior.push_back(d);
    else
      for (int sdx : ss) op.subs[static_cast<size_t>(sdx)].boundary.push_back(d);
  }
  for (int sdx = 0; sdx < p; ++sdx) {
    BddcSub& sd = op.subs[static_cast<size_t>(sdx)];
    const int nI = sd.nI = static_cast<int>(sd.interior.size());
    const int nB = sd.nB = static_cast<int>(sd.boundary.size());
    sd.boundary_index.resize(static_cast<size_t>(nB));
    sd.scaling.resize(static_cast<size_t>(nB));
    for (int k = 0; k < nB; ++k) {
      const int d = sd.boundary[static_cast<size_t>(k)];
      sd.boundary_index[static_cast<size_t>(k)] = op.interface_index[static_cast<size_t>(d)];
      sd.scaling[static_cast<size_t>(k)] = 1.0 / static_cast<double>(part.dof_subdomains[static_cast<size_t>(d)].size());
    }
    // assemble_subdomain_matrix (assembly.cpp:250-263): rho K + M over the subdomain's tets
    std::vector<int> dofs = sd.interior;
    dofs.insert(dofs.end(), sd.boundary.begin(), sd.boundary.end());
    std::vector<uint8_t> mask(static_cast<size_t>(mesh.nt()), 0);
    for (int t : sd.tets) mask[static_cast<size_t>(t)] = 1;
    std::vector<int> row_of_vert(static_cast<size_t>(mesh.nv()), -1), vert_of_row(dofs.size());
    for (size_t i = 0; i < dofs.size(); ++i) {
      const int v = dm.dof_to_vertex[static_cast<size_t>(dofs[i])];
      row_of_vert[static_cast<size_t>(v)] = static_cast<int>(i);
      vert_of_row[i] = v;
    }
    const Csr Asub = assemble_matrix(mesh, row_of_vert, vert_of_row, sys.rho, 1.0, &mask);
    Dense AII(static_cast<size_t>(nI) * nI, 0.0), BB(static_cast<size_t>(nB) * nB, 0.0);
    sd.A_IB.rows = nI; sd.A_IB.cols = nB; sd.A_IB.rp.assign(static_cast<size_t>(nI) + 1, 0);
    sd.A_BI.rows = nB; sd.A_BI.cols = nI; sd.A_BI.rp.assign(static_cast<size_t>(nB) + 1, 0);
    for (int r = 0; r < nI + nB; ++r) {
      for (int k = Asub.rp[static_cast<size_t>(r)]; k < Asub.rp[static_cast<size_t>(r) + 1]; ++k) {
        const int c = Asub.ci[static_cast<size_t>(k)];
        const double v = Asub.v[static_cast<size_t>(k)];
        if (r < nI && c < nI) AII[static_cast<size_t>(r) * nI + c] = v;
        else if (r < nI) { sd.A_IB.ci.push_back(c - nI); sd.A_IB.v.push_back(v); }
        else if (c < nI) { sd.A_BI.ci.push_back(c); sd.A_BI.v.push_back(v); }
        else BB[static_cast<size_t>(r - nI) * nB + (c - nI)] = v;
      }
      if (r < nI) sd.A_IB.rp[static_cast<size_t>(r) + 1] = static_cast<int>(sd.A_IB.ci.size());
      else sd.A_BI.rp[static_cast<size_t>(r - nI) + 1] = static_cast<int>(sd.A_BI.ci.size());
    }
    Dense X(static_cast<size_t>(nI) * nB, 0.0);  // A_II^-1 A_IB
    if (nI > 0) {
      sd.llt = llt_compute(nI, AII);
      if (!sd.llt.ok) throw std::runtime_error("build_bddc: interior factorization failed in subdomain " + std::to_string(sdx));
      const std::vector<double> dIB = to_dense(sd.A_IB);
      for (int j = 0; j < nB; ++j) {
        Vec col(static_cast<size_t>(nI));
        for (int i = 0; i < nI; ++i) col[static_cast<size_t>(i)] = dIB[static_cast<size_t>(i) * nB + j];
        const Vec x = llt_solve(sd.llt, col);
        for (int i = 0; i < nI; ++i) X[static_cast<size_t>(i) * nB + j] = x[static_cast<size_t>(i)];
      }
    }
    const std::vector<double> dBI = nI > 0 ? to_dense(sd.A_BI) : std::vector<double>();
    Dense S(static_cast<size_t>(nB) * nB);
    for (int a = 0; a < nB; ++a)
      for (int b = 0; b < nB; ++b) {
        double acc = 0.0;
        for (int k = 0; k < nI; ++k) acc += dBI[static_cast<size_t>(a) * nI + k] * X[static_cast<size_t>(k) * nB + b];
        S[static_cast<size_t>(a) * nB + b] = BB[static_cast<size_t>(a) * nB + b] - acc;
      }
    sd.S.resize(S.size());
    for (int a = 0; a < nB; ++a)
      for (int b = 0; b < nB; ++b)
        sd.S[static_cast<size_t>(a) * nB + b] = 0.5 * (S[static_cast<size_t>(a) * nB + b] + S[static_cast<size_t>(b) * nB + a]);
    // constraints: local corners then face classes (bddc.cpp:233-254)
    std::vector<int> local_corners;
    for (int d : sd.boundary)
      if (is_corner[static_cast<size_t>(d)]) local_corners.push_back(d);
    const auto& cls = sub_classes[static_cast<size_t>(sdx)];
    const int ncon = sd.ncon = static_cast<int>(local_corners.size() + cls.size());
    sd.C.assign(static_cast<size_t>(ncon) * nB, 0.0);
    auto lbi = [&](int d) {
      return static_cast<int>(std::lower_bound(sd.boundary.begin(), sd.boundary.end(), d) - sd.boundary.begin());
    };
    int row = 0;
    for (int d : local_corners) {
      sd.C[static_cast<size_t>(row) * nB + lbi(d)] = 1.0;
      sd.primal_index.push_back(corner_primal[static_cast<size_t>(d)]);
      ++row;
    }
    for (int c : cls) {
      const auto& members = class_dofs[static_cast<size_t>(c)];
      const double w = 1.0 / static_cast<double>(members.size());
      for (int d : members) sd.C[static_cast<size_t>(row) * nB + lbi(d)] = w;
      sd.primal_index.push_back(first_class + c);
      ++row;
    }
    const int m = nB + ncon;
    if (m > 0) {
      Dense sad(static_cast<size_t>(m) * m, 0.0);
      for (int a = 0; a < nB; ++a)
        for (int b = 0; b < nB; ++b) sad[static_cast<size_t>(a) * m + b] = sd.S[static_cast<size_t>(a) * nB + b];
      for (int r = 0; r < ncon; ++r)
        for (int b = 0; b < nB; ++b) {
          sad[static_cast<size_t>(b) * m + nB + r] = sd.C[static_cast<size_t>(r) * nB + b];
          sad[static_cast<size_t>(nB + r) * m + b] = sd.C[static_cast<size_t>(r) * nB + b];
        }
      sd.saddle = lu_compute(m, sad);
      sd.Phi.assign(static_cast<size_t>(nB) * ncon, 0.0);
      for (int c = 0; c < ncon; ++c) {
        Vec rhs(static_cast<size_t>(m), 0.0);
        rhs[static_cast<size_t>(nB + c)] = 1.0;
        const Vec sol = lu_solve(sd.saddle, rhs);
        for (int b = 0; b < nB; ++b) sd.Phi[static_cast<size_t>(b) * ncon + c] = sol[static_cast<size_t>(b)];
      }
    }
  }
  op.coarse.assign(static_cast<size_t>(np) * np, 0.0);
  for (const auto& sd : op.subs) {
    const int nc = sd.ncon, nB = sd.nB;
    if (!nc) continue;
    Dense SP(static_cast<size_t>(nB) * nc, 0.0);  // S Phi
    for (int a = 0; a < nB; ++a)
      for (int c = 0; c < nc; ++c) {
        double acc = 0.0;
        for (int k = 0; k < nB; ++k) acc += sd.S[static_cast<size_t>(a) * nB + k] * sd.Phi[static_cast<size_t>(k) * nc + c];
        SP[static_cast<size_t>(a) * nc + c] = acc;
      }
    for (int r = 0; r < nc; ++r)
      for (int c = 0; c < nc; ++c) {
        double acc = 0.0;
        for (int k = 0; k < nB; ++k) acc += sd.Phi[static_cast<size_t>(k) * nc + r] * SP[static_cast<size_t>(k) * nc + c];
        op.coarse[static_cast<size_t>(sd.primal_index[static_cast<size_t>(r)]) * np + sd.primal_index[static_cast<size_t>(c)]] += acc;
      }
  }
  if (np > 0) {
    op.coarse_llt = llt_compute(np, op.coarse);
    if (!op.coarse_llt.ok) throw std::runtime_error("build_bddc: coarse matrix not positive definite");
  }
  return op;
}

Vec gather_v(const Vec& x, const std::vector<int>& idx) {
  Vec o(idx.size());
  for (size_t k = 0; k < idx.size(); ++k) o[k] = x[static_cast<size_t>(idx[k])];
  return o;
}

Vec schur_apply(const Bddc& op, const Vec& x) {  // bddc.cpp:303-324
  Vec y = spmv(op.A_CC, x);
  for (const auto& sd : op.subs) {
    if (sd.boundary.empty() || sd.interior.empty()) continue;
    const Vec w = llt_solve(sd.llt, spmv(sd.A_IB, gather_v(x, sd.boundary_index)));
    const Vec c = spmv(sd.A_BI, w);
    for (size_t k = 0; k < c.size(); ++k) y[static_cast<size_t>(sd.boundary_index[k])] -= c[k];
  }
  return y;
}
Vec reduce_rhs(const Bddc& op, const Vec& f) {  // bddc.cpp:326-345
  Vec g = gather_v(f, op.interface_dofs);
  for (const auto& sd : op.subs) {
    if (sd.boundary.empty() || sd.interior.empty()) continue;
    const Vec c = spmv(sd.A_BI, llt_solve(sd.llt, gather_v(f, sd.interior)));
    for (size_t k = 0; k < c.size(); ++k) g[static_cast<size_t>(sd.boundary_index[k])] -= c[k];
  }
  return g;
}
Vec expand_solution(const Bddc& op, const Vec& uC, const Vec& f) {  // bddc.cpp:347-370
  Vec u(f.size(), 0.0);
  for (size_t k = 0; k < op.interface_dofs.size(); ++k) u[static_cast<size_t>(op.interface_dofs[k])] = uC[k];
  for (const auto& sd : op.subs) {
    if (sd.interior.empty()) continue;
    Vec rhs = gather_v(f, sd.interior);
    if (!sd.boundary.empty()) {
      const Vec t = spmv(sd.A_IB, gather_v(uC, sd.boundary_index));
      for (size_t k = 0; k < rhs.size(); ++k) rhs[k] -= t[k];
    }
    const Vec w = llt_solve(sd.llt, rhs);
    for (size_t k = 0; k < sd.interior.size(); ++k) u[static_cast<size_t>(sd.interior[k])] = w[k];
  }
  return u;
}
Vec bddc_apply(const Bddc& op, const Vec& r) {  // bddc.cpp:372-430
  const int nC = static_cast<int>(op.interface_dofs.size());
  Vec z(static_cast<size_t>(nC), 0.0), rp(static_cast<size_t>(op.n_primal), 0.0);
  std::vector<Vec> rbs(op.subs.size());
  for (size_t s = 0; s < op.subs.size(); ++s) {
    const BddcSub& sd = op.subs[s];
    if (!sd.nB) continue;
    Vec rb = gather_v(r, sd.boundary_index);
    for (int k = 0; k < sd.nB; ++k) rb[static_cast<size_t>(k)] = sd.scaling[static_cast<size_t>(k)] * rb[static_cast<size_t>(k)];
    Vec rhs(static_cast<size_t>(sd.nB + sd.ncon), 0.0);
    for (int k = 0; k < sd.nB; ++k) rhs[static_cast<size_t>(k)] = rb[static_cast<size_t>(k)];
    const Vec sol = lu_solve(sd.saddle, rhs);
    for (int k = 0; k < sd.nB; ++k)
      z[static_cast<size_t>(sd.boundary_index[static_cast<size_t>(k)])] += sd.scaling[static_cast<size_t>(k)] * sol[static_cast<size_t>(k)];
    for (int c = 0; c < sd.ncon; ++c) {
      double acc = 0.0;
      for (int k = 0; k < sd.nB; ++k) acc += sd.Phi[static_cast<size_t>(k) * sd.ncon + c] * rb[static_cast<size_t>(k)];
      rp[static_cast<size_t>(sd.primal_index[static_cast<size_t>(c)])] += acc;
    }
  }
  if (op.n_primal > 0) {
    const Vec lam = llt_solve(op.coarse_llt, rp);
    for (const auto& sd : op.subs) {
      if (!sd.ncon) continue;
      for (int k = 0; k < sd.nB; ++k) {
        double acc = 0.0;
        for (int c = 0; c < sd.ncon; ++c)
          acc += sd.Phi[static_cast<size_t>(k) * sd.ncon + c] * lam[static_cast<size_t>(sd.primal_index[static_cast<size_t>(c)])];
        z[static_cast<size_t>(sd.boundary_index[static_cast<size_t>(k)])] += sd.scaling[static_cast<size_t>(k)] * acc;
      }
    }
  }
  return z;
}

template <class F>
int guard(F&& fn) {
  try {
    fn();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}

}  // namespace

// ---------------------------------------------------------------------------
// C surface
struct or_mesh {
  Mesh m;
};
struct or_csr {
  Csr a;
};
struct or_system {
  System s;
  or_csr views[3];
};
struct or_amg {
  Amg h;
  std::vector<or_csr> views;  // 3 per level
};
struct or_bddc {
  Bddc op;
};

extern "C" {

const char* or_last_error(void) { return g_err.c_str(); }
void or_set_num_threads(int n) { g_threads = n < 1 ? 1 : n; }
int or_num_threads(void) { return g_threads; }

int or_build_structured_cube(int n, or_mesh** out) {
  return guard([&] { *out = new or_mesh{build_structured_cube(n)}; });
}
void or_mesh_free(or_mesh* m) { delete m; }
int or_mesh_new(int nv, const double* xyz, int nt, const int* tets, const uint8_t* boundary, or_mesh** out) {
  return guard([&] {
    auto* m = new or_mesh;
    for (int v = 0; v < nv; ++v) {
      m->m.vertices.push_back(V3{{xyz[3 * v], xyz[3 * v + 1], xyz[3 * v + 2]}});
      m->m.boundary.push_back(boundary[v]);
    }
    for (int t = 0; t < nt; ++t) {
      m->m.tets.push_back({tets[4 * t], tets[4 * t + 1], tets[4 * t + 2], tets[4 * t + 3]});
      m->m.refinement_edge.push_back(3);
      m->m.generation.push_back(0);
    }
    *out = m;
  });
}
void or_mesh_info(const or_mesh* m, int* nv, int* nt) {
  *nv = m->m.nv();
  *nt = m->m.nt();
}
void or_mesh_get(const or_mesh* m, double* xyz, int* tets, uint8_t* bnd, uint8_t* re, int* gen) {
  const Mesh& M = m->m;
  for (int v = 0; v < M.nv(); ++v)
    for (int c = 0; c < 3; ++c) {
      if (xyz) xyz[3 * v + c] = M.vertices[static_cast<size_t>(v)].c[c];
    }
  for (int t = 0; t < M.nt(); ++t)
    for (int c = 0; c < 4; ++c)
      if (tets) tets[4 * t + c] = M.tets[static_cast<size_t>(t)][static_cast<size_t>(c)];
  if (bnd) std::memcpy(bnd, M.boundary.data(), M.boundary.size());
  if (re) std::memcpy(re, M.refinement_edge.data(), M.refinement_edge.size());
  if (gen) std::memcpy(gen, M.generation.data(), M.generation.size() * sizeof(int));
}
double or_tet_volume(const or_mesh* m, int t) { return tet_volume(m->m, t); }

int or_rule_size(int rule) { return rule_by_id(rule).size(); }
void or_rule_get(int rule, double* pts, double* w) {
  const Rule& r = rule_by_id(rule);
  for (int q = 0; q < r.size(); ++q) {
    for (int k = 0; k < 4; ++k) pts[4 * q + k] = r.pts[static_cast<size_t>(q)][static_cast<size_t>(k)];
    w[q] = r.w[static_cast<size_t>(q)];
  }
}

int or_target_eval(int kind, int n, uint64_t seed, int npts, const double* xyz, double* out) {
  return guard([&] {
    const Target t = make_target(kind, n, seed);
    for (int i = 0; i < npts; ++i) out[i] = t(V3{{xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2]}});
  });
}
void or_pseudo_random_vec(int n, uint64_t seed, double* out) { pseudo_random(n, seed, out); }

static int mesh_resolution(const Mesh& m) {
  // structured cube: (n+1)^3 vertices
  int n = 0;
  while ((n + 1) * (n + 1) * (n + 1) < m.nv()) ++n;
  return n;
}

int or_build_system(const or_mesh* m, double rho, int kind, uint64_t seed, or_system** out) {
  return guard([&] {
    const Target t = make_target(kind, kind == OR_TARGET_SINE_RANDOM ? mesh_resolution(m->m) : 0, seed);
    auto* s = new or_system;
    s->s = build_system(m->m, rho, t);
    *out = s;
  });
}
void or_system_free(or_system* s) { delete s; }
int or_system_n_dofs(const or_system* s) { return s->s.dm.n_dofs(); }
or_csr* or_system_csr(or_system* s, int which) {
  const Csr& c = which == 0 ? s->s.K : which == 1 ? s->s.M : s->s.A;
  s->views[which].a = c;
  return &s->views[which];
}
void or_system_get_f(const or_system* s, double* f) { std::memcpy(f, s->s.f.data(), s->s.f.size() * sizeof(double)); }
void or_system_get_dofmap(const or_system* s, int* v2d, int* d2v) {
  if (v2d) std::memcpy(v2d, s->s.dm.vertex_to_dof.data(), s->s.dm.vertex_to_dof.size() * sizeof(int));
  if (d2v) std::memcpy(d2v, s->s.dm.dof_to_vertex.data(), s->s.dm.dof_to_vertex.size() * sizeof(int));
}
int or_assemble_full(const or_mesh* m, int which, or_csr** out) {
  return guard([&] {
    std::vector<int> rows(static_cast<size_t>(m->m.nv()));
    for (int i = 0; i < m->m.nv(); ++i) rows[static_cast<size_t>(i)] = i;
    *out = new or_csr{assemble_matrix(m->m, rows, rows, which == 0 ? 1.0 : 0.0, which == 1 ? 1.0 : 0.0)};
  });
}
int or_assemble_load(const or_mesh* m, int kind, uint64_t seed, double* f) {
  return guard([&] {
    const Target t = make_target(kind, kind == OR_TARGET_SINE_RANDOM ? mesh_resolution(m->m) : 0, seed);
    const DofMap dm = interior_dof_map(m->m);
    const Vec v = load_vector(m->m, dm, t);
    std::memcpy(f, v.data(), v.size() * sizeof(double));
  });
}

int or_csr_new(int rows, int cols, int64_t nnz, const int* rp, const int* ci, const double* v, or_csr** out) {
  return guard([&] {
    auto* c = new or_csr;
    c->a.rows = rows;
    c->a.cols = cols;
    c->a.rp.assign(rp, rp + rows + 1);
    c->a.ci.assign(ci, ci + nnz);
    c->a.v.assign(v, v + nnz);
    *out = c;
  });
}
int or_from_triplets(int rows, int cols, int64_t n, const int* ti, const int* tj, const double* tv, or_csr** out) {
  return guard([&] {
    *out = new or_csr{from_triplets(rows, cols, std::vector<int>(ti, ti + n), std::vector<int>(tj, tj + n),
                                    std::vector<double>(tv, tv + n))};
  });
}
void or_csr_free(or_csr* a) { delete a; }
void or_csr_info(const or_csr* a, int* rows, int* cols, int64_t* nnz) {
  *rows = a->a.rows;
  *cols = a->a.cols;
  *nnz = a->a.nnz();
}
void or_csr_get(const or_csr* a, int* rp, int* ci, double* v) {
  if (rp) std::memcpy(rp, a->a.rp.data(), a->a.rp.size() * sizeof(int));
  if (ci) std::memcpy(ci, a->a.ci.data(), a->a.ci.size() * sizeof(int));
  if (v) std::memcpy(v, a->a.v.data(), a->a.v.size() * sizeof(double));
}

int or_spmv(const or_csr* a, int nx, const double* x, double* y) {
  return guard([&] {
    const Vec r = spmv(a->a, Vec(x, x + nx));
    std::memcpy(y, r.data(), r.size() * sizeof(double));
  });
}
int or_dense_cholesky_solve(int n, const double* A, const double* b, double* x) {
  return guard([&] {
    const Llt f = llt_compute(n, std::vector<double>(A, A + static_cast<size_t>(n) * n));
    if (!f.ok) throw std::runtime_error("dense_cholesky_solve: matrix not positive definite");
    const Vec r = llt_solve(f, Vec(b, b + n));
    std::memcpy(x, r.data(), r.size() * sizeof(double));
  });
}
double or_dot(int n, const double* a, const double* b) { return eigen_dot(a, b, n); }

int or_coarsen_redblack(const or_csr* a, uint8_t* flags, or_csr** p_out) {
  return guard([&] {
    auto fp = coarsen_redblack(a->a);
    std::memcpy(flags, fp.first.data(), fp.first.size());
    *p_out = new or_csr{std::move(fp.second)};
  });
}
int or_galerkin_coarse(const or_csr* a, const or_csr* p, or_csr** out) {
  return guard([&] { *out = new or_csr{galerkin_coarse(a->a, p->a)}; });
}
int or_sgs_sweep(const or_csr* a, const double* f, const double* u, double* out) {
  return guard([&] {
    const int n = a->a.rows;
    const Vec r = sgs_sweep(a->a, Vec(f, f + n), Vec(u, u + n));
    std::memcpy(out, r.data(), r.size() * sizeof(double));
  });
}
int or_build_amg(const or_csr* a, int thr, int m, or_amg** out) {
  return guard([&] {
    auto* h = new or_amg;
    h->h = build_amg(a->a, thr, m);
    h->views.resize(h->h.levels.size() * 3);
    *out = h;
  });
}
void or_amg_free(or_amg* h) { delete h; }
int or_amg_num_levels(const or_amg* h) { return static_cast<int>(h->h.levels.size()); }
or_csr* or_amg_level_csr(or_amg* h, int level, int which) {
  if (level < 0 || level >= static_cast<int>(h->h.levels.size())) return nullptr;
  const Level& lv = h->h.levels[static_cast<size_t>(level)];
  if (which != 0 && !lv.has_p) return nullptr;
  or_csr* v = &h->views[static_cast<size_t>(level) * 3 + static_cast<size_t>(which)];
  v->a = which == 0 ? lv.A : which == 1 ? lv.P : lv.Pt;
  return v;
}
int or_amg_level_flags(const or_amg* h, int level, uint8_t* flags) {
  const Level& lv = h->h.levels[static_cast<size_t>(level)];
  if (!lv.has_p) return 1;
  std::memcpy(flags, lv.flags.data(), lv.flags.size());
  return 0;
}
int or_amg_apply(const or_amg* h, int n, const double* r, double* z) {
  return guard([&] {
    const Vec out = amg_apply(h->h, Vec(r, r + n));
    std::memcpy(z, out.data(), out.size() * sizeof(double));
  });
}
// the V-cycle entered at `level` (amg.cpp:121-132 recursion from level l): checks the
// coarse tail that rank 0 runs in the distributed solve
int or_amg_apply_from(const or_amg* h, int level, int n, const double* r, double* z) {
  return guard([&] {
    if (level < 0 || (size_t)level >= h->h.levels.size()) throw std::invalid_argument("amg_apply_from: level");
    const Vec out = vcycle(h->h, static_cast<size_t>(level), Vec(r, r + n));
    std::memcpy(z, out.data(), out.size() * sizeof(double));
  });
}

int or_pcg(const or_csr* a, int precond, const or_amg* h, const double* f, double tol, int max_iter, double* x,
           int* iterations, int* converged, double* history) {
  return guard([&] {
    const Csr& A = a->a;
    const int n = A.rows;
    std::function<Vec(const Vec&)> P;
    if (precond == 0) {
      P = [](const Vec& r) { return r; };
    } else if (precond == 1) {
      Vec d(static_cast<size_t>(n), 0.0);
      for (int i = 0; i < n; ++i)
        for (int k = A.rp[static_cast<size_t>(i)]; k < A.rp[static_cast<size_t>(i) + 1]; ++k)
          if (A.ci[static_cast<size_t>(k)] == i) d[static_cast<size_t>(i)] = A.v[static_cast<size_t>(k)];
      for (double v : d)
        if (v <= 0.0) throw std::runtime_error("jacobi_precond: non-positive diagonal");
      P = [d](const Vec& r) {
        Vec z(r.size());
        for (size_t i = 0; i < r.size(); ++i) z[i] = r[i] / d[i];
        return z;
      };
    } else {
      if (!h) throw std::invalid_argument("pcg: amg preconditioner requires a hierarchy");
      P = [h](const Vec& r) { return amg_apply(h->h, r); };
    }
    const PcgOut o = pcg([&A](const Vec& v) { return spmv(A, v); }, P, Vec(f, f + n), tol, max_iter);
    std::memcpy(x, o.x.data(), o.x.size() * sizeof(double));
    *iterations = o.iterations;
    *converged = o.converged ? 1 : 0;
    if (history) std::memcpy(history, o.history.data(), o.history.size() * sizeof(double));
  });
}

int or_solve_system_amg(const or_system* s, double tol, double* u, int* iterations, int* converged,
                        double* setup_seconds, double* solve_seconds) {
  return guard([&] {
    using clk = std::chrono::steady_clock;
    *iterations = 0;
    *converged = 0;
    *setup_seconds = *solve_seconds = 0.0;
    if (s->s.f.empty()) {
      *converged = 1;
      return;
    }
    const auto t0 = clk::now();
    const Amg h = build_amg(s->s.A, 64, 1);
    const auto t1 = clk::now();
    const Csr& A = s->s.A;
    const PcgOut o = pcg([&A](const Vec& v) { return spmv(A, v); }, [&h](const Vec& r) { return amg_apply(h, r); },
                         s->s.f, tol, 500);
    const auto t2 = clk::now();
    std::memcpy(u, o.x.data(), o.x.size() * sizeof(double));
    *iterations = o.iterations;
    *converged = o.converged ? 1 : 0;
    *setup_seconds = std::chrono::duration<double>(t1 - t0).count();
    *solve_seconds = std::chrono::duration<double>(t2 - t1).count();
  });
}

// The whole BASELINE step on the CPU, timed in C++ like bench.cpp:193-224:
// build_structured_cube + build_system [t_build], build_amg [t_setup], pcg [t_solve].
int or_pipeline(int n, double rho, int kind, uint64_t seed, double tol, int* iterations, int* converged,
                int* n_dofs, double* t_build, double* t_setup, double* t_solve) {
  return guard([&] {
    using clk = std::chrono::steady_clock;
    const auto t0 = clk::now();
    const Mesh m = build_structured_cube(n);
    const Target t = make_target(kind, kind == OR_TARGET_SINE_RANDOM ? n : 0, seed);
    const System s = build_system(m, rho, t);
    const auto t1 = clk::now();
    const Amg h = build_amg(s.A, 64, 1);
    const auto t2 = clk::now();
    const Csr& A = s.A;
    const PcgOut o = pcg([&A](const Vec& v) { return spmv(A, v); }, [&h](const Vec& r) { return amg_apply(h, r); },
                         s.f, tol, 500);
    const auto t3 = clk::now();
    *iterations = o.iterations;
    *converged = o.converged ? 1 : 0;
    *n_dofs = s.dm.n_dofs();
    *t_build = std::chrono::duration<double>(t1 - t0).count();
    *t_setup = std::chrono::duration<double>(t2 - t1).count();
    *t_solve = std::chrono::duration<double>(t3 - t2).count();
  });
}

int or_l2_error_manufactured(const or_mesh* m, const or_system* s, const double* coeffs, double rho, double* out) {
  return guard([&] { *out = l2_error(m->m, s->s.dm, coeffs, manufactured_exact(rho)); });
}
int or_target_dual_norm(const or_system* s, const double* coeffs, double* out) {
  return guard([&] { *out = target_dual_norm(s->s, coeffs); });
}
int or_l2_error_target_squared(const or_mesh* m, const or_system* s, const double* coeffs, int kind, int n,
                               uint64_t seed, double* out) {
  return guard([&] { *out = l2_error_target_squared(m->m, s->s.dm, coeffs, make_target(kind, n, seed)); });
}
int or_h1_semi_error_manufactured(const or_mesh* m, const or_system* s, const double* coeffs, double rho,
                                  double* out) {
  return guard([&] { *out = h1_semi_error(m->m, s->s.dm, coeffs, manufactured_exact(rho)); });
}
int or_error_norms_target(const or_mesh* m, const or_system* s, const double* coeffs, int kind, int n,
                          uint64_t seed, double* l2, double* h1) {
  return guard([&] {
    const Target t = make_target(kind, n, seed);
    const TargetExact ex{t};
    if (l2) *l2 = l2_error(m->m, s->s.dm, coeffs, ex);
    if (h1) *h1 = h1_semi_error(m->m, s->s.dm, coeffs, ex);
  });
}
// §8(f)3 -- adaptivity (adapt.hpp, mesh.hpp:40-44)
int or_estimate(const or_mesh* m, const or_system* s, const double* coeffs, int kind, uint64_t seed,
                double* per_tet, double* global) {
  return guard([&] {
    if (kind == OR_TARGET_SINE_RANDOM) throw std::invalid_argument("estimate: the sine+random target needs a lattice");
    const Estimate e = estimate(m->m, s->s.dm, coeffs, s->s.rho, make_target(kind, 0, seed));
    std::memcpy(per_tet, e.per_tet.data(), e.per_tet.size() * sizeof(double));
    *global = e.global;
  });
}
int or_mark_dorfler(int n, const double* eta, double theta, int* marked, int* n_marked) {
  return guard([&] {
    const std::vector<int> mk = mark_dorfler(Vec(eta, eta + n), theta);
    std::memcpy(marked, mk.data(), mk.size() * sizeof(int));
    *n_marked = static_cast<int>(mk.size());
  });
}
int or_bisect_marked(const or_mesh* m, int n_marked, const int* marked, or_mesh** out) {
  return guard([&] { *out = new or_mesh{bisect_marked(m->m, std::vector<int>(marked, marked + n_marked))}; });
}
int or_uniform_refine(const or_mesh* m, or_mesh** out) {
  return guard([&] { *out = new or_mesh{uniform_refine(m->m)}; });
}
/* history rows: level, dofs, iterations (int[3]) and eta, err_l2_sq, err_hm1_sq (double[3]) */
int or_adaptive_solve(const or_mesh* initial, int kind, uint64_t seed, double rho, int dof_budget, double tol,
                      double theta, int cap, int* n_levels, int* hist_i, double* hist_d, or_mesh** final_mesh,
                      double* coeffs, int coeffs_cap) {
  return guard([&] {
    if (kind == OR_TARGET_SINE_RANDOM) throw std::invalid_argument("adaptive_solve: the sine+random target needs a lattice");
    Mesh fm;
    Vec fc;
    const auto h = adaptive_solve(initial->m, make_target(kind, 0, seed), rho, dof_budget, tol, theta, &fm, &fc);
    *n_levels = static_cast<int>(h.size());
    for (int k = 0; k < static_cast<int>(h.size()) && k < cap; ++k) {
      hist_i[3 * k] = h[static_cast<size_t>(k)].level;
      hist_i[3 * k + 1] = h[static_cast<size_t>(k)].dofs;
      hist_i[3 * k + 2] = h[static_cast<size_t>(k)].iterations;
      hist_d[3 * k] = h[static_cast<size_t>(k)].eta;
      hist_d[3 * k + 1] = h[static_cast<size_t>(k)].err_l2_sq;
      hist_d[3 * k + 2] = h[static_cast<size_t>(k)].err_hm1_sq;
    }
    if (coeffs && static_cast<int>(fc.size()) <= coeffs_cap) std::memcpy(coeffs, fc.data(), fc.size() * sizeof(double));
    if (final_mesh) *final_mesh = new or_mesh{std::move(fm)};
  });
}

// §8(f)4 BDDC (bddc.hpp)
int or_partition_geometric(const or_mesh* m, const or_system* s, int p, int* owner, int* n_subdomains_per_dof,
                           int* subdomains /* n_dofs * 8 */) {
  return guard([&] {
    const Partition part = partition_geometric(m->m, s->s.dm, p);
    std::memcpy(owner, part.owner.data(), part.owner.size() * sizeof(int));
    for (size_t d = 0; d < part.dof_subdomains.size(); ++d) {
      const auto& ss = part.dof_subdomains[d];
      n_subdomains_per_dof[d] = static_cast<int>(ss.size());
      for (size_t k = 0; k < ss.size() && k < 8; ++k) subdomains[8 * d + k] = ss[k];
    }
  });
}
int or_bddc_create(const or_mesh* m, const or_system* s, int p, or_bddc** out) {
  return guard([&] {
    const Partition part = partition_geometric(m->m, s->s.dm, p);
    *out = new or_bddc{build_bddc(m->m, s->s, part)};
  });
}
void or_bddc_free(or_bddc* b) { delete b; }
void or_bddc_info(const or_bddc* b, int* n_interface, int* n_primal, int* p) {
  *n_interface = static_cast<int>(b->op.interface_dofs.size());
  *n_primal = b->op.n_primal;
  *p = b->op.part.p;
}
void or_bddc_interface(const or_bddc* b, int* dofs) {
  std::memcpy(dofs, b->op.interface_dofs.data(), b->op.interface_dofs.size() * sizeof(int));
}
void or_bddc_coarse(const or_bddc* b, double* out) {
  std::memcpy(out, b->op.coarse.data(), b->op.coarse.size() * sizeof(double));
}
void or_bddc_sub_info(const or_bddc* b, int s, int* nI, int* nB, int* ncon) {
  const auto& sd = b->op.subs[static_cast<size_t>(s)];
  *nI = sd.nI;
  *nB = sd.nB;
  *ncon = sd.ncon;
}
/* boundary dofs, boundary_index, primal_index (int), scaling (nB), C (ncon x nB), Phi (nB x ncon), S (nB x nB) */
void or_bddc_sub_get(const or_bddc* b, int s, int* boundary, int* bidx, int* pidx, double* scaling, double* C,
                     double* Phi, double* S) {
  const auto& sd = b->op.subs[static_cast<size_t>(s)];
  if (boundary) std::memcpy(boundary, sd.boundary.data(), sd.boundary.size() * sizeof(int));
  if (bidx) std::memcpy(bidx, sd.boundary_index.data(), sd.boundary_index.size() * sizeof(int));
  if (pidx) std::memcpy(pidx, sd.primal_index.data(), sd.primal_index.size() * sizeof(int));
  if (scaling) std::memcpy(scaling, sd.scaling.data(), sd.scaling.size() * sizeof(double));
  if (C) std::memcpy(C, sd.C.data(), sd.C.size() * sizeof(double));
  if (Phi) std::memcpy(Phi, sd.Phi.data(), sd.Phi.size() * sizeof(double));
  if (S) std::memcpy(S, sd.S.data(), sd.S.size() * sizeof(double));
}
int or_bddc_op(const or_bddc* b, int which, int n_in, const double* in, const double* f, double* out) {
  return guard([&] {
    const Vec x(in, in + n_in);
    Vec y;
    switch (which) {
      case 0: y = schur_apply(b->op, x); break;
      case 1: y = reduce_rhs(b->op, x); break;
      case 2: y = expand_solution(b->op, x, Vec(f, f + b->op.interface_index.size())); break;
      case 3: y = bddc_apply(b->op, x); break;
      default: throw std::invalid_argument("or_bddc_op: which");
    }
    std::memcpy(out, y.data(), y.size() * sizeof(double));
  });
}
/* bddc.cpp:440-456 bddc_solve */
int or_bddc_solve(const or_mesh* m, const or_system* s, int p, double tol, int max_iter, double* u, int* iterations,
                  int* converged, double* history) {
  return guard([&] {
    const Partition part = partition_geometric(m->m, s->s.dm, p);
    const Bddc op = build_bddc(m->m, s->s, part);
    const Vec g = reduce_rhs(op, s->s.f);
    const PcgOut o = pcg([&op](const Vec& x) { return schur_apply(op, x); },
                         [&op](const Vec& r) { return bddc_apply(op, r); }, g, tol, max_iter);
    const Vec uu = expand_solution(op, o.x, s->s.f);
    std::memcpy(u, uu.data(), uu.size() * sizeof(double));
    *iterations = o.iterations;
    *converged = o.converged ? 1 : 0;
    if (history) std::memcpy(history, o.history.data(), o.history.size() * sizeof(double));
  });
}

int or_target_grad(int kind, int n, uint64_t seed, int npts, const double* xyz, double* g) {
  return guard([&] {
    const Target t = make_target(kind, n, seed);
    for (int i = 0; i < npts; ++i) t.grad(V3{{xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2]}}, g + 3 * i);
  });
}

}  // extern "C"
