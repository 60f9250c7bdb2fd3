// Host setup for the B200 path. See setup.hpp. Reference counterparts:
// sphere_mesh.cpp (tree, refinement, two-irregular closure, coarsening),
// quadrature.cpp (Duffy-collapsed Gauss rule), angular_disc.cpp:40-59
// (Const patch mass / Jacobians), scatter.cpp:33-99 (harmonics, couplings),
// spatial_disc.cpp:45-88 (element matrices; 2D bilinear here),
// transport.cpp:23-64 (fused blocks), sweeps.cpp:61-72 (GS blocks),
// multigrid.cpp:51-98 (hierarchy), transport.cpp:110-179 (rhs).
#include "setup.hpp"

#include <algorithm>
#include <cmath>
#include <map>
#include <numbers>
#include <stdexcept>
#include <unordered_map>

namespace stamg_b200 {

namespace {

constexpr double kPi = std::numbers::pi;

void normalize3(const std::int64_t* f, double* out) {
  const double x = double(f[0]), y = double(f[1]), z = double(f[2]);
  const double inv = 1.0 / std::sqrt(x * x + y * y + z * z);
  out[0] = x * inv, out[1] = y * inv, out[2] = z * inv;
}

// Segment key of one atomic edge piece: endpoints in lexicographic order.
struct Seg {
  std::array<std::int64_t, 6> k;
  bool operator==(const Seg&) const = default;
};
struct SegHash {  // same mixing as the reference table so the split order matches
  std::size_t operator()(const Seg& s) const {
    std::size_t h = 0xcbf29ce484222325ull;
    for (std::int64_t x : s.k) h ^= std::size_t(x) + 0x9e3779b97f4a7c15ull + (h << 6) + (h >> 2);
    return h;
  }
};

}  // namespace

void SphereTree::add(int lvl, int oct, int par, const std::int64_t* a, const std::int64_t* b,
                     const std::int64_t* c) {
  level.push_back(lvl);
  octant.push_back(oct);
  parent.push_back(par);
  kids.push_back({-1, -1, -1, -1});
  leaf.push_back(1);
  std::array<std::int64_t, 9> f{a[0], a[1], a[2], b[0], b[1], b[2], c[0], c[1], c[2]};
  flat.push_back(f);
  std::array<double, 9> u{};
  for (int v = 0; v < 3; ++v) normalize3(&f[3 * v], &u[3 * v]);
  unit.push_back(u);
}

// 1 -> 4 split on the lattice; daughters (a,mab,mca), (mab,b,mbc),
// (mca,mbc,c), (mab,mbc,mca) as sphere_mesh.cpp:44-58.
void SphereTree::split(int id) {
  if (!leaf[id]) throw std::invalid_argument("refine: patch is not a leaf");
  const auto f = flat[id];
  std::int64_t m[3][3];
  for (int r = 0; r < 3; ++r) {
    m[0][r] = (f[0 + r] + f[3 + r]) / 2;  // ab
    m[1][r] = (f[3 + r] + f[6 + r]) / 2;  // bc
    m[2][r] = (f[6 + r] + f[0 + r]) / 2;  // ca
  }
  const int base = size(), lvl = level[id] + 1, oct = octant[id];
  leaf[id] = 0;
  kids[id] = {base, base + 1, base + 2, base + 3};
  add(lvl, oct, id, &f[0], m[0], m[2]);
  add(lvl, oct, id, m[0], &f[3], m[1]);
  add(lvl, oct, id, m[2], m[1], &f[6]);
  add(lvl, oct, id, m[0], m[1], m[2]);
  max_level = std::max(max_level, lvl);
}

void SphereTree::relist() {
  leaves.clear();
  max_level = 0;
  for (int id = 0; id < size(); ++id)
    if (leaf[id]) leaves.push_back(id), max_level = std::max(max_level, level[id]);
}

// Repeatedly split the coarser side of any edge shared by leaves more than two
// levels apart (sphere_mesh.cpp:82-120).
void SphereTree::close_two_irregular() {
  for (bool again = true; again;) {
    again = false;
    relist();
    std::unordered_map<Seg, std::array<int, 2>, SegHash> segs;
    segs.reserve(leaves.size() * 6);
    for (int id : leaves) {
      const std::int64_t pieces = std::int64_t(1) << (max_level - level[id]);
      const auto& f = flat[id];
      for (int e = 0; e < 3; ++e) {
        const std::int64_t* u = &f[3 * e];
        const std::int64_t* v = &f[3 * ((e + 1) % 3)];
        std::int64_t step[3];
        for (int r = 0; r < 3; ++r) step[r] = (v[r] - u[r]) / pieces;
        for (std::int64_t t = 0; t < pieces; ++t) {
          std::array<std::int64_t, 3> p0{u[0] + step[0] * t, u[1] + step[1] * t, u[2] + step[2] * t};
          std::array<std::int64_t, 3> p1{p0[0] + step[0], p0[1] + step[1], p0[2] + step[2]};
          if (p1 < p0) std::swap(p0, p1);
          Seg s{{p0[0], p0[1], p0[2], p1[0], p1[1], p1[2]}};
          auto [it, fresh] = segs.try_emplace(s, std::array<int, 2>{id, -1});
          if (!fresh) it->second[1] = id;
        }
      }
    }
    for (const auto& [s, pr] : segs) {
      if (pr[1] < 0) continue;
      if (std::abs(level[pr[0]] - level[pr[1]]) > 2) {
        split(level[pr[0]] < level[pr[1]] ? pr[0] : pr[1]);
        again = true;
        break;
      }
    }
  }
  relist();
}

bool in_cone(const SphereTree& t, int id, double half_angle_deg) {
  const auto& u = t.unit[id];
  double c[3] = {u[0] + u[3] + u[6], u[1] + u[4] + u[7], u[2] + u[5] + u[8]};
  const double n = std::sqrt(c[0] * c[0] + c[1] * c[1] + c[2] * c[2]);
  return c[0] / n >= std::cos(half_angle_deg * kPi / 180.0);
}

SphereTree make_sphere(int kind, int level, int extra, double cone_half_angle_deg) {
  if (level < 0) throw std::invalid_argument("angular level < 0");
  SphereTree t;
  const std::int64_t S = SphereTree::kScale;
  for (int oct = 0; oct < 8; ++oct) {  // octahedron faces (sphere_mesh.cpp:141-153)
    const std::int64_t sx = (oct & 1) ? -1 : 1, sy = (oct & 2) ? -1 : 1, sz = (oct & 4) ? -1 : 1;
    std::int64_t a[3] = {sx * S, 0, 0}, b[3] = {0, sy * S, 0}, c[3] = {0, 0, sz * S};
    if (sx * sy * sz < 0) t.add(0, oct, -1, a, c, b);
    else t.add(0, oct, -1, a, b, c);
  }
  t.relist();
  if (kind == 0 || kind == 2) {
    for (int l = 0; l < level; ++l) {
      const std::vector<int> cur = t.leaves;
      for (int id : cur) t.split(id);
      t.relist();
    }
    if (kind == 2) {  // cone refinement around +x (EXTENSION for config 4)
      for (int e = 0; e < extra; ++e) {
        const std::vector<int> cur = t.leaves;
        for (int id : cur)
          if (t.level[id] == level + e && in_cone(t, id, cone_half_angle_deg)) t.split(id);
        t.relist();
      }
      t.close_two_irregular();
    }
    return t;
  }
  if (kind == 1) {  // polar band (sphere_mesh.cpp:122-131,173-189)
    if (level < 1) throw std::invalid_argument("build_banded_mesh: l_max < 1");
    auto target = [&](int id) {
      const auto& u = t.unit[id];
      const double z = std::max({u[2], u[5], u[8]});
      const int tl = z > 0.9875 ? level : z > 0.9 ? level - 1 : z > 0.8 ? level - 2 : z > 0.6 ? level - 3 : level - 4;
      return std::max(tl, 0);
    };
    for (bool changed = true; changed;) {
      changed = false;
      const std::vector<int> cur = t.leaves;
      for (int id : cur)
        if (t.level[id] < target(id)) t.split(id), changed = true;
      t.relist();
    }
    t.close_two_irregular();
    return t;
  }
  throw std::invalid_argument("unknown angular mesh kind");
}

SphereTree coarsen(const SphereTree& t, int level) {  // sphere_mesh.cpp:191-203
  SphereTree out = t;
  if (level >= t.max_level) return out;
  std::fill(out.leaf.begin(), out.leaf.end(), 0);
  for (int id : t.leaves) {
    int a = id;
    while (out.level[a] > level) a = out.parent[a];
    out.leaf[a] = 1;
  }
  out.relist();
  return out;
}

// ------------------------------------------------------------ quadrature
namespace {

struct Rule1D {
  std::vector<double> x, w;
};

const Rule1D& gauss01(int n) {  // Newton on P_n, mapped to [0,1] (quadrature.cpp:13-57)
  static std::map<int, Rule1D> cache;
  auto it = cache.find(n);
  if (it != cache.end()) return it->second;
  Rule1D r;
  r.x.resize(n);
  r.w.resize(n);
  auto legendre = [n](double t, double& pn, double& pn1) {
    double a = 1.0, b = t;
    for (int k = 2; k <= n; ++k) {
      const double c = ((2 * k - 1) * t * b - (k - 1) * a) / k;
      a = b, b = c;
    }
    pn = b, pn1 = a;
  };
  for (int i = 0; i < n; ++i) {
    double t = std::cos(kPi * (i + 0.75) / (n + 0.5));
    double pn = 0, pn1 = 0;
    for (int it2 = 0; it2 < 100; ++it2) {
      legendre(t, pn, pn1);
      const double dp = n * (t * pn - pn1) / (t * t - 1.0);
      const double dt = pn / dp;
      t -= dt;
      if (std::abs(dt) < 1e-15) break;
    }
    legendre(t, pn, pn1);
    const double dp = n * (t * pn - pn1) / (t * t - 1.0);
    r.x[i] = 0.5 * (1.0 - t);
    r.w[i] = 1.0 / ((1.0 - t * t) * dp * dp);
  }
  return cache.emplace(n, std::move(r)).first->second;
}


// Visit every node of the Duffy-collapsed rule of one patch
// (quadrature.cpp:59-92): f(unit direction, weight).
template <class F>
void for_each_node(const SphereTree& t, int id, int order, F&& f) {
  const Rule1D& g = gauss01(order);
  const double inv = 1.0 / double(SphereTree::kScale);
  double a[3], b[3], c[3];
  for (int r = 0; r < 3; ++r)
    a[r] = double(t.flat[id][r]) * inv, b[r] = double(t.flat[id][3 + r]) * inv, c[r] = double(t.flat[id][6 + r]) * inv;
  const double e1[3] = {b[0] - a[0], b[1] - a[1], b[2] - a[2]}, e2[3] = {c[0] - a[0], c[1] - a[1], c[2] - a[2]};
  const double cr[3] = {e1[1] * e2[2] - e1[2] * e2[1], e1[2] * e2[0] - e1[0] * e2[2], e1[0] * e2[1] - e1[1] * e2[0]};
  const double two_area = std::sqrt(cr[0] * cr[0] + cr[1] * cr[1] + cr[2] * cr[2]);
  const double hplane = (a[0] * cr[0] + a[1] * cr[1] + a[2] * cr[2]) / two_area;
  for (int iu = 0; iu < order; ++iu) {
    const double u = g.x[iu];
    for (int iv = 0; iv < order; ++iv) {
      const double v = g.x[iv];
      double x[3];
      for (int r = 0; r < 3; ++r) x[r] = (1.0 - u) * a[r] + u * ((1.0 - v) * b[r] + v * c[r]);
      const double rr = std::sqrt(x[0] * x[0] + x[1] * x[1] + x[2] * x[2]);
      const double w = g.w[iu] * g.w[iv] * u * two_area * hplane / (rr * rr * rr);
      const double om[3] = {x[0] / rr, x[1] / rr, x[2] / rr};
      f(om, w);
    }
  }
}

}  // namespace

// The same rule with its flat-triangle barycentric coordinates (1-u, u(1-v), uv), the nodal
// Lin basis of angular_disc.cpp:40-59 (quadrature.cpp:84).
void patch_rule(const SphereTree& t, int id, int order, std::vector<double>& om, std::vector<double>& bary,
                std::vector<double>& w) {
  const Rule1D& g = gauss01(order);
  om.clear(), bary.clear(), w.clear();
  for_each_node(t, id, order, [&](const double* o, double wt) {
    om.insert(om.end(), o, o + 3);
    w.push_back(wt);
  });
  for (int iu = 0; iu < order; ++iu)
    for (int iv = 0; iv < order; ++iv) {
      const double u = g.x[iu], v = g.x[iv];
      bary.push_back(1.0 - u), bary.push_back(u * (1.0 - v)), bary.push_back(u * v);
    }
}

int patch_order(int level, int base) {  // quadrature.hpp:31-34
  const int bump = level == 0 ? 20 : level == 1 ? 12 : 8;
  return std::max(base, bump);
}

void gauss_rule01(int n, const double** x, const double** w) {
  const Rule1D& r = gauss01(n);
  *x = r.x.data(), *w = r.w.data();
}

namespace {

// Real orthonormal spherical harmonics up to degree N, h = n^2 + n + o
// (associated-Legendre recurrence along each order m; scatter.cpp:33-65).
void harmonics(int N, const double* om, double* out) {
  const double z = om[2];
  const double rxy = std::hypot(om[0], om[1]);
  const double phi = std::atan2(om[1], om[0]);
  double pmm = 1.0 / std::sqrt(4.0 * kPi);
  for (int m = 0; m <= N; ++m) {
    const double cm = m == 0 ? 1.0 : std::numbers::sqrt2 * std::cos(m * phi);
    const double sm = m == 0 ? 0.0 : std::numbers::sqrt2 * std::sin(m * phi);
    double prev = 0.0, cur = pmm;
    for (int n = m; n <= N; ++n) {
      const int base = n * n + n;
      out[base + m] = cm * cur;
      if (m > 0) out[base - m] = sm * cur;
      if (n < N) {
        const double nn = n + 1;
        const double ca = std::sqrt((4.0 * nn * nn - 1.0) / (nn * nn - double(m) * m));
        const double cb = std::sqrt(((nn - 1) * (nn - 1) - double(m) * m) / (4.0 * (nn - 1) * (nn - 1) - 1.0));
        const double next = ca * (z * cur - cb * prev);
        prev = cur, cur = next;
      }
    }
    if (m < N) pmm *= -std::sqrt((2.0 * m + 3.0) / (2.0 * m + 2.0)) * rxy;
  }
}

// 4x4 products of the 2x2 Kronecker factors, dof i = ix + 2*iy
inline double kron22(const double* A, const double* B, int r, int c) {
  return A[(r >> 1) * 2 + (c >> 1)] * B[(r & 1) * 2 + (c & 1)];
}

}  // namespace

void real_harmonics(int N, const double* om, double* out) { harmonics(N, om, out); }

void inverse4(const double* A, double* Ainv) {  // partial-pivot Gauss-Jordan
  double m[4][8];
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < 8; ++j) m[i][j] = j < 4 ? A[i * 4 + j] : (j - 4 == i ? 1.0 : 0.0);
  for (int k = 0; k < 4; ++k) {
    int p = k;
    for (int i = k + 1; i < 4; ++i)
      if (std::abs(m[i][k]) > std::abs(m[p][k])) p = i;
    if (m[p][k] == 0.0) throw std::invalid_argument("singular diagonal block");
    if (p != k)
      for (int j = 0; j < 8; ++j) std::swap(m[k][j], m[p][j]);
    const double d = 1.0 / m[k][k];
    for (int j = 0; j < 8; ++j) m[k][j] *= d;
    for (int i = 0; i < 4; ++i)
      if (i != k) {
        const double f = m[i][k];
        for (int j = 0; j < 8; ++j) m[i][j] -= f * m[k][j];
      }
  }
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < 4; ++j) Ainv[i * 4 + j] = m[i][4 + j];
}

Problem copy_problem(const stamg_problem& s) {
  Problem p;
  p.spec = s;
  if (s.n_mat < 1 || !s.sigma_t || !s.moments) throw std::invalid_argument("problem: no materials");
  p.sigma_t.assign(s.sigma_t, s.sigma_t + s.n_mat);
  p.moments.assign(s.moments, s.moments + size_t(s.n_mat) * (s.N + 1));
  p.n_el = s.nx * s.ny * (s.dim == 3 ? s.nz : 1);
  if (s.mat_of_el) p.mat.assign(s.mat_of_el, s.mat_of_el + p.n_el);
  else p.mat.assign(p.n_el, 0);
  if (s.q_el) p.q_el.assign(s.q_el, s.q_el + p.n_el);
  p.h = s.box / s.nx;
  p.spec.sigma_t = nullptr, p.spec.moments = nullptr, p.spec.mat_of_el = nullptr, p.spec.q_el = nullptr;
  return p;
}

void validate(const Problem& p) {
  const auto& s = p.spec;
  if (s.dim != 2) throw std::invalid_argument("B200 path supports dim = 2 only");
  if (s.basis != 0 || s.p != 1) throw std::invalid_argument("B200 path supports the Const basis with bilinear cells only");
  if (s.nx < 1 || s.ny < 1) throw std::invalid_argument("build_hex_mesh: zero element count");
  if (s.box <= 0) throw std::invalid_argument("build_hex_mesh: box must be positive");
  if (s.nx != s.ny) throw std::invalid_argument("B200 path expects a square grid (nx == ny)");
  if (s.N < 0) throw std::invalid_argument("scatter order < 0");
  if (s.nr > s.N) throw std::invalid_argument("build_hierarchy: nr exceeds N");
  for (int m : p.mat)
    if (m < 0 || m >= s.n_mat) throw std::invalid_argument("build_operators: bad material id");
  if (s.beam != 0 && s.beam != 2) throw std::invalid_argument("B200 path supports beam = 0 or 2 (x=0 cone)");
}

std::vector<int> range_subset(int q_begin, int q_end) {
  std::vector<int> v;
  for (int q = q_begin; q < q_end; ++q) v.push_back(q);
  return v;
}

LevelTables build_level(const Problem& pb, const SphereTree& t, int order, bool with_gs, const std::vector<int>* subset) {
  LevelTables L;
  const auto& s = pb.spec;
  const int Pg = int(t.leaves.size());
  if (subset) {
    for (size_t k = 0; k < subset->size(); ++k)
      if ((*subset)[k] < 0 || (*subset)[k] >= Pg || (k && (*subset)[k] <= (*subset)[k - 1]))
        throw std::invalid_argument("build_level: bad patch subset");
    L.qpos = *subset;
  } else {
    L.qpos = range_subset(0, Pg);
  }
  L.P_global = Pg, L.q_begin = L.qpos.empty() ? 0 : L.qpos[0];
  L.n_el = pb.n_el, L.P = int(L.qpos.size()), L.order = order, L.H = (order + 1) * (order + 1);
  L.n_mat = s.n_mat, L.nx = s.nx, L.ny = s.ny;
  const int P = L.P, H = L.H;
  const double hx = s.box / s.nx, hy = s.box / s.ny;
  // spatial factors (spatial_disc.cpp:11-15,62-69)
  const double mx[4] = {2 * hx / 6, hx / 6, hx / 6, 2 * hx / 6}, my[4] = {2 * hy / 6, hy / 6, hy / 6, 2 * hy / 6};
  const double g[4] = {-0.5, -0.5, 0.5, 0.5};
  const double t_lo[4] = {1, 0, 0, 0}, t_hi[4] = {0, 0, 0, 1}, c_lo[4] = {0, 1, 0, 0}, c_hi[4] = {0, 0, 1, 0};
  double Nm[16], V[2][16], Fs[4][16], Fn[4][16];
  for (int r = 0; r < 4; ++r)
    for (int c = 0; c < 4; ++c) {
      const int k = r * 4 + c;
      Nm[k] = kron22(my, mx, r, c);
      V[0][k] = kron22(my, g, r, c), V[1][k] = kron22(g, mx, r, c);
      Fs[0][k] = kron22(my, t_lo, r, c), Fs[1][k] = kron22(my, t_hi, r, c);
      Fs[2][k] = kron22(t_lo, mx, r, c), Fs[3][k] = kron22(t_hi, mx, r, c);
      Fn[0][k] = kron22(my, c_lo, r, c), Fn[1][k] = kron22(my, c_hi, r, c);
      Fn[2][k] = kron22(c_lo, mx, r, c), Fn[3][k] = kron22(c_hi, mx, r, c);
    }
  std::copy(Nm, Nm + 16, L.Nmat);

  L.leaf_id.resize(L.P);
  for (int q = 0; q < L.P; ++q) L.leaf_id[q] = t.leaves[L.qpos[q]];
  L.octant.resize(P);
  L.area.resize(P);
  L.Aflow.resize(size_t(P) * 3);
  L.X.assign(size_t(P) * H, 0.0);
  L.sig.assign(size_t(L.n_mat) * H, 0.0);
  for (int m = 0; m < L.n_mat; ++m)
    for (int n = 0; n <= order; ++n)
      for (int o = -n; o <= n; ++o) L.sig[size_t(m) * H + n * n + n + o] = pb.moments[size_t(m) * (s.N + 1) + n];
  L.B.resize(size_t(L.n_mat) * P * 16);
  L.Binv.resize(size_t(L.n_mat) * P * 16);
  L.C.resize(size_t(P) * 32);
  L.cxy.resize(size_t(P) * 8);
  const int xorder_base = order > 12 ? 12 : 8;  // scatter.hpp:42
  std::vector<double> Y(H);
  // the couplings are ~all of the setup time (1e9 harmonic evaluations at config 5): on the device
  const bool device_X = pb.device_setup && device_couplings_supported(order);
  if (device_X) device_couplings(t, L.leaf_id, order, xorder_base, L.X.data());
  for (int q = 0; q < P; ++q) L.octant[q] = t.octant[L.leaf_id[q]];
  // operator blocks on the device too (build_operators, transport.cpp:43-57); the host loop below
  // is the STAMG_HOST_SETUP=1 path and the test oracle for the kernel
  const bool device_blocks = pb.device_setup;
  if (device_blocks) {
    double el16[176];
    std::copy(Nm, Nm + 16, el16);
    std::copy(&V[0][0], &V[0][0] + 32, el16 + 16);
    std::copy(&Fs[0][0], &Fs[0][0] + 64, el16 + 48);
    std::copy(&Fn[0][0], &Fn[0][0] + 64, el16 + 112);
    device_patch_blocks(t, L.leaf_id, pb.sigma_t, el16, L.area.data(), L.Aflow.data(), L.B.data(), L.Binv.data(),
                        L.C.data(), L.cxy.data());
  }
  for (int q = 0; q < P && !(device_blocks && device_X); ++q) {
    const int id = L.leaf_id[q];
    L.octant[q] = t.octant[id];
    // Const patch operators: M = sum w, A^xi = sum w Omega_xi (angular_disc.cpp:40-59)
    double M = 0, A[3] = {0, 0, 0};
    for_each_node(t, id, patch_order(t.level[id], 8), [&](const double* om, double w) {
      M += w;
      for (int xi = 0; xi < 3; ++xi) A[xi] += om[xi] * w;
    });
    L.area[q] = M;
    for (int xi = 0; xi < 3; ++xi) L.Aflow[q * 3 + xi] = A[xi];
    // couplings X_q(h) = int_patch Y_h (scatter.cpp:74-99)
    if (!device_X) {
      double* Xq = &L.X[size_t(q) * H];
      for_each_node(t, id, patch_order(t.level[id], xorder_base), [&](const double* om, double w) {
        harmonics(order, om, Y.data());
        for (int h = 0; h < H; ++h) Xq[h] += w * Y[h];
      });
    }
    // fused blocks (transport.cpp:46-56)
    const int oct = t.octant[id];
    double sgn[2], Cq[2][16];
    int fin[2], fout[2];
    for (int xi = 0; xi < 2; ++xi) {
      sgn[xi] = (oct >> xi) & 1 ? -1.0 : 1.0;
      fout[xi] = 2 * xi + (sgn[xi] > 0 ? 1 : 0);
      fin[xi] = 2 * xi + (sgn[xi] > 0 ? 0 : 1);
      for (int k = 0; k < 16; ++k) Cq[xi][k] = -sgn[xi] * (A[xi] * Fn[fin[xi]][k]);
    }
    for (int m = 0; m < L.n_mat; ++m) {
      double* B = &L.B[(size_t(m) * P + q) * 16];
      for (int k = 0; k < 16; ++k) B[k] = pb.sigma_t[m] * (M * Nm[k]);
      for (int xi = 0; xi < 2; ++xi)
        for (int k = 0; k < 16; ++k) {
          B[k] += -1.0 * (A[xi] * V[xi][k]);
          B[k] += sgn[xi] * (A[xi] * Fs[fout[xi]][k]);
        }
      inverse4(B, &L.Binv[(size_t(m) * P + q) * 16]);
    }
    for (int xi = 0; xi < 2; ++xi) std::copy(Cq[xi], Cq[xi] + 16, &L.C[size_t(q) * 32 + xi * 16]);
    // nonzero 2x2 sub-blocks: rows = inflow-face dofs, cols = upwind trace dofs
    const int ix_in = sgn[0] > 0 ? 0 : 1, jx = 1 - ix_in;
    const int iy_in = sgn[1] > 0 ? 0 : 1, jy = 1 - iy_in;
    double* cxy = &L.cxy[size_t(q) * 8];
    for (int a = 0; a < 2; ++a)
      for (int b = 0; b < 2; ++b) {
        cxy[a * 2 + b] = Cq[0][(ix_in + 2 * a) * 4 + (jx + 2 * b)];
        cxy[4 + a * 2 + b] = Cq[1][(2 * iy_in + a) * 4 + (2 * jy + b)];
      }
  }
  // sweep plan: patches per octant (sweeps.cpp:14) and groups of 4 equal-octant patches
  L.oct_ptr.assign(9, 0);
  for (int oct = 0; oct < 8; ++oct) {
    L.oct_ptr[oct] = int(L.oct_patches.size());
    std::vector<int> mine;
    for (int q = 0; q < P; ++q)
      if (L.octant[q] == oct) mine.push_back(q);
    L.oct_patches.insert(L.oct_patches.end(), mine.begin(), mine.end());
    for (size_t k = 0; k < mine.size(); k += 4) {
      for (int j = 0; j < 4; ++j) L.groups.push_back(k + j < mine.size() ? mine[k + j] : -1);
      L.group_oct.push_back(oct);
    }
  }
  L.oct_ptr[8] = int(L.oct_patches.size());
  // 8-direction groups; an octant whose count is not a multiple of 8 (the config-4 cone
  // mesh: 466 = 58*8 + 2) ends with a padded group (-1 lanes idle)
  L.groups8_padded = false;
  for (int oct = 0; oct < 8; ++oct)
    for (int k = L.oct_ptr[oct]; k < L.oct_ptr[oct + 1]; k += 8) {
      for (int j = 0; j < 8; ++j) {
        const bool in = k + j < L.oct_ptr[oct + 1];
        L.groups8.push_back(in ? L.oct_patches[k + j] : -1);
        L.groups8_padded = L.groups8_padded || !in;
      }
      L.group8_oct.push_back(oct);
    }
  if (with_gs) {  // scatter-implicit blocks of the coarse solver (sweeps.cpp:60-72)
    L.sq.resize(size_t(L.n_mat) * P);
    L.BinvGS.resize(size_t(L.n_mat) * P * 16);
    for (int m = 0; m < L.n_mat; ++m)
      for (int q = 0; q < P; ++q) {
        double sq = 0;
        const double* Xq = &L.X[size_t(q) * H];
        for (int h = 0; h < H; ++h) sq += Xq[h] * L.sig[size_t(m) * H + h] * Xq[h];
        L.sq[size_t(m) * P + q] = sq;
        double Bp[16];
        const double* B = &L.B[(size_t(m) * P + q) * 16];
        for (int k = 0; k < 16; ++k) Bp[k] = B[k] - sq * Nm[k];
        inverse4(Bp, &L.BinvGS[(size_t(m) * P + q) * 16]);
      }
  }
  find_symmetry(L, t);
  return L;
}

// Reflections (axis-aligned mirror maps) that map the leaf set of `t` onto itself:
// per symmetric axis the leaf position of each leaf's mirror image. With `only`
// non-empty, just those axes are tried.
void leaf_mirrors(const SphereTree& t, std::vector<int>& axes, std::vector<std::vector<int>>& mirror,
                  const std::vector<int>& only) {
  const int Pg = int(t.leaves.size());
  using Key = std::array<std::int64_t, 9>;
  auto key_of = [](std::array<std::int64_t, 9> f) {
    std::array<std::array<std::int64_t, 3>, 3> v{{{f[0], f[1], f[2]}, {f[3], f[4], f[5]}, {f[6], f[7], f[8]}}};
    std::sort(v.begin(), v.end());
    Key k;
    for (int i = 0; i < 3; ++i)
      for (int r = 0; r < 3; ++r) k[3 * i + r] = v[i][r];
    return k;
  };
  std::map<Key, int> pos;
  for (int q = 0; q < Pg; ++q) pos[key_of(t.flat[t.leaves[q]])] = q;
  axes.clear(), mirror.clear();
  for (int axis = 0; axis < 3; ++axis) {
    if (!only.empty() && std::find(only.begin(), only.end(), axis) == only.end()) continue;
    std::vector<int> mq(Pg, -1);
    bool ok = true;
    for (int q = 0; ok && q < Pg; ++q) {
      auto f = t.flat[t.leaves[q]];
      for (int v = 0; v < 3; ++v) f[3 * v + axis] = -f[3 * v + axis];
      auto it = pos.find(key_of(f));
      if (it == pos.end()) ok = false;
      else mq[q] = it->second;
    }
    if (ok) axes.push_back(axis), mirror.push_back(mq);
  }
}

std::vector<int> throughput_shard(const SphereTree& t, int rank, int world) {
  const int Pg = int(t.leaves.size());
  std::vector<int> axes;
  std::vector<std::vector<int>> mirror;
  leaf_mirrors(t, axes, mirror, {});
  std::vector<int> reps;  // orbit representatives: octant bits 0 on every symmetric axis
  for (int q = 0; q < Pg; ++q) {
    bool rep = true;
    for (int axis : axes)
      if ((t.octant[t.leaves[q]] >> axis) & 1) rep = false;
    if (rep) reps.push_back(q);
  }
  const int G = 1 << int(axes.size());
  if (axes.empty() || int(reps.size()) * G != Pg) {  // no reflection symmetry: contiguous slices of 4
    const int quads = (Pg + 3) / 4;
    const int q0 = std::min(Pg, 4 * int((int64_t(quads) * rank) / world));
    const int q1 = std::min(Pg, 4 * int((int64_t(quads) * (rank + 1)) / world));
    return range_subset(q0, q1);
  }
  // whole orbits, in slices of 8 representatives when possible (full 8-direction groups per octant)
  const int R = int(reps.size()), unit = R % (8 * world) == 0 ? 8 : 1, units = R / unit;
  const int r0 = unit * int((int64_t(units) * rank) / world), r1 = unit * int((int64_t(units) * (rank + 1)) / world);
  std::vector<int> out;
  for (int r = r0; r < r1; ++r)
    for (int g = 0; g < G; ++g) {
      int m = reps[r];
      for (size_t k = 0; k < axes.size(); ++k)
        if ((g >> k) & 1) m = mirror[k][m];
      out.push_back(m);
    }
  std::sort(out.begin(), out.end());
  return out;
}

void find_symmetry(LevelTables& L, const SphereTree& t) {
  // key of a patch: its three lattice vertices, sorted
  using Key = std::array<std::int64_t, 9>;
  auto key_of = [](std::array<std::int64_t, 9> f) {
    std::array<std::array<std::int64_t, 3>, 3> v{{{f[0], f[1], f[2]}, {f[3], f[4], f[5]}, {f[6], f[7], f[8]}}};
    std::sort(v.begin(), v.end());
    Key k;
    for (int i = 0; i < 3; ++i)
      for (int r = 0; r < 3; ++r) k[3 * i + r] = v[i][r];
    return k;
  };
  std::map<Key, int> pos;
  for (int q = 0; q < L.P; ++q) pos[key_of(t.flat[L.leaf_id[q]])] = q;
  std::vector<std::vector<int>> mirror;  // per symmetric axis: q -> mirror q
  L.n_sym_axes = 0;
  for (int axis = 0; axis < 3; ++axis) {
    std::vector<int> mq(L.P, -1);
    bool ok = true;  // a rank's slice must be closed under the reflection (lookup among its own patches)
    for (int q = 0; ok && q < L.P; ++q) {
      auto f = t.flat[L.leaf_id[q]];
      for (int v = 0; v < 3; ++v) f[3 * v + axis] = -f[3 * v + axis];
      auto it = pos.find(key_of(f));
      if (it == pos.end()) ok = false;
      else mq[q] = it->second;
    }
    if (!ok) continue;
    L.sym_axes[L.n_sym_axes++] = axis;
    mirror.push_back(mq);
  }
  const int G = 1 << L.n_sym_axes;
  L.orbit.clear();
  if (L.n_sym_axes == 0) return;
  // representatives: patches whose octant bits on the symmetric axes are all 0
  for (int q = 0; q < L.P; ++q) {
    bool rep = true;
    for (int k = 0; k < L.n_sym_axes; ++k)
      if ((L.octant[q] >> L.sym_axes[k]) & 1) rep = false;
    if (!rep) continue;
    for (int g = 0; g < G; ++g) {
      int m = q;
      for (int k = 0; k < L.n_sym_axes; ++k)
        if ((g >> k) & 1) m = mirror[k][m];
      L.orbit.push_back(m);
    }
  }
  if (int(L.orbit.size()) != L.P) {  // every patch must lie in exactly one orbit
    L.orbit.clear();
    L.n_sym_axes = 0;
    return;
  }
  // harmonic parity classes: Y_{n,o} under x: (-1)^m (cos) / -(-1)^m (sin); y: +1 (cos) / -1 (sin);
  // z: (-1)^(n+m); class bit k set when odd under sym_axes[k]
  L.hclass.assign(L.H, 0);
  for (int n = 0; n <= L.order; ++n)
    for (int o = -n; o <= n; ++o) {
      const int m = o < 0 ? -o : o;
      const int px = o >= 0 ? (m & 1) : ((m + 1) & 1);
      const int py = o >= 0 ? 0 : 1;
      const int pz = (n + m) & 1;
      const int par[3] = {px, py, pz};
      int c = 0;
      for (int k = 0; k < L.n_sym_axes; ++k) c |= par[L.sym_axes[k]] << k;
      L.hclass[n * n + n + o] = c;
    }
  // the fold's exactness is a property of the coupling table, not only of the lattice:
  // measure the reflection defect of X over every orbit member and harmonic
  double xmax = 0, dmax = 0;
  for (double v : L.X) xmax = std::max(xmax, std::abs(v));
  const int R = L.P / G;
  for (int r = 0; r < R; ++r) {
    const double* Xr = &L.X[size_t(L.orbit[size_t(r) * G]) * L.H];
    for (int g = 1; g < G; ++g) {
      const double* Xg = &L.X[size_t(L.orbit[size_t(r) * G + g]) * L.H];
      for (int h = 0; h < L.H; ++h) {
        const double chi = (__builtin_popcount(unsigned(g) & unsigned(L.hclass[h])) & 1) ? -1.0 : 1.0;
        dmax = std::max(dmax, std::abs(Xg[h] - chi * Xr[h]));
      }
    }
  }
  L.sym_defect = xmax > 0 ? dmax / xmax : 0.0;
}

std::vector<std::vector<int>> partition_levels(const SphereTree& fine, int nlev, int rank, int world) {
  const int Lmax = fine.max_level;
  nlev = nlev <= 0 ? Lmax + 1 : std::min(nlev, Lmax + 1);
  const int lmin = Lmax + 1 - nlev;
  std::vector<SphereTree> trees;
  for (int i = 0; i < nlev; ++i) trees.push_back(lmin + i == Lmax ? fine : coarsen(fine, lmin + i));
  // root (coarsest-level position) of every leaf of every level
  std::unordered_map<int, int> root_pos;
  for (int c = 0; c < int(trees[0].leaves.size()); ++c) root_pos[trees[0].leaves[c]] = c;
  auto root_of = [&](int id) {
    while (!root_pos.count(id)) id = fine.parent[id];
    return root_pos[id];
  };
  const int R = int(trees[0].leaves.size());
  std::vector<long> weight(R, 0);
  for (int id : trees.back().leaves) weight[root_of(id)]++;
  long total = 0;
  for (long w : weight) total += w;
  // units of assignment: whole reflection orbits of roots when the finest mesh is mirror
  // symmetric (a rank's subtrees are then closed under the reflections at every level and
  // its scatter folds, as on one GPU), else single roots
  std::vector<int> axes, axes0;
  std::vector<std::vector<int>> mf, m0;
  leaf_mirrors(fine, axes, mf, {});
  std::vector<std::vector<int>> units;  // roots of each unit, in root order of the unit's first member
  if (!axes.empty()) {
    leaf_mirrors(trees[0], axes0, m0, axes);
    if (axes0 == axes) {
      std::vector<int> seen(R, 0);
      for (int c = 0; c < R; ++c) {
        if (seen[c]) continue;
        std::vector<int> orb{c};
        for (size_t k = 0; k < axes0.size(); ++k) {
          const size_t n = orb.size();
          for (size_t i = 0; i < n; ++i) orb.push_back(m0[k][orb[i]]);
        }
        std::sort(orb.begin(), orb.end());
        orb.erase(std::unique(orb.begin(), orb.end()), orb.end());
        for (int q : orb) seen[q] = 1;
        units.push_back(orb);
      }
      if (int(units.size()) < world) units.clear();  // too few orbits to give every rank one
    }
  }
  if (units.empty())
    for (int c = 0; c < R; ++c) units.push_back({c});
  // balance the finest-level directions: heaviest unit first onto the least-loaded rank
  // (deterministic: ties by first root, then by rank); the cone mesh of config 4 has
  // orbits of very different weight, so contiguous cuts were 1.25x imbalanced at 8 ranks
  (void)total;
  std::vector<long> uw(units.size(), 0);
  for (size_t u = 0; u < units.size(); ++u)
    for (int c : units[u]) uw[u] += weight[c];
  std::vector<int> order(units.size());
  for (size_t u = 0; u < units.size(); ++u) order[u] = int(u);
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return uw[a] > uw[b]; });
  std::vector<long> load(world, 0);
  std::vector<int> owner(R, 0);
  for (int u : order) {
    const int o = int(std::min_element(load.begin(), load.end()) - load.begin());
    load[o] += uw[u];
    for (int c : units[u]) owner[c] = o;
  }
  std::vector<std::vector<int>> parts(nlev);
  for (int i = 0; i < nlev; ++i)
    for (int q = 0; q < int(trees[i].leaves.size()); ++q)
      if (i == 0 || owner[root_of(trees[i].leaves[q])] == rank) parts[i].push_back(q);
  return parts;
}

std::vector<LevelTables> build_hierarchy(const Problem& pb, const SphereTree& fine, int nr, int nlev,
                                         const std::vector<std::vector<int>>* parts) {
  const int Lmax = fine.max_level;
  nlev = nlev <= 0 ? Lmax + 1 : std::min(nlev, Lmax + 1);
  const int lmin = Lmax + 1 - nlev;
  std::vector<SphereTree> trees;
  std::vector<LevelTables> lv;
  for (int i = 0; i < nlev; ++i) {
    const int l = lmin + i;
    trees.push_back(l == Lmax ? fine : coarsen(fine, l));
    lv.push_back(build_level(pb, trees.back(), nr, i == 0, parts && i > 0 ? &(*parts)[i] : nullptr));
  }
  for (int i = 1; i < nlev; ++i) {  // transfer maps (multigrid.cpp:68-96), Const: B = [1]
    const auto& ct = trees[i - 1];
    const auto& ft = trees[i];
    const LevelTables& C = lv[i - 1];
    std::unordered_map<int, int> pos;  // coarse leaf id -> position in the coarse level's (local) list
    for (int c = 0; c < C.P; ++c) pos[C.leaf_id[c]] = c;
    auto& L = lv[i];
    L.up.resize(L.P);
    L.up_w.assign(L.P, 1.0);
    for (int q = 0; q < L.P; ++q) {
      const int id = L.leaf_id[q];
      auto it = pos.find(id);
      if (it == pos.end()) it = pos.find(ft.parent[id]);
      if (it == pos.end()) throw std::logic_error("build_hierarchy: meshes are not nested");
      L.up[q] = it->second;
    }
    (void)ct;
    const int Pc = C.P;
    L.child_ptr.assign(Pc + 1, 0);
    for (int q = 0; q < L.P; ++q) L.child_ptr[L.up[q] + 1]++;
    for (int c = 0; c < Pc; ++c) L.child_ptr[c + 1] += L.child_ptr[c];
    L.child_idx.resize(L.P);
    std::vector<int> fillp(L.child_ptr.begin(), L.child_ptr.end() - 1);
    for (int q = 0; q < L.P; ++q) L.child_idx[fillp[L.up[q]]++] = q;  // ascending q per parent
  }
  return lv;
}

std::vector<double> assemble_rhs(const Problem& pb, const LevelTables& lev, const SphereTree& tree) {
  const int P = lev.P;
  std::vector<double> f(size_t(pb.n_el) * P * kS, 0.0);
  double nsum[4] = {0, 0, 0, 0};
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < 4; ++j) nsum[i] += lev.Nmat[i * 4 + j];
  if (!pb.q_el.empty()) {  // isotropic volume source (transport.cpp:114-127)
    for (int el = 0; el < pb.n_el; ++el) {
      if (pb.q_el[el] == 0.0) continue;
      const double c = pb.q_el[el] / (4.0 * kPi);
      for (int q = 0; q < P; ++q)
        for (int i = 0; i < 4; ++i) f[(size_t(el) * P + q) * 4 + i] += (c * lev.area[q]) * nsum[i];
    }
  }
  if (pb.spec.beam == 2) {  // unit incoming flux on in-cone patches at x = 0
    for (int q = 0; q < P; ++q) {
      if (!in_cone(tree, lev.leaf_id[q], pb.spec.cone_half_angle_deg)) continue;
      if (lev.octant[q] & 1) continue;
      const double* Cx = &lev.C[size_t(q) * 32];
      for (int iy = 0; iy < pb.spec.ny; ++iy) {
        const int el = iy * pb.spec.nx;
        for (int i = 0; i < 4; ++i) {
          double acc = 0;
          for (int j = 0; j < 4; ++j) acc += Cx[i * 4 + j];
          f[(size_t(el) * P + q) * 4 + i] += -pb.spec.strength * acc;
        }
      }
    }
  }
  return f;
}

}  // namespace stamg_b200
