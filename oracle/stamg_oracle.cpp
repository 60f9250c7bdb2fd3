// ORACLE — TEST INFRASTRUCTURE ONLY (see stamg_oracle.hpp). CPU restatement of
// /root/reference/proj/src/*.cpp; each block cites the lines it follows.
#include "stamg_oracle.hpp"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <map>
#include <mutex>
#include <numbers>
#include <unordered_map>

namespace oracle {

namespace {
inline Vec3 sub(const Vec3& a, const Vec3& b) { return {a[0] - b[0], a[1] - b[1], a[2] - b[2]}; }
inline Vec3 add(const Vec3& a, const Vec3& b) { return {a[0] + b[0], a[1] + b[1], a[2] + b[2]}; }
inline Vec3 mul(double s, const Vec3& a) { return {s * a[0], s * a[1], s * a[2]}; }
inline double dot(const Vec3& a, const Vec3& b) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; }
inline Vec3 cross(const Vec3& a, const Vec3& b) {
  return {a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0]};
}
inline double norm(const Vec3& a) { return std::sqrt(dot(a, a)); }
inline Vec3 to_double(const IVec3& f, double s = 1.0) {
  return {double(f[0]) * s, double(f[1]) * s, double(f[2]) * s};
}
double vnorm(const Vec& v) {
  double s = 0;
  for (double x : v) s += x * x;
  return std::sqrt(s);
}
double vdot(const Vec& a, const Vec& b) {
  double s = 0;
  for (size_t i = 0; i < a.size(); ++i) s += a[i] * b[i];
  return s;
}
}  // namespace

// kron.hpp:7-14
Mat kron(const Mat& A, const Mat& B) {
  Mat K(A.r * B.r, A.c * B.c);
  for (int i = 0; i < A.r; ++i)
    for (int j = 0; j < A.c; ++j)
      for (int k = 0; k < B.r; ++k)
        for (int l = 0; l < B.c; ++l) K(i * B.r + k, j * B.c + l) = A(i, j) * B(k, l);
  return K;
}

// Doolittle LU with partial (row) pivoting, as Eigen::PartialPivLU.
LU::LU(const Mat& A) : n(A.r), lu(A), piv(A.r) {
  for (int i = 0; i < n; ++i) piv[i] = i;
  for (int k = 0; k < n; ++k) {
    int p = k;
    double best = std::abs(lu(k, k));
    for (int i = k + 1; i < n; ++i)
      if (std::abs(lu(i, k)) > best) best = std::abs(lu(i, k)), p = i;
    if (p != k) {
      for (int j = 0; j < n; ++j) std::swap(lu(k, j), lu(p, j));
      std::swap(piv[k], piv[p]);
    }
    const double d = lu(k, k);
    if (d == 0.0) continue;
    for (int i = k + 1; i < n; ++i) {
      const double l = lu(i, k) / d;
      lu(i, k) = l;
      for (int j = k + 1; j < n; ++j) lu(i, j) -= l * lu(k, j);
    }
  }
}

void LU::solve(const double* b, double* x) const {
  double tmp[64];
  std::vector<double> big;
  double* t = tmp;
  if (n > 64) big.resize(n), t = big.data();
  for (int i = 0; i < n; ++i) t[i] = b[piv[i]];
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < i; ++j) t[i] -= lu(i, j) * t[j];
  for (int i = n - 1; i >= 0; --i) {
    for (int j = i + 1; j < n; ++j) t[i] -= lu(i, j) * t[j];
    t[i] /= lu(i, i);
  }
  for (int i = 0; i < n; ++i) x[i] = t[i];
}

// ============================================================ sphere_mesh.cpp
namespace {

Vec3 to_unit(const IVec3& f) {  // sphere_mesh.cpp:14-18
  Vec3 v = to_double(f);
  return mul(1.0 / norm(v), v);
}

Patch make_patch(int id, int level, int octant, int parent, const IVec3& a, const IVec3& b,
                 const IVec3& c) {  // :20-30
  Patch p;
  p.id = id, p.level = level, p.octant = octant, p.parent = parent;
  p.flat = {a, b, c};
  p.vert = {to_unit(a), to_unit(b), to_unit(c)};
  return p;
}

void rebuild_leaf_list(AngularMesh& mesh) {  // :32-41
  mesh.leaves.clear();
  mesh.max_level = 0;
  for (const Patch& p : mesh.all)
    if (p.leaf) {
      mesh.leaves.push_back(p.id);
      mesh.max_level = std::max(mesh.max_level, p.level);
    }
}

IVec3 half_sum(const IVec3& a, const IVec3& b) {
  return {(a[0] + b[0]) / 2, (a[1] + b[1]) / 2, (a[2] + b[2]) / 2};
}

void split_patch(AngularMesh& mesh, int id) {  // :44-58
  if (!mesh.all[id].leaf) throw std::invalid_argument("refine: patch is not a leaf");
  const IVec3 a = mesh.all[id].flat[0], b = mesh.all[id].flat[1], c = mesh.all[id].flat[2];
  const IVec3 mab = half_sum(a, b), mbc = half_sum(b, c), mca = half_sum(c, a);
  const int base = int(mesh.all.size());
  const int lvl = mesh.all[id].level + 1, oct = mesh.all[id].octant;
  mesh.all[id].leaf = false;
  mesh.all[id].kids = {base, base + 1, base + 2, base + 3};
  mesh.all.push_back(make_patch(base + 0, lvl, oct, id, a, mab, mca));
  mesh.all.push_back(make_patch(base + 1, lvl, oct, id, mab, b, mbc));
  mesh.all.push_back(make_patch(base + 2, lvl, oct, id, mca, mbc, c));
  mesh.all.push_back(make_patch(base + 3, lvl, oct, id, mab, mbc, mca));
  mesh.max_level = std::max(mesh.max_level, lvl);
}

struct SegKey {  // :60-79
  std::array<std::int64_t, 6> v;
  bool operator==(const SegKey&) const = default;
};
struct SegKeyHash {
  std::size_t operator()(const SegKey& k) const {
    std::size_t h = 0xcbf29ce484222325ull;
    for (std::int64_t x : k.v) h ^= static_cast<std::size_t>(x) + 0x9e3779b97f4a7c15ull + (h << 6) + (h >> 2);
    return h;
  }
};
SegKey make_seg_key(const IVec3& u, const IVec3& v) {
  std::array<std::int64_t, 3> a{u[0], u[1], u[2]}, b{v[0], v[1], v[2]};
  if (b < a) std::swap(a, b);
  return SegKey{{a[0], a[1], a[2], b[0], b[1], b[2]}};
}

using SegTable = std::unordered_map<SegKey, std::array<int, 2>, SegKeyHash>;

SegTable segment_table(const AngularMesh& mesh) {  // :82-101
  SegTable table;
  table.reserve(mesh.leaves.size() * 6);
  for (int id : mesh.leaves) {
    const Patch& p = mesh.all[id];
    const std::int64_t k = std::int64_t(1) << (mesh.max_level - p.level);
    for (int e = 0; e < 3; ++e) {
      const IVec3 u = p.flat[e], v = p.flat[(e + 1) % 3];
      const IVec3 step = {(v[0] - u[0]) / k, (v[1] - u[1]) / k, (v[2] - u[2]) / k};
      for (std::int64_t t = 0; t < k; ++t) {
        const IVec3 s0 = {u[0] + step[0] * t, u[1] + step[1] * t, u[2] + step[2] * t};
        const IVec3 s1 = {s0[0] + step[0], s0[1] + step[1], s0[2] + step[2]};
        auto [it, fresh] = table.try_emplace(make_seg_key(s0, s1), std::array<int, 2>{id, -1});
        if (!fresh) it->second[1] = id;
      }
    }
  }
  return table;
}

void enforce_two_irregularity(AngularMesh& mesh) {  // :103-120
  for (bool changed = true; changed;) {
    changed = false;
    rebuild_leaf_list(mesh);
    auto table = segment_table(mesh);
    for (const auto& [key, pair] : table) {
      if (pair[1] < 0) continue;
      const Patch& x = mesh.all[pair[0]];
      const Patch& y = mesh.all[pair[1]];
      if (std::abs(x.level - y.level) > 2) {
        split_patch(mesh, x.level < y.level ? x.id : y.id);
        changed = true;
        break;
      }
    }
  }
  rebuild_leaf_list(mesh);
}

int banded_target(const Patch& p, int l_max) {  // :122-131
  double z = std::max({p.vert[0][2], p.vert[1][2], p.vert[2][2]});
  int t;
  if (z > 0.9875) t = l_max;
  else if (z > 0.9) t = l_max - 1;
  else if (z > 0.8) t = l_max - 2;
  else if (z > 0.6) t = l_max - 3;
  else t = l_max - 4;
  return std::max(t, 0);
}

}  // namespace

int AngularMesh::leaf_pos(int id) const {  // :135-139
  auto it = std::lower_bound(leaves.begin(), leaves.end(), id);
  if (it == leaves.end() || *it != id) return -1;
  return int(it - leaves.begin());
}

AngularMesh build_base_mesh() {  // :141-153
  AngularMesh mesh;
  for (int oct = 0; oct < 8; ++oct) {
    const std::int64_t sx = (oct & 1) ? -1 : 1, sy = (oct & 2) ? -1 : 1, sz = (oct & 4) ? -1 : 1;
    IVec3 a{sx * kFlatScale, 0, 0}, b{0, sy * kFlatScale, 0}, c{0, 0, sz * kFlatScale};
    if (sx * sy * sz < 0) std::swap(b, c);
    mesh.all.push_back(make_patch(oct, 0, oct, -1, a, b, c));
  }
  rebuild_leaf_list(mesh);
  return mesh;
}

void refine(AngularMesh& mesh, int patch_id) {  // :155-160
  if (patch_id < 0 || patch_id >= int(mesh.all.size()))
    throw std::invalid_argument("refine: unknown patch id");
  split_patch(mesh, patch_id);
  enforce_two_irregularity(mesh);
}

AngularMesh build_uniform_mesh(int level) {  // :162-171
  if (level < 0) throw std::invalid_argument("build_uniform_mesh: level < 0");
  AngularMesh mesh = build_base_mesh();
  for (int l = 0; l < level; ++l) {
    std::vector<int> current = mesh.leaves;
    for (int id : current) split_patch(mesh, id);
    rebuild_leaf_list(mesh);
  }
  return mesh;
}

AngularMesh build_banded_mesh(int l_max) {  // :173-189
  if (l_max < 1) throw std::invalid_argument("build_banded_mesh: l_max < 1");
  AngularMesh mesh = build_base_mesh();
  for (bool changed = true; changed;) {
    changed = false;
    std::vector<int> current = mesh.leaves;
    for (int id : current)
      if (mesh.all[id].level < banded_target(mesh.all[id], l_max)) {
        split_patch(mesh, id);
        changed = true;
      }
    rebuild_leaf_list(mesh);
  }
  enforce_two_irregularity(mesh);
  return mesh;
}

// EXTENSION (BASELINE config 4): centroid-in-cone rule, recorded in DESIGN.md.
bool patch_in_cone(const Patch& p, double half_angle_deg) {
  Vec3 c = add(add(p.vert[0], p.vert[1]), p.vert[2]);
  c = mul(1.0 / norm(c), c);
  return c[0] >= std::cos(half_angle_deg * std::numbers::pi / 180.0);
}

AngularMesh build_cone_mesh(int base_level, int extra, double half_angle_deg) {
  AngularMesh mesh = build_uniform_mesh(base_level);
  for (int e = 0; e < extra; ++e) {
    std::vector<int> current = mesh.leaves;
    for (int id : current)
      if (mesh.all[id].level == base_level + e && patch_in_cone(mesh.all[id], half_angle_deg))
        split_patch(mesh, id);
    rebuild_leaf_list(mesh);
  }
  enforce_two_irregularity(mesh);
  return mesh;
}

AngularMesh coarsen_to_level(const AngularMesh& mesh, int level) {  // :191-203
  if (level < 0) throw std::invalid_argument("coarsen_to_level: level < 0");
  AngularMesh out = mesh;
  if (level >= mesh.max_level) return out;
  for (Patch& p : out.all) p.leaf = false;
  for (int id : mesh.leaves) {
    int a = id;
    while (out.all[a].level > level) a = out.all[a].parent;
    out.all[a].leaf = true;
  }
  rebuild_leaf_list(out);
  return out;
}

double patch_area(const Patch& p) {  // :205-210
  const Vec3 &a = p.vert[0], &b = p.vert[1], &c = p.vert[2];
  const double num = std::abs(dot(a, cross(b, c)));
  const double den = 1.0 + dot(a, b) + dot(b, c) + dot(c, a);
  return 2.0 * std::atan2(num, den);
}

double total_area(const AngularMesh& mesh) {
  double s = 0;
  for (int id : mesh.leaves) s += patch_area(mesh.all[id]);
  return s;
}

std::vector<std::vector<int>> leaf_neighbors(const AngularMesh& mesh) {  // :218-230
  std::vector<std::vector<int>> nbr(mesh.leaves.size());
  for (const auto& [key, pair] : segment_table(mesh)) {
    if (pair[1] < 0) continue;
    nbr[mesh.leaf_pos(pair[0])].push_back(pair[1]);
    nbr[mesh.leaf_pos(pair[1])].push_back(pair[0]);
  }
  for (auto& v : nbr) {
    std::sort(v.begin(), v.end());
    v.erase(std::unique(v.begin(), v.end()), v.end());
  }
  return nbr;
}

bool two_irregular(const AngularMesh& mesh) {  // :232-240
  auto nbr = leaf_neighbors(mesh);
  for (size_t i = 0; i < nbr.size(); ++i) {
    const int li = mesh.all[mesh.leaves[i]].level;
    for (int id : nbr[i])
      if (std::abs(li - mesh.all[id].level) > 2) return false;
  }
  return true;
}

// ============================================================ quadrature.cpp
namespace {
Gauss1D compute_gauss(int n) {  // quadrature.cpp:13-45
  Gauss1D g;
  g.x.resize(n);
  g.w.resize(n);
  for (int i = 0; i < n; ++i) {
    double t = std::cos(std::numbers::pi * (i + 0.75) / (n + 0.5));
    double p0 = 0, p1 = 0;
    for (int it = 0; it < 100; ++it) {
      p0 = 1.0;
      p1 = t;
      for (int k = 2; k <= n; ++k) {
        double p2 = ((2 * k - 1) * t * p1 - (k - 1) * p0) / k;
        p0 = p1;
        p1 = p2;
      }
      double dp = n * (t * p1 - p0) / (t * t - 1.0);
      double dt = p1 / dp;
      t -= dt;
      if (std::abs(dt) < 1e-15) break;
    }
    p0 = 1.0;
    p1 = t;
    for (int k = 2; k <= n; ++k) {
      double p2 = ((2 * k - 1) * t * p1 - (k - 1) * p0) / k;
      p0 = p1;
      p1 = p2;
    }
    double dp = n * (t * p1 - p0) / (t * t - 1.0);
    g.x[i] = 0.5 * (1.0 - t);
    g.w[i] = 1.0 / ((1.0 - t * t) * dp * dp);
  }
  return g;
}
}  // namespace

const Gauss1D& gauss_legendre_01(int n) {  // :49-57
  if (n < 1 || n > 64) throw std::invalid_argument("gauss_legendre_01: bad order");
  static std::map<int, Gauss1D> cache;
  static std::mutex mtx;
  std::lock_guard<std::mutex> lock(mtx);
  auto it = cache.find(n);
  if (it == cache.end()) it = cache.emplace(n, compute_gauss(n)).first;
  return it->second;
}

QuadratureRule patch_quadrature(const Patch& patch, int order) {  // :59-92
  if (order < 1 || order > 64) throw std::invalid_argument("patch_quadrature: unsupported order");
  const int n = order;
  const Gauss1D& g = gauss_legendre_01(n);
  const double inv = 1.0 / double(kFlatScale);
  const Vec3 a = to_double(patch.flat[0], inv), b = to_double(patch.flat[1], inv),
             c = to_double(patch.flat[2], inv);
  const Vec3 cr = cross(sub(b, a), sub(c, a));
  const double two_area = norm(cr);
  const Vec3 nrm = mul(1.0 / two_area, cr);
  const double h = dot(a, nrm);
  QuadratureRule rule;
  rule.nodes.resize(n * n);
  rule.bary.resize(n * n);
  rule.weights.resize(n * n);
  int idx = 0;
  for (int iu = 0; iu < n; ++iu) {
    const double u = g.x[iu];
    for (int iv = 0; iv < n; ++iv, ++idx) {
      const double v = g.x[iv];
      const Vec3 x = add(mul(1.0 - u, a), mul(u, add(mul(1.0 - v, b), mul(v, c))));
      const double r = norm(x);
      const double wf = g.w[iu] * g.w[iv] * u * two_area;
      rule.nodes[idx] = mul(1.0 / r, x);
      rule.bary[idx] = {1.0 - u, u * (1.0 - v), u * v};
      rule.weights[idx] = wf * h / (r * r * r);
    }
  }
  return rule;
}

// ============================================================ angular_disc.cpp
namespace {
// solve V mu = omega with V = flat vertices as columns (angular_disc.cpp:10-24)
Vec3 flat_solve(const Patch& patch, const Vec3& omega) {
  const double inv = 1.0 / double(kFlatScale);
  Mat V(3, 3);
  for (int i = 0; i < 3; ++i)
    for (int r = 0; r < 3; ++r) V(r, i) = double(patch.flat[i][r]) * inv;
  LU lu(V);
  Vec3 mu;
  lu.solve(omega.data(), mu.data());
  return mu;
}
}  // namespace

Vec3 barycentric(const Patch& patch, const Vec3& omega) {
  Vec3 mu = flat_solve(patch, omega);
  const double s = mu[0] + mu[1] + mu[2];
  return mul(1.0 / s, mu);
}

bool patch_contains(const Patch& patch, const Vec3& omega, double tol) {  // :26-32
  Vec3 mu = flat_solve(patch, omega);
  const double s = mu[0] + mu[1] + mu[2];
  if (s <= 0) return false;
  mu = mul(1.0 / s, mu);
  return std::min({mu[0], mu[1], mu[2]}) >= -tol;
}

PatchOperators build_patch_operators(BasisKind kind, const Patch& patch, int order) {  // :40-59
  if (order <= 0) order = default_patch_order(patch.level);
  const int dofs = dofs_per_patch(kind);
  const QuadratureRule rule = patch_quadrature(patch, order);
  PatchOperators ops;
  ops.M = Mat(dofs, dofs);
  for (auto& a : ops.A) a = Mat(dofs, dofs);
  double psi[3];
  for (int g = 0; g < rule.size(); ++g) {
    if (kind == BasisKind::Const) psi[0] = 1.0;
    else for (int d = 0; d < 3; ++d) psi[d] = rule.bary[g][d];
    for (int i = 0; i < dofs; ++i)
      for (int j = 0; j < dofs; ++j) {
        const double o = rule.weights[g] * (psi[i] * psi[j]);
        ops.M(i, j) += o;
        for (int xi = 0; xi < 3; ++xi) ops.A[xi](i, j) += rule.nodes[g][xi] * o;
      }
  }
  return ops;
}

std::pair<Mat, Mat> face_split(BasisKind kind, const Patch& patch, const Vec3& normal,
                               int order) {  // :61-96
  const int dofs = dofs_per_patch(kind);
  int axis = -1;
  for (int xi = 0; xi < 3; ++xi)
    if (std::abs(std::abs(normal[xi]) - 1.0) < 1e-14) axis = xi;
  if (axis >= 0) {
    const PatchOperators ops = build_patch_operators(kind, patch, 0);
    Mat face = ops.A[axis];
    for (double& v : face.a) v *= normal[axis];
    const double sgn = (patch.octant >> axis) & 1 ? -1.0 : 1.0;
    if (normal[axis] * sgn > 0) return {face, Mat(dofs, dofs)};
    return {Mat(dofs, dofs), face};
  }
  if (order < 20) order = 20;
  const QuadratureRule rule = patch_quadrature(patch, order);
  Mat face(dofs, dofs), out(dofs, dofs);
  double psi[3];
  for (int g = 0; g < rule.size(); ++g) {
    if (kind == BasisKind::Const) psi[0] = 1.0;
    else for (int d = 0; d < 3; ++d) psi[d] = rule.bary[g][d];
    const double on = dot(rule.nodes[g], normal);
    for (int i = 0; i < dofs; ++i)
      for (int j = 0; j < dofs; ++j) {
        const double t = rule.weights[g] * on * (psi[i] * psi[j]);
        face(i, j) += t;
        if (on > 0) out(i, j) += t;
      }
  }
  Mat in = face;
  for (size_t i = 0; i < in.a.size(); ++i) in.a[i] -= out.a[i];
  return {out, in};
}

// ============================================================ scatter.cpp
ScatterKernel fp_equivalent_moments(int N, double alpha, double sigma_a) {  // scatter.cpp:9-21
  if (N < 1) throw std::invalid_argument("fp_equivalent_moments: N < 1");
  if (alpha <= 0) throw std::invalid_argument("fp_equivalent_moments: alpha <= 0");
  ScatterKernel k;
  k.N = N;
  k.sigma_a = sigma_a;
  k.moments.resize(N + 1);
  for (int n = 0; n <= N; ++n) k.moments[n] = 0.5 * alpha * (double(N) * (N + 1) - double(n) * (n + 1));
  k.sigma_t = sigma_a + k.moments[0];
  return k;
}

ScatterKernel absorber_kernel(double sigma_a) {  // :23-31
  ScatterKernel k;
  k.N = 0;
  k.sigma_a = sigma_a;
  k.sigma_t = sigma_a;
  k.moments = Vec(1, 0.0);
  return k;
}

// EXTENSION: Henyey-Greenstein, sigma_{s,n} = c sigma_t g^n
ScatterKernel hg_moments(int N, double sigma_t, double c, double g) {
  ScatterKernel k;
  k.N = N;
  k.sigma_t = sigma_t;
  k.moments.resize(N + 1);
  double gn = 1.0;
  for (int n = 0; n <= N; ++n, gn *= g) k.moments[n] = c * sigma_t * gn;
  k.sigma_a = sigma_t - k.moments[0];
  return k;
}

void eval_real_harmonics(int N, const Vec3& omega, double* out) {  // :33-65
  const double z = omega[2];
  const double rxy = std::hypot(omega[0], omega[1]);
  const double phi = std::atan2(omega[1], omega[0]);
  const double inv_sqrt4pi = 1.0 / std::sqrt(4.0 * std::numbers::pi);
  double pmm = inv_sqrt4pi;
  for (int m = 0; m <= N; ++m) {
    const double cm = m == 0 ? 1.0 : std::numbers::sqrt2 * std::cos(m * phi);
    const double sm = m == 0 ? 0.0 : std::numbers::sqrt2 * std::sin(m * phi);
    double p_prev = 0.0, p = pmm;
    for (int n = m; n <= N; ++n) {
      const int base = n * n + n;
      out[base + m] = cm * p;
      if (m > 0) out[base - m] = sm * p;
      if (n < N) {
        const double nn = n + 1;
        const double a = std::sqrt((4.0 * nn * nn - 1.0) / (nn * nn - double(m) * m));
        const double b = std::sqrt(((nn - 1) * (nn - 1) - double(m) * m) / (4.0 * (nn - 1) * (nn - 1) - 1.0));
        const double p_next = a * (z * p - b * p_prev);
        p_prev = p;
        p = p_next;
      }
    }
    if (m < N) pmm *= -std::sqrt((2.0 * m + 3.0) / (2.0 * m + 2.0)) * rxy;
  }
}

HarmonicCouplings build_couplings(const AngularMesh& mesh, BasisKind kind, int N, int order) {  // :74-99
  HarmonicCouplings coup;
  coup.N = N;
  coup.kind = kind;
  coup.D = dofs_per_patch(kind);
  const int H = harmonic_count(N);
  coup.X = Mat(mesh.n_leaves() * coup.D, H);
  std::vector<double> Y(H);
  for (int lp = 0; lp < mesh.n_leaves(); ++lp) {
    const Patch& patch = mesh.patch(mesh.leaves[lp]);
    const int ord = order > 0 ? order : default_patch_order(patch.level, default_quad_order(N));
    const QuadratureRule rule = patch_quadrature(patch, ord);
    for (int g = 0; g < rule.size(); ++g) {
      eval_real_harmonics(N, rule.nodes[g], Y.data());
      for (int d = 0; d < coup.D; ++d) {
        const double psi = kind == BasisKind::Const ? 1.0 : rule.bary[g][d];
        const double w = rule.weights[g] * psi;
        double* row = &coup.X(lp * coup.D + d, 0);
        for (int h = 0; h < H; ++h) row[h] += w * Y[h];
      }
    }
  }
  return coup;
}

Vec sigma_by_harmonic(const ScatterKernel& k, int max_order) {  // :101-108
  if (max_order > k.N) throw std::invalid_argument("sigma_by_harmonic: max_order exceeds kernel order");
  Vec s(harmonic_count(std::max(max_order, 0)), 0.0);
  for (int n = 0; n <= max_order; ++n)
    for (int o = -n; o <= n; ++o) s[n * n + n + o] = k.moments[n];
  return s;
}

// ============================================================ spatial_disc.cpp
int Grid::neighbor(int el, int f) const {  // spatial_disc.cpp:19-27
  auto [ix, iy, iz] = coords(el);
  const int axis = f / 2, dir = (f % 2) ? 1 : -1;
  int c[3] = {ix, iy, iz};
  c[axis] += dir;
  const int n[3] = {nx, ny, nz};
  if (c[axis] < 0 || c[axis] >= n[axis]) return -1;
  return index(c[0], c[1], c[2]);
}

Grid build_grid(int dim, int nx, int ny, int nz, double box) {  // :29-43
  if (dim != 2 && dim != 3) throw std::invalid_argument("build_grid: dim must be 2 or 3");
  if (dim == 2) nz = 1;
  if (nx < 1 || ny < 1 || nz < 1) throw std::invalid_argument("build_hex_mesh: zero element count");
  if (box <= 0) throw std::invalid_argument("build_hex_mesh: box must be positive");
  Grid g;
  g.dim = dim, g.nx = nx, g.ny = ny, g.nz = nz, g.box = box;
  g.hx = box / nx, g.hy = box / ny, g.hz = dim == 3 ? box / nz : 0.0;
  g.n_el = nx * ny * nz;
  return g;
}

namespace {
Mat m2(double a, double b, double c, double d) {
  Mat m(2, 2);
  m(0, 0) = a, m(0, 1) = b, m(1, 0) = c, m(1, 1) = d;
  return m;
}
Mat mass1d(double h) { return m2(2 * h / 6.0, h / 6.0, h / 6.0, 2 * h / 6.0); }  // :11-15
Mat scalar(double v) { return Mat(1, 1, v); }
}  // namespace

ElementMatrices element_matrices(const Grid& mesh, int p) {  // :45-88 (+ 2D EXTENSION)
  if (p != 0 && p != 1) throw std::invalid_argument("element_matrices: p must be 0 or 1");
  ElementMatrices em;
  if (p == 0) {
    em.S = 1;
    em.N = scalar(mesh.volume());
    double areas[3];
    if (mesh.dim == 3) areas[0] = mesh.hy * mesh.hz, areas[1] = mesh.hx * mesh.hz, areas[2] = mesh.hx * mesh.hy;
    else areas[0] = mesh.hy, areas[1] = mesh.hx, areas[2] = 0.0;
    for (int xi = 0; xi < 3; ++xi) {
      em.V[xi] = scalar(0.0);
      for (int s = 0; s < 2; ++s) {
        em.F_self[2 * xi + s] = scalar(areas[xi]);
        em.F_neigh[2 * xi + s] = scalar(areas[xi]);
      }
    }
    return em;
  }
  const Mat mx = mass1d(mesh.hx), my = mass1d(mesh.hy);
  const Mat g = m2(-0.5, -0.5, 0.5, 0.5);
  const Mat t_lo = m2(1, 0, 0, 0), t_hi = m2(0, 0, 0, 1), c_lo = m2(0, 1, 0, 0), c_hi = m2(0, 0, 1, 0);
  if (mesh.dim == 3) {
    em.S = 8;
    const Mat mz = mass1d(mesh.hz);
    em.N = kron(mz, kron(my, mx));
    em.V[0] = kron(mz, kron(my, g));
    em.V[1] = kron(mz, kron(g, mx));
    em.V[2] = kron(g, kron(my, mx));
    for (int xi = 0; xi < 3; ++xi) {
      auto assemble = [&](const Mat& t) {
        switch (xi) {
          case 0: return kron(mz, kron(my, t));
          case 1: return kron(mz, kron(t, mx));
          default: return kron(t, kron(my, mx));
        }
      };
      em.F_self[2 * xi] = assemble(t_lo);
      em.F_self[2 * xi + 1] = assemble(t_hi);
      em.F_neigh[2 * xi] = assemble(c_lo);
      em.F_neigh[2 * xi + 1] = assemble(c_hi);
    }
    return em;
  }
  // EXTENSION: 2D bilinear, dof i = ix + 2*iy
  em.S = 4;
  em.N = kron(my, mx);
  em.V[0] = kron(my, g);
  em.V[1] = kron(g, mx);
  em.V[2] = Mat(4, 4);
  em.F_self[0] = kron(my, t_lo), em.F_self[1] = kron(my, t_hi);
  em.F_self[2] = kron(t_lo, mx), em.F_self[3] = kron(t_hi, mx);
  em.F_neigh[0] = kron(my, c_lo), em.F_neigh[1] = kron(my, c_hi);
  em.F_neigh[2] = kron(c_lo, mx), em.F_neigh[3] = kron(c_hi, mx);
  em.F_self[4] = em.F_self[5] = em.F_neigh[4] = em.F_neigh[5] = Mat(4, 4);
  return em;
}

std::vector<int> sweep_order(const Grid& mesh, int octant) {  // :90-106
  if (octant < 0 || octant > 7) throw std::invalid_argument("sweep_order: bad octant");
  auto axis_range = [](int n, bool reversed) {
    std::vector<int> r(n);
    for (int i = 0; i < n; ++i) r[i] = reversed ? n - 1 - i : i;
    return r;
  };
  const auto xs = axis_range(mesh.nx, octant & 1);
  const auto ys = axis_range(mesh.ny, octant & 2);
  const auto zs = axis_range(mesh.nz, mesh.dim == 3 && (octant & 4));
  std::vector<int> order;
  order.reserve(mesh.n_el);
  for (int iz : zs)
    for (int iy : ys)
      for (int ix : xs) order.push_back(mesh.index(ix, iy, iz));
  return order;
}

// ============================================================ transport.cpp
namespace {
int axis_sign(int octant, int xi) { return (octant >> xi) & 1 ? -1 : 1; }  // transport.cpp:13
std::array<double, 2> shape_integrals(double a, double b, double h) {     // :16-19
  const double len = b - a, quad = (b * b - a * a) / (2 * h);
  return {len - quad, quad};
}
void axpy_mat(Mat& B, double s, const Mat& K) {
  for (size_t i = 0; i < B.a.size(); ++i) B.a[i] += s * K.a[i];
}
void matvec_add(const Mat& A, const double* x, double* y, double s = 1.0) {
  for (int i = 0; i < A.r; ++i) {
    double acc = 0;
    for (int j = 0; j < A.c; ++j) acc += A(i, j) * x[j];
    y[i] += s * acc;
  }
}
}  // namespace

ProblemOperators build_operators(const Grid& mesh, const AngularMesh& angular, BasisKind kind,
                                 int p, const std::vector<ScatterKernel>& kernels,
                                 const std::vector<int>& mat) {  // transport.cpp:23-64
  if (kernels.empty()) throw std::invalid_argument("build_operators: no kernels");
  ProblemOperators ops;
  ops.mesh = mesh;
  ops.angular = angular;
  ops.kind = kind;
  ops.p = p;
  ops.kernels = kernels;
  ops.N = kernels[0].N;
  for (const auto& k : kernels)
    if (k.N != ops.N) throw std::invalid_argument("build_operators: kernels differ in order");
  ops.mat = mat.empty() ? std::vector<int>(mesh.n_el, 0) : mat;
  if (int(ops.mat.size()) != mesh.n_el) throw std::invalid_argument("build_operators: material map size");
  for (int m : ops.mat)
    if (m < 0 || m >= int(kernels.size())) throw std::invalid_argument("build_operators: bad material id");
  ops.em = element_matrices(mesh, p);
  const int D = dofs_per_patch(kind);
  ops.layout = Layout{mesh.n_el, angular.n_leaves(), ops.em.S, D};
  ops.coup = build_couplings(angular, kind, ops.N);
  const int P = angular.n_leaves();
  const int nmat = int(kernels.size());
  ops.diag.assign(nmat, {});
  for (int lp = 0; lp < P; ++lp) {
    const Patch& patch = angular.patch(angular.leaves[lp]);
    PatchOperators po = build_patch_operators(kind, patch);
    std::array<Mat, 3> C;
    std::array<int, 3> fin{-1, -1, -1}, fout{-1, -1, -1};
    const Mat MN = kron(po.M, ops.em.N);
    for (int m = 0; m < nmat; ++m) {
      Mat B = MN;
      for (double& v : B.a) v *= kernels[m].sigma_t;
      for (int xi = 0; xi < mesh.dim; ++xi) {
        const double s = axis_sign(patch.octant, xi);
        const int fo = 2 * xi + (s > 0 ? 1 : 0);
        axpy_mat(B, -1.0, kron(po.A[xi], ops.em.V[xi]));
        axpy_mat(B, s, kron(po.A[xi], ops.em.F_self[fo]));
      }
      ops.diag[m].push_back(std::move(B));
    }
    for (int xi = 0; xi < mesh.dim; ++xi) {
      const double s = axis_sign(patch.octant, xi);
      fout[xi] = 2 * xi + (s > 0 ? 1 : 0);
      fin[xi] = 2 * xi + (s > 0 ? 0 : 1);
      C[xi] = kron(po.A[xi], ops.em.F_neigh[fin[xi]]);
      for (double& v : C[xi].a) v *= -s;
    }
    ops.pops.push_back(std::move(po));
    ops.inflow.push_back(std::move(C));
    ops.inflow_face.push_back(fin);
    ops.outflow_face.push_back(fout);
  }
  return ops;
}

void apply_L_into(const ProblemOperators& ops, const double* phi, double* y) {  // :66-88
  const Layout& lo = ops.layout;
  const int bs = lo.D * lo.S;
#pragma omp parallel for schedule(static)
  for (int el = 0; el < lo.n_el; ++el) {
    std::array<int, 6> nb{-1, -1, -1, -1, -1, -1};
    for (int f = 0; f < ops.mesh.n_faces(); ++f) nb[f] = ops.mesh.neighbor(el, f);
    const auto& diag = ops.diag[ops.mat[el]];
    for (int q = 0; q < lo.n_patch; ++q) {
      double* yb = y + lo.block(el, q);
      const double* xb = phi + lo.block(el, q);
      for (int i = 0; i < bs; ++i) yb[i] = 0.0;
      matvec_add(diag[q], xb, yb);
      for (int xi = 0; xi < ops.mesh.dim; ++xi) {
        const int up = nb[ops.inflow_face[q][xi]];
        if (up < 0) continue;
        matvec_add(ops.inflow[q][xi], phi + lo.block(up, q), yb);
      }
    }
  }
}

void apply_scatter_into(const ProblemOperators& ops, const double* phi, int max_order,
                        double scale, double* y) {  // scatter.cpp:110-135
  const Layout& lo = ops.layout;
  std::vector<Vec> sig;
  for (const auto& k : ops.kernels) sig.push_back(sigma_by_harmonic(k, max_order));
  const int Hr = int(sig[0].size());
  const int PD = lo.n_patch * lo.D, S = lo.S;
  const Mat& X = ops.coup.X;
  const int H = X.c;
#pragma omp parallel
  {
    std::vector<double> mom(size_t(Hr) * S), src(size_t(Hr) * S);
#pragma omp for schedule(static)
    for (int el = 0; el < lo.n_el; ++el) {
      const double* Phi = phi + lo.element(el);
      double* Yel = y + lo.element(el);
      const Vec& sg = sig[ops.mat[el]];
      std::fill(mom.begin(), mom.end(), 0.0);
      for (int r = 0; r < PD; ++r) {  // mom = Xr^T Phi
        const double* xr = &X.a[size_t(r) * H];
        for (int h = 0; h < Hr; ++h) {
          const double xv = xr[h];
          for (int i = 0; i < S; ++i) mom[h * S + i] += xv * Phi[r * S + i];
        }
      }
      for (int h = 0; h < Hr; ++h)  // src = diag(sig) mom N
        for (int i = 0; i < S; ++i) {
          double acc = 0;
          for (int j = 0; j < S; ++j) acc += mom[h * S + j] * ops.em.N(j, i);
          src[h * S + i] = sg[h] * acc;
        }
      for (int r = 0; r < PD; ++r) {  // Y += scale Xr src
        const double* xr = &X.a[size_t(r) * H];
        for (int i = 0; i < S; ++i) {
          double acc = 0;
          for (int h = 0; h < Hr; ++h) acc += xr[h] * src[h * S + i];
          Yel[r * S + i] += scale * acc;
        }
      }
    }
  }
}

void apply_A_into(const ProblemOperators& ops, const double* phi, int order, double* y) {  // :96-101
  apply_L_into(ops, phi, y);
  apply_scatter_into(ops, phi, order, -1.0, y);
}

Vec assemble_rhs(const ProblemOperators& ops, const SourceSpec& spec) {  // :110-179
  const Layout& lo = ops.layout;
  Vec f(lo.size(), 0.0);
  Vec nsum(lo.S, 0.0);
  for (int i = 0; i < lo.S; ++i)
    for (int j = 0; j < lo.S; ++j) nsum[i] += ops.em.N(i, j);
  if (!spec.q_el.empty()) {
    if (int(spec.q_el.size()) != lo.n_el) throw std::invalid_argument("assemble_rhs: q_el size");
    for (int el = 0; el < lo.n_el; ++el) {
      if (spec.q_el[el] == 0.0) continue;
      const double c = spec.q_el[el] / (4.0 * std::numbers::pi);
      for (int q = 0; q < lo.n_patch; ++q)
        for (int d = 0; d < lo.D; ++d) {
          double msum = 0;
          for (int e = 0; e < lo.D; ++e) msum += ops.pops[q].M(d, e);
          for (int i = 0; i < lo.S; ++i) f[lo.block(el, q) + d * lo.S + i] += (c * msum) * nsum[i];
        }
    }
  }
  const Grid& m = ops.mesh;
  if (spec.beam == 1) {  // +z pencil beam, transport.cpp:129-178 (3D only)
    if (m.dim != 3) throw std::invalid_argument("assemble_rhs: pencil beam needs 3D");
    if (!(spec.x0 >= 0 && spec.x0 < spec.x1 && spec.x1 <= m.box && spec.y0 >= 0 &&
          spec.y0 < spec.y1 && spec.y1 <= m.box))
      throw std::invalid_argument("assemble_rhs: beam footprint outside boundary");
    const Vec3 pole{0, 0, 1};
    std::vector<std::pair<int, Vec3>> recv;
    for (int q = 0; q < lo.n_patch; ++q) {
      const Patch& patch = ops.angular.patch(ops.angular.leaves[q]);
      if (!patch_contains(patch, pole)) continue;
      Vec3 psi{1.0, 0, 0};
      if (ops.kind == BasisKind::Lin) psi = barycentric(patch, pole);
      recv.push_back({q, psi});
    }
    if (recv.empty()) throw std::logic_error("assemble_rhs: no patch holds the beam");
    const double share = spec.strength / double(recv.size());
    for (int iy = 0; iy < m.ny; ++iy) {
      const double ylo = iy * m.hy, yhi = ylo + m.hy;
      const double b0 = std::max(ylo, spec.y0), b1 = std::min(yhi, spec.y1);
      if (b1 <= b0) continue;
      for (int ix = 0; ix < m.nx; ++ix) {
        const double xlo = ix * m.hx, xhi = xlo + m.hx;
        const double a0 = std::max(xlo, spec.x0), a1 = std::min(xhi, spec.x1);
        if (a1 <= a0) continue;
        const int el = m.index(ix, iy, 0);
        Vec t(lo.S);
        if (ops.p == 0) t[0] = (a1 - a0) * (b1 - b0);
        else {
          const auto tx = shape_integrals(a0 - xlo, a1 - xlo, m.hx);
          const auto ty = shape_integrals(b0 - ylo, b1 - ylo, m.hy);
          for (int i = 0; i < 8; ++i) t[i] = ((i >> 2) & 1) ? 0.0 : tx[i & 1] * ty[(i >> 1) & 1];
        }
        for (const auto& [q, psi] : recv)
          for (int d = 0; d < lo.D; ++d)
            for (int i = 0; i < lo.S; ++i) f[lo.block(el, q) + d * lo.S + i] += (share * psi[d]) * t[i];
      }
    }
  } else if (spec.beam == 2) {
    // EXTENSION (config 4): unit incoming angular flux on every in-cone patch
    // through the x = 0 face; enters as the upwind term -C_{q,x} psi_b with a
    // ghost neighbour whose every dof is 1.
    Vec ones(size_t(lo.D) * lo.S, 1.0);
    for (int q = 0; q < lo.n_patch; ++q) {
      const Patch& patch = ops.angular.patch(ops.angular.leaves[q]);
      if (!patch_in_cone(patch, spec.cone_half_angle_deg)) continue;
      if (ops.inflow_face[q][0] != 0) continue;  // needs Omega_x > 0
      for (int iz = 0; iz < m.nz; ++iz)
        for (int iy = 0; iy < m.ny; ++iy) {
          const int el = m.index(0, iy, iz);
          matvec_add(ops.inflow[q][0], ones.data(), f.data() + lo.block(el, q), -spec.strength);
        }
    }
  }
  return f;
}

Vec scalar_flux(const ProblemOperators& ops, const double* phi) {  // harness.cpp:183-205
  const Layout& lay = ops.layout;
  Vec nsum(lay.S, 0.0), out(lay.n_el, 0.0);
  for (int i = 0; i < lay.S; ++i)
    for (int j = 0; j < lay.S; ++j) nsum[i] += ops.em.N(i, j);
  std::vector<Vec> msum(lay.n_patch, Vec(lay.D, 0.0));
  for (int q = 0; q < lay.n_patch; ++q)
    for (int d = 0; d < lay.D; ++d)
      for (int e = 0; e < lay.D; ++e) msum[q][d] += ops.pops[q].M(d, e);
  const double vol = ops.mesh.volume();
  for (int el = 0; el < lay.n_el; ++el) {
    double integral = 0;
    for (int q = 0; q < lay.n_patch; ++q) {
      const double* blk = phi + lay.block(el, q);
      for (int d = 0; d < lay.D; ++d) {
        double bn = 0;
        for (int i = 0; i < lay.S; ++i) bn += blk[d * lay.S + i] * nsum[i];
        integral += msum[q][d] * bn;
      }
    }
    out[el] = integral / vol;
  }
  return out;
}

// ============================================================ sweeps.cpp
SweepPlan build_sweep_plan(const ProblemOperators& ops) {  // sweeps.cpp:7-18
  SweepPlan plan;
  for (int oct = 0; oct < 8; ++oct) plan.order[oct] = sweep_order(ops.mesh, oct);
  const int P = ops.layout.n_patch;
  for (int q = 0; q < P; ++q) plan.patches[ops.angular.patch(ops.angular.leaves[q]).octant].push_back(q);
  plan.lu.resize(ops.diag.size());
  for (size_t m = 0; m < ops.diag.size(); ++m)
    for (int q = 0; q < P; ++q) plan.lu[m].emplace_back(ops.diag[m][q]);
  return plan;
}

void standard_sweep(const SweepPlan& plan, const ProblemOperators& ops, const double* rhs,
                    double* z, int q_begin, int q_end) {  // :20-42
  const Layout& lo = ops.layout;
  const int bs = lo.D * lo.S;
  if (q_end < 0) q_end = lo.n_patch;
#pragma omp parallel for schedule(dynamic)
  for (int q = q_begin; q < q_end; ++q) {
    const int oct = ops.angular.patch(ops.angular.leaves[q]).octant;
    std::vector<double> r(bs);
    for (const int el : plan.order[oct]) {
      for (int i = 0; i < bs; ++i) r[i] = rhs[lo.block(el, q) + i];
      for (int xi = 0; xi < ops.mesh.dim; ++xi) {
        const int up = ops.mesh.neighbor(el, ops.inflow_face[q][xi]);
        if (up < 0) continue;
        matvec_add(ops.inflow[q][xi], z + lo.block(up, q), r.data(), -1.0);
      }
      plan.lu[ops.mat[el]][q].solve(r.data(), z + lo.block(el, q));
    }
  }
}

void coarse_scatter_sweep(const SweepPlan& plan, const ProblemOperators& ops, const double* rhs,
                          int nu, double* phi) {  // :51-104
  const Layout& lo = ops.layout;
  if (nu <= 0) return;
  const int D = lo.D, S = lo.S, bs = D * S;
  const int nmat = int(ops.kernels.size());
  std::vector<Vec> sig;
  for (const auto& k : ops.kernels) sig.push_back(sigma_by_harmonic(k, k.N));
  const int H = int(sig[0].size());
  const Mat& X = ops.coup.X;
  // fold the self-scatter block into each diagonal solve (:60-72)
  std::vector<std::vector<LU>> lu(nmat);
  for (int m = 0; m < nmat; ++m)
    for (int q = 0; q < lo.n_patch; ++q) {
      Mat B = ops.diag[m][q];
      for (int a = 0; a < D; ++a)
        for (int d = 0; d < D; ++d) {
          double sq = 0;
          for (int h = 0; h < H; ++h) sq += X(q * D + a, h) * sig[m][h] * X(q * D + d, h);
          for (int l = 0; l < S; ++l)
            for (int i = 0; i < S; ++i) B(a * S + l, d * S + i) -= sq * ops.em.N(l, i);
        }
      lu[m].emplace_back(B);
    }
  // per-element moments (:74-79)
  std::vector<Vec> mom(lo.n_el, Vec(size_t(H) * S, 0.0));
  for (int el = 0; el < lo.n_el; ++el) {
    const double* chunk = phi + lo.element(el);
    for (int r = 0; r < lo.n_patch * D; ++r)
      for (int h = 0; h < H; ++h)
        for (int i = 0; i < S; ++i) mom[el][h * S + i] += X(r, h) * chunk[r * S + i];
  }
  std::vector<double> r(bs), znew(bs), t(size_t(H) * S);
  for (int pass = 0; pass < nu; ++pass)  // :83-103
    for (int oct = 0; oct < 8; ++oct)
      for (const int el : plan.order[oct])
        for (const int q : plan.patches[oct]) {
          const Vec& sg = sig[ops.mat[el]];
          for (int i = 0; i < bs; ++i) r[i] = rhs[lo.block(el, q) + i];
          for (int xi = 0; xi < ops.mesh.dim; ++xi) {
            const int up = ops.mesh.neighbor(el, ops.inflow_face[q][xi]);
            if (up < 0) continue;
            matvec_add(ops.inflow[q][xi], phi + lo.block(up, q), r.data(), -1.0);
          }
          double* zold = phi + lo.block(el, q);
          // t = sig * (mom - X_q^T zold)   (H x S)
          for (int h = 0; h < H; ++h)
            for (int i = 0; i < S; ++i) {
              double xz = 0;
              for (int d = 0; d < D; ++d) xz += X(q * D + d, h) * zold[d * S + i];
              t[h * S + i] = sg[h] * (mom[el][h * S + i] - xz);
            }
          // r += X_q t N
          for (int a = 0; a < D; ++a) {
            double xt[8] = {0};
            for (int i = 0; i < S; ++i)
              for (int h = 0; h < H; ++h) xt[i] += X(q * D + a, h) * t[h * S + i];
            for (int i = 0; i < S; ++i) {
              double acc = 0;
              for (int j = 0; j < S; ++j) acc += xt[j] * ops.em.N(j, i);
              r[a * S + i] += acc;
            }
          }
          lu[ops.mat[el]][q].solve(r.data(), znew.data());
          for (int h = 0; h < H; ++h)
            for (int i = 0; i < S; ++i) {
              double dz = 0;
              for (int d = 0; d < D; ++d) dz += X(q * D + d, h) * (znew[d * S + i] - zold[d * S + i]);
              mom[el][h * S + i] += dz;
            }
          for (int i = 0; i < bs; ++i) zold[i] = znew[i];
        }
}

void smoother_step(const SweepPlan& plan, const ProblemOperators& ops, const double* f, int order,
                   double* phi) {  // :106-113
  const size_t n = ops.layout.size();
  Vec r(n);
  apply_A_into(ops, phi, order, r.data());
  for (size_t i = 0; i < n; ++i) r[i] = f[i] - r[i];
  standard_sweep(plan, ops, r.data(), r.data());
  for (size_t i = 0; i < n; ++i) phi[i] += r[i];
}

// ============================================================ multigrid.cpp
namespace {
std::vector<ScatterKernel> truncate_kernels(const std::vector<ScatterKernel>& ks, int nr) {  // :11-16
  std::vector<ScatterKernel> out;
  for (const auto& k : ks) {
    ScatterKernel t = k;
    t.N = nr;
    t.moments.assign(k.moments.begin(), k.moments.begin() + nr + 1);
    out.push_back(t);  // sigma_t keeps the full-order removal
  }
  return out;
}

std::array<double, 3> corner_weights(const Patch& parent, const IVec3& v) {  // :20-35
  const auto& a = parent.flat[0];
  const auto& b = parent.flat[1];
  const auto& c = parent.flat[2];
  if (v == a) return {1, 0, 0};
  if (v == b) return {0, 1, 0};
  if (v == c) return {0, 0, 1};
  const IVec3 w{2 * v[0], 2 * v[1], 2 * v[2]};
  auto s = [](const IVec3& x, const IVec3& y) { return IVec3{x[0] + y[0], x[1] + y[1], x[2] + y[2]}; };
  if (w == s(a, b)) return {0.5, 0.5, 0};
  if (w == s(b, c)) return {0, 0.5, 0.5};
  if (w == s(a, c)) return {0.5, 0, 0.5};
  throw std::logic_error("corner_weights: vertex not nested in parent");
}
}  // namespace

int nr_default(int N) {  // :39-49
  switch (N) {
    case 4: return 2;
    case 8: return 4;
    case 12: return 6;
    case 16: return 7;
    case 20: return 8;
    case 24: return 9;
    default: return std::min(9, (N + 1) / 2);
  }
}

MgHierarchy build_hierarchy(const ProblemOperators& fine, const CycleSpec& cycle) {  // :51-98
  MgHierarchy h;
  h.cycle = cycle;
  h.nr = cycle.nr < 0 ? fine.N : cycle.nr;
  if (h.nr > fine.N) throw std::invalid_argument("build_hierarchy: nr exceeds N");
  const auto kr = truncate_kernels(fine.kernels, h.nr);
  const int L = fine.angular.max_level;
  // EXTENSION: keep only the n_levels finest angular levels
  const int nlev = cycle.n_levels <= 0 ? L + 1 : std::min(cycle.n_levels, L + 1);
  const int lmin = L + 1 - nlev;
  h.level.resize(nlev);
  for (int i = 0; i < nlev; ++i) {
    const int l = lmin + i;
    const AngularMesh mesh = l == L ? fine.angular : coarsen_to_level(fine.angular, l);
    h.level[i].ops = build_operators(fine.mesh, mesh, fine.kind, fine.p, kr, fine.mat);
    h.level[i].plan = build_sweep_plan(h.level[i].ops);
  }
  const int D = dofs_per_patch(fine.kind);
  for (int i = 1; i < nlev; ++i) {
    const AngularMesh& cm = h.level[i - 1].ops.angular;
    const AngularMesh& fm = h.level[i].ops.angular;
    std::unordered_map<int, int> coarse_pos;
    for (int c = 0; c < cm.n_leaves(); ++c) coarse_pos[cm.leaves[c]] = c;
    auto& up = h.level[i].up;
    up.resize(fm.n_leaves());
    for (int q = 0; q < fm.n_leaves(); ++q) {
      const Patch& p = fm.patch(fm.leaves[q]);
      if (auto it = coarse_pos.find(p.id); it != coarse_pos.end()) {
        up[q] = {it->second, Mat::identity(D)};
        continue;
      }
      const auto it = coarse_pos.find(p.parent);
      if (it == coarse_pos.end()) throw std::logic_error("build_hierarchy: meshes are not nested");
      Mat B(D, D);
      if (fine.kind == BasisKind::Const) B(0, 0) = 1.0;
      else {
        const Patch& parent = cm.patch(p.parent);
        for (int d = 0; d < 3; ++d) {
          auto w = corner_weights(parent, p.flat[d]);
          for (int e = 0; e < 3; ++e) B(d, e) = w[e];
        }
      }
      up[q] = {it->second, std::move(B)};
    }
  }
  return h;
}

Vec prolongate(const MgHierarchy& h, int l, const double* coarse) {  // :100-117
  if (l < 1 || l >= int(h.level.size())) throw std::invalid_argument("prolongate: level out of range");
  const Layout& lf = h.level[l].ops.layout;
  const Layout& lc = h.level[l - 1].ops.layout;
  Vec fine(lf.size(), 0.0);
#pragma omp parallel for schedule(static)
  for (int el = 0; el < lf.n_el; ++el)
    for (int q = 0; q < lf.n_patch; ++q) {
      const TransferBlock& t = h.level[l].up[q];
      double* dst = fine.data() + lf.block(el, q);
      const double* src = coarse + lc.block(el, t.coarse);
      for (int d = 0; d < lf.D; ++d)
        for (int i = 0; i < lf.S; ++i) {
          double acc = 0;
          for (int e = 0; e < lc.D; ++e) acc += t.B(d, e) * src[e * lc.S + i];
          dst[d * lf.S + i] = acc;
        }
    }
  return fine;
}

Vec restrict_residual(const MgHierarchy& h, int l, const double* fine) {  // :119-136
  if (l < 1 || l >= int(h.level.size())) throw std::invalid_argument("restrict_residual: level out of range");
  const Layout& lf = h.level[l].ops.layout;
  const Layout& lc = h.level[l - 1].ops.layout;
  Vec coarse(lc.size(), 0.0);
#pragma omp parallel for schedule(static)
  for (int el = 0; el < lf.n_el; ++el)
    for (int q = 0; q < lf.n_patch; ++q) {
      const TransferBlock& t = h.level[l].up[q];
      const double* src = fine + lf.block(el, q);
      double* dst = coarse.data() + lc.block(el, t.coarse);
      for (int e = 0; e < lc.D; ++e)
        for (int i = 0; i < lf.S; ++i) {
          double acc = 0;
          for (int d = 0; d < lf.D; ++d) acc += t.B(d, e) * src[d * lf.S + i];
          dst[e * lc.S + i] += acc;
        }
    }
  return coarse;
}

void lmg_vcycle(const MgHierarchy& h, int l, const double* f, double* phi) {  // :138-170
  const MgLevel& lev = h.level[l];
  const size_t n = lev.ops.layout.size();
  if (l == 0) {
    if (h.cycle.coarse_tol > 0) {
      double fnorm = 0;
      for (size_t i = 0; i < n; ++i) fnorm += f[i] * f[i];
      fnorm = std::sqrt(fnorm);
      Vec r(n);
      for (int s = 0; s < 200; ++s) {
        coarse_scatter_sweep(lev.plan, lev.ops, f, 1, phi);
        apply_A_into(lev.ops, phi, lev.ops.N, r.data());
        double rn = 0;
        for (size_t i = 0; i < n; ++i) rn += (f[i] - r[i]) * (f[i] - r[i]);
        if (std::sqrt(rn) <= h.cycle.coarse_tol * fnorm) break;
      }
    } else {
      coarse_scatter_sweep(lev.plan, lev.ops, f, h.cycle.coarse_sweeps, phi);
    }
    return;
  }
  for (int s = 0; s < h.cycle.nu_pre; ++s) smoother_step(lev.plan, lev.ops, f, h.nr, phi);
  Vec r(n);
  apply_A_into(lev.ops, phi, h.nr, r.data());
  for (size_t i = 0; i < n; ++i) r[i] = f[i] - r[i];
  const Vec rc = restrict_residual(h, l, r.data());
  Vec ec(rc.size(), 0.0);
  lmg_vcycle(h, l - 1, rc.data(), ec.data());
  const Vec pe = prolongate(h, l, ec.data());
  for (size_t i = 0; i < n; ++i) phi[i] += pe[i];
  for (int s = 0; s < h.cycle.nu_post; ++s) smoother_step(lev.plan, lev.ops, f, h.nr, phi);
}

Vec mg_apply(const MgHierarchy& h, const double* r) {  // :172-176
  Vec phi(h.level.back().ops.layout.size(), 0.0);
  lmg_vcycle(h, int(h.level.size()) - 1, r, phi.data());
  return phi;
}

// ============================================================ krylov.cpp
std::pair<Vec, SolveReport> bicgstab(const LinearOp& apply_op, const LinearOp& precond,
                                     const Vec& b, double tol, int max_iter) {  // krylov.cpp:9-93
  if (tol <= 0) throw std::invalid_argument("bicgstab: tol must be positive");
  const auto t0 = std::chrono::steady_clock::now();
  SolveReport rep;
  const size_t n = b.size();
  Vec x(n, 0.0);
  const double bnorm = vnorm(b);
  auto finish = [&](const Vec& sol) {
    if (bnorm > 0) {
      Vec ax = apply_op(sol);
      for (size_t i = 0; i < n; ++i) ax[i] = b[i] - ax[i];
      rep.final_residual = vnorm(ax) / bnorm;
    } else rep.final_residual = 0.0;
    rep.converged = rep.final_residual < tol;
    rep.wall_time = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return std::make_pair(sol, rep);
  };
  if (bnorm == 0.0) {
    rep.converged = true;
    return {x, rep};
  }
  Vec r = b;
  const Vec rhat = r;
  Vec p(n, 0.0), v(n, 0.0), s(n);
  double rho = 1, alpha = 1, omega = 1;
  for (int it = 1; it <= max_iter; ++it) {
    const double rho1 = vdot(rhat, r);
    if (rho1 == 0.0 || omega == 0.0) {
      rep.breakdown = true;
      return finish(x);
    }
    const double beta = (rho1 / rho) * (alpha / omega);
    rho = rho1;
    for (size_t i = 0; i < n; ++i) p[i] = r[i] + beta * (p[i] - omega * v[i]);
    const Vec phat = precond(p);
    ++rep.preconditioner_applications;
    v = apply_op(phat);
    const double rv = vdot(rhat, v);
    if (rv == 0.0) {
      rep.breakdown = true;
      return finish(x);
    }
    alpha = rho / rv;
    for (size_t i = 0; i < n; ++i) s[i] = r[i] - alpha * v[i];
    for (size_t i = 0; i < n; ++i) x[i] += alpha * phat[i];
    const double snorm = vnorm(s) / bnorm;
    if (std::isnan(snorm)) throw std::runtime_error("bicgstab: NaN residual");
    if (snorm < tol) {
      rep.iterations = it;
      rep.residual_history.push_back(snorm);
      return finish(x);
    }
    const Vec shat = precond(s);
    ++rep.preconditioner_applications;
    const Vec t = apply_op(shat);
    const double tt = vdot(t, t);
    if (tt == 0.0) {
      rep.breakdown = true;
      return finish(x);
    }
    omega = vdot(t, s) / tt;
    for (size_t i = 0; i < n; ++i) x[i] += omega * shat[i];
    for (size_t i = 0; i < n; ++i) r[i] = s[i] - omega * t[i];
    const double rnorm = vnorm(r) / bnorm;
    if (std::isnan(rnorm)) throw std::runtime_error("bicgstab: NaN residual");
    rep.iterations = it;
    rep.residual_history.push_back(rnorm);
    if (rnorm < tol) return finish(x);
  }
  return finish(x);
}

// EXTENSION: right-preconditioned GMRES(m) with classical Gram-Schmidt and one
// reorthogonalisation pass (CGS2), Givens rotations, x0 = 0. The GPU solver
// runs exactly this algorithm; reporting follows krylov.hpp:15-24.
std::pair<Vec, SolveReport> gmres(const LinearOp& A, const LinearOp& M, const Vec& b, double tol,
                                  int max_iter, int restart, double) {
  if (tol <= 0) throw std::invalid_argument("gmres: tol must be positive");
  if (restart < 1) throw std::invalid_argument("gmres: restart must be positive");
  const auto t0 = std::chrono::steady_clock::now();
  SolveReport rep;
  const size_t n = b.size();
  Vec x(n, 0.0);
  const double bnorm = vnorm(b);
  if (bnorm == 0.0) {
    rep.converged = true;
    return {x, rep};
  }
  const int m = restart;
  std::vector<Vec> V(m + 1, Vec(n));
  Vec r = b, w(n);
  int it = 0;
  bool done = false;
  while (!done) {
    const double beta = vnorm(r);
    for (size_t i = 0; i < n; ++i) V[0][i] = r[i] / beta;
    std::vector<double> g(m + 1, 0.0), cs(m, 0.0), sn(m, 0.0);
    std::vector<std::vector<double>> H(m, std::vector<double>(m + 1, 0.0));  // H[j][i]
    g[0] = beta;
    int k = 0;
    for (int j = 0; j < m; ++j) {
      ++it;
      const Vec z = M(V[j]);
      ++rep.preconditioner_applications;
      w = A(z);
      auto& h = H[j];
      for (int pass = 0; pass < 2; ++pass) {  // CGS2
        std::vector<double> c(j + 1);
        for (int i = 0; i <= j; ++i) c[i] = vdot(V[i], w);
        for (int i = 0; i <= j; ++i) {
          for (size_t t = 0; t < n; ++t) w[t] -= c[i] * V[i][t];
          h[i] += c[i];
        }
      }
      h[j + 1] = vnorm(w);
      if (h[j + 1] != 0.0)
        for (size_t t = 0; t < n; ++t) V[j + 1][t] = w[t] / h[j + 1];
      for (int i = 0; i < j; ++i) {  // apply previous rotations
        const double tmp = cs[i] * h[i] + sn[i] * h[i + 1];
        h[i + 1] = -sn[i] * h[i] + cs[i] * h[i + 1];
        h[i] = tmp;
      }
      const double den = std::hypot(h[j], h[j + 1]);
      cs[j] = den == 0.0 ? 1.0 : h[j] / den;
      sn[j] = den == 0.0 ? 0.0 : h[j + 1] / den;
      const double hj1 = h[j + 1];
      h[j] = cs[j] * h[j] + sn[j] * hj1;
      h[j + 1] = 0.0;
      g[j + 1] = -sn[j] * g[j];
      g[j] = cs[j] * g[j];
      const double res = std::abs(g[j + 1]) / bnorm;
      if (std::isnan(res)) throw std::runtime_error("gmres: NaN residual");
      rep.iterations = it;
      rep.residual_history.push_back(res);
      k = j + 1;
      if (res < tol || it >= max_iter || hj1 == 0.0) {
        done = res < tol || it >= max_iter;
        if (hj1 == 0.0 && !(res < tol)) rep.breakdown = true, done = true;
        break;
      }
    }
    // y = H^{-1} g (upper triangular k x k), x += M (V y)
    std::vector<double> y(k, 0.0);
    for (int i = k - 1; i >= 0; --i) {
      double s = g[i];
      for (int jj = i + 1; jj < k; ++jj) s -= H[jj][i] * y[jj];
      y[i] = s / H[i][i];
    }
    Vec u(n, 0.0);
    for (int jj = 0; jj < k; ++jj)
      for (size_t t = 0; t < n; ++t) u[t] += y[jj] * V[jj][t];
    const Vec du = M(u);
    ++rep.preconditioner_applications;
    for (size_t t = 0; t < n; ++t) x[t] += du[t];
    if (done) break;
    const Vec ax = A(x);
    for (size_t t = 0; t < n; ++t) r[t] = b[t] - ax[t];
  }
  Vec ax = A(x);
  for (size_t t = 0; t < n; ++t) ax[t] = b[t] - ax[t];
  rep.final_residual = vnorm(ax) / bnorm;
  rep.converged = rep.final_residual < tol;
  rep.wall_time = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return {x, rep};
}

// ============================================================ tests/support/oracles.cpp
Mat dense_transport_matrix(const ProblemOperators& ops) {  // oracles.cpp:29-70
  const Layout& lo = ops.layout;
  const int S = lo.S, D = lo.D;
  const int n = int(lo.size());
  Mat L(n, n);
  for (int el = 0; el < lo.n_el; ++el)
    for (int q = 0; q < lo.n_patch; ++q) {
      const Patch& patch = ops.angular.patch(ops.angular.leaves[q]);
      const PatchOperators& po = ops.pops[q];
      const int row0 = int(lo.block(el, q));
      const double st = ops.kernels[ops.mat[el]].sigma_t;
      for (int m = 0; m < D; ++m)
        for (int d = 0; d < D; ++d)
          for (int l = 0; l < S; ++l)
            for (int i = 0; i < S; ++i) {
              double v = st * po.M(m, d) * ops.em.N(l, i);
              for (int xi = 0; xi < ops.mesh.dim; ++xi) v -= po.A[xi](m, d) * ops.em.V[xi](l, i);
              L(row0 + m * S + l, row0 + d * S + i) += v;
            }
      for (int f = 0; f < ops.mesh.n_faces(); ++f) {
        Vec3 normal{0, 0, 0};
        normal[f / 2] = (f % 2) ? 1.0 : -1.0;
        const auto [a_out, a_in] = face_split(ops.kind, patch, normal);
        for (int m = 0; m < D; ++m)
          for (int d = 0; d < D; ++d)
            for (int l = 0; l < S; ++l)
              for (int i = 0; i < S; ++i) L(row0 + m * S + l, row0 + d * S + i) += a_out(m, d) * ops.em.F_self[f](l, i);
        const int nb = ops.mesh.neighbor(el, f);
        if (nb < 0) continue;
        const int col0 = int(lo.block(nb, q));
        for (int m = 0; m < D; ++m)
          for (int d = 0; d < D; ++d)
            for (int l = 0; l < S; ++l)
              for (int i = 0; i < S; ++i) L(row0 + m * S + l, col0 + d * S + i) += a_in(m, d) * ops.em.F_neigh[f](l, i);
      }
    }
  return L;
}

Mat dense_scatter_matrix(const ProblemOperators& ops, int max_order) {  // oracles.cpp:72-91
  const Layout& lo = ops.layout;
  const int S = lo.S, D = lo.D;
  const int n = int(lo.size());
  Mat Sm(n, n);
  for (int el = 0; el < lo.n_el; ++el) {
    const Vec sig = sigma_by_harmonic(ops.kernels[ops.mat[el]], max_order);
    for (int q = 0; q < lo.n_patch; ++q)
      for (int p = 0; p < lo.n_patch; ++p)
        for (int m = 0; m < D; ++m)
          for (int d = 0; d < D; ++d) {
            double ang = 0;
            for (size_t h = 0; h < sig.size(); ++h) ang += sig[h] * ops.coup.X(q * D + m, h) * ops.coup.X(p * D + d, h);
            for (int l = 0; l < S; ++l)
              for (int i = 0; i < S; ++i) Sm(int(lo.block(el, q)) + m * S + l, int(lo.block(el, p)) + d * S + i) += ang * ops.em.N(l, i);
          }
  }
  return Sm;
}

}  // namespace oracle
