// Host tables of the reference-shape path (generic.hpp): build_operators,
// build_sweep_plan, build_hierarchy and assemble_rhs for 2D / 3D cells with p0 or linear
// dofs and the Const or Lin angular basis. Dense per-patch blocks of size bs = D*S, row
// (d, i) -> d*S + i, as the reference's kron(angular, spatial) products give them.
#include "generic.hpp"

#include <algorithm>
#include <cmath>
#include <numbers>
#include <stdexcept>
#include <unordered_map>

namespace stamg_b200 {
namespace gen {

namespace {

constexpr double kPi = std::numbers::pi;

using Mat = std::vector<double>;  // row-major square or rectangular, sizes carried by the caller

// C (ra*rb x ca*cb) = A (ra x ca) kron B (rb x cb)   (kron.hpp:7-14)
Mat kron(const Mat& A, int ra, int ca, const Mat& B, int rb, int cb) {
  Mat C(size_t(ra) * rb * ca * cb);
  for (int i = 0; i < ra; ++i)
    for (int j = 0; j < ca; ++j)
      for (int k = 0; k < rb; ++k)
        for (int l = 0; l < cb; ++l) C[(size_t(i) * rb + k) * (ca * cb) + j * cb + l] = A[i * ca + j] * B[k * cb + l];
  return C;
}

// element matrices (spatial_disc.cpp:45-88; 2D: the same 1D factors without the z factor)
struct Element {
  int S = 1;
  Mat N, V[3], Fs[6], Fn[6];
};

Element element_matrices(int dim, int p, double hx, double hy, double hz) {
  Element e;
  if (p == 0) {
    e.S = 1;
    const double vol = dim == 3 ? hx * hy * hz : hx * hy;
    const double area[3] = {dim == 3 ? hy * hz : hy, dim == 3 ? hx * hz : hx, hx * hy};
    e.N = {vol};
    for (int xi = 0; xi < dim; ++xi) {
      e.V[xi] = {0.0};
      for (int s = 0; s < 2; ++s) e.Fs[2 * xi + s] = {area[xi]}, e.Fn[2 * xi + s] = {area[xi]};
    }
    return e;
  }
  auto mass = [](double h) { return Mat{2 * h / 6, h / 6, h / 6, 2 * h / 6}; };
  const Mat mx = mass(hx), my = mass(hy), mz = mass(hz);
  const Mat g{-0.5, -0.5, 0.5, 0.5};  // int phi_l' phi_i
  const Mat t_lo{1, 0, 0, 0}, t_hi{0, 0, 0, 1}, c_lo{0, 1, 0, 0}, c_hi{0, 0, 1, 0};
  // dof i = ix + 2 iy (+ 4 iz): the x factor is innermost
  auto prod = [&](const Mat& az, const Mat& ay, const Mat& ax) {
    const Mat yx = kron(ay, 2, 2, ax, 2, 2);
    return dim == 3 ? kron(az, 2, 2, yx, 4, 4) : yx;
  };
  e.S = dim == 3 ? 8 : 4;
  e.N = prod(mz, my, mx);
  e.V[0] = prod(mz, my, g), e.V[1] = prod(mz, g, mx);
  if (dim == 3) e.V[2] = prod(g, my, mx);
  for (int xi = 0; xi < dim; ++xi) {
    auto face = [&](const Mat& t) { return xi == 0 ? prod(mz, my, t) : xi == 1 ? prod(mz, t, mx) : prod(t, my, mx); };
    e.Fs[2 * xi] = face(t_lo), e.Fs[2 * xi + 1] = face(t_hi);
    e.Fn[2 * xi] = face(c_lo), e.Fn[2 * xi + 1] = face(c_hi);
  }
  return e;
}

// dense inverse by partial-pivot Gauss-Jordan (the reference solves with PartialPivLU,
// sweeps.cpp:15,39; applying the inverse differs from it at rounding level)
Mat inverse(const Mat& A, int n) {
  std::vector<long double> m(size_t(n) * 2 * n, 0.0L);
  for (int i = 0; i < n; ++i) {
    for (int j = 0; j < n; ++j) m[size_t(i) * 2 * n + j] = A[size_t(i) * n + j];
    m[size_t(i) * 2 * n + n + i] = 1.0L;
  }
  for (int k = 0; k < n; ++k) {
    int p = k;
    for (int i = k + 1; i < n; ++i)
      if (std::abs(m[size_t(i) * 2 * n + k]) > std::abs(m[size_t(p) * 2 * n + k])) p = i;
    if (m[size_t(p) * 2 * n + k] == 0.0L) throw std::invalid_argument("singular diagonal block");
    if (p != k)
      for (int j = 0; j < 2 * n; ++j) std::swap(m[size_t(k) * 2 * n + j], m[size_t(p) * 2 * n + j]);
    const long double d = 1.0L / m[size_t(k) * 2 * n + k];
    for (int j = 0; j < 2 * n; ++j) m[size_t(k) * 2 * n + j] *= d;
    for (int i = 0; i < n; ++i) {
      if (i == k) continue;
      const long double f = m[size_t(i) * 2 * n + k];
      if (f == 0.0L) continue;
      for (int j = 0; j < 2 * n; ++j) m[size_t(i) * 2 * n + j] -= f * m[size_t(k) * 2 * n + j];
    }
  }
  Mat R(size_t(n) * n);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) R[size_t(i) * n + j] = double(m[size_t(i) * 2 * n + n + j]);
  return R;
}

// barycentric coordinates of a direction in a patch's flat triangle (angular_disc.cpp:19-33):
// solve [a b c] mu = omega, normalise; false when omega is outside (mu sum <= 0 or min < -tol)
bool barycentric(const SphereTree& t, int id, const double* om, double* mu, double tol = 1e-12) {
  const double inv = 1.0 / double(SphereTree::kScale);
  double V[9];
  for (int c = 0; c < 3; ++c)
    for (int r = 0; r < 3; ++r) V[r * 3 + c] = double(t.flat[id][3 * c + r]) * inv;
  const Mat Vi = inverse(Mat(V, V + 9), 3);
  double s = 0;
  for (int r = 0; r < 3; ++r) {
    mu[r] = Vi[r * 3] * om[0] + Vi[r * 3 + 1] * om[1] + Vi[r * 3 + 2] * om[2];
    s += mu[r];
  }
  if (s <= 0) return false;
  for (int r = 0; r < 3; ++r) mu[r] /= s;
  return std::min({mu[0], mu[1], mu[2]}) >= -tol;
}

// integral of the 1D nodal shapes over [a, b] inside [0, h] (transport.cpp:16-19)
void shape_integrals(double a, double b, double h, double* out) {
  const double len = b - a, quad = (b * b - a * a) / (2 * h);
  out[0] = len - quad, out[1] = quad;
}

}  // namespace

bool handles(const stamg_problem& s) { return !(s.dim == 2 && s.p == 1 && s.basis == 0); }

void validate(const Problem& pb) {
  const auto& s = pb.spec;
  if (s.dim != 2 && s.dim != 3) throw std::invalid_argument("build_hex_mesh: dim must be 2 or 3");
  if (s.p != 0 && s.p != 1) throw std::invalid_argument("element_matrices: p must be 0 or 1");
  if (s.basis != 0 && s.basis != 1) throw std::invalid_argument("unknown angular basis");
  if (s.nx < 1 || s.ny < 1 || (s.dim == 3 && s.nz < 1)) throw std::invalid_argument("build_hex_mesh: zero element count");
  if (s.box <= 0) throw std::invalid_argument("build_hex_mesh: box must be positive");
  if (s.N < 0) throw std::invalid_argument("scatter order < 0");
  if (s.nr > s.N) throw std::invalid_argument("build_hierarchy: nr exceeds N");
  if (s.n_mat != 1) throw std::invalid_argument("the reference-shape path has one global scatter kernel (transport.hpp:34)");
  if (s.beam != 0 && s.beam != 1) throw std::invalid_argument("the reference-shape path supports beam = 0 or 1 (+z pencil)");
  if (s.beam == 1 && s.dim != 3) throw std::invalid_argument("the +z pencil beam needs a 3D grid");
}

Tables build_level(const Problem& pb, const SphereTree& tree, int order, bool with_gs) {
  const auto& s = pb.spec;
  Tables L;
  L.dim = s.dim, L.nx = s.nx, L.ny = s.ny, L.nz = s.dim == 3 ? s.nz : 1;
  L.n_el = L.nx * L.ny * L.nz;
  L.D = s.basis == 1 ? 3 : 1;
  const double hx = s.box / s.nx, hy = s.box / s.ny, hz = s.dim == 3 ? s.box / s.nz : 1.0;
  const Element em = element_matrices(s.dim, s.p, hx, hy, hz);
  L.S = em.S, L.bs = L.D * L.S;
  L.P = int(tree.leaves.size()), L.order = order, L.H = (order + 1) * (order + 1);
  L.Nmat = em.N;
  const int P = L.P, D = L.D, S = L.S, bs = L.bs, H = L.H;
  L.leaf_id = tree.leaves;
  L.octant.resize(P);
  L.sig.assign(H, 0.0);
  for (int n = 0; n <= order; ++n)
    for (int o = -n; o <= n; ++o) L.sig[n * n + n + o] = pb.moments[n];
  L.X.assign(size_t(P) * D * H, 0.0);
  L.Bd.resize(size_t(P) * bs * bs);
  L.Binv.resize(size_t(P) * bs * bs);
  L.C.assign(size_t(P) * 3 * bs * bs, 0.0);
  L.M1.assign(size_t(P) * D, 0.0);
  if (with_gs) L.BinvGS.resize(size_t(P) * bs * bs);
  const int xbase = order > 12 ? 12 : 8;  // scatter.hpp:42
  std::vector<double> om, bary, w, Y(H);
  L.oct_ptr.assign(9, 0);
  for (int q = 0; q < P; ++q) {
    const int id = L.leaf_id[q], oct = tree.octant[id];
    L.octant[q] = oct;
    // patch operators M, A^xi (angular_disc.cpp:40-59)
    Mat M(size_t(D) * D, 0.0), A[3] = {Mat(size_t(D) * D, 0.0), Mat(size_t(D) * D, 0.0), Mat(size_t(D) * D, 0.0)};
    patch_rule(tree, id, patch_order(tree.level[id], 8), om, bary, w);
    for (size_t g = 0; g < w.size(); ++g) {
      double psi[3] = {1.0, 0.0, 0.0};
      if (D == 3) psi[0] = bary[3 * g], psi[1] = bary[3 * g + 1], psi[2] = bary[3 * g + 2];
      for (int a = 0; a < D; ++a)
        for (int b = 0; b < D; ++b) {
          const double outer = w[g] * (psi[a] * psi[b]);
          M[a * D + b] += outer;
          for (int xi = 0; xi < 3; ++xi) A[xi][a * D + b] += om[3 * g + xi] * outer;
        }
    }
    for (int a = 0; a < D; ++a)
      for (int b = 0; b < D; ++b) L.M1[size_t(q) * D + a] += M[a * D + b];
    // couplings X_q(d, h) = int psi_d Y_h (scatter.cpp:74-99)
    patch_rule(tree, id, patch_order(tree.level[id], xbase), om, bary, w);
    for (size_t g = 0; g < w.size(); ++g) {
      real_harmonics(order, &om[3 * g], Y.data());
      for (int d = 0; d < D; ++d) {
        const double pw = w[g] * (D == 3 ? bary[3 * g + d] : 1.0);
        double* Xr = &L.X[(size_t(q) * D + d) * H];
        for (int h = 0; h < H; ++h) Xr[h] += pw * Y[h];
      }
    }
    // fused blocks (transport.cpp:43-57)
    Mat B = kron(M, D, D, em.N, S, S);
    for (double& v : B) v *= pb.sigma_t[0];
    for (int xi = 0; xi < s.dim; ++xi) {
      const double sg = (oct >> xi) & 1 ? -1.0 : 1.0;
      const int fout = 2 * xi + (sg > 0 ? 1 : 0), fin = 2 * xi + (sg > 0 ? 0 : 1);
      const Mat kv = kron(A[xi], D, D, em.V[xi], S, S), kf = kron(A[xi], D, D, em.Fs[fout], S, S);
      const Mat kc = kron(A[xi], D, D, em.Fn[fin], S, S);
      for (int k = 0; k < bs * bs; ++k) {
        B[k] -= kv[k];
        B[k] += sg * kf[k];
        L.C[(size_t(q) * 3 + xi) * bs * bs + k] = -sg * kc[k];
      }
    }
    std::copy(B.begin(), B.end(), &L.Bd[size_t(q) * bs * bs]);
    const Mat Bi = inverse(B, bs);
    std::copy(Bi.begin(), Bi.end(), &L.Binv[size_t(q) * bs * bs]);
    if (with_gs) {  // self-scatter folded into the block (sweeps.cpp:61-72)
      Mat Bg = B;
      for (int m = 0; m < D; ++m)
        for (int d = 0; d < D; ++d) {
          double sq = 0;
          for (int h = 0; h < H; ++h) sq += L.X[(size_t(q) * D + m) * H + h] * L.sig[h] * L.X[(size_t(q) * D + d) * H + h];
          for (int i = 0; i < S; ++i)
            for (int j = 0; j < S; ++j) Bg[size_t(m * S + i) * bs + d * S + j] -= sq * em.N[i * S + j];
        }
      const Mat Bgi = inverse(Bg, bs);
      std::copy(Bgi.begin(), Bgi.end(), &L.BinvGS[size_t(q) * bs * bs]);
    }
  }
  for (int oct = 0; oct < 8; ++oct) {  // plan.patches (sweeps.cpp:14)
    L.oct_ptr[oct] = int(L.oct_patches.size());
    for (int q = 0; q < P; ++q)
      if (L.octant[q] == oct) L.oct_patches.push_back(q);
  }
  L.oct_ptr[8] = int(L.oct_patches.size());
  return L;
}

std::vector<Tables> build_hierarchy(const Problem& pb, const SphereTree& fine, int nr, int nlev) {
  const int Lmax = fine.max_level;
  nlev = nlev <= 0 ? Lmax + 1 : std::min(nlev, Lmax + 1);
  const int lmin = Lmax + 1 - nlev;
  std::vector<SphereTree> trees;
  std::vector<Tables> lv;
  for (int i = 0; i < nlev; ++i) {
    const int l = lmin + i;
    trees.push_back(l == Lmax ? fine : coarsen(fine, l));
    lv.push_back(gen::build_level(pb, trees.back(), nr, i == 0));
  }
  for (int i = 1; i < nlev; ++i) {  // transfer blocks (multigrid.cpp:68-96)
    const SphereTree& ft = trees[i];
    const Tables& C = lv[i - 1];
    Tables& L = lv[i];
    const int D = L.D;
    std::unordered_map<int, int> pos;
    for (int c = 0; c < C.P; ++c) pos[C.leaf_id[c]] = c;
    L.up.resize(L.P);
    L.upB.assign(size_t(L.P) * D * D, 0.0);
    for (int q = 0; q < L.P; ++q) {
      const int id = L.leaf_id[q];
      double* B = &L.upB[size_t(q) * D * D];
      auto it = pos.find(id);
      if (it != pos.end()) {  // the leaf is also a leaf of the coarser mesh: identity
        L.up[q] = it->second;
        for (int d = 0; d < D; ++d) B[d * D + d] = 1.0;
        continue;
      }
      const int par = ft.parent[id];
      it = pos.find(par);
      if (it == pos.end()) throw std::logic_error("build_hierarchy: meshes are not nested");
      L.up[q] = it->second;
      if (D == 1) {
        B[0] = 1.0;
        continue;
      }
      // Lin: exact barycentric coordinates of the child's corners in the parent triangle,
      // resolved on the integer lattice (vertex or edge midpoint; multigrid.cpp:20-35)
      const auto& pf = ft.flat[par];
      const auto& cf = ft.flat[id];
      for (int d = 0; d < 3; ++d) {
        const std::int64_t* v = &cf[3 * d];
        auto eq = [&](const std::int64_t* x, std::int64_t s0, const std::int64_t* a, const std::int64_t* b) {
          for (int r = 0; r < 3; ++r)
            if (s0 * x[r] != a[r] + (b ? b[r] : 0)) return false;
          return true;
        };
        const std::int64_t *a = &pf[0], *b = &pf[3], *c = &pf[6];
        double* row = &B[d * 3];
        if (eq(v, 1, a, nullptr)) row[0] = 1;
        else if (eq(v, 1, b, nullptr)) row[1] = 1;
        else if (eq(v, 1, c, nullptr)) row[2] = 1;
        else if (eq(v, 2, a, b)) row[0] = row[1] = 0.5;
        else if (eq(v, 2, b, c)) row[1] = row[2] = 0.5;
        else if (eq(v, 2, a, c)) row[0] = row[2] = 0.5;
        else throw std::logic_error("corner_weights: vertex not nested in parent");
      }
    }
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

std::vector<double> assemble_rhs(const Problem& pb, const Tables& t, const SphereTree& tree) {
  const auto& s = pb.spec;
  const int P = t.P, D = t.D, S = t.S, bs = t.bs;
  std::vector<double> f(size_t(t.n_el) * P * bs, 0.0);
  std::vector<double> nsum(S, 0.0);
  for (int i = 0; i < S; ++i)
    for (int j = 0; j < S; ++j) nsum[i] += t.Nmat[i * S + j];
  if (!pb.q_el.empty()) {  // isotropic volume source (transport.cpp:114-127)
    for (int el = 0; el < t.n_el; ++el) {
      if (pb.q_el[el] == 0.0) continue;
      const double c = pb.q_el[el] / (4.0 * kPi);
      for (int q = 0; q < P; ++q)
        for (int d = 0; d < D; ++d)
          for (int i = 0; i < S; ++i) f[(size_t(el) * P + q) * bs + d * S + i] += (c * t.M1[size_t(q) * D + d]) * nsum[i];
    }
  }
  if (s.beam == 1) {  // pencil beam along +z through the z = 0 footprint (transport.cpp:129-178)
    if (!(s.x0 >= 0 && s.x0 < s.x1 && s.x1 <= s.box && s.y0 >= 0 && s.y0 < s.y1 && s.y1 <= s.box))
      throw std::invalid_argument("assemble_rhs: beam footprint outside boundary");
    const double pole[3] = {0, 0, 1};
    std::vector<int> rq;
    std::vector<std::array<double, 3>> rpsi;
    for (int q = 0; q < P; ++q) {
      double mu[3];
      if (!barycentric(tree, t.leaf_id[q], pole, mu)) continue;
      rq.push_back(q);
      rpsi.push_back(D == 3 ? std::array<double, 3>{mu[0], mu[1], mu[2]} : std::array<double, 3>{1.0, 0.0, 0.0});
    }
    if (rq.empty()) throw std::logic_error("assemble_rhs: no patch holds the beam");
    const double share = s.strength / double(rq.size());
    const double hx = s.box / s.nx, hy = s.box / s.ny;
    for (int iy = 0; iy < s.ny; ++iy) {
      const double ylo = iy * hy, yhi = ylo + hy;
      const double b0 = std::max(ylo, s.y0), b1 = std::min(yhi, s.y1);
      if (b1 <= b0) continue;
      for (int ix = 0; ix < s.nx; ++ix) {
        const double xlo = ix * hx, xhi = xlo + hx;
        const double a0 = std::max(xlo, s.x0), a1 = std::min(xhi, s.x1);
        if (a1 <= a0) continue;
        const int el = iy * s.nx + ix;  // iz = 0
        std::vector<double> tv(S, 0.0);
        if (s.p == 0) {
          tv[0] = (a1 - a0) * (b1 - b0);
        } else {
          double tx[2], ty[2];
          shape_integrals(a0 - xlo, a1 - xlo, hx, tx);
          shape_integrals(b0 - ylo, b1 - ylo, hy, ty);
          for (int i = 0; i < S; ++i) tv[i] = ((i >> 2) & 1) ? 0.0 : tx[i & 1] * ty[(i >> 1) & 1];
        }
        for (size_t r = 0; r < rq.size(); ++r)
          for (int d = 0; d < D; ++d)
            for (int i = 0; i < S; ++i) f[(size_t(el) * P + rq[r]) * bs + d * S + i] += (share * rpsi[r][d]) * tv[i];
      }
    }
  }
  return f;
}

}  // namespace gen
}  // namespace stamg_b200
