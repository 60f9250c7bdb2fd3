// ORACLE — TEST INFRASTRUCTURE ONLY.
//
// Plain C++20 CPU restatement of the reference solver `stamg`
// (/root/reference/proj, arXiv 2010.04559 companion code) used as the parity
// checker for the B200 path. Only tests/, __graft_entry__.smoke() and
// bench.py's cpu_baseline / --impl reference leg may load it. The product
// library (paper_2010_04559_b200/) never links or calls anything here.
//
// The reference cannot be compiled in this image (Eigen3 and vendor/ are
// absent), so this file restates it without Eigen, following
// the cited reference lines. It keeps the reference's 3D / Lin generality so
// the reference's own unit-test identities can be re-run against it, and adds
// the extensions BASELINE.json needs (2D bilinear cells, HG moments, per-cell
// materials, GMRES, MG depth, cone mesh + x-face beam, block sources), each
// marked "EXTENSION".
#pragma once

#include <array>
#include <cstdint>
#include <functional>
#include <stdexcept>
#include <string>
#include <vector>

namespace oracle {

using Vec = std::vector<double>;
using IVec3 = std::array<std::int64_t, 3>;
using Vec3 = std::array<double, 3>;

// Row-major dense matrix (stands in for Eigen::MatrixXd / RowMat).
struct Mat {
  int r = 0, c = 0;
  std::vector<double> a;
  Mat() = default;
  Mat(int rows, int cols, double v = 0.0) : r(rows), c(cols), a(size_t(rows) * cols, v) {}
  double& operator()(int i, int j) { return a[size_t(i) * c + j]; }
  double operator()(int i, int j) const { return a[size_t(i) * c + j]; }
  static Mat identity(int n) {
    Mat m(n, n);
    for (int i = 0; i < n; ++i) m(i, i) = 1.0;
    return m;
  }
};

Mat kron(const Mat& A, const Mat& B);  // kron.hpp:7-14

// Partial-pivot LU (stands in for Eigen::PartialPivLU, sweeps.cpp:15,39).
struct LU {
  int n = 0;
  Mat lu;
  std::vector<int> piv;
  LU() = default;
  explicit LU(const Mat& A);
  void solve(const double* b, double* x) const;  // x may alias b
};

// ---------------------------------------------------------------- sphere mesh
// sphere_mesh.hpp:20-63
inline constexpr std::int64_t kFlatScale = std::int64_t(1) << 20;

struct Patch {
  int id = -1, level = 0, octant = 0, parent = -1;
  std::array<int, 4> kids{-1, -1, -1, -1};
  bool leaf = true;
  std::array<IVec3, 3> flat{};
  std::array<Vec3, 3> vert{};
};

struct AngularMesh {
  std::vector<Patch> all;
  std::vector<int> leaves;
  int max_level = 0;
  const Patch& patch(int id) const { return all[id]; }
  int n_leaves() const { return int(leaves.size()); }
  int leaf_pos(int id) const;
};

AngularMesh build_base_mesh();
void refine(AngularMesh& mesh, int patch_id);
AngularMesh build_uniform_mesh(int level);
AngularMesh build_banded_mesh(int l_max);
// EXTENSION: uniform `base_level` plus `extra` refinement levels of every leaf
// whose centroid lies within `half_angle_deg` of +x (BASELINE config 4).
AngularMesh build_cone_mesh(int base_level, int extra, double half_angle_deg);
bool patch_in_cone(const Patch& p, double half_angle_deg);
AngularMesh coarsen_to_level(const AngularMesh& mesh, int level);
double patch_area(const Patch& p);
double total_area(const AngularMesh& mesh);
std::vector<std::vector<int>> leaf_neighbors(const AngularMesh& mesh);
bool two_irregular(const AngularMesh& mesh);

// ---------------------------------------------------------------- quadrature
struct Gauss1D {
  std::vector<double> x, w;
};
const Gauss1D& gauss_legendre_01(int n);
inline int default_patch_order(int level, int base = 8) {  // quadrature.hpp:31-34
  const int bump = level == 0 ? 20 : level == 1 ? 12 : 8;
  return base > bump ? base : bump;
}
struct QuadratureRule {
  std::vector<Vec3> nodes, bary;
  std::vector<double> weights;
  int size() const { return int(weights.size()); }
};
QuadratureRule patch_quadrature(const Patch& patch, int order);

// ---------------------------------------------------------------- angular disc
enum class BasisKind { Const = 0, Lin = 1 };
inline int dofs_per_patch(BasisKind k) { return k == BasisKind::Const ? 1 : 3; }
Vec3 barycentric(const Patch& patch, const Vec3& omega);
bool patch_contains(const Patch& patch, const Vec3& omega, double tol = 1e-12);
struct PatchOperators {
  Mat M;
  std::array<Mat, 3> A;
};
PatchOperators build_patch_operators(BasisKind kind, const Patch& patch, int order = 0);
std::pair<Mat, Mat> face_split(BasisKind kind, const Patch& patch, const Vec3& normal,
                               int order = 24);

// ---------------------------------------------------------------- scatter
// scatter.hpp:14-20; per material (EXTENSION: materials, HG moments)
struct ScatterKernel {
  int N = 0;
  double sigma_a = 0, sigma_t = 0;
  Vec moments;  // sigma_{s,n}, n = 0..N
};
ScatterKernel fp_equivalent_moments(int N, double alpha, double sigma_a = 0.0);
ScatterKernel absorber_kernel(double sigma_a);
ScatterKernel hg_moments(int N, double sigma_t, double c, double g);  // EXTENSION
inline int harmonic_count(int N) { return (N + 1) * (N + 1); }
void eval_real_harmonics(int N, const Vec3& omega, double* out);
inline int default_quad_order(int N) { return N > 12 ? 12 : 8; }
struct HarmonicCouplings {
  int N = 0, D = 1;
  BasisKind kind = BasisKind::Const;
  Mat X;  // (P*D) x H
};
HarmonicCouplings build_couplings(const AngularMesh& mesh, BasisKind kind, int N, int order = 0);
Vec sigma_by_harmonic(const ScatterKernel& k, int max_order);

// ---------------------------------------------------------------- spatial disc
// HexMesh (spatial_disc.hpp:12-25) generalised to dim 2 (EXTENSION: nz = 1,
// faces 0..3, S = 4 bilinear with dof i = ix + 2*iy).
struct Grid {
  int dim = 3, nx = 0, ny = 0, nz = 0;
  double box = 0, hx = 0, hy = 0, hz = 0;
  int n_el = 0;
  int index(int ix, int iy, int iz) const { return (iz * ny + iy) * nx + ix; }
  std::array<int, 3> coords(int el) const { return {el % nx, (el / nx) % ny, el / (nx * ny)}; }
  int neighbor(int el, int f) const;
  double volume() const { return dim == 3 ? hx * hy * hz : hx * hy; }
  int n_faces() const { return 2 * dim; }
};
Grid build_grid(int dim, int nx, int ny, int nz, double box);
struct ElementMatrices {
  int S = 0;
  Mat N;
  std::array<Mat, 3> V;
  std::array<Mat, 6> F_self, F_neigh;
};
ElementMatrices element_matrices(const Grid& g, int p);
std::vector<int> sweep_order(const Grid& g, int octant);

// ---------------------------------------------------------------- layout
struct Layout {  // layout.hpp:16-32
  int n_el = 0, n_patch = 0, S = 1, D = 1;
  std::int64_t size() const { return std::int64_t(n_el) * n_patch * S * D; }
  std::int64_t block(int el, int q) const { return (std::int64_t(el) * n_patch + q) * D * S; }
  std::int64_t element(int el) const { return std::int64_t(el) * n_patch * D * S; }
};

// ---------------------------------------------------------------- transport
struct ProblemOperators {  // transport.hpp:29-45 (+ materials)
  Grid mesh;
  AngularMesh angular;
  BasisKind kind = BasisKind::Const;
  int p = 0;
  std::vector<ScatterKernel> kernels;  // per material
  std::vector<int> mat;                // per element (EXTENSION)
  int N = 0;                           // common scatter order of the kernels
  Layout layout;
  ElementMatrices em;
  HarmonicCouplings coup;
  std::vector<PatchOperators> pops;
  std::vector<std::vector<Mat>> diag;          // [material][q]
  std::vector<std::array<Mat, 3>> inflow;      // [q][xi]
  std::vector<std::array<int, 3>> inflow_face, outflow_face;
};
ProblemOperators build_operators(const Grid& mesh, const AngularMesh& angular, BasisKind kind,
                                 int p, const std::vector<ScatterKernel>& kernels,
                                 const std::vector<int>& mat);

void apply_L_into(const ProblemOperators& ops, const double* phi, double* y);
void apply_scatter_into(const ProblemOperators& ops, const double* phi, int max_order,
                        double scale, double* y);
void apply_A_into(const ProblemOperators& ops, const double* phi, int order, double* y);

struct SourceSpec {
  // isotropic volume source density per element (empty: none); reference
  // "uniform" is q_el == strength everywhere (transport.cpp:114-127)
  Vec q_el;
  int beam = 0;  // 0 none, 1 +z pencil (transport.cpp:129-178), 2 x=0 cone (EXTENSION)
  double strength = 1.0;
  double x0 = 2, x1 = 3, y0 = 2, y1 = 3;
  double cone_half_angle_deg = 15.0;
};
Vec assemble_rhs(const ProblemOperators& ops, const SourceSpec& spec);
// per-element scalar flux (harness.cpp:183-205): integral / volume
Vec scalar_flux(const ProblemOperators& ops, const double* phi);

// ---------------------------------------------------------------- sweeps
struct SweepPlan {  // sweeps.hpp:16-20
  std::array<std::vector<int>, 8> order, patches;
  std::vector<std::vector<LU>> lu;  // [material][q]
};
SweepPlan build_sweep_plan(const ProblemOperators& ops);
void standard_sweep(const SweepPlan& plan, const ProblemOperators& ops, const double* rhs,
                    double* z, int q_begin = 0, int q_end = -1);
void coarse_scatter_sweep(const SweepPlan& plan, const ProblemOperators& ops, const double* rhs,
                          int nu, double* phi);
void smoother_step(const SweepPlan& plan, const ProblemOperators& ops, const double* f,
                   int order, double* phi);

// ---------------------------------------------------------------- multigrid
struct CycleSpec {
  int nu_pre = 1, nu_post = 1, nr = -1, coarse_sweeps = 10;
  double coarse_tol = 0;
  int n_levels = 0;  // EXTENSION: 0 = all levels (reference behaviour)
};
int nr_default(int N);
struct TransferBlock {
  int coarse = -1;
  Mat B;
};
struct MgLevel {
  ProblemOperators ops;
  SweepPlan plan;
  std::vector<TransferBlock> up;
};
struct MgHierarchy {
  std::vector<MgLevel> level;  // 0 = coarsest used level
  CycleSpec cycle;
  int nr = 0;
};
MgHierarchy build_hierarchy(const ProblemOperators& fine, const CycleSpec& cycle);
Vec prolongate(const MgHierarchy& h, int l, const double* coarse);
Vec restrict_residual(const MgHierarchy& h, int l, const double* fine);
void lmg_vcycle(const MgHierarchy& h, int l, const double* f, double* phi);
Vec mg_apply(const MgHierarchy& h, const double* r);

// ---------------------------------------------------------------- krylov
using LinearOp = std::function<Vec(const Vec&)>;
struct SolveReport {
  int iterations = 0;
  std::vector<double> residual_history;
  bool converged = false, breakdown = false;
  double final_residual = 0, wall_time = 0;
  int preconditioner_applications = 0;
};
std::pair<Vec, SolveReport> bicgstab(const LinearOp& A, const LinearOp& M, const Vec& b,
                                     double tol, int max_iter);
// EXTENSION: right-preconditioned restarted GMRES(m), CGS2, Givens.
std::pair<Vec, SolveReport> gmres(const LinearOp& A, const LinearOp& M, const Vec& b, double tol,
                                  int max_iter, int restart, double atol_breakdown = 0.0);

// dense oracles (tests/support/oracles.cpp:29-91)
Mat dense_transport_matrix(const ProblemOperators& ops);
Mat dense_scatter_matrix(const ProblemOperators& ops, int max_order);

}  // namespace oracle
