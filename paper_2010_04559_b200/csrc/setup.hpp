// Host-side setup for the B200 path (the reference's L0/L1: angular mesh,
// patch quadrature, couplings, fused-block operator tables, hierarchy
// transfers). Runs once per problem on the host and produces flat,
// device-ready arrays. Specialised to what the B200 kernels execute:
// 2D cells with bilinear dofs (S = 4, i = ix + 2*iy) and the Const angular
// basis (D = 1). Reference counterparts are cited per function.
#pragma once

#include <array>
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/stamg_b200.h"

namespace stamg_b200 {

constexpr int kS = 4;  // spatial dofs per cell (2D bilinear)

// ---- angular mesh (sphere_mesh.hpp:20-63), struct-of-arrays tree ----
struct SphereTree {
  static constexpr std::int64_t kScale = std::int64_t(1) << 20;  // flat lattice scale
  std::vector<int> level, octant, parent;
  std::vector<std::array<int, 4>> kids;
  std::vector<char> leaf;
  std::vector<std::array<std::int64_t, 9>> flat;  // 3 lattice vertices
  std::vector<std::array<double, 9>> unit;        // 3 unit-sphere vertices
  std::vector<int> leaves;                        // ascending ids
  int max_level = 0;

  int size() const { return int(level.size()); }
  void add(int lvl, int oct, int par, const std::int64_t* a, const std::int64_t* b, const std::int64_t* c);
  void split(int id);
  void relist();
  void close_two_irregular();
};

SphereTree make_sphere(int kind, int level, int extra, double cone_half_angle_deg);
SphereTree coarsen(const SphereTree& t, int level);
bool in_cone(const SphereTree& t, int id, double half_angle_deg);

// ---- per-level device tables ----
struct LevelTables {
  int n_el = 0, P = 0, order = 0, H = 0, n_mat = 1;
  int P_global = 0, q_begin = 0;      // direction sharding: leaf-order positions of the local patches
  std::vector<int> qpos;              // [P] position of each local patch in the level's full leaf order
  int nx = 0, ny = 0;
  std::vector<int> leaf_id, octant;   // per patch
  std::vector<double> X;              // [P][H] couplings (scatter.hpp:32-39)
  std::vector<double> sig;            // [n_mat][H] sigma per harmonic
  std::vector<double> B;              // [n_mat][P][16] diag blocks (transport.cpp:46-54)
  std::vector<double> Binv;           // [n_mat][P][16]
  std::vector<double> C;              // [P][2][16] full inflow blocks (transport.cpp:55)
  std::vector<double> cxy;            // [P][8] nonzero 2x2 sub-blocks of C_x, C_y
  std::vector<double> BinvGS;         // [n_mat][P][16] inverse of B - (X sig X^T) N (sweeps.cpp:61-72)
  std::vector<double> sq;             // [n_mat][P] X_q sig X_q^T
  std::vector<double> area;           // [P] patch mass M_q
  std::vector<double> Aflow;          // [P][3] A^x, A^y, A^z
  std::vector<int> groups;            // [n_groups][4] patch ids of equal octant (-1 pad)
  std::vector<int> group_oct;         // [n_groups]
  std::vector<int> groups8;           // [n_groups8][8] equal-octant patches (-1 pads an octant's last group)
  std::vector<int> group8_oct;
  bool groups8_padded = false;        // some group holds -1 lanes (no wavefront layout then)
  std::vector<int> oct_patches;       // patches listed by octant (plan.patches)
  std::vector<int> oct_ptr;           // [9]
  // transfers to the next coarser level (multigrid.cpp:68-96); empty on level 0
  std::vector<int> up;                // [P] coarse position
  std::vector<double> up_w;           // [P] Const transfer block B = [1]
  std::vector<int> child_ptr, child_idx;  // CSR children of each coarse patch, ascending
  double Nmat[16];                    // spatial mass matrix
  // ---- reflection symmetry of the scatter operator (exact algebra: X[g(q)][h] = chi_h(g) X[q][h])
  int n_sym_axes = 0;                 // |G| = 2^n_sym_axes
  int sym_axes[3] = {0, 0, 0};
  std::vector<int> orbit;             // [R][|G|] patch index of member g of orbit r (r = representative)
  std::vector<int> hclass;            // [H] parity class of each harmonic under the symmetric axes
  // max_{r,g,h} |X[orbit(r,g)][h] - chi_h(g) X[orbit(r,0)][h]| / max|X|: how far the
  // coupling table is from the exact reflection identity the fold relies on
  double sym_defect = 0.0;
};

// The folded scatter is used only when the coupling table satisfies the
// reflection identity to this relative accuracy (the quadrature of build_couplings
// is exact only up to its order; level-2 meshes miss it by ~2e-9).
constexpr double kFoldMaxDefect = 1e-14;

// Reflections (x, y, z) that map the leaf set onto itself; fills n_sym_axes,
// sym_axes, orbit, hclass and sym_defect (an empty orbit table means no folding).
void find_symmetry(LevelTables& L, const SphereTree& tree);

struct Problem {
  stamg_problem spec{};
  std::vector<double> sigma_t, moments;
  std::vector<int> mat;
  std::vector<double> q_el;
  int n_el = 0;
  double h = 0;
  bool device_setup = false;  // build_couplings on the current CUDA device (couplings.cu)
};

Problem copy_problem(const stamg_problem& p);
void validate(const Problem& p);

// build_operators + build_sweep_plan for one angular mesh and scatter order
// `subset` (ascending leaf-order positions) restricts the level to a rank's
// directions; nullptr = all leaves.
LevelTables build_level(const Problem& pb, const SphereTree& tree, int order, bool with_gs,
                        const std::vector<int>* subset = nullptr);
// contiguous leaf-order range [q_begin, q_end) as a subset
std::vector<int> range_subset(int q_begin, int q_end);
// Direction shard of `rank` for contexts without a hierarchy (config 5): whole orbits of
// the mesh's reflection symmetry group (so each rank can fold its scatter), balanced in
// slices of 8 orbit representatives; contiguous slices of 4 patches without symmetry.
std::vector<int> throughput_shard(const SphereTree& tree, int rank, int world);

// Mirror maps of the reflections (x, y, z; or only the axes in `only`) that map the
// leaf set onto itself: axes[k] and mirror[k][leaf position] = its mirror's position.
void leaf_mirrors(const SphereTree& t, std::vector<int>& axes, std::vector<std::vector<int>>& mirror,
                  const std::vector<int>& only);
// Direction sharding of a hierarchy: rank r owns whole subtrees rooted at the
// coarsest used level's patches, assigned in whole reflection orbits of the roots
// when the finest mesh is mirror symmetric and there are at least `world` orbits (so
// every rank's levels are closed under the reflections and fold their scatter), else
// root by root; units balanced by the number of finest-level descendants (heaviest
// first onto the least-loaded rank), so a rank's roots need not be contiguous.
// Returns per level (0 = coarsest) the ascending leaf positions held by `rank`;
// level 0 is replicated (all positions).
std::vector<std::vector<int>> partition_levels(const SphereTree& fine, int nlev, int rank, int world);

// build_hierarchy: nlev levels, index 0 coarsest; fills up/child maps. With
// `parts` (from partition_levels) levels >= 1 hold only the rank's patches and
// up[] indexes the coarser level's local list (level 0: the full list).
std::vector<LevelTables> build_hierarchy(const Problem& pb, const SphereTree& fine, int nr, int nlev,
                                         const std::vector<std::vector<int>>* parts = nullptr);
// assemble_rhs (transport.cpp:110-179 + cone beam EXTENSION)
std::vector<double> assemble_rhs(const Problem& pb, const LevelTables& lev, const SphereTree& tree);

// quadrature helpers (quadrature.hpp:31-34, quadrature.cpp:13-57): per-patch
// 1D order, cached Gauss-Legendre rule on [0, 1]
int patch_order(int level, int base);
void gauss_rule01(int n, const double** x, const double** w);
// build_couplings (scatter.cpp:74-99) on the current CUDA device: X [P][H] for
// the given leaves, written to host memory; orders up to 32
bool device_couplings_supported(int order);
void device_couplings(const SphereTree& t, const std::vector<int>& leaf_id, int order, int xorder_base, double* X);
// build_operators (transport.cpp:43-57) on the current CUDA device: patch mass and Jacobians by
// quadrature, fused blocks, their inverses, inflow blocks; el16 = N | V0 | V1 | F_self[4] | F_neigh[4]
void device_patch_blocks(const SphereTree& t, const std::vector<int>& leaf_id, const std::vector<double>& sigma_t,
                         const double* el16, double* area, double* Aflow, double* B, double* Binv, double* C, double* cxy);

// every node of a patch's Duffy-collapsed rule: unit directions [n][3], flat barycentric
// coordinates [n][3], weights [n] (quadrature.cpp:59-92); real orthonormal harmonics
void patch_rule(const SphereTree& t, int id, int order, std::vector<double>& om, std::vector<double>& bary,
                std::vector<double>& w);
void real_harmonics(int N, const double* om, double* out);

// 4x4 helpers
void inverse4(const double* A, double* Ainv);

}  // namespace stamg_b200
