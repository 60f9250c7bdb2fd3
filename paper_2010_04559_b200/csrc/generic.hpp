// Reference-shape path: every discretisation the reference solver itself supports --
// 2D / 3D structured cells with p0 or (bi/tri)linear dofs (S = 1, 4, 8), the Const or the
// nodal Lin angular basis (D = 1, 3) -- for problems outside the tuned 2D-bilinear-Const
// kernels (angular_disc.cpp:40-59, spatial_disc.cpp:45-88).
//
// Vectors are in the reference Layout, index ((el*P + q)*D + d)*S + i (layout.hpp:16-32); a
// (cell, patch) block is bs = D*S doubles, a cell is a (P*D) x S row-major slab. Host setup
// (generic_setup.cpp) builds dense per-patch tables; the kernels (generic.cu) are written
// for any bs <= 24: block operators as dense bs x bs products, hyperplane-ordered sweeps,
// one warp per cell for the scatter-implicit coarse Gauss-Seidel.
#pragma once

#include <cstdint>
#include <vector>

#include <cuda_runtime.h>

#include "setup.hpp"

namespace stamg_b200 {
namespace gen {

constexpr int kMaxBs = 24;  // D * S <= 3 * 8

// ---- host tables of one level (build_operators + build_sweep_plan, transport.cpp:23-64,
//      sweeps.cpp:7-18; one material: the reference's kernel is global, transport.hpp:34) ----
struct Tables {
  int dim = 3, nx = 0, ny = 0, nz = 1, n_el = 0;
  int S = 1, D = 1, bs = 1, P = 0, order = 0, H = 0;
  std::vector<int> leaf_id, octant;
  std::vector<double> X;        // [P*D][H] couplings (scatter.cpp:74-99)
  std::vector<double> sig;      // [H] sigma per harmonic
  std::vector<double> Bd;       // [P][bs*bs] diagonal blocks B_q
  std::vector<double> Binv;     // [P][bs*bs] B_q^-1
  std::vector<double> C;        // [P][3][bs*bs] inflow blocks C_{q,xi}
  std::vector<double> BinvGS;   // [P][bs*bs] (B_q - (X_q sig X_q^T) x N)^-1 (sweeps.cpp:61-72)
  std::vector<double> Nmat;     // [S*S]
  std::vector<double> M1;       // [P][D] row sums of the patch mass matrix
  std::vector<int> oct_patches, oct_ptr;
  // transfers to the next coarser level (multigrid.cpp:68-96): parent position and the D x D
  // block B (Const: 1; Lin: barycentric coordinates of the child's corners in the parent)
  std::vector<int> up;
  std::vector<double> upB;      // [P][D*D]
  std::vector<int> child_ptr, child_idx;
};

bool handles(const stamg_problem& s);  // problems routed to this path
void validate(const Problem& pb);
Tables build_level(const Problem& pb, const SphereTree& tree, int order, bool with_gs);
std::vector<Tables> build_hierarchy(const Problem& pb, const SphereTree& fine, int nr, int nlev);
// assemble_rhs (transport.cpp:110-179): isotropic volume source and the +z pencil beam
std::vector<double> assemble_rhs(const Problem& pb, const Tables& t, const SphereTree& tree);

// ---- device side ----
struct Dev {
  int dim = 3, nx = 0, ny = 0, nz = 1, n_el = 0, S = 1, D = 1, bs = 1, P = 0, H = 0, order = 0;
  double* XT = nullptr;  // [H][P*D] transposed couplings (M2D reads them coalesced over rows)
  double *X = nullptr, *sig = nullptr, *Bd = nullptr, *Binv = nullptr, *C = nullptr, *BinvGS = nullptr;
  double *Nmat = nullptr, *upB = nullptr, *src = nullptr, *mom = nullptr;
  int *octant = nullptr, *oct_patches = nullptr, *oct_ptr = nullptr, *up = nullptr, *child_ptr = nullptr,
      *child_idx = nullptr;
  int max_np = 0;
  // cells listed hyperplane by hyperplane in frame coordinates (fi | fj << 10 | fk << 20), for the
  // tensor-core sweep; null when a grid side exceeds 1023
  int *plane_cells = nullptr, *plane_ptr = nullptr;
  int* gs_prog = nullptr;  // [ny*nz] per-line progress counters of the dataflow coarse GS
};

// y = alpha (B x + sum_xi C_xi x_up) + beta f   (apply_L_into, transport.cpp:66-88)
void launch_apply_L(const Dev& L, const double* x, double* y, double alpha, double beta, const double* f,
                    cudaStream_t s);
// exact L^-1 (standard_sweep, sweeps.cpp:20-42); z may alias rhs
void launch_sweep(const Dev& L, const double* rhs, double* z, cudaStream_t s);
// y += scale X_r diag(sig) (X_r^T phi) N with the first (order+1)^2 harmonics
// (apply_scatter_into, scatter.cpp:110-135): D2M + sigma N epilogue into L.src, then M2D
void launch_d2m(const Dev& L, const double* phi, int order, bool apply_sigma_N, double* out, cudaStream_t s);
void launch_m2d(const Dev& L, const double* src, int order, double scale, double* y, cudaStream_t s);
// prolongate / restrict_residual (multigrid.cpp:100-136)
void launch_prolong(const Dev& F, const double* coarse, double* fine, int Pc, bool add, cudaStream_t s);
void launch_restrict(const Dev& F, const double* fine, double* coarse, int Pc, cudaStream_t s);
// coarse_scatter_sweep (sweeps.cpp:51-104), the reference's (pass, octant, cell, patch) order
void launch_coarse_gs(const Dev& L, const double* rhs, int nu, double* phi, cudaStream_t s);

}  // namespace gen
}  // namespace stamg_b200
