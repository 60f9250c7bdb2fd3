// ORACLE — TEST INFRASTRUCTURE ONLY.
//
// C API over the UNMODIFIED reference solver (/root/reference/proj/src/*.cpp,
// compiled against the Eigen-subset shim in oracle/eigen_shim/ by
// `make -C oracle ref`; outputs only under oracle/_ref/). It exists to pin the
// CPU restatement (oracle/stamg_oracle.cpp) to the reference itself: the
// tests run both on the reference's own 3D problems and compare
// (tests/test_oracle_vs_reference.py; golden vectors in tests/golden/ref_*.npz,
// made by tests/golden/make_golden_ref.py). Every entry point is a direct call
// of a reference function; nothing here re-implements the algorithm.
//
//   ref_create        build_hex_mesh / build_uniform_mesh | build_banded_mesh /
//                     build_operators / build_sweep_plan / build_hierarchy
//                     (spatial_disc.hpp, sphere_mesh.hpp, transport.hpp:47-49,
//                      sweeps.hpp:22, multigrid.hpp:50)
//   ref_apply_L/A     transport.hpp:52-60
//   ref_apply_scatter scatter.hpp:51-57
//   ref_sweep         sweeps.hpp:24-28
//   ref_coarse_gs     sweeps.hpp:32-33
//   ref_smoother      sweeps.hpp:36-37
//   ref_prolong/restrict, ref_vcycle, ref_mg_apply   multigrid.hpp:52-60
//   ref_bicgstab      krylov.hpp:27-30 with the harness's closures
//                     (harness.cpp:211-231)
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>

#include "stamg/krylov.hpp"
#include "stamg/multigrid.hpp"
#include "stamg/scatter.hpp"
#include "stamg/sphere_mesh.hpp"
#include "stamg/sweeps.hpp"
#include "stamg/transport.hpp"

using namespace stamg;

namespace {
thread_local std::string g_err;

struct Ref {
  ProblemOperators ops;
  SweepPlan plan;
  MgHierarchy h;
  SourceSpec src;
};

template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = std::string("invalid_argument: ") + e.what();
    return 1;
  } catch (const std::logic_error& e) {
    g_err = std::string("logic_error: ") + e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 3;
  }
}

const ProblemOperators& ops_of(const Ref* r, int level) {
  if (level < 0) return r->ops;
  if (level >= int(r->h.level.size())) throw std::invalid_argument("level out of range");
  return r->h.level[level].ops;
}
const SweepPlan& plan_of(const Ref* r, int level) {
  if (level < 0) return r->plan;
  if (level >= int(r->h.level.size())) throw std::invalid_argument("level out of range");
  return r->h.level[level].plan;
}
FluxVector vec_in(const double* p, std::ptrdiff_t n) {
  FluxVector v(n);
  std::memcpy(v.data(), p, sizeof(double) * size_t(n));
  return v;
}
void vec_out(const FluxVector& v, double* p) { std::memcpy(p, v.data(), sizeof(double) * size_t(v.size())); }
}  // namespace

extern "C" {

struct ref_spec {
  int nx, ny, nz;
  double box;
  int basis;          // 0 Const, 1 Lin
  int p;              // spatial order 0 / 1
  int angular_kind;   // 0 uniform, 1 banded (+z)
  int angular_level;  // uniform level or banded l_max
  int N;
  const double* moments;  // [N+1]
  double sigma_t, sigma_a;
  int source_kind;  // 0 uniform, 1 +z beam
  double strength, x0, x1, y0, y1;
  int nu_pre, nu_post, nr, coarse_sweeps;
  double coarse_tol;
};

struct ref_report {
  int iterations, converged, breakdown, preconditioner_applications;
  double final_residual, wall_time;
};

const char* ref_last_error(void) { return g_err.c_str(); }

int ref_create(const ref_spec* s, void** out) {
  return guard([&] {
    auto r = std::make_unique<Ref>();
    const HexMesh mesh = build_hex_mesh(s->nx, s->ny, s->nz, s->box);
    const AngularMesh ang =
        s->angular_kind == 0 ? build_uniform_mesh(s->angular_level) : build_banded_mesh(s->angular_level);
    ScatterKernel k;
    k.N = s->N;
    k.sigma_t = s->sigma_t;
    k.sigma_a = s->sigma_a;
    k.moments.resize(s->N + 1);
    for (int n = 0; n <= s->N; ++n) k.moments[n] = s->moments[n];
    r->ops = build_operators(mesh, ang, s->basis == 0 ? BasisKind::Const : BasisKind::Lin, s->p, k);
    r->plan = build_sweep_plan(r->ops);
    CycleSpec cyc;
    cyc.nu_pre = s->nu_pre;
    cyc.nu_post = s->nu_post;
    cyc.nr = s->nr;
    cyc.coarse_sweeps = s->coarse_sweeps;
    cyc.coarse_tol = s->coarse_tol;
    r->h = build_hierarchy(r->ops, cyc);
    r->src.kind = s->source_kind == 0 ? SourceSpec::Kind::Uniform : SourceSpec::Kind::Beam;
    r->src.strength = s->strength;
    r->src.x0 = s->x0, r->src.x1 = s->x1, r->src.y0 = s->y0, r->src.y1 = s->y1;
    *out = r.release();
  });
}

int ref_destroy(void* h) {
  delete static_cast<Ref*>(h);
  return 0;
}

int ref_layout(void* h, int level, int out4[4]) {
  return guard([&] {
    const Layout& lo = ops_of(static_cast<Ref*>(h), level).layout;
    out4[0] = lo.n_el, out4[1] = lo.n_patch, out4[2] = lo.S, out4[3] = lo.D;
  });
}

int ref_n_levels(void* h, int* n, int* nr) {
  return guard([&] {
    *n = int(static_cast<Ref*>(h)->h.level.size());
    *nr = static_cast<Ref*>(h)->h.nr;
  });
}

int ref_rhs(void* h, double* f) {
  return guard([&] {
    const Ref* r = static_cast<Ref*>(h);
    vec_out(assemble_rhs(r->ops, r->src), f);
  });
}

int ref_X(void* h, int level, double* out, int* rows, int* cols) {
  return guard([&] {
    const auto& X = ops_of(static_cast<Ref*>(h), level).coup.X;
    *rows = int(X.rows()), *cols = int(X.cols());
    if (out)
      for (int i = 0; i < X.rows(); ++i)
        for (int j = 0; j < X.cols(); ++j) out[size_t(i) * X.cols() + j] = X(i, j);
  });
}

int ref_diag(void* h, int level, int q, double* out, int* n) {
  return guard([&] {
    const auto& B = ops_of(static_cast<Ref*>(h), level).diag.at(size_t(q));
    *n = int(B.rows());
    if (out)
      for (int i = 0; i < B.rows(); ++i)
        for (int j = 0; j < B.cols(); ++j) out[size_t(i) * B.cols() + j] = B(i, j);
  });
}

int ref_apply_L(void* h, int level, const double* x, double* y) {
  return guard([&] {
    const auto& ops = ops_of(static_cast<Ref*>(h), level);
    FluxVector out;
    apply_L_into(ops, vec_in(x, ops.layout.size()), out);
    vec_out(out, y);
  });
}

int ref_apply_A(void* h, int level, const double* x, int order, double* y) {
  return guard([&] {
    const auto& ops = ops_of(static_cast<Ref*>(h), level);
    FluxVector out(ops.layout.size());
    apply_A_into(ops, vec_in(x, ops.layout.size()), order, out);
    vec_out(out, y);
  });
}

// y (in/out) += scale * S_order x
int ref_apply_scatter(void* h, int level, const double* x, int order, double scale, double* y) {
  return guard([&] {
    const auto& ops = ops_of(static_cast<Ref*>(h), level);
    FluxVector yy = vec_in(y, ops.layout.size());
    apply_scatter_into(ops.kernel, ops.coup, ops.em.N, ops.layout, vec_in(x, ops.layout.size()), order, scale, yy);
    vec_out(yy, y);
  });
}

int ref_sweep(void* h, int level, const double* rhs, double* z) {
  return guard([&] {
    const Ref* r = static_cast<Ref*>(h);
    const auto& ops = ops_of(r, level);
    FluxVector out(ops.layout.size());
    standard_sweep(plan_of(r, level), ops, vec_in(rhs, ops.layout.size()), out);
    vec_out(out, z);
  });
}

int ref_coarse_gs(void* h, int level, const double* rhs, int nu, double* phi) {
  return guard([&] {
    const Ref* r = static_cast<Ref*>(h);
    const auto& ops = ops_of(r, level);
    FluxVector p = vec_in(phi, ops.layout.size());
    coarse_scatter_sweep(plan_of(r, level), ops, vec_in(rhs, ops.layout.size()), nu, p);
    vec_out(p, phi);
  });
}

int ref_smoother(void* h, int level, const double* f, int order, double* phi) {
  return guard([&] {
    const Ref* r = static_cast<Ref*>(h);
    const auto& ops = ops_of(r, level);
    FluxVector p = vec_in(phi, ops.layout.size());
    smoother_step(plan_of(r, level), ops, vec_in(f, ops.layout.size()), order, p);
    vec_out(p, phi);
  });
}

int ref_prolong(void* h, int l, const double* coarse, double* fine) {
  return guard([&] {
    const Ref* r = static_cast<Ref*>(h);
    if (l < 1 || l >= int(r->h.level.size())) throw std::invalid_argument("prolongate: level out of range");
    vec_out(prolongate(r->h, l, vec_in(coarse, r->h.level[l - 1].ops.layout.size())), fine);
  });
}

int ref_restrict(void* h, int l, const double* fine, double* coarse) {
  return guard([&] {
    const Ref* r = static_cast<Ref*>(h);
    if (l < 1 || l >= int(r->h.level.size())) throw std::invalid_argument("restrict_residual: level out of range");
    vec_out(restrict_residual(r->h, l, vec_in(fine, r->h.level[l].ops.layout.size())), coarse);
  });
}

int ref_vcycle(void* h, int l, const double* f, double* phi) {
  return guard([&] {
    const Ref* r = static_cast<Ref*>(h);
    const auto& ops = ops_of(r, l);
    FluxVector p = vec_in(phi, ops.layout.size());
    lmg_vcycle(r->h, l, vec_in(f, ops.layout.size()), p);
    vec_out(p, phi);
  });
}

int ref_mg_apply(void* h, const double* rv, double* z) {
  return guard([&] {
    const Ref* r = static_cast<Ref*>(h);
    vec_out(mg_apply(r->h, vec_in(rv, r->ops.layout.size())), z);
  });
}

// precond: 0 standard_sweep, 1 mg_apply, 2 identity (harness.cpp:211-231)
int ref_bicgstab(void* h, int precond, double tol, int max_iter, double* x, ref_report* rep, double* hist, int cap) {
  return guard([&] {
    const Ref* r = static_cast<Ref*>(h);
    const LinearOp apply = [r](const FluxVector& v) { return apply_A(r->ops, v, r->ops.kernel.N); };
    LinearOp pc;
    if (precond == 0) pc = [r](const FluxVector& v) { return standard_sweep(r->plan, r->ops, v); };
    else if (precond == 1) pc = [r](const FluxVector& v) { return mg_apply(r->h, v); };
    else pc = [](const FluxVector& v) { return v; };
    const FluxVector b = assemble_rhs(r->ops, r->src);
    auto [sol, sr] = bicgstab(apply, pc, b, tol, max_iter);
    vec_out(sol, x);
    rep->iterations = sr.iterations, rep->converged = sr.converged, rep->breakdown = sr.breakdown;
    rep->preconditioner_applications = sr.preconditioner_applications;
    rep->final_residual = sr.final_residual, rep->wall_time = sr.wall_time;
    for (int i = 0; hist && i < cap && i < int(sr.residual_history.size()); ++i) hist[i] = sr.residual_history[i];
  });
}

}  // extern "C"
