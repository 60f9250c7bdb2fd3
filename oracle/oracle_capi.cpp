// ORACLE — TEST INFRASTRUCTURE ONLY. ctypes-facing C ABI over the CPU
// restatement in stamg_oracle.cpp. Loaded by tests/ (parity checker),
// __graft_entry__.smoke() and bench.py's CPU baseline arm; never by the
// product library.
#include <cmath>
#include <cstring>
#include <memory>
#include <numbers>
#include <string>

#include "stamg_oracle.hpp"

using namespace oracle;

extern "C" {

typedef struct {
  int dim, nx, ny, nz;
  double box;
  int basis, p;
  int angular_kind;  // 0 uniform, 1 banded, 2 cone
  int angular_level, cone_levels;
  double cone_half_angle_deg;
  int N, n_mat;
  const double* sigma_t;  // n_mat
  const double* moments;  // n_mat * (N + 1)
  const int* mat_of_el;   // n_el or NULL
  const double* q_el;     // n_el or NULL
  int beam;
  double strength, x0, x1, y0, y1;
  int nr, n_levels, nu_pre, nu_post, coarse_sweeps;
  double coarse_tol;
} orc_spec;

typedef struct {
  int iterations, converged, breakdown, preconditioner_applications;
  double final_residual, wall_time;
} orc_report;
}

namespace {
thread_local std::string g_err;

struct Handle {
  ProblemOperators ops;
  SweepPlan plan;
  SourceSpec src;
  CycleSpec cycle;
  std::unique_ptr<MgHierarchy> hier;
  const MgHierarchy& h() {
    if (!hier) hier = std::make_unique<MgHierarchy>(build_hierarchy(ops, cycle));
    return *hier;
  }
  // level -1 = the fine problem itself; otherwise a hierarchy level
  const ProblemOperators& lops(int l) { return l < 0 ? ops : h().level.at(l).ops; }
  const SweepPlan& lplan(int l) { return l < 0 ? plan : h().level.at(l).plan; }
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
  } catch (const std::runtime_error& e) {
    g_err = std::string("runtime_error: ") + e.what();
    return 3;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 4;
  }
}

AngularMesh make_mesh(int kind, int level, int extra, double angle) {
  if (kind == 0) return build_uniform_mesh(level);
  if (kind == 1) return build_banded_mesh(level);
  if (kind == 2) return build_cone_mesh(level, extra, angle);
  throw std::invalid_argument("unknown angular kind");
}
}  // namespace

extern "C" {

const char* orc_last_error() { return g_err.c_str(); }

int orc_create(const orc_spec* s, void** out) {
  return guard([&] {
    auto hd = std::make_unique<Handle>();
    const Grid g = build_grid(s->dim, s->nx, s->ny, s->nz, s->box);
    const AngularMesh am = make_mesh(s->angular_kind, s->angular_level, s->cone_levels, s->cone_half_angle_deg);
    std::vector<ScatterKernel> ks;
    for (int m = 0; m < s->n_mat; ++m) {
      ScatterKernel k;
      k.N = s->N;
      k.sigma_t = s->sigma_t[m];
      k.moments.assign(s->moments + size_t(m) * (s->N + 1), s->moments + size_t(m + 1) * (s->N + 1));
      k.sigma_a = k.sigma_t - k.moments[0];
      ks.push_back(k);
    }
    std::vector<int> mat;
    if (s->mat_of_el) mat.assign(s->mat_of_el, s->mat_of_el + g.n_el);
    hd->ops = build_operators(g, am, BasisKind(s->basis), s->p, ks, mat);
    hd->plan = build_sweep_plan(hd->ops);
    if (s->q_el) hd->src.q_el.assign(s->q_el, s->q_el + g.n_el);
    hd->src.beam = s->beam;
    hd->src.strength = s->strength;
    hd->src.x0 = s->x0, hd->src.x1 = s->x1, hd->src.y0 = s->y0, hd->src.y1 = s->y1;
    hd->src.cone_half_angle_deg = s->cone_half_angle_deg;
    hd->cycle.nr = s->nr;
    hd->cycle.n_levels = s->n_levels;
    hd->cycle.nu_pre = s->nu_pre;
    hd->cycle.nu_post = s->nu_post;
    hd->cycle.coarse_sweeps = s->coarse_sweeps;
    hd->cycle.coarse_tol = s->coarse_tol;
    *out = hd.release();
  });
}

void orc_destroy(void* h) { delete static_cast<Handle*>(h); }

int orc_n_levels(void* hp, int* n, int* nr) {
  return guard([&] {
    auto* h = static_cast<Handle*>(hp);
    *n = int(h->h().level.size());
    *nr = h->h().nr;
  });
}

int orc_layout(void* hp, int l, int* out4) {
  return guard([&] {
    const Layout& lo = static_cast<Handle*>(hp)->lops(l).layout;
    out4[0] = lo.n_el, out4[1] = lo.n_patch, out4[2] = lo.S, out4[3] = lo.D;
  });
}

int orc_rhs(void* hp, double* f) {
  return guard([&] {
    auto* h = static_cast<Handle*>(hp);
    const Vec v = assemble_rhs(h->ops, h->src);
    std::memcpy(f, v.data(), v.size() * sizeof(double));
  });
}

int orc_apply_L(void* hp, int l, const double* x, double* y) {
  return guard([&] { apply_L_into(static_cast<Handle*>(hp)->lops(l), x, y); });
}
int orc_apply_A(void* hp, int l, const double* x, int order, double* y) {
  return guard([&] { apply_A_into(static_cast<Handle*>(hp)->lops(l), x, order, y); });
}
int orc_apply_scatter(void* hp, int l, const double* x, int order, double scale, double* y) {
  return guard([&] {
    const auto& ops = static_cast<Handle*>(hp)->lops(l);
    if (order > ops.N) throw std::invalid_argument("sigma_by_harmonic: max_order exceeds kernel order");
    apply_scatter_into(ops, x, order, scale, y);
  });
}
int orc_sweep(void* hp, int l, const double* rhs, double* z, int q0, int q1) {
  return guard([&] {
    auto* h = static_cast<Handle*>(hp);
    standard_sweep(h->lplan(l), h->lops(l), rhs, z, q0, q1);
  });
}
int orc_coarse_gs(void* hp, int l, const double* rhs, int nu, double* phi) {
  return guard([&] {
    auto* h = static_cast<Handle*>(hp);
    coarse_scatter_sweep(h->lplan(l), h->lops(l), rhs, nu, phi);
  });
}
int orc_smoother(void* hp, int l, const double* f, int order, double* phi) {
  return guard([&] {
    auto* h = static_cast<Handle*>(hp);
    smoother_step(h->lplan(l), h->lops(l), f, order, phi);
  });
}
int orc_prolong(void* hp, int l, const double* coarse, double* fine) {
  return guard([&] {
    const Vec v = prolongate(static_cast<Handle*>(hp)->h(), l, coarse);
    std::memcpy(fine, v.data(), v.size() * sizeof(double));
  });
}
int orc_restrict(void* hp, int l, const double* fine, double* coarse) {
  return guard([&] {
    const Vec v = restrict_residual(static_cast<Handle*>(hp)->h(), l, fine);
    std::memcpy(coarse, v.data(), v.size() * sizeof(double));
  });
}
int orc_vcycle(void* hp, int l, const double* f, double* phi) {
  return guard([&] { lmg_vcycle(static_cast<Handle*>(hp)->h(), l, f, phi); });
}
int orc_mg_apply(void* hp, const double* r, double* z) {
  return guard([&] {
    const Vec v = mg_apply(static_cast<Handle*>(hp)->h(), r);
    std::memcpy(z, v.data(), v.size() * sizeof(double));
  });
}

// D2M restricted to patches [q0, q1): mom (n_el x H x S) = X_r^T Phi_el
int orc_d2m(void* hp, int l, const double* phi, int order, int q0, int q1, double* mom) {
  return guard([&] {
    const auto& ops = static_cast<Handle*>(hp)->lops(l);
    const Layout& lo = ops.layout;
    const int H = harmonic_count(order), S = lo.S, Hf = ops.coup.X.c;
    for (int el = 0; el < lo.n_el; ++el) {
      double* m = mom + size_t(el) * H * S;
      std::fill(m, m + size_t(H) * S, 0.0);
      for (int q = q0; q < q1; ++q)
        for (int h = 0; h < H; ++h)
          for (int i = 0; i < S; ++i) m[h * S + i] += ops.coup.X.a[size_t(q) * Hf + h] * phi[lo.block(el, q) + i];
    }
  });
}
// M2D restricted to patches [q0, q1): y_el,q += scale X_q diag(sig) mom_el N
int orc_m2d(void* hp, int l, const double* mom, int order, double scale, int q0, int q1, double* y) {
  return guard([&] {
    const auto& ops = static_cast<Handle*>(hp)->lops(l);
    const Layout& lo = ops.layout;
    const int H = harmonic_count(order), S = lo.S, Hf = ops.coup.X.c;
    std::vector<double> src(size_t(H) * S);
    for (int el = 0; el < lo.n_el; ++el) {
      const Vec sg = sigma_by_harmonic(ops.kernels[ops.mat[el]], order);
      const double* m = mom + size_t(el) * H * S;
      for (int h = 0; h < H; ++h)
        for (int i = 0; i < S; ++i) {
          double acc = 0;
          for (int j = 0; j < S; ++j) acc += m[h * S + j] * ops.em.N(j, i);
          src[h * S + i] = sg[h] * acc;
        }
      for (int q = q0; q < q1; ++q)
        for (int i = 0; i < S; ++i) {
          double acc = 0;
          for (int h = 0; h < H; ++h) acc += ops.coup.X.a[size_t(q) * Hf + h] * src[h * S + i];
          y[lo.block(el, q) + i] += scale * acc;
        }
    }
  });
}

int orc_solve(void* hp, int method, int precond, double tol, int max_iter, int restart, double* x,
              orc_report* rep, double* history, int history_cap) {
  return guard([&] {
    auto* h = static_cast<Handle*>(hp);
    const Vec b = assemble_rhs(h->ops, h->src);
    const size_t n = b.size();
    LinearOp A = [h, n](const Vec& v) {
      Vec y(n);
      apply_A_into(h->ops, v.data(), h->ops.N, y.data());
      return y;
    };
    LinearOp M;
    if (precond == 0)
      M = [h, n](const Vec& v) {
        Vec z(n);
        standard_sweep(h->plan, h->ops, v.data(), z.data());
        return z;
      };
    else if (precond == 1)
      M = [h](const Vec& v) { return mg_apply(h->h(), v.data()); };
    else
      M = [](const Vec& v) { return v; };
    auto [sol, r] = method == 0 ? bicgstab(A, M, b, tol, max_iter) : gmres(A, M, b, tol, max_iter, restart);
    std::memcpy(x, sol.data(), n * sizeof(double));
    rep->iterations = r.iterations;
    rep->converged = r.converged;
    rep->breakdown = r.breakdown;
    rep->preconditioner_applications = r.preconditioner_applications;
    rep->final_residual = r.final_residual;
    rep->wall_time = r.wall_time;
    for (int i = 0; i < history_cap && i < int(r.residual_history.size()); ++i) history[i] = r.residual_history[i];
  });
}

int orc_scalar_flux(void* hp, const double* phi, double* out) {
  return guard([&] {
    const Vec v = scalar_flux(static_cast<Handle*>(hp)->ops, phi);
    std::memcpy(out, v.data(), v.size() * sizeof(double));
  });
}

// ------------------------------------------------------------------ tables
int orc_X(void* hp, int l, double* out, int* rows, int* cols) {
  return guard([&] {
    const Mat& X = static_cast<Handle*>(hp)->lops(l).coup.X;
    *rows = X.r, *cols = X.c;
    if (out) std::memcpy(out, X.a.data(), X.a.size() * sizeof(double));
  });
}
int orc_diag(void* hp, int l, int m, int q, double* out) {
  return guard([&] {
    const Mat& B = static_cast<Handle*>(hp)->lops(l).diag.at(m).at(q);
    std::memcpy(out, B.a.data(), B.a.size() * sizeof(double));
  });
}
int orc_inflow(void* hp, int l, int q, int xi, double* out) {
  return guard([&] {
    const Mat& C = static_cast<Handle*>(hp)->lops(l).inflow.at(q)[xi];
    std::memcpy(out, C.a.data(), C.a.size() * sizeof(double));
  });
}
int orc_patch_ops(void* hp, int l, int q, double* m_a_out /* M, Ax, Ay, Az for D=1 */) {
  return guard([&] {
    const auto& po = static_cast<Handle*>(hp)->lops(l).pops.at(q);
    m_a_out[0] = po.M(0, 0);
    for (int xi = 0; xi < 3; ++xi) m_a_out[1 + xi] = po.A[xi](0, 0);
  });
}
int orc_patch_info(void* hp, int l, int* octant, int* level, int* id, int* parent_coarse) {
  return guard([&] {
    auto* h = static_cast<Handle*>(hp);
    const auto& ops = h->lops(l);
    for (int q = 0; q < ops.layout.n_patch; ++q) {
      const Patch& p = ops.angular.patch(ops.angular.leaves[q]);
      octant[q] = p.octant, level[q] = p.level, id[q] = p.id;
      parent_coarse[q] = (l >= 1) ? h->h().level[l].up[q].coarse : -1;
    }
  });
}
int orc_dense_L(void* hp, double* out) {
  return guard([&] {
    const Mat L = dense_transport_matrix(static_cast<Handle*>(hp)->ops);
    std::memcpy(out, L.a.data(), L.a.size() * sizeof(double));
  });
}
int orc_dense_S(void* hp, int order, double* out) {
  return guard([&] {
    const Mat S = dense_scatter_matrix(static_cast<Handle*>(hp)->ops, order);
    std::memcpy(out, S.a.data(), S.a.size() * sizeof(double));
  });
}

// ------------------------------------------------------------------ meshes
int orc_mesh_stats(int kind, int level, int extra, double angle, int* n_leaves, int* max_level,
                   double* area, int* two_irr, int* min_nbrs, int* max_nbrs) {
  return guard([&] {
    const AngularMesh m = make_mesh(kind, level, extra, angle);
    *n_leaves = m.n_leaves();
    *max_level = m.max_level;
    *area = total_area(m);
    *two_irr = two_irregular(m);
    auto nb = leaf_neighbors(m);
    int lo = 1 << 30, hi = 0;
    for (auto& v : nb) lo = std::min(lo, int(v.size())), hi = std::max(hi, int(v.size()));
    *min_nbrs = lo, *max_nbrs = hi;
  });
}
int orc_mesh_coarsen_count(int kind, int level, int extra, double angle, int to_level, int* n) {
  return guard([&] { *n = coarsen_to_level(make_mesh(kind, level, extra, angle), to_level).n_leaves(); });
}
int orc_refine_count(int patch_id, int* n_leaves) {
  return guard([&] {
    AngularMesh m = build_base_mesh();
    refine(m, patch_id);
    *n_leaves = m.n_leaves();
  });
}
int orc_gauss(int n, double* x, double* w) {
  return guard([&] {
    const Gauss1D& g = gauss_legendre_01(n);
    std::memcpy(x, g.x.data(), n * sizeof(double));
    std::memcpy(w, g.w.data(), n * sizeof(double));
  });
}
int orc_harmonics(int N, const double* omega, double* out) {
  return guard([&] { eval_real_harmonics(N, Vec3{omega[0], omega[1], omega[2]}, out); });
}
int orc_fp_moments(int N, double alpha, double sigma_a, double* moments, double* sigma_t) {
  return guard([&] {
    const ScatterKernel k = fp_equivalent_moments(N, alpha, sigma_a);
    std::memcpy(moments, k.moments.data(), (N + 1) * sizeof(double));
    *sigma_t = k.sigma_t;
  });
}
int orc_nr_default(int N) { return nr_default(N); }
}
