// ref_driver.cpp — TEST INFRASTRUCTURE ONLY (oracle/, never on the product path).
//
// A thin extern "C" shim over the UNMODIFIED reference library, compiled from
// the sources where they lie under /root/reference/proj/src by oracle/Makefile
// into oracle/_ref/libcavity_ref.so. It exposes the reference's own run_case,
// kernels and host logic with the plain-C structs of include/cavity_b200.h so
// that tests, the golden-fixture generator and bench.py's CPU baseline can
// call the real reference through ctypes. No reference source is copied here.
#include <cmath>
#include <cstring>
#include <exception>
#include <limits>
#include <stdexcept>
#include <string>
#include <vector>

#include "cavity/decomp.hpp"
#include "cavity/exchange.hpp"
#include "cavity/kernels.hpp"
#include "cavity/overlap.hpp"
#include "cavity/runner.hpp"
#include "cavity/slab.hpp"
#include "cavity/solver.hpp"
#include "cavity/util/dump.hpp"
#include "cavity/metrics.hpp"
#include "cavity/util/repro_sum.hpp"
#include "cavity_b200.h"

using namespace cavity;

namespace {

thread_local std::string g_err;

template <typename Fn>
int guard(Fn&& fn) {
  try {
    fn();
    return CAV_OK;
  } catch (const transport::TransportTimeout& e) {
    g_err = e.what();
    return CAV_ETIMEOUT;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return CAV_EINVAL;
  } catch (const std::length_error& e) {
    g_err = e.what();
    return CAV_ELENGTH;
  } catch (const std::logic_error& e) {
    g_err = e.what();
    return CAV_ELOGIC;
  } catch (const std::exception& e) {
    g_err = e.what();
    return CAV_ERUNTIME;
  }
}

FluidParams to_fluid(const cav_fluid_params& f) {
  FluidParams p;
  p.rho = f.rho;
  p.nu = f.nu;
  p.alpha = f.alpha;
  p.sigma = f.sigma;
  p.gravity = {f.gravity[0], f.gravity[1], f.gravity[2]};
  p.u_ref = f.u_ref;
  p.kappa = f.kappa;
  p.t_hot = f.t_hot;
  p.t_cold = f.t_cold;
  p.t_inf = f.t_inf;
  p.length = f.length;
  return p;
}

RunConfig to_config(const cav_run_config& c) {
  RunConfig r;
  r.grid = GridSize3{c.nx, c.ny, c.nz};
  r.np = c.np;
  r.mode = static_cast<DecompMode>(c.mode);
  if (c.dims[0] > 0) r.dims = Dims3{c.dims[0], c.dims[1], c.dims[2]};
  r.strategy = static_cast<Strategy>(c.strategy);
  r.overlap = c.overlap != 0;
  r.steps = static_cast<long>(c.steps);
  r.fluid = to_fluid(c.fluid);
  r.solver.cfl = c.cfl;
  r.solver.max_steps = static_cast<long>(c.max_steps);
  r.solver.conv_tol = c.conv_tol;
  r.solver.rescale = c.rescale != 0;
  r.solver.check_every = c.check_every;
  r.seed = c.seed;
  r.timeout_ms = c.timeout_ms;
  r.monitor_every = c.monitor_every;
  r.verify_tol = c.verify_tol;
  return r;
}

Box to_box(const cav_box& b) {
  return Box{{b.lo[0], b.lo[1], b.lo[2]}, {b.hi[0], b.hi[1], b.hi[2]}};
}

kernels::StencilParams to_sp(const cav_stencil_params& s) {
  static_assert(sizeof(kernels::StencilParams) == sizeof(cav_stencil_params));
  kernels::StencilParams out;
  std::memcpy(&out, &s, sizeof out);
  return out;
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

const char* ref_backend(void) { return kernels::backend_name(kernels::active_backend()); }

int ref_force_backend(int which) {  // -1 auto, 0 scalar, 1 avx2
  return guard([&] {
    if (which < 0) kernels::force_backend(std::nullopt);
    else kernels::force_backend(static_cast<kernels::Backend>(which));
  });
}

int ref_run_case(const cav_run_config* c, const cav_case_options* o, cav_case_result* out) {
  return guard([&] {
    const RunConfig cfg = to_config(*c);
    CaseOptions opt;
    opt.collect_fields = o->collect_fields != 0;
    opt.collect_history = o->collect_history != 0;
    opt.corrupt_exchange = o->corrupt_exchange != 0;
    const CaseResult r = run_case(cfg, opt);
    out->steps_marched = r.steps_marched;
    out->steps_timed = r.steps_timed;
    out->converged = r.converged ? 1 : 0;
    out->np = r.record.np;
    const auto dims = parse_dims(r.record.dims);
    out->dims[0] = dims->pi;
    out->dims[1] = dims->pj;
    out->dims[2] = dims->pk;
    out->wall_time_s = r.record.wall_time_s;
    out->ssspnt = r.record.ssspnt;
    out->bytes_sent = r.record.bytes_sent;
    out->hist_count = static_cast<long long>(r.history.size());
    for (std::size_t n = 0; n < r.history.size() && static_cast<long long>(n) < out->hist_capacity; ++n) {
      out->hist_iter[n] = r.history[n].iteration;
      for (int v = 0; v < 5; ++v) out->hist_l2[5 * n + v] = r.history[n].l2[v];
    }
    for (std::size_t rk = 0; rk < r.ledgers.size() && static_cast<int>(rk) < out->ledger_capacity; ++rk) {
      const ByteLedger& l = r.ledgers[rk];
      cav_ledger& d = out->ledgers[rk];
      for (int f = 0; f < 6; ++f) {
        d.face_bytes[f] = l.face_bytes[f];
        d.face_messages[f] = l.face_messages[f];
        d.last_face_bytes[f] = l.last_face_bytes[f];
      }
      d.bytes_sent = l.bytes_sent;
      d.messages_sent = l.messages_sent;
      d.exchanges = l.exchanges;
    }
    if (out->fields && r.fields) {
      const std::size_t n = r.fields->nodes();
      const std::vector<double>* f[5] = {&r.fields->p, &r.fields->u, &r.fields->v, &r.fields->w,
                                         &r.fields->t};
      for (int v = 0; v < 5; ++v) std::memcpy(out->fields + v * n, f[v]->data(), n * sizeof(double));
    }
  });
}

void ref_run_config_default(cav_run_config* c) {
  const RunConfig r;
  std::memset(c, 0, sizeof *c);
  c->nx = r.grid.nx;
  c->ny = r.grid.ny;
  c->nz = r.grid.nz;
  c->np = r.np;
  c->mode = static_cast<int>(r.mode);
  c->strategy = static_cast<int>(r.strategy);
  c->overlap = r.overlap;
  c->steps = r.steps;
  c->fluid.rho = r.fluid.rho;
  c->fluid.nu = r.fluid.nu;
  c->fluid.alpha = r.fluid.alpha;
  c->fluid.sigma = r.fluid.sigma;
  for (int a = 0; a < 3; ++a) c->fluid.gravity[a] = r.fluid.gravity[a];
  c->fluid.u_ref = r.fluid.u_ref;
  c->fluid.kappa = r.fluid.kappa;
  c->fluid.t_hot = r.fluid.t_hot;
  c->fluid.t_cold = r.fluid.t_cold;
  c->fluid.t_inf = r.fluid.t_inf;
  c->fluid.length = r.fluid.length;
  c->cfl = r.solver.cfl;
  c->max_steps = r.solver.max_steps;
  c->conv_tol = r.solver.conv_tol;
  c->rescale = r.solver.rescale;
  c->check_every = r.solver.check_every;
  c->seed = r.seed;
  c->timeout_ms = r.timeout_ms;
  c->monitor_every = r.monitor_every;
  c->verify_tol = r.verify_tol;
}

// ---- op level (reference kernels on host pointers) ------------------------

void ref_make_stencil_params(double dx, double dy, double dz, const cav_fluid_params* prm,
                             cav_stencil_params* out) {
  Grid3 g;
  g.nx = g.ny = g.nz = 5;
  g.dx = dx;
  g.dy = dy;
  g.dz = dz;
  const kernels::StencilParams sp = make_stencil_params(g, to_fluid(*prm));
  std::memcpy(out, &sp, sizeof *out);
}

int ref_residual_box(const cav_field_ptrs* in, const cav_residual_ptrs* out, int X, int Y,
                     const cav_box* box, const cav_stencil_params* sp, int backend) {
  return guard([&] {
    const kernels::FieldPtrs fi{in->p, in->u, in->v, in->w, in->t};
    const kernels::ResidualPtrs ro{out->p, out->u, out->v, out->w, out->t};
    if (backend == 0) {
      kernels::residual_box_scalar(fi, ro, X, Y, to_box(*box), to_sp(*sp));
    } else {
      kernels::residual_box(fi, ro, X, Y, to_box(*box), to_sp(*sp));
    }
  });
}

int ref_update_box(double* q, const double* r, double dt, int X, int Y, const cav_box* box) {
  return guard([&] { kernels::update_box_scalar(q, r, dt, X, Y, to_box(*box)); });
}

namespace {
// Wraps caller storage (Field3 layout) into a FieldSet and back.
FieldSet load_set(const Grid3& g, double* const ptrs[5]) {
  FieldSet f(g);
  for (int v = 0; v < 5; ++v) std::memcpy(f[static_cast<Var>(v)].data(), ptrs[v], g.cells() * sizeof(double));
  return f;
}
void store_set(const FieldSet& f, double* const ptrs[5]) {
  for (int v = 0; v < 5; ++v)
    std::memcpy(ptrs[v], f[static_cast<Var>(v)].data(), f.grid.cells() * sizeof(double));
}
Grid3 grid_of(int nx, int ny, int nz, double dx, double dy, double dz) {
  Grid3 g;
  g.nx = nx;
  g.ny = ny;
  g.nz = nz;
  g.dx = dx;
  g.dy = dy;
  g.dz = dz;
  return g;
}
}  // namespace

int ref_apply_boundary_conditions(const cav_residual_ptrs* fp, int nx, int ny, int nz,
                                  const int walls[6], const cav_fluid_params* prm) {
  return guard([&] {
    const Grid3 g = grid_of(nx, ny, nz, 1.0, 1.0, 1.0);
    double* const ptrs[5] = {fp->p, fp->u, fp->v, fp->w, fp->t};
    FieldSet f = load_set(g, ptrs);
    WallSet ws;
    for (int i = 0; i < 6; ++i) ws.wall[i] = walls[i] != 0;
    apply_boundary_conditions(f, ws, to_fluid(*prm));
    store_set(f, ptrs);
  });
}

int ref_compute_dt(const cav_field_ptrs* fp, int nx, int ny, int nz, double dx, double dy,
                   double dz, const cav_fluid_params* prm, double cfl, double* dt_out) {
  return guard([&] {
    const Grid3 g = grid_of(nx, ny, nz, dx, dy, dz);
    double* const ptrs[5] = {const_cast<double*>(fp->p), const_cast<double*>(fp->u),
                             const_cast<double*>(fp->v), const_cast<double*>(fp->w),
                             const_cast<double*>(fp->t)};
    const FieldSet f = load_set(g, ptrs);
    *dt_out = compute_dt(f, to_fluid(*prm), cfl);
  });
}

int ref_residual_norm_partials(const cav_field_ptrs* fp, int nx, int ny, int nz, uint64_t* out) {
  return guard([&] {
    const Grid3 g = grid_of(nx, ny, nz, 1.0, 1.0, 1.0);
    double* const ptrs[5] = {const_cast<double*>(fp->p), const_cast<double*>(fp->u),
                             const_cast<double*>(fp->v), const_cast<double*>(fp->w),
                             const_cast<double*>(fp->t)};
    const FieldSet f = load_set(g, ptrs);
    const auto sums = residual_norm_partials(f);
    for (int v = 0; v < 5; ++v) sums[v].serialize(out + v * ReproSum::kSerializedWords);
  });
}

double ref_repro_sum(const double* terms, long long n, int* status) {
  double out = 0.0;
  *status = guard([&] {
    ReproSum s;
    for (long long i = 0; i < n; ++i) s.add(terms[i]);
    out = s.value();
  });
  return out;
}

double ref_repro_value(const uint64_t* limbs70) {
  return ReproSum::deserialize(limbs70).value();
}

int ref_copy_box_to(const double* f, int nx, int ny, int nz, const cav_box* box, double* out) {
  return guard([&] {
    const Grid3 g = grid_of(nx, ny, nz, 1.0, 1.0, 1.0);
    Field3 q(g);
    std::memcpy(q.data(), f, g.cells() * sizeof(double));
    copy_box_to(q, to_box(*box), out);
  });
}

int ref_face_boxes(int nx, int ny, int nz, int face, int depth, cav_box* interior, cav_box* ghost) {
  return guard([&] {
    const Grid3 g = grid_of(nx, ny, nz, 1.0, 1.0, 1.0);
    const Box a = face_interior_box(g, face_from_id(face), depth);
    const Box b = face_ghost_box(g, face_from_id(face), depth);
    for (int i = 0; i < 3; ++i) {
      interior->lo[i] = a.lo[i];
      interior->hi[i] = a.hi[i];
      ghost->lo[i] = b.lo[i];
      ghost->hi[i] = b.hi[i];
    }
  });
}

// ---- host logic ------------------------------------------------------------

int ref_choose_dims(int np, int mode, int out[3]) {
  return guard([&] {
    const Dims3 d = choose_dims(np, static_cast<DecompMode>(mode));
    out[0] = d.pi;
    out[1] = d.pj;
    out[2] = d.pk;
  });
}

int ref_partition(int nx, int ny, int nz, const int dims[3], int* ext) {
  return guard([&] {
    const auto e = partition(GridSize3{nx, ny, nz}, Dims3{dims[0], dims[1], dims[2]});
    for (std::size_t r = 0; r < e.size(); ++r)
      for (int a = 0; a < 3; ++a) {
        ext[6 * r + a] = e[r].lo[a];
        ext[6 * r + 3 + a] = e[r].hi[a];
      }
  });
}

int ref_center_owner(int nx, int ny, int nz, const int dims[3], int node[3], int* owner) {
  return guard([&] {
    const BlockMap m = make_block_map(GridSize3{nx, ny, nz}, Dims3{dims[0], dims[1], dims[2]});
    const auto c = m.center_node();
    for (int a = 0; a < 3; ++a) node[a] = c[a];
    *owner = m.owner_of(c);
  });
}

int ref_grow_grid(int nx, int ny, int nz, int np, int mode, int type, int out[3]) {
  return guard([&] {
    const GridSize3 g = grow_grid(GridSize3{nx, ny, nz}, np, static_cast<DecompMode>(mode), type);
    out[0] = g.nx;
    out[1] = g.ny;
    out[2] = g.nz;
  });
}

int ref_build_plan(int nx, int ny, int nz, const int rank_at[6], int strategy,
                   cav_plan_entry* out, int capacity, int* count) {
  return guard([&] {
    const Grid3 g = grid_of(nx, ny, nz, 1.0, 1.0, 1.0);
    NeighborTable t;
    for (int f = 0; f < 6; ++f) t.rank_at[f] = rank_at[f];
    const ExchangePlan p = build_plan(g, t, static_cast<Strategy>(strategy));
    *count = static_cast<int>(p.entries.size());
    for (std::size_t n = 0; n < p.entries.size() && static_cast<int>(n) < capacity; ++n) {
      const PlanEntry& e = p.entries[n];
      cav_plan_entry& d = out[n];
      std::memset(&d, 0, sizeof d);
      d.face = face_id(e.face);
      d.neighbor = e.neighbor;
      d.nvars = static_cast<int>(e.vars.size());
      for (std::size_t v = 0; v < e.vars.size(); ++v) {
        d.var[v] = static_cast<int>(e.vars[v].var);
        d.depth[v] = e.vars[v].depth;
      }
      d.scalars = static_cast<long long>(e.scalars);
      d.send_tag = e.send_tag;
      d.recv_tag = e.recv_tag;
    }
  });
}

int ref_overlap_regions(int nx, int ny, int nz, const int rank_at[6], cav_box* internal,
                        cav_box external[6], int* n_external) {
  return guard([&] {
    const Grid3 g = grid_of(nx, ny, nz, 1.0, 1.0, 1.0);
    NeighborTable t;
    for (int f = 0; f < 6; ++f) t.rank_at[f] = rank_at[f];
    const OverlapRegions r = compute_overlap_regions(g, t);
    for (int a = 0; a < 3; ++a) {
      internal->lo[a] = r.internal_box.lo[a];
      internal->hi[a] = r.internal_box.hi[a];
    }
    *n_external = static_cast<int>(r.external.size());
    for (std::size_t n = 0; n < r.external.size(); ++n)
      for (int a = 0; a < 3; ++a) {
        external[n].lo[a] = r.external[n].lo[a];
        external[n].hi[a] = r.external[n].hi[a];
      }
  });
}

int ref_write_solution(const char* path, int nx, int ny, int nz, const double* fields) {
  return guard([&] {
    GlobalFields g;
    g.size = GridSize3{nx, ny, nz};
    const std::size_t n = g.nodes();
    std::vector<double>* f[5] = {&g.p, &g.u, &g.v, &g.w, &g.t};
    for (int v = 0; v < 5; ++v) f[v]->assign(fields + v * n, fields + (v + 1) * n);
    write_solution(path, g);
  });
}

int ref_csv_row(int np, const char* mode, const char* dims, const char* strategy, int overlap,
                long long size, long steps, double wall, double ss, double sp, double eff,
                unsigned long long bytes, char* out, int cap) {
  return guard([&] {
    metrics::RunRecord r;
    r.np = np;
    r.mode = mode;
    r.dims = dims;
    r.strategy = strategy;
    r.overlap = overlap;
    r.size = size;
    r.steps = steps;
    r.wall_time_s = wall;
    r.ssspnt = ss;
    r.speedup = sp;
    r.efficiency = eff;
    r.bytes_sent = bytes;
    const std::string s = metrics::csv_header() + "\n" + metrics::csv_row(r);
    std::snprintf(out, static_cast<std::size_t>(cap), "%s", s.c_str());
  });
}

}  // extern "C"
