// ops.cu — op-level sm_100a kernels behind the reference's backend seam
// (include/cavity/kernels.hpp:42-46 residual_box/update_box, plus the solver
// ops of src/solver.cpp and the slab copies of src/slab.cpp). They operate on
// device arrays in the reference Field3 layout and exist so every op can be
// checked bitwise against the CPU oracle in isolation (tests/test_gpu_ops.py,
// mirroring tests/test_kernels.cpp:77-167 and tests/test_solver.cpp). The
// production path is the fused block pipeline in block.cu, which shares the
// same per-cell arithmetic (cell.cuh).
#include <cuda_runtime.h>

#include <cstring>
#include <vector>

#include "device.cuh"
#include "host.hpp"
#include "ops.hpp"
#include "status.hpp"

namespace cav {

namespace {

Geo field3_geo(int X, int Y, int nz_storage) {
  Geo g{};
  g.nx = X - 4;
  g.ny = Y - 4;
  g.nz = nz_storage - 4;
  g.pitch = X;
  g.ypitch = Y;
  g.off = 0;
  g.fstride = 0;
  return g;
}

struct BoxIter {
  int lo0, lo1, lo2, w, h;
  long long n;
  __device__ __forceinline__ void at(long long q, int& i, int& j, int& k) const {
    i = lo0 + static_cast<int>(q % w);
    const long long r = q / w;
    j = lo1 + static_cast<int>(r % h);
    k = lo2 + static_cast<int>(r / h);
  }
};

BoxIter box_iter(const cav_box& b) {
  BoxIter it{b.lo[0], b.lo[1], b.lo[2], b.hi[0] - b.lo[0], b.hi[1] - b.lo[1], host::box_volume(b)};
  return it;
}

int blocks_for(long long n, int nt) {
  long long b = (n + nt - 1) / nt;
  return static_cast<int>(b < 1 ? 1 : b);
}

__global__ void k_residual_box(cav_field_ptrs in, cav_residual_ptrs out, Geo g, BoxIter it,
                               cav_stencil_params sp) {
  const long long q = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (q >= it.n) return;
  int i, j, k;
  it.at(q, i, j, k);
  const Star s = load_star(in.p, in.u, in.v, in.w, in.t, g, i, j, k, 0.0);
  const Res r = residual_of(s, sp);
  const long long c = g.idx(i, j, k);
  out.p[c] = r.p;
  out.u[c] = r.u;
  out.v[c] = r.v;
  out.w[c] = r.w;
  out.t[c] = r.t;
}

__global__ void k_update_box(double* q, const double* r, double dt, Geo g, BoxIter it) {
  const long long n = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (n >= it.n) return;
  int i, j, k;
  it.at(n, i, j, k);
  const long long c = g.idx(i, j, k);
  q[c] = q[c] + dt * r[c];  // euler_step / update_box_scalar
}

__global__ void k_rescale(double* p, Geo g, BoxIter it, double pc) {
  const long long n = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (n >= it.n) return;
  int i, j, k;
  it.at(n, i, j, k);
  const long long c = g.idx(i, j, k);
  p[c] = p[c] - pc;
}

__global__ void k_copy_box(double* f, Geo g, BoxIter it, double* buf, int to_buf) {
  const long long n = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (n >= it.n) return;
  int i, j, k;
  it.at(n, i, j, k);
  const long long c = g.idx(i, j, k);
  if (to_buf) buf[n] = f[c];
  else f[c] = buf[n];
}

// compute_dt's two scans (src/solver.cpp:200-227) as one pass: non-finite
// mask per field plus the exact max of the CFL denominators.
constexpr int kScanThreads = 256;
__global__ void __launch_bounds__(kScanThreads) k_dt_scan(cav_field_ptrs f, Geo g, BoxIter it,
                                                          double u_ref, Acc* acc, long long it_no,
                                                          int rank) {
  double a = 0.0, b = 0.0, c = 0.0;
  unsigned m = 0;
  for (long long n = blockIdx.x * static_cast<long long>(kScanThreads) + threadIdx.x; n < it.n;
       n += static_cast<long long>(gridDim.x) * kScanThreads) {
    int i, j, k;
    it.at(n, i, j, k);
    const long long q = g.idx(i, j, k);
    const double u = f.u[q], v = f.v[q], w = f.w[q];
    m |= nonfinite(f.p[q]) | (nonfinite(u) << 1) | (nonfinite(v) << 2) | (nonfinite(w) << 3) |
         (nonfinite(f.t[q]) << 4);
    const Denoms d = cfl_denoms(u, v, w, u_ref);
    a = dmax_d(a, d.du);
    b = dmax_d(b, d.dv);
    c = dmax_d(c, d.dw);
  }
  block_reduce_max3_or<kScanThreads>(a, b, c, m);
  if (threadIdx.x == 0) acc_publish(acc, a, b, c, m, it_no, rank);
}

// Exact residual-norm digits (see cell.cuh): per-CTA shared carry-save
// accumulator, flushed with global atomics.
constexpr int kNormThreads = 256;
__global__ void __launch_bounds__(kNormThreads) k_norm_digits(cav_field_ptrs f, Geo g, BoxIter it,
                                                              unsigned long long* dig,
                                                              unsigned* bad) {
  __shared__ unsigned long long sd[5 * kDigits];
  for (int x = threadIdx.x; x < 5 * kDigits; x += kNormThreads) sd[x] = 0;
  __syncthreads();
  unsigned nf = 0;
  for (long long n = blockIdx.x * static_cast<long long>(kNormThreads) + threadIdx.x; n < it.n;
       n += static_cast<long long>(gridDim.x) * kNormThreads) {
    int i, j, k;
    it.at(n, i, j, k);
    const long long q = g.idx(i, j, k);
    const double r[5] = {f.p[q], f.u[q], f.v[q], f.w[q], f.t[q]};
#pragma unroll
    for (int v = 0; v < 5; ++v) {
      const double x = r[v] * r[v];
      nf |= nonfinite(x);
      if (!nonfinite(x)) add_term_digits(sd + v * kDigits, x);
    }
  }
  __syncthreads();
  for (int x = threadIdx.x; x < 5 * kDigits; x += kNormThreads)
    if (sd[x]) atomicAdd(&dig[x], sd[x]);
  if (nf) atomicOr(bad, 1u);
}

// apply_boundary_conditions (src/solver.cpp:129-191): one thread per
// (wall face, transverse interior position); writes both ghost layers of all
// five fields. Faces write disjoint cells and read only the interior, so the
// kernel is order-free.
struct BcArgs {
  double* f[5];
  int step_only;  // 1: only the ghosts a step reads (u,v,w,T first layer)
  Geo g;
  int nfaces;
  int face[6];
  long long start[7];  // prefix sums of transverse counts
  double t_hot, t_cold;
  const IterScalars* sc;
};

__global__ void k_bc(BcArgs a) {
  const long long q = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (q >= a.start[a.nfaces]) return;
  int s = 0;
  while (q >= a.start[s + 1]) ++s;
  const int fid = a.face[s];
  const int ax = fid >> 1, high = fid & 1;
  const int n[3] = {a.g.nx, a.g.ny, a.g.nz};
  const int a1 = ax == 0 ? 1 : 0, a2 = ax == 2 ? 1 : 2;
  const long long r = q - a.start[s];
  int idx[3];
  idx[a1] = 2 + static_cast<int>(r % n[a1]);
  idx[a2] = 2 + static_cast<int>(r / n[a1]);
  const int nn = n[ax];
  const int g1 = high ? nn + 3 : 0, g0 = high ? nn + 2 : 1;
  const int i0 = high ? nn + 1 : 2, i1 = high ? nn : 3, i2 = high ? nn - 1 : 4;
  auto at = [&](int normal) {
    int c[3] = {idx[0], idx[1], idx[2]};
    c[ax] = normal;
    return a.g.idx(c[0], c[1], c[2]);
  };
  const long long cg0 = at(g0), cg1 = at(g1), ci0 = at(i0), ci1 = at(i1), ci2 = at(i2);
#pragma unroll
  for (int v = 1; v <= 3; ++v) {  // no-slip: antisymmetric velocity
    a.f[v][cg0] = -a.f[v][ci0];
    if (!a.step_only) a.f[v][cg1] = -a.f[v][ci1];
  }
  double* T = a.f[4];
  if (ax == 0) {  // isothermal x walls
    const double tw = high ? a.t_cold : a.t_hot;
    T[cg0] = 2.0 * tw - T[ci0];
    if (!a.step_only) T[cg1] = 2.0 * tw - T[ci1];
  } else {  // adiabatic y/z walls
    T[cg0] = T[ci0];
    if (!a.step_only) T[cg1] = T[ci1];
  }
  double* P = a.f[0];
  const double pc = a.sc ? a.sc->pc : 0.0;
  const double p0 = P[ci0] - pc, p1 = P[ci1] - pc, p2 = P[ci2] - pc;
  const double pg0 = (3.0 * p0 - 3.0 * p1) + p2;  // cubic extrapolation
  P[cg0] = pg0;
  P[cg1] = (3.0 * pg0 - 3.0 * p0) + p1;
}

}  // namespace

namespace ops {

void launch_bc(double* const fields[5], const Geo& g, const int walls[6], const cav_fluid_params& prm,
               const IterScalars* sc, cudaStream_t st, bool step_only) {
  BcArgs a{};
  a.step_only = step_only ? 1 : 0;
  for (int v = 0; v < 5; ++v) a.f[v] = fields[v];
  a.g = g;
  a.t_hot = prm.t_hot;
  a.t_cold = prm.t_cold;
  a.sc = sc;
  const int n[3] = {g.nx, g.ny, g.nz};
  a.start[0] = 0;
  for (int f = 0; f < 6; ++f) {
    if (!walls[f]) continue;
    const int ax = f >> 1;
    const int a1 = ax == 0 ? 1 : 0, a2 = ax == 2 ? 1 : 2;
    a.face[a.nfaces] = f;
    a.start[a.nfaces + 1] = a.start[a.nfaces] + static_cast<long long>(n[a1]) * n[a2];
    ++a.nfaces;
  }
  if (a.nfaces == 0) return;
  k_bc<<<blocks_for(a.start[a.nfaces], 256), 256, 0, st>>>(a);
  CAV_CUDA(cudaGetLastError());
}


void residual_box(const cav_field_ptrs& in, const cav_residual_ptrs& out, int X, int Y,
                  const cav_box& box, const cav_stencil_params& sp, cudaStream_t st) {
  const BoxIter it = box_iter(box);
  if (it.n == 0) return;
  k_residual_box<<<blocks_for(it.n, 128), 128, 0, st>>>(in, out, field3_geo(X, Y, 1 << 20), it, sp);
  CAV_CUDA(cudaGetLastError());
}

void update_box(double* q, const double* r, double dt, int X, int Y, const cav_box& box,
                cudaStream_t st) {
  const BoxIter it = box_iter(box);
  if (it.n == 0) return;
  k_update_box<<<blocks_for(it.n, 256), 256, 0, st>>>(q, r, dt, field3_geo(X, Y, 1 << 20), it);
  CAV_CUDA(cudaGetLastError());
}

void preload_kernels() {
  cudaFuncAttributes fa;
  CAV_CUDA(cudaFuncGetAttributes(&fa, k_residual_box));
  CAV_CUDA(cudaFuncGetAttributes(&fa, k_update_box));
  CAV_CUDA(cudaFuncGetAttributes(&fa, k_rescale));
  CAV_CUDA(cudaFuncGetAttributes(&fa, k_copy_box));
  CAV_CUDA(cudaFuncGetAttributes(&fa, k_dt_scan));
  CAV_CUDA(cudaFuncGetAttributes(&fa, k_norm_digits));
  CAV_CUDA(cudaFuncGetAttributes(&fa, k_bc));
}

void launch_dt_scan(const cav_field_ptrs& f, const Geo& g, const cav_box& box, double u_ref, Acc* acc,
                    long long it_no, int rank, cudaStream_t st) {
  const BoxIter it = box_iter(box);
  const int nb = std::min(blocks_for(it.n, kScanThreads), 148 * 8);
  k_dt_scan<<<nb, kScanThreads, 0, st>>>(f, g, it, u_ref, acc, it_no, rank);
  CAV_CUDA(cudaGetLastError());
}

}  // namespace ops
}  // namespace cav

using namespace cav;

extern "C" {

int cav_residual_box(const cav_field_ptrs* in, const cav_residual_ptrs* out, int X, int Y,
                     const cav_box* box, const cav_stencil_params* sp, void* stream) {
  return guarded([&] { ops::residual_box(*in, *out, X, Y, *box, *sp, static_cast<cudaStream_t>(stream)); });
}

int cav_update_box(double* q, const double* r, double dt, int X, int Y, const cav_box* box,
                   void* stream) {
  return guarded([&] { ops::update_box(q, r, dt, X, Y, *box, static_cast<cudaStream_t>(stream)); });
}

int cav_apply_boundary_conditions(const cav_residual_ptrs* f, int nx, int ny, int nz, const int walls[6],
                                  const cav_fluid_params* prm, void* stream) {
  return guarded([&] {
    const Geo g = field3_geo(nx + 4, ny + 4, nz + 4);
    double* fields[5] = {f->p, f->u, f->v, f->w, f->t};
    ops::launch_bc(fields, g, walls, *prm, nullptr, static_cast<cudaStream_t>(stream));
  });
}

int cav_compute_dt(const cav_field_ptrs* f, int nx, int ny, int nz, double dx, double dy, double dz,
                   const cav_fluid_params* prm, double cfl, double* dt_out, void* stream) {
  return guarded([&] {
    if (!(cfl > 0.0) || !std::isfinite(cfl))
      throw std::invalid_argument("compute_dt: cfl must be positive, got " + host::fmt_double_f(cfl));
    const cudaStream_t st = static_cast<cudaStream_t>(stream);
    const Geo g = field3_geo(nx + 4, ny + 4, nz + 4);
    const cav_box ib{{2, 2, 2}, {nx + 2, ny + 2, nz + 2}};
    const BoxIter it = box_iter(ib);
    Acc* acc = nullptr;
    CAV_CUDA(cudaMallocAsync(&acc, sizeof(Acc), st));
    Acc init{};
    init.err = ~0ull;
    CAV_CUDA(cudaMemcpyAsync(acc, &init, sizeof init, cudaMemcpyHostToDevice, st));
    const int nb = std::min(blocks_for(it.n, kScanThreads), 148 * 8);
    k_dt_scan<<<nb, kScanThreads, 0, st>>>(*f, g, it, prm->u_ref, acc, 0, 0);
    CAV_CUDA(cudaGetLastError());
    Acc got{};
    CAV_CUDA(cudaMemcpyAsync(&got, acc, sizeof got, cudaMemcpyDeviceToHost, st));
    CAV_CUDA(cudaFreeAsync(acc, st));
    CAV_CUDA(cudaStreamSynchronize(st));
    if (got.err != ~0ull) {
      static const char* names[5] = {"p", "u", "v", "w", "T"};
      throw std::runtime_error(std::string("compute_dt: non-finite value in field ") +
                               names[(got.err & 15) - 1]);
    }
    *dt_out = ops::dt_from_maxima(got.dmax, dx, dy, dz, *prm, cfl);
  });
}

int cav_rescale_pressure(double* p, int nx, int ny, int nz, double pc, void* stream) {
  return guarded([&] {
    const cav_box ib{{2, 2, 2}, {nx + 2, ny + 2, nz + 2}};
    const BoxIter it = box_iter(ib);
    k_rescale<<<blocks_for(it.n, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
        p, field3_geo(nx + 4, ny + 4, nz + 4), it, pc);
    CAV_CUDA(cudaGetLastError());
  });
}

int cav_residual_norm_partials(const cav_field_ptrs* r, int nx, int ny, int nz, uint64_t* limbs_out,
                               void* stream) {
  return guarded([&] {
    const cudaStream_t st = static_cast<cudaStream_t>(stream);
    const cav_box ib{{2, 2, 2}, {nx + 2, ny + 2, nz + 2}};
    const BoxIter it = box_iter(ib);
    unsigned long long* dig = nullptr;
    const size_t bytes = 5 * kDigits * sizeof(unsigned long long) + 16;
    CAV_CUDA(cudaMallocAsync(&dig, bytes, st));
    CAV_CUDA(cudaMemsetAsync(dig, 0, bytes, st));
    unsigned* bad = reinterpret_cast<unsigned*>(dig + 5 * kDigits);
    const int nb = std::min(blocks_for(it.n, kNormThreads), 148 * 4);
    k_norm_digits<<<nb, kNormThreads, 0, st>>>(*r, field3_geo(nx + 4, ny + 4, nz + 4), it, dig, bad);
    CAV_CUDA(cudaGetLastError());
    std::vector<unsigned long long> h(5 * kDigits + 2);
    CAV_CUDA(cudaMemcpyAsync(h.data(), dig, bytes, cudaMemcpyDeviceToHost, st));
    CAV_CUDA(cudaFreeAsync(dig, st));
    CAV_CUDA(cudaStreamSynchronize(st));
    unsigned badv;
    std::memcpy(&badv, &h[5 * kDigits], sizeof badv);
    if (badv) throw std::invalid_argument("repro_sum: non-finite term");
    for (int v = 0; v < 5; ++v)
      host::digits_to_limbs(reinterpret_cast<const uint64_t*>(&h[v * kDigits]), limbs_out + 70 * v);
  });
}

int cav_copy_box_to(const double* f, int X, int Y, const cav_box* box, double* out, void* stream) {
  return guarded([&] {
    const BoxIter it = box_iter(*box);
    if (it.n == 0) return;
    k_copy_box<<<blocks_for(it.n, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
        const_cast<double*>(f), field3_geo(X, Y, 1 << 20), it, out, 1);
    CAV_CUDA(cudaGetLastError());
  });
}

int cav_copy_box_from(double* f, int X, int Y, const cav_box* box, const double* in, void* stream) {
  return guarded([&] {
    const BoxIter it = box_iter(*box);
    if (it.n == 0) return;
    k_copy_box<<<blocks_for(it.n, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
        f, field3_geo(X, Y, 1 << 20), it, const_cast<double*>(in), 0);
    CAV_CUDA(cudaGetLastError());
  });
}

}  // extern "C"
