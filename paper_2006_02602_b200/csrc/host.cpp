// host.cpp — host-side logic of the B200 cavity driver and its C-ABI exports.
// Written fresh against the reference's documented behaviour; each function
// cites the reference lines whose semantics it keeps.
#include "host.hpp"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <limits>
#include <stdexcept>

#include "status.hpp"

namespace cav {

namespace {
thread_local std::string g_last_error;
}
void set_last_error(const std::string& msg) { g_last_error = msg; }
const char* last_error_cstr() { return g_last_error.c_str(); }

}  // namespace cav

namespace cav::host {

namespace {
const char* kAxis[3] = {"i", "j", "k"};

bool is_prime(int n) {
  if (n < 2) return false;
  for (int d = 2; d * d <= n; ++d)
    if (n % d == 0) return false;
  return true;
}
}  // namespace

std::string fmt_double_f(double v) {
  char buf[64];
  std::snprintf(buf, sizeof buf, "%f", v);
  return buf;
}

void validate_grid(int nx, int ny, int nz, double dx, double dy, double dz) {
  const int n[3] = {nx, ny, nz};
  const double h[3] = {dx, dy, dz};
  for (int a = 0; a < 3; ++a) {
    if (n[a] < 5)
      throw std::invalid_argument(std::string("grid: axis ") + kAxis[a] + " has " + std::to_string(n[a]) +
                                  " nodes, minimum is 5");
    if (!(h[a] > 0.0) || !std::isfinite(h[a]))
      throw std::invalid_argument(std::string("grid: spacing along ") + kAxis[a] + " must be positive and finite");
  }
}

std::array<double, 3> cavity_spacing(int nx, int ny, int nz, double lx, double ly, double lz) {
  if (nx < 2 || ny < 2 || nz < 2)
    throw std::invalid_argument("grid: need at least 2 nodes per axis to define spacing");
  const std::array<double, 3> h{lx / (nx - 1), ly / (ny - 1), lz / (nz - 1)};
  validate_grid(nx, ny, nz, h[0], h[1], h[2]);
  return h;
}

void validate_params(const cav_fluid_params& p) {
  auto positive = [](double v, const char* name) {
    if (!(v > 0.0) || !std::isfinite(v))
      throw std::invalid_argument(std::string("params: ") + name + " must be positive and finite");
  };
  positive(p.rho, "rho");
  positive(p.nu, "nu");
  positive(p.alpha, "alpha");
  positive(p.u_ref, "u_ref");
  positive(p.length, "length");
  if (!(p.kappa >= 0.0) || !std::isfinite(p.kappa)) throw std::invalid_argument("params: kappa must be >= 0");
  for (double g : p.gravity)
    if (!std::isfinite(g)) throw std::invalid_argument("params: gravity must be finite");
  if (!std::isfinite(p.sigma) || !std::isfinite(p.t_hot) || !std::isfinite(p.t_cold) || !std::isfinite(p.t_inf))
    throw std::invalid_argument("params: temperatures and sigma must be finite");
  if (p.t_hot < p.t_cold) throw std::invalid_argument("params: t_hot must be >= t_cold");
}

cav_fluid_params for_rayleigh(double ra) {
  cav_fluid_params p{};
  p.rho = 1.0;
  p.nu = 1.5e-5;
  p.alpha = 1.5e-5 / 0.71;
  p.gravity[0] = 0.0;
  p.gravity[1] = 0.0;
  p.gravity[2] = -9.81;
  p.u_ref = 0.03;
  p.kappa = 0.01;
  p.t_hot = 300.5;
  p.t_cold = 299.5;
  p.t_inf = 300.0;
  p.length = 0.05;
  const double g = std::sqrt((p.gravity[0] * p.gravity[0] + p.gravity[1] * p.gravity[1]) +
                             p.gravity[2] * p.gravity[2]);
  const double l3 = (p.length * p.length) * p.length;
  p.sigma = ra * p.nu * p.alpha / (g * (p.t_hot - p.t_cold) * l3);
  return p;
}

cav_stencil_params stencil_params(double dx, double dy, double dz, const cav_fluid_params& p) {
  cav_stencil_params s{};
  s.inv2dx = 1.0 / (2.0 * dx);
  s.inv2dy = 1.0 / (2.0 * dy);
  s.inv2dz = 1.0 / (2.0 * dz);
  s.invdx2 = 1.0 / (dx * dx);
  s.invdy2 = 1.0 / (dy * dy);
  s.invdz2 = 1.0 / (dz * dz);
  const double x2 = dx * dx, y2 = dy * dy, z2 = dz * dz;
  s.invdx4 = 1.0 / (x2 * x2);
  s.invdy4 = 1.0 / (y2 * y2);
  s.invdz4 = 1.0 / (z2 * z2);
  s.kdx3 = p.kappa * (x2 * dx);
  s.kdy3 = p.kappa * (y2 * dy);
  s.kdz3 = p.kappa * (z2 * dz);
  s.u_ref = p.u_ref;
  s.nu = p.nu;
  s.alpha = p.alpha;
  s.rho = p.rho;
  s.inv_rho = 1.0 / p.rho;
  s.sigma = p.sigma;
  s.t_inf = p.t_inf;
  s.gx = p.gravity[0];
  s.gy = p.gravity[1];
  s.gz = p.gravity[2];
  return s;
}

double beta_fast_s2(double u_ref) {
  if (!(u_ref > 0.0) || !std::isfinite(u_ref)) return -1.0;
  const double inf = std::numeric_limits<double>::infinity();
  double s = u_ref * u_ref;
  while (s > 0.0 && !(std::sqrt(s) < u_ref)) s = std::nextafter(s, 0.0);
  for (;;) {
    const double t = std::nextafter(s, inf);
    if (!(std::sqrt(t) < u_ref)) break;
    s = t;
  }
  return s;
}

BetaFast beta_fast(double u_ref) {
  BetaFast bf{beta_fast_s2(u_ref), 0u};
  if (u_ref >= 1e-100 && u_ref <= 1e100) {  // u_ref/2 and its squares stay normal
    const double h = u_ref * 0.5;
    uint64_t bits;
    std::memcpy(&bits, &h, sizeof bits);
    bf.hb = static_cast<unsigned>(bits >> 32);
  }
  return bf;
}

std::array<int, 3> choose_dims(int np, int mode) {
  if (np < 1) throw std::invalid_argument("choose_dims: np must be >= 1");
  switch (mode) {
    case CAV_MODE_1D_I: return {np, 1, 1};
    case CAV_MODE_1D_J: return {1, np, 1};
    case CAV_MODE_1D_K: return {1, 1, np};
    case CAV_MODE_2D: {
      if (np > 2 && is_prime(np))
        throw std::invalid_argument("choose_dims: 2d cannot split a prime rank count " + std::to_string(np) +
                                    " into pencils; use 1d-k, or a composite np such as " +
                                    std::to_string(np - 1) + " or " + std::to_string(np + 1));
      int pj = 1;  // largest divisor <= sqrt(np): most balanced pj <= pk
      for (int d = 1; d * d <= np; ++d)
        if (np % d == 0) pj = d;
      return {1, pj, np / pj};
    }
    default: {
      // prime factors, largest first, each onto the smallest running product
      std::vector<int> f;
      int m = np;
      for (int d = 2; d * d <= m; ++d)
        while (m % d == 0) {
          f.push_back(d);
          m /= d;
        }
      if (m > 1) f.push_back(m);
      std::sort(f.rbegin(), f.rend());
      std::array<long long, 3> prod{1, 1, 1};
      for (int x : f) *std::min_element(prod.begin(), prod.end()) *= x;
      std::sort(prod.begin(), prod.end());
      return {static_cast<int>(prod[0]), static_cast<int>(prod[1]), static_cast<int>(prod[2])};
    }
  }
}

std::array<int, 3> decomp_dims(int np, int mode, const int ov[3]) {
  if (ov && ov[0] > 0) {
    if (ov[0] * ov[1] * ov[2] != np) {
      char buf[64];
      std::snprintf(buf, sizeof buf, "%dx%dx%d", ov[0], ov[1], ov[2]);
      throw std::invalid_argument(std::string("decomp: dims ") + buf + " do not multiply to np=" +
                                  std::to_string(np));
    }
    return {ov[0], ov[1], ov[2]};
  }
  return choose_dims(np, mode);
}

std::vector<Extent> partition(std::array<int, 3> n, std::array<int, 3> p) {
  std::array<std::vector<int>, 3> starts;
  for (int a = 0; a < 3; ++a) {
    if (p[a] < 1) throw std::invalid_argument("partition: block counts must be >= 1");
    if (n[a] < p[a])
      throw std::invalid_argument(std::string("partition: axis ") + kAxis[a] + " has fewer nodes than blocks");
  }
  for (int a = 0; a < 3; ++a) {
    const int base = n[a] / p[a], rem = n[a] % p[a];
    if (p[a] > 1 && base < 5)
      throw std::invalid_argument(std::string("partition: axis ") + kAxis[a] + ": " + std::to_string(n[a]) +
                                  " nodes over " + std::to_string(p[a]) + " blocks gives " +
                                  std::to_string(base) + "-node blocks; minimum is 5");
    int pos = 0;
    for (int c = 0; c <= p[a]; ++c) {
      starts[a].push_back(pos);
      pos += base + (c < rem ? 1 : 0);  // remainder to the low blocks
    }
  }
  std::vector<Extent> out(static_cast<std::size_t>(p[0] * p[1] * p[2]));
  for (int ck = 0; ck < p[2]; ++ck)
    for (int cj = 0; cj < p[1]; ++cj)
      for (int ci = 0; ci < p[0]; ++ci) {
        const int r = ci + p[0] * (cj + p[1] * ck);  // ranks i-fastest
        const int c[3] = {ci, cj, ck};
        for (int a = 0; a < 3; ++a) {
          out[r].lo[a] = starts[a][c[a]];
          out[r].hi[a] = starts[a][c[a] + 1];
        }
      }
  return out;
}

std::array<int, 6> neighbors(std::array<int, 3> d, int rank) {
  if (rank < 0 || rank >= d[0] * d[1] * d[2]) throw std::invalid_argument("rank out of range");
  const int c[3] = {rank % d[0], (rank / d[0]) % d[1], rank / (d[0] * d[1])};
  std::array<int, 6> t{CAV_WALL, CAV_WALL, CAV_WALL, CAV_WALL, CAV_WALL, CAV_WALL};
  for (int a = 0; a < 3; ++a)
    for (int s = 0; s < 2; ++s) {
      int nc[3] = {c[0], c[1], c[2]};
      nc[a] += s == 0 ? -1 : 1;
      if (nc[a] < 0 || nc[a] >= d[a]) continue;  // cavity walls, no wrap
      t[2 * a + s] = nc[0] + d[0] * (nc[1] + d[1] * nc[2]);
    }
  return t;
}

std::array<int, 3> center_node(std::array<int, 3> n) { return {(n[0] - 1) / 2, (n[1] - 1) / 2, (n[2] - 1) / 2}; }

int owner_of(const std::vector<Extent>& ext, std::array<int, 3> node) {
  for (std::size_t r = 0; r < ext.size(); ++r) {
    bool in = true;
    for (int a = 0; a < 3; ++a) in = in && node[a] >= ext[r].lo[a] && node[a] < ext[r].hi[a];
    if (in) return static_cast<int>(r);
  }
  throw std::invalid_argument("block map: node outside the global interior");
}

std::array<int, 3> grow_grid(std::array<int, 3> b, int np, int mode, int type) {
  if (type != 1 && type != 2) throw std::invalid_argument("grow_grid: growth type must be 1 or 2");
  if (np < 1 || (np & (np - 1)) != 0)
    throw std::invalid_argument("grow_grid: np must be a power of two, got " + std::to_string(np));
  int m = 0;
  while ((1 << m) < np) ++m;
  int fx = 1, fy = 1, fz = 1;
  if (type == 1 || mode == CAV_MODE_3D) {
    fz = 1 << ((m + 2) / 3);  // doubling round-robin z, y, x
    fy = 1 << ((m + 1) / 3);
    fx = 1 << (m / 3);
  } else if (mode == CAV_MODE_1D_I) {
    fx = np;
  } else if (mode == CAV_MODE_1D_J) {
    fy = np;
  } else if (mode == CAV_MODE_1D_K) {
    fz = np;
  } else if (mode == CAV_MODE_2D) {
    fz = 1 << ((m + 1) / 2);
    fy = 1 << (m / 2);
  }
  return {b[0] * fx, b[1] * fy, b[2] * fz};
}

std::vector<cav_plan_entry> build_plan(std::array<int, 3> n, const std::array<int, 6>& rank_at, int s) {
  validate_grid(n[0], n[1], n[2], 1.0, 1.0, 1.0);
  std::vector<cav_plan_entry> plan;
  for (int f = 0; f < 6; ++f) {
    if (rank_at[f] == CAV_WALL) continue;
    const int axis = f / 2;
    const bool i_face = axis == 0;
    const bool packed = s == CAV_V3 || ((s == CAV_V1 || s == CAV_V2) && i_face);
    const bool sized = s == CAV_V3 || (s == CAV_V2 && i_face);
    long long area = 1;
    for (int a = 0; a < 3; ++a)
      if (a != axis) area *= n[a];
    const int opp = f ^ 1;
    auto depth = [&](int v) { return sized && v != 0 ? 1 : 2; };  // p keeps 2 layers
    if (packed) {
      cav_plan_entry e{};
      e.face = f;
      e.neighbor = rank_at[f];
      e.nvars = 5;
      for (int v = 0; v < 5; ++v) {
        e.var[v] = v;
        e.depth[v] = depth(v);
        e.scalars += area * e.depth[v];
      }
      e.send_tag = opp * 8;  // receiver face * 8 + group 0
      e.recv_tag = f * 8;
      plan.push_back(e);
    } else {
      for (int v = 0; v < 5; ++v) {
        cav_plan_entry e{};
        e.face = f;
        e.neighbor = rank_at[f];
        e.nvars = 1;
        e.var[0] = v;
        e.depth[0] = depth(v);
        e.scalars = area * e.depth[0];
        e.send_tag = opp * 8 + 1 + v;
        e.recv_tag = f * 8 + 1 + v;
        plan.push_back(e);
      }
    }
  }
  return plan;
}

cav_box face_box(std::array<int, 3> n, int face, int depth, bool ghost) {
  if (depth < 1 || depth > 2)
    throw std::invalid_argument("slab: depth must be 1..2, got " + std::to_string(depth));
  const int a = face / 2;
  const bool high = face % 2;
  if (n[a] < depth) throw std::invalid_argument("slab: block too thin for requested depth");
  cav_box b{};
  for (int x = 0; x < 3; ++x) {
    b.lo[x] = 2;  // transverse extent: interior only, corners never travel
    b.hi[x] = n[x] + 2;
  }
  if (!ghost) {
    b.lo[a] = high ? n[a] + 2 - depth : 2;
    b.hi[a] = high ? n[a] + 2 : 2 + depth;
  } else {
    b.lo[a] = high ? n[a] + 2 : 2 - depth;
    b.hi[a] = high ? n[a] + 2 + depth : 2;
  }
  return b;
}

long long box_volume(const cav_box& b) {
  long long v = 1;
  for (int a = 0; a < 3; ++a) {
    if (b.hi[a] <= b.lo[a]) return 0;
    v *= b.hi[a] - b.lo[a];
  }
  return v;
}

void overlap_regions(std::array<int, 3> n, const std::array<int, 6>& rank_at, cav_box* internal,
                     std::vector<cav_box>& external) {
  cav_box rest{{2, 2, 2}, {n[0] + 2, n[1] + 2, n[2] + 2}};
  external.clear();
  for (int f = 0; f < 6; ++f) {  // face-id order keeps the shells disjoint
    if (rank_at[f] == CAV_WALL) continue;
    const int a = f / 2;
    const int depth = std::min(2, rest.hi[a] - rest.lo[a]);
    if (depth <= 0) continue;
    cav_box shell = rest;
    if (f % 2 == 0) {
      shell.hi[a] = rest.lo[a] + depth;
      rest.lo[a] += depth;
    } else {
      shell.lo[a] = rest.hi[a] - depth;
      rest.hi[a] -= depth;
    }
    if (box_volume(shell) > 0) external.push_back(shell);
  }
  *internal = rest;
}

// ---- exact sums ------------------------------------------------------------
constexpr int kLimbs = 35;

void digits_to_limbs(const uint64_t* dig, uint64_t* limbs70) {
  // value = sum_d dig[d] * 2^(32 d); propagate carries in radix 2^32.
  uint32_t w[2 * kLimbs] = {};
  unsigned __int128 carry = 0;
  for (int d = 0; d < 2 * kLimbs; ++d) {
    carry += dig[d];
    w[d] = static_cast<uint32_t>(carry);
    carry >>= 32;
  }
  if (carry != 0) throw std::runtime_error("repro_sum: accumulator overflow");
  for (int l = 0; l < kLimbs; ++l) {
    limbs70[l] = static_cast<uint64_t>(w[2 * l]) | (static_cast<uint64_t>(w[2 * l + 1]) << 32);
    limbs70[kLimbs + l] = 0;  // every norm term is >= 0
  }
}

void repro_merge(uint64_t* a, const uint64_t* b) {
  for (int half = 0; half < 2; ++half) {
    unsigned __int128 c = 0;
    for (int l = 0; l < kLimbs; ++l) {
      c += static_cast<unsigned __int128>(a[half * kLimbs + l]) + b[half * kLimbs + l];
      a[half * kLimbs + l] = static_cast<uint64_t>(c);
      c >>= 64;
    }
  }
}

double repro_value(const uint64_t* limbs70) {
  const uint64_t* pos = limbs70;
  const uint64_t* neg = limbs70 + kLimbs;
  int sign = 0;
  for (int l = kLimbs - 1; l >= 0 && sign == 0; --l)
    if (pos[l] != neg[l]) sign = pos[l] > neg[l] ? 1 : -1;
  if (sign == 0) return 0.0;
  const uint64_t* a = sign > 0 ? pos : neg;
  const uint64_t* b = sign > 0 ? neg : pos;
  uint64_t mag[kLimbs];
  uint64_t borrow = 0;
  for (int l = 0; l < kLimbs; ++l) {
    const unsigned __int128 d = static_cast<unsigned __int128>(a[l]) - b[l] - borrow;
    mag[l] = static_cast<uint64_t>(d);
    borrow = static_cast<uint64_t>(d >> 64) & 1;
  }
  int top = -1;
  for (int l = kLimbs - 1; l >= 0 && top < 0; --l)
    if (mag[l]) top = l * 64 + 63 - __builtin_clzll(mag[l]);
  auto bit = [&](int x) { return static_cast<int>((mag[x >> 6] >> (x & 63)) & 1); };
  const int lo = top <= 52 ? 0 : top - 52;
  uint64_t m = 0;
  for (int x = top; x >= lo; --x) m = (m << 1) | static_cast<uint64_t>(bit(x));
  int e2 = -1140;
  if (top > 52) {  // round to nearest, ties to even, with guard and sticky
    const int g = bit(top - 53);
    bool sticky = false;
    for (int x = top - 54; x >= 0 && !sticky; --x) sticky = bit(x) != 0;
    if (g && (sticky || (m & 1))) {
      if (++m == (1ull << 53)) {
        m >>= 1;
        ++top;
      }
    }
    e2 = top - 52 - 1140;
  }
  const double r = std::ldexp(static_cast<double>(m), e2);
  return sign > 0 ? r : -r;
}

}  // namespace cav::host

// ---- C ABI -----------------------------------------------------------------
using namespace cav;

namespace {
std::array<int, 3> arr3(const int* d) { return {d[0], d[1], d[2]}; }
std::array<int, 6> arr6(const int* d) { return {d[0], d[1], d[2], d[3], d[4], d[5]}; }
}  // namespace

extern "C" {

const char* cav_last_error(void) { return cav::last_error_cstr(); }

void cav_fluid_for_rayleigh(double ra, cav_fluid_params* out) { *out = host::for_rayleigh(ra); }

int cav_validate_params(const cav_fluid_params* p) {
  return guarded([&] { host::validate_params(*p); });
}

int cav_make_cavity_grid(int nx, int ny, int nz, double lx, double ly, double lz, double h[3]) {
  return guarded([&] {
    const auto s = host::cavity_spacing(nx, ny, nz, lx, ly, lz);
    for (int a = 0; a < 3; ++a) h[a] = s[a];
  });
}

void cav_make_stencil_params(double dx, double dy, double dz, const cav_fluid_params* prm,
                             cav_stencil_params* out) {
  *out = host::stencil_params(dx, dy, dz, *prm);
}

int cav_choose_dims(int np, int mode, int out[3]) {
  return guarded([&] {
    const auto d = host::choose_dims(np, mode);
    for (int a = 0; a < 3; ++a) out[a] = d[a];
  });
}

int cav_partition(int nx, int ny, int nz, const int dims[3], int* ext) {
  return guarded([&] {
    const auto e = host::partition({nx, ny, nz}, arr3(dims));
    for (std::size_t r = 0; r < e.size(); ++r)
      for (int a = 0; a < 3; ++a) {
        ext[6 * r + a] = e[r].lo[a];
        ext[6 * r + 3 + a] = e[r].hi[a];
      }
  });
}

int cav_neighbors(const int dims[3], int rank, int rank_at[6]) {
  return guarded([&] {
    const auto t = host::neighbors(arr3(dims), rank);
    for (int f = 0; f < 6; ++f) rank_at[f] = t[f];
  });
}

int cav_center_owner(int nx, int ny, int nz, const int dims[3], int node[3], int* owner) {
  return guarded([&] {
    const auto c = host::center_node({nx, ny, nz});
    *owner = host::owner_of(host::partition({nx, ny, nz}, arr3(dims)), c);
    for (int a = 0; a < 3; ++a) node[a] = c[a];
  });
}

int cav_grow_grid(int nx, int ny, int nz, int np, int mode, int type, int out[3]) {
  return guarded([&] {
    const auto g = host::grow_grid({nx, ny, nz}, np, mode, type);
    for (int a = 0; a < 3; ++a) out[a] = g[a];
  });
}

int cav_build_plan(int nx, int ny, int nz, const int rank_at[6], int strategy, cav_plan_entry* out,
                   int capacity, int* count) {
  return guarded([&] {
    if (strategy < CAV_BASELINE || strategy > CAV_V3) throw std::invalid_argument("plan: unknown strategy");
    const auto p = host::build_plan({nx, ny, nz}, arr6(rank_at), strategy);
    *count = static_cast<int>(p.size());
    if (out)
      for (std::size_t n = 0; n < p.size() && static_cast<int>(n) < capacity; ++n) out[n] = p[n];
  });
}

int cav_overlap_regions(int nx, int ny, int nz, const int rank_at[6], cav_box* internal,
                        cav_box external[6], int* n_external) {
  return guarded([&] {
    std::vector<cav_box> ext;
    host::overlap_regions({nx, ny, nz}, arr6(rank_at), internal, ext);
    *n_external = static_cast<int>(ext.size());
    for (std::size_t n = 0; n < ext.size(); ++n) external[n] = ext[n];
  });
}

int cav_face_interior_box(int nx, int ny, int nz, int face, int depth, cav_box* out) {
  return guarded([&] { *out = host::face_box({nx, ny, nz}, face, depth, false); });
}

int cav_face_ghost_box(int nx, int ny, int nz, int face, int depth, cav_box* out) {
  return guarded([&] { *out = host::face_box({nx, ny, nz}, face, depth, true); });
}

double cav_repro_value(const uint64_t* limbs70) { return host::repro_value(limbs70); }

void cav_repro_merge(uint64_t* a70, const uint64_t* b70) { host::repro_merge(a70, b70); }

void cav_run_config_default(cav_run_config* c) {
  std::memset(c, 0, sizeof *c);
  c->nx = c->ny = c->nz = 32;
  c->np = 1;
  c->mode = CAV_MODE_3D;
  c->strategy = CAV_V3;
  c->overlap = 0;
  c->steps = -1;
  c->fluid = host::for_rayleigh(1e5);
  c->cfl = 0.4;
  c->max_steps = 200000;
  c->conv_tol = 1e-8;
  c->rescale = 1;
  c->check_every = 10;
  c->seed = 0;
  c->timeout_ms = 20000.0;
  c->monitor_every = 0;
  c->verify_tol = 1e-12;
}

}  // extern "C"
