// cell.cuh — per-cell arithmetic shared by every sm_100a kernel in this
// library, so the tiled fused step, the shell/pointwise step and the op-level
// parity kernels produce identical bits.
//
// Operation order follows residual_cell (/root/reference/proj/src/kernels_cell.hpp:14-79)
// exactly. The library is compiled with --fmad=false (no contraction, like the
// reference's -ffp-contract=off, P/CMakeLists.txt:14), IEEE div/sqrt and no
// flush-to-zero, so every +,-,*,/,sqrt rounds exactly as the CPU's does.
#pragma once

#include <cstdint>

#include "cavity_b200.h"

namespace cav {

// std::max / std::min semantics: (a < b) ? b : a and (b < a) ? b : a.
__host__ __device__ __forceinline__ double smax(double a, double b) { return a < b ? b : a; }
__host__ __device__ __forceinline__ double smin(double a, double b) { return b < a ? b : a; }

// Values one cell's residual reads: the 13-point pressure star (+-2 per axis)
// and the 7-point stars (+-1) of u, v, w, T. Corners are never read.
struct Star {
  double p, pxm, pxp, pxm2, pxp2, pym, pyp, pym2, pyp2, pzm, pzp, pzm2, pzp2;
  double u, uxm, uxp, uym, uyp, uzm, uzp;
  double v, vxm, vxp, vym, vyp, vzm, vzp;
  double w, wxm, wxp, wym, wyp, wzm, wzp;
  double t, txm, txp, tym, typ, tzm, tzp;
};

struct Res {
  double p, u, v, w, t;
};

// residual_cell (kernels_cell.hpp:22-78), written once against an accessor S
// that yields the star's values (S::p(), S::pxm(), ...). Every expression and
// its parenthesisation is the reference's; only the order in which independent
// expressions are evaluated is grouped per equation, which keeps fewer values
// live and cannot change any result.
//
// beta = max(sqrt(s2), u_ref) (compute_beta, include/cavity/solver.hpp:73-75)
// with two exact shortcuts (BetaFast, host: host::beta_fast):
//  * hb: when |u|, |v|, |w| all have a high word below hi(u_ref/2), each is
//    below u_ref/2, so s2 <= 3/4 u_ref^2 (+ rounding) < s2 and beta is u_ref:
//    decided with integer ops on the high words, s2 itself is never formed;
//  * s2: the largest double whose correctly rounded square root is still
//    below u_ref; for s2' <= s2 beta is u_ref (sqrt is monotone), so the IEEE
//    sqrt sequence is skipped. NaN always takes the full path.
// {-1, 0} disables both.
struct BetaFast {
  double s2;
  unsigned hb;
};

// The square root is volatile inline PTX (sqrt.rn.f64, the same correctly
// rounded operation) so the compiler cannot hoist it above the branch and
// if-convert: at quiescent cells s2 == 0, which would otherwise run the IEEE
// sequence's special-case call on every cell.
__device__ __forceinline__ double sqrt_rn(double x) {
  double r;
  asm volatile("sqrt.rn.f64 %0, %1;" : "=d"(r) : "d"(x));
  return r;
}
// true unless |u|, |v|, |w| < u_ref/2 is certain from the high words
__device__ __forceinline__ bool speed_not_small(double u, double v, double w, unsigned hb) {
  const unsigned a = static_cast<unsigned>(__double2hiint(u)) & 0x7FFFFFFFu;
  const unsigned b = static_cast<unsigned>(__double2hiint(v)) & 0x7FFFFFFFu;
  const unsigned c = static_cast<unsigned>(__double2hiint(w)) & 0x7FFFFFFFu;
  return max(max(a, b), c) >= hb;
}
__device__ __forceinline__ double beta_of(double u, double v, double w, double u_ref, const BetaFast& bf) {
  double b = u_ref;
  if (speed_not_small(u, v, w, bf.hb)) {
    const double s2 = (u * u + v * v) + w * w;
    if (!(s2 <= bf.s2)) b = smax(sqrt_rn(s2), u_ref);
  }
  return b;
}

template <class S>
__device__ __forceinline__ Res residual_t(const S& s, const cav_stencil_params& q, const BetaFast& bf = {-1.0, 0u}) {
  const double uc = s.u(), vc = s.v(), wc = s.w(), tc = s.t();
  const double b = beta_of(uc, vc, wc, q.u_ref, bf);
  const double b2 = b * b;
  Res r;
  // continuity + fourth-difference damping
  const double ux = (s.uxp() - s.uxm()) * q.inv2dx;
  const double vy = (s.vyp() - s.vym()) * q.inv2dy;
  const double wz = (s.wzp() - s.wzm()) * q.inv2dz;
  const double dv = (ux + vy) + wz;
  const double pc = s.p();
  const double p6 = 6.0 * pc;
  const double pxm = s.pxm(), pxp = s.pxp();
  const double fx = ((((s.pxm2() - 4.0 * pxm) + p6) - 4.0 * pxp) + s.pxp2()) * q.invdx4;
  const double px = (pxp - pxm) * q.inv2dx;
  const double pym = s.pym(), pyp = s.pyp();
  const double fy = ((((s.pym2() - 4.0 * pym) + p6) - 4.0 * pyp) + s.pyp2()) * q.invdy4;
  const double py = (pyp - pym) * q.inv2dy;
  const double pzm = s.pzm(), pzp = s.pzp();
  const double fz = ((((s.pzm2() - 4.0 * pzm) + p6) - 4.0 * pzp) + s.pzp2()) * q.invdz4;
  const double pz = (pzp - pzm) * q.inv2dz;
  const double dmp = b * ((q.kdx3 * fx + q.kdy3 * fy) + q.kdz3 * fz);
  r.p = -b2 * (q.rho * dv + dmp);
  const double by = q.sigma * (tc - q.t_inf);
  // x momentum
  {
    const double uxm = s.uxm(), uxp = s.uxp(), uym = s.uym(), uyp = s.uyp(), uzm = s.uzm(), uzp = s.uzp();
    const double uy = (uyp - uym) * q.inv2dy;
    const double uz = (uzp - uzm) * q.inv2dz;
    const double u2 = 2.0 * uc;
    const double lu = ((uxp - u2) + uxm) * q.invdx2 + ((uyp - u2) + uym) * q.invdy2 + ((uzp - u2) + uzm) * q.invdz2;
    const double cu = (uc * ux + vc * uy) + wc * uz;
    r.u = ((-cu - q.inv_rho * px) + q.nu * lu) + by * q.gx;
  }
  // y momentum
  {
    const double vxm = s.vxm(), vxp = s.vxp(), vym = s.vym(), vyp = s.vyp(), vzm = s.vzm(), vzp = s.vzp();
    const double vx = (vxp - vxm) * q.inv2dx;
    const double vz = (vzp - vzm) * q.inv2dz;
    const double v2 = 2.0 * vc;
    const double lv = ((vxp - v2) + vxm) * q.invdx2 + ((vyp - v2) + vym) * q.invdy2 + ((vzp - v2) + vzm) * q.invdz2;
    const double cv = (uc * vx + vc * vy) + wc * vz;
    r.v = ((-cv - q.inv_rho * py) + q.nu * lv) + by * q.gy;
  }
  // z momentum
  {
    const double wxm = s.wxm(), wxp = s.wxp(), wym = s.wym(), wyp = s.wyp(), wzm = s.wzm(), wzp = s.wzp();
    const double wx = (wxp - wxm) * q.inv2dx;
    const double wy = (wyp - wym) * q.inv2dy;
    const double w2 = 2.0 * wc;
    const double lw = ((wxp - w2) + wxm) * q.invdx2 + ((wyp - w2) + wym) * q.invdy2 + ((wzp - w2) + wzm) * q.invdz2;
    const double cw = (uc * wx + vc * wy) + wc * wz;
    r.w = ((-cw - q.inv_rho * pz) + q.nu * lw) + by * q.gz;
  }
  // energy
  {
    const double txm = s.txm(), txp = s.txp(), tym = s.tym(), typ = s.typ(), tzm = s.tzm(), tzp = s.tzp();
    const double tx = (txp - txm) * q.inv2dx;
    const double ty = (typ - tym) * q.inv2dy;
    const double tz = (tzp - tzm) * q.inv2dz;
    const double t2 = 2.0 * tc;
    const double lt = ((txp - t2) + txm) * q.invdx2 + ((typ - t2) + tym) * q.invdy2 + ((tzp - t2) + tzm) * q.invdz2;
    const double ct = (uc * tx + vc * ty) + wc * tz;
    r.t = -ct + q.alpha * lt;
  }
  return r;
}

// Accessor over a Star value (pointwise kernels).
struct StarAcc {
  const Star& s;
#define CAV_A(n) \
  __device__ __forceinline__ double n() const { return s.n; }
  CAV_A(p) CAV_A(pxm) CAV_A(pxp) CAV_A(pxm2) CAV_A(pxp2) CAV_A(pym) CAV_A(pyp) CAV_A(pym2) CAV_A(pyp2)
  CAV_A(pzm) CAV_A(pzp) CAV_A(pzm2) CAV_A(pzp2)
  CAV_A(u) CAV_A(uxm) CAV_A(uxp) CAV_A(uym) CAV_A(uyp) CAV_A(uzm) CAV_A(uzp)
  CAV_A(v) CAV_A(vxm) CAV_A(vxp) CAV_A(vym) CAV_A(vyp) CAV_A(vzm) CAV_A(vzp)
  CAV_A(w) CAV_A(wxm) CAV_A(wxp) CAV_A(wym) CAV_A(wyp) CAV_A(wzm) CAV_A(wzp)
  CAV_A(t) CAV_A(txm) CAV_A(txp) CAV_A(tym) CAV_A(typ) CAV_A(tzm) CAV_A(tzp)
#undef CAV_A
};

__device__ __forceinline__ Res residual_of(const Star& s, const cav_stencil_params& q,
                                          const BetaFast& bf = {-1.0, 0u}) {
  return residual_t(StarAcc{s}, q, bf);
}

// compute_beta (include/cavity/solver.hpp:73-75) and the per-cell CFL
// denominators |u|+beta, |v|+beta, |w|+beta of compute_dt (src/solver.cpp:220-224).
// dt = cfl*min(min_c h/d_c, visc, therm); because correctly rounded division
// is monotone in d > 0, min_c fl(h/d_c) == fl(h / max_c d_c), so the device
// only needs max_c d_c per axis (an exact, order-free reduction).
struct Denoms {
  double du, dv, dw;
};
__device__ __forceinline__ Denoms cfl_denoms(double u, double v, double w, double u_ref,
                                             const BetaFast& bf = {-1.0, 0u}) {
  const double b = beta_of(u, v, w, u_ref, bf);
  return {fabs(u) + b, fabs(v) + b, fabs(w) + b};
}

// Exponent field all ones <=> inf or NaN (the isfinite test of compute_dt).
__device__ __forceinline__ unsigned nonfinite(double x) {
  return (static_cast<unsigned>(__double2hiint(x)) & 0x7FF00000u) == 0x7FF00000u;
}

// Device storage geometry. Element (i,j,k) of field f (storage coordinates,
// interior at [2, n+2)) lives at base + f*fstride + off + i + pitch*(j + ypitch*k).
// The op-level kernels use the reference Field3 layout (off 0, pitch X, ypitch Y);
// blocks use a padded layout whose interior rows start 128-byte aligned.
struct Geo {
  int nx, ny, nz;
  int pitch, ypitch;
  int off;
  long long fstride;
  __host__ __device__ __forceinline__ long long idx(int i, int j, int k) const {
    return static_cast<long long>(off) + i +
           static_cast<long long>(pitch) * (j + static_cast<long long>(ypitch) * k);
  }
  __host__ __device__ __forceinline__ bool interior(int i, int j, int k) const {
    return i >= 2 && i < nx + 2 && j >= 2 && j < ny + 2 && k >= 2 && k < nz + 2;
  }
};

// ---- exact norm digits -----------------------------------------------------
// ReproSum (inc/util/repro_sum.hpp:19-40) holds value*2^1140 in 64-bit limbs.
// On the device each variable's sum is kept as 70 radix-2^32 digits stored in
// u64 words (carry-save: a word can absorb 2^32 pieces before overflowing).
// A term x >= 0 with exponent field e lands at bit offset e+65 (normal) or 66
// (subnormal), exactly as ReproSum::add; its <= 85-bit shifted mantissa is
// split into three 32-bit pieces added to consecutive digits. The host
// propagates carries into ReproSum limbs and rounds with ReproSum::value.
constexpr int kDigits = 70;
// Per check iteration: 5 x 70 digit words, then the 5 L-inf maxima (bits of
// max |R_v|), padded (CAV_NORM_WORDS in cavity_b200.h).
constexpr int kNormWords = CAV_NORM_WORDS;
static_assert(kNormWords >= 5 * kDigits + 5, "norm words");

struct TermPieces {
  int d;            // first digit
  uint32_t a, b, c; // pieces for digits d, d+1, d+2
};

__device__ __forceinline__ TermPieces term_pieces(double x) {
  const uint64_t bits = static_cast<uint64_t>(__double_as_longlong(x));
  const int e = static_cast<int>((bits >> 52) & 0x7FF);
  uint64_t m = bits & ((1ull << 52) - 1);
  int off = 66;
  if (e != 0) {
    m |= 1ull << 52;
    off = e + 65;
  }
  const int s = off & 31;
  const uint64_t lo = m << s;                       // low 64 bits of m*2^s
  const uint64_t hi = s ? (m >> (64 - s)) : 0ull;   // bits 64.. (< 2^21)
  return {off >> 5, static_cast<uint32_t>(lo), static_cast<uint32_t>(lo >> 32),
          static_cast<uint32_t>(hi)};
}

}  // namespace cav
