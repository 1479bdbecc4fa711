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

// residual_cell, value form (kernels_cell.hpp:22-78).
__device__ __forceinline__ Res residual_of(const Star& s, const cav_stencil_params& q) {
  const double uc = s.u, vc = s.v, wc = s.w, tc = s.t;
  const double speed = sqrt((uc * uc + vc * vc) + wc * wc);
  const double b = smax(speed, q.u_ref);
  const double b2 = b * b;

  const double ux = (s.uxp - s.uxm) * q.inv2dx;
  const double uy = (s.uyp - s.uym) * q.inv2dy;
  const double uz = (s.uzp - s.uzm) * q.inv2dz;
  const double vx = (s.vxp - s.vxm) * q.inv2dx;
  const double vy = (s.vyp - s.vym) * q.inv2dy;
  const double vz = (s.vzp - s.vzm) * q.inv2dz;
  const double wx = (s.wxp - s.wxm) * q.inv2dx;
  const double wy = (s.wyp - s.wym) * q.inv2dy;
  const double wz = (s.wzp - s.wzm) * q.inv2dz;
  const double tx = (s.txp - s.txm) * q.inv2dx;
  const double ty = (s.typ - s.tym) * q.inv2dy;
  const double tz = (s.tzp - s.tzm) * q.inv2dz;
  const double px = (s.pxp - s.pxm) * q.inv2dx;
  const double py = (s.pyp - s.pym) * q.inv2dy;
  const double pz = (s.pzp - s.pzm) * q.inv2dz;

  Res r;
  const double dv = (ux + vy) + wz;
  const double p6 = 6.0 * s.p;
  const double fx = ((((s.pxm2 - 4.0 * s.pxm) + p6) - 4.0 * s.pxp) + s.pxp2) * q.invdx4;
  const double fy = ((((s.pym2 - 4.0 * s.pym) + p6) - 4.0 * s.pyp) + s.pyp2) * q.invdy4;
  const double fz = ((((s.pzm2 - 4.0 * s.pzm) + p6) - 4.0 * s.pzp) + s.pzp2) * q.invdz4;
  const double dmp = b * ((q.kdx3 * fx + q.kdy3 * fy) + q.kdz3 * fz);
  r.p = -b2 * (q.rho * dv + dmp);

  const double u2 = 2.0 * uc, v2 = 2.0 * vc, w2 = 2.0 * wc, t2 = 2.0 * tc;
  const double lu = ((s.uxp - u2) + s.uxm) * q.invdx2 + ((s.uyp - u2) + s.uym) * q.invdy2 +
                    ((s.uzp - u2) + s.uzm) * q.invdz2;
  const double lv = ((s.vxp - v2) + s.vxm) * q.invdx2 + ((s.vyp - v2) + s.vym) * q.invdy2 +
                    ((s.vzp - v2) + s.vzm) * q.invdz2;
  const double lw = ((s.wxp - w2) + s.wxm) * q.invdx2 + ((s.wyp - w2) + s.wym) * q.invdy2 +
                    ((s.wzp - w2) + s.wzm) * q.invdz2;
  const double cu = (uc * ux + vc * uy) + wc * uz;
  const double cv = (uc * vx + vc * vy) + wc * vz;
  const double cw = (uc * wx + vc * wy) + wc * wz;
  const double by = q.sigma * (tc - q.t_inf);
  r.u = ((-cu - q.inv_rho * px) + q.nu * lu) + by * q.gx;
  r.v = ((-cv - q.inv_rho * py) + q.nu * lv) + by * q.gy;
  r.w = ((-cw - q.inv_rho * pz) + q.nu * lw) + by * q.gz;

  const double lt = ((s.txp - t2) + s.txm) * q.invdx2 + ((s.typ - t2) + s.tym) * q.invdy2 +
                    ((s.tzp - t2) + s.tzm) * q.invdz2;
  const double ct = (uc * tx + vc * ty) + wc * tz;
  r.t = -ct + q.alpha * lt;
  return r;
}

// compute_beta (include/cavity/solver.hpp:73-75) and the per-cell CFL
// denominators |u|+beta, |v|+beta, |w|+beta of compute_dt (src/solver.cpp:220-224).
// dt = cfl*min(min_c h/d_c, visc, therm); because correctly rounded division
// is monotone in d > 0, min_c fl(h/d_c) == fl(h / max_c d_c), so the device
// only needs max_c d_c per axis (an exact, order-free reduction).
struct Denoms {
  double du, dv, dw;
};
__device__ __forceinline__ Denoms cfl_denoms(double u, double v, double w, double u_ref) {
  const double b = smax(sqrt((u * u + v * v) + w * w), u_ref);
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
