// device.cuh — device building blocks shared by the op-level parity kernels
// (ops.cu) and the block-level fused pipeline (block.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "cell.cuh"

namespace cav {

// Per-iteration scalars every kernel of iteration n reads: the step dt_n and
// the centre-pressure shift pcs_n. Every block stores the rescaled pressure
// directly: the updated p' of iteration n is written as fl(p' - pcs_n), where
// pcs_n = p'(centre) is computed ahead of the step from the same inputs with
// the same arithmetic (center_p_update on one rank; k_fold over the gathered
// centre stencil on many). That is exactly rescale_pressure
// (src/solver.cpp:248-257), so stored states are always final.
struct IterScalars {
  double dt;
  double pc;   // 0: no shift is ever pending (kept for the op-level k_bc signature)
  double pcs;  // shift the step applies on store (pc_n; 0 with rescale off)
  double pad;
};

// Per-iteration accumulators written by the fused step (and the prologue scan).
struct Acc {
  unsigned long long dmax[3];  // bit patterns of max(|u|+beta), ... (all >= u_ref > 0)
  unsigned long long err;      // min error code, ~0 = none
  unsigned long long pad[4];
};

// Error code ordering = the reference's reporting order: earliest iteration,
// then lowest rank (run_case prefers the lowest non-echo rank,
// src/runner.cpp:294-309), then kind (norms are evaluated before compute_dt,
// src/runner.cpp:200-223): kind 0 = "repro_sum: non-finite term",
// 1..5 = "compute_dt: non-finite value in field p,u,v,w,T".
__host__ __device__ __forceinline__ unsigned long long err_code(long long it, int rank, int kind) {
  return (static_cast<unsigned long long>(it) << 24) | (static_cast<unsigned long long>(rank) << 4) |
         static_cast<unsigned long long>(kind);
}

__device__ __forceinline__ double dmax_d(double a, double b) { return a < b ? b : a; }

// |x| as bits: for non-negative doubles (and +inf, then NaN) the unsigned
// order of the bit patterns is the numeric order, so an integer max is the
// exact L-inf maximum (any grouping, any order).
__device__ __forceinline__ unsigned long long abs_bits(double x) {
  return static_cast<unsigned long long>(__double_as_longlong(x)) & 0x7FFFFFFFFFFFFFFFull;
}
__device__ __forceinline__ unsigned long long warp_max_u64(unsigned long long x) {
  for (int o = 16; o > 0; o >>= 1) x = max(x, __shfl_xor_sync(0xffffffffu, x, o));
  return x;
}

// Loads one cell's star from global memory (layout g). Pressure values of
// interior cells get the pending rescale shift fl(p - pc); ghost values are
// already final. Subtracting +0.0 is the exact identity, so shift==0.0 means
// "no rescale pending".
__device__ __forceinline__ Star load_star(const double* __restrict__ P, const double* __restrict__ U,
                                          const double* __restrict__ V, const double* __restrict__ W,
                                          const double* __restrict__ T, const Geo& g, int i, int j,
                                          int k, double pc) {
  const long long c = g.idx(i, j, k);
  const long long sj = g.pitch, sk = static_cast<long long>(g.pitch) * g.ypitch;
  auto ps = [&](long long off, int ii, int jj, int kk) {
    const double x = P[c + off];
    return x - (g.interior(ii, jj, kk) ? pc : 0.0);
  };
  Star s;
  s.p = ps(0, i, j, k);
  s.pxm = ps(-1, i - 1, j, k);
  s.pxp = ps(1, i + 1, j, k);
  s.pxm2 = ps(-2, i - 2, j, k);
  s.pxp2 = ps(2, i + 2, j, k);
  s.pym = ps(-sj, i, j - 1, k);
  s.pyp = ps(sj, i, j + 1, k);
  s.pym2 = ps(-2 * sj, i, j - 2, k);
  s.pyp2 = ps(2 * sj, i, j + 2, k);
  s.pzm = ps(-sk, i, j, k - 1);
  s.pzp = ps(sk, i, j, k + 1);
  s.pzm2 = ps(-2 * sk, i, j, k - 2);
  s.pzp2 = ps(2 * sk, i, j, k + 2);
#define CAV_Q7(F, A)           \
  s.F = A[c];                  \
  s.F##xm = A[c - 1];          \
  s.F##xp = A[c + 1];          \
  s.F##ym = A[c - sj];         \
  s.F##yp = A[c + sj];         \
  s.F##zm = A[c - sk];         \
  s.F##zp = A[c + sk];
  CAV_Q7(u, U)
  CAV_Q7(v, V)
  CAV_Q7(w, W)
  CAV_Q7(t, T)
#undef CAV_Q7
  return s;
}

// Wall ghosts on the fly (apply_boundary_conditions, src/solver.cpp:158-191):
// a cell next to a wall face gets the ghost values the reference's BC pass
// would have stored, computed from the same (lazily shifted) interior values
// the star already holds, so no separate BC pass touches HBM.
//   u,v,w: g0 = -i0;  T: g0 = 2*t_wall - i0 (x walls) or i0 (y, z walls)
//   p: g0 = (3*i0 - 3*i1) + i2,  g1 = (3*g0 - 3*i0) + i1
struct WallInfo {
  unsigned char wall[6];
  double t_hot, t_cold;
};

__device__ __forceinline__ double cubic_g0(double i0, double i1, double i2) { return (3.0 * i0 - 3.0 * i1) + i2; }
__device__ __forceinline__ double cubic_g1(double g0, double i0, double i1) { return (3.0 * g0 - 3.0 * i0) + i1; }

__device__ __forceinline__ void apply_wall_ghosts(Star& s, const WallInfo& w, const Geo& g, int i, int j, int k) {
  // x walls (isothermal)
  if (w.wall[0] && i == 2) {
    const double g0 = cubic_g0(s.p, s.pxp, s.pxp2);
    s.pxm2 = cubic_g1(g0, s.p, s.pxp);
    s.pxm = g0;
    s.uxm = -s.u;
    s.vxm = -s.v;
    s.wxm = -s.w;
    s.txm = 2.0 * w.t_hot - s.t;
  } else if (w.wall[0] && i == 3) {
    s.pxm2 = cubic_g0(s.pxm, s.p, s.pxp);
  }
  if (w.wall[1] && i == g.nx + 1) {
    const double g0 = cubic_g0(s.p, s.pxm, s.pxm2);
    s.pxp2 = cubic_g1(g0, s.p, s.pxm);
    s.pxp = g0;
    s.uxp = -s.u;
    s.vxp = -s.v;
    s.wxp = -s.w;
    s.txp = 2.0 * w.t_cold - s.t;
  } else if (w.wall[1] && i == g.nx) {
    s.pxp2 = cubic_g0(s.pxp, s.p, s.pxm);
  }
  // y walls (adiabatic)
  if (w.wall[2] && j == 2) {
    const double g0 = cubic_g0(s.p, s.pyp, s.pyp2);
    s.pym2 = cubic_g1(g0, s.p, s.pyp);
    s.pym = g0;
    s.uym = -s.u;
    s.vym = -s.v;
    s.wym = -s.w;
    s.tym = s.t;
  } else if (w.wall[2] && j == 3) {
    s.pym2 = cubic_g0(s.pym, s.p, s.pyp);
  }
  if (w.wall[3] && j == g.ny + 1) {
    const double g0 = cubic_g0(s.p, s.pym, s.pym2);
    s.pyp2 = cubic_g1(g0, s.p, s.pym);
    s.pyp = g0;
    s.uyp = -s.u;
    s.vyp = -s.v;
    s.wyp = -s.w;
    s.typ = s.t;
  } else if (w.wall[3] && j == g.ny) {
    s.pyp2 = cubic_g0(s.pyp, s.p, s.pym);
  }
  // z walls (adiabatic)
  if (w.wall[4] && k == 2) {
    const double g0 = cubic_g0(s.p, s.pzp, s.pzp2);
    s.pzm2 = cubic_g1(g0, s.p, s.pzp);
    s.pzm = g0;
    s.uzm = -s.u;
    s.vzm = -s.v;
    s.wzm = -s.w;
    s.tzm = s.t;
  } else if (w.wall[4] && k == 3) {
    s.pzm2 = cubic_g0(s.pzm, s.p, s.pzp);
  }
  if (w.wall[5] && k == g.nz + 1) {
    const double g0 = cubic_g0(s.p, s.pzm, s.pzm2);
    s.pzp2 = cubic_g1(g0, s.p, s.pzm);
    s.pzp = g0;
    s.uzp = -s.u;
    s.vzp = -s.v;
    s.wzp = -s.w;
    s.tzp = s.t;
  } else if (w.wall[5] && k == g.nz) {
    s.pzp2 = cubic_g0(s.pzp, s.p, s.pzm);
  }
}

// true when the cell touches a wall's two-layer ghost band on any axis
__device__ __forceinline__ bool near_wall(const WallInfo& w, const Geo& g, int i, int j, int k) {
  return (w.wall[0] && i <= 3) || (w.wall[1] && i >= g.nx) || (w.wall[2] && j <= 3) ||
         (w.wall[3] && j >= g.ny) || (w.wall[4] && k <= 3) || (w.wall[5] && k >= g.nz);
}

// p' at one interior cell of `state` (layout g): the cell's residual and
// Euler update exactly as the fused step computes them (compute_residual +
// euler_step, src/solver.cpp:105-120, :234-246), with wall ghosts formed on
// the fly. Used to obtain the centre pressure pc_n before the step that
// stores fl(p' - pc_n) (rescale_pressure, src/solver.cpp:248-257).
__device__ __forceinline__ double center_p_update(const double* state, const Geo& g, const WallInfo& w,
                                                  const cav_stencil_params& sp, const BetaFast& bf, double dt,
                                                  double pc_lazy, int i, int j, int k) {
  const long long fs = g.fstride;
  Star st = load_star(state, state + fs, state + 2 * fs, state + 3 * fs, state + 4 * fs, g, i, j, k, pc_lazy);
  if (near_wall(w, g, i, j, k)) apply_wall_ghosts(st, w, g, i, j, k);
  const Res r = residual_of(st, sp, bf);
  return st.p + dt * r.p;
}

// Block-wide max of three doubles and OR of a mask; thread 0 gets the result.
template <int NT>
__device__ __forceinline__ void block_reduce_max3_or(double& a, double& b, double& c, unsigned& m) {
  __shared__ double sred[3][NT / 32];
  __shared__ unsigned smask[NT / 32];
  for (int o = 16; o > 0; o >>= 1) {
    a = dmax_d(a, __shfl_xor_sync(0xffffffffu, a, o));
    b = dmax_d(b, __shfl_xor_sync(0xffffffffu, b, o));
    c = dmax_d(c, __shfl_xor_sync(0xffffffffu, c, o));
  }
  m = __reduce_or_sync(0xffffffffu, m);
  const int tid = threadIdx.x + blockDim.x * (threadIdx.y + blockDim.y * threadIdx.z);
  const int warp = tid >> 5, lane = tid & 31;
  if (lane == 0) {
    sred[0][warp] = a;
    sred[1][warp] = b;
    sred[2][warp] = c;
    smask[warp] = m;
  }
  __syncthreads();
  if (tid == 0) {
    for (int w = 1; w < NT / 32; ++w) {
      a = dmax_d(a, sred[0][w]);
      b = dmax_d(b, sred[1][w]);
      c = dmax_d(c, sred[2][w]);
      m |= smask[w];
    }
  }
}

// Publishes a block's CFL maxima / non-finite mask into an accumulator.
// Non-negative doubles order like their bit patterns, so an unsigned atomicMax
// on the bits is an exact max.
__device__ __forceinline__ void acc_publish(Acc* acc, double a, double b, double c, unsigned mask,
                                            long long it_for_dt, int rank) {
  atomicMax(&acc->dmax[0], static_cast<unsigned long long>(__double_as_longlong(a)));
  atomicMax(&acc->dmax[1], static_cast<unsigned long long>(__double_as_longlong(b)));
  atomicMax(&acc->dmax[2], static_cast<unsigned long long>(__double_as_longlong(c)));
  if (mask) atomicMin(&acc->err, err_code(it_for_dt, rank, 1 + __ffs(mask) - 1));
}

__device__ __forceinline__ void add_term_digits(unsigned long long* dig, double x) {
  if (x == 0.0) return;
  const TermPieces tp = term_pieces(x);
  atomicAdd(&dig[tp.d], static_cast<unsigned long long>(tp.a));
  atomicAdd(&dig[tp.d + 1], static_cast<unsigned long long>(tp.b));
  if (tp.c) atomicAdd(&dig[tp.d + 2], static_cast<unsigned long long>(tp.c));
}

// ---- exact norms on the device (single thread) -------------------------------
// The host's digits_to_limbs + repro_value (host.cpp, ReproSum::value,
// inc/util/repro_sum.hpp:48-77) for a positive accumulator: carry-save
// radix-2^32 digits -> binary magnitude * 2^-1140, rounded to nearest even.
// NaN on accumulator overflow (the host fold of the same digits throws).
__device__ inline double repro_value_from_digits(const unsigned long long* dig) {
  constexpr int kLimbs = 35;
  unsigned long long mag[kLimbs];
  unsigned __int128 carry = 0;
  for (int l = 0; l < kLimbs; ++l) {
    carry += dig[2 * l];
    const unsigned long long lo = static_cast<unsigned long long>(carry) & 0xFFFFFFFFull;
    carry >>= 32;
    carry += dig[2 * l + 1];
    const unsigned long long hi = static_cast<unsigned long long>(carry) & 0xFFFFFFFFull;
    carry >>= 32;
    mag[l] = lo | (hi << 32);
  }
  if (carry != 0) return __longlong_as_double(0x7FF8000000000000ll);
  int top = -1;
  for (int l = kLimbs - 1; l >= 0 && top < 0; --l)
    if (mag[l]) top = l * 64 + 63 - __clzll(static_cast<long long>(mag[l]));
  if (top < 0) return 0.0;
  auto bit = [&](int x) { return static_cast<int>((mag[x >> 6] >> (x & 63)) & 1); };
  const int lo = top <= 52 ? 0 : top - 52;
  unsigned long long m = 0;
  for (int x = top; x >= lo; --x) m = (m << 1) | static_cast<unsigned long long>(bit(x));
  int e2 = -1140;
  if (top > 52) {  // round to nearest, ties to even, with guard and sticky
    const int gb = bit(top - 53);
    bool sticky = false;
    for (int x = top - 54; x >= 0 && !sticky; --x) sticky = bit(x) != 0;
    if (gb && (sticky || (m & 1))) {
      if (++m == (1ull << 53)) {
        m >>= 1;
        ++top;
      }
    }
    e2 = top - 52 - 1140;
  }
  return ldexp(static_cast<double>(m), e2);
}

// ---- cross-GPU flag protocol (system scope: peers may be other GPUs) ----
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

}  // namespace cav
