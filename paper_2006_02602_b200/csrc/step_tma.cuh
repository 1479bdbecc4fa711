// step_tma.cuh — the fused pseudo-time step (K4), TMA-fed and warp-specialised.
//
// One persistent CTA per SM: TY consumer warps (a 32 x TY tile of cells per
// plane, one cell per consumer thread), one TMA issuer warp, one patcher warp.
//
// Issuer (one lane): streams 36 x (TY+4) plane tiles of all five fields (tile
// plus a 2-cell halo ring) into a ring of R shared-memory slots with
// cp.async.bulk.tensor.4d (completion = the slot's `full` mbarrier transaction
// count); it only waits for a slot to be released (`empty`).
// Patcher (whole warp): as each plane lands it finalises it in place — the
// lazy rescale fl(p - pc) on interior pressure, and the wall ghosts of
// apply_boundary_conditions (src/solver.cpp:158-191) for x/y walls — and
// arrives on the slot's `ready` mbarrier. So consumers read final values only.
//
// Consumer warps: keep their column's k-window in registers (p: k-2..k+2,
// u,v,w,T: k-1..k+1; z-wall ghosts are formed there), read in-plane
// neighbours from the ready slot of plane k, compute residual_t (cell.cuh,
// the reference's arithmetic), the Euler update, the next step's CFL maxima
// and the non-finite flags, store, and release the slot (`empty` mbarrier).
// There is no CTA-wide barrier per plane.
//
// Work: items are (k-chunk, tile) in chunk-major order; CTA c takes items
// c, c+G, c+2G, ... so the ~G items in flight at any time are neighbouring
// tiles of the same chunk: their halo rows are L2 hits, every SM gets the same
// number of items (+-1), and each item restarts the k-window once.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include "device.cuh"
#include "ops.hpp"

namespace cav {

namespace tma {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// try_wait with a suspend-time hint: a waiting warp sleeps in hardware until
// the phase completes (or the hint elapses) instead of re-issuing the probe,
// which keeps idle consumers off the issue slots.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n"
      "@!P1 bra WAIT;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity), "r"(1000000u)
      : "memory");
}
__device__ __forceinline__ void load_4d(void* dst, const CUtensorMap* map, int x, int y, int z, int f,
                                        uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
      "[%6];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(f), "r"(smem_u32(bar))
      : "memory");
}
// L2-only prefetch of one box (no shared-memory destination, no completion).
__device__ __forceinline__ void prefetch_4d(const CUtensorMap* map, int x, int y, int z, int f) {
  asm volatile("cp.async.bulk.prefetch.tensor.4d.L2.global.tile [%0, {%1, %2, %3, %4}];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(x), "r"(y), "r"(z), "r"(f)
               : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void named_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

}  // namespace tma

constexpr int kTmaBW = 36;  // 32 + 2x2 halo
constexpr int kPrefetch = 8;       // L2 prefetch distance, in plane entries

// Tile height TY (= consumer warps), ring depth R and CTAs per SM.
template <int TY_, int R_, int CTAS_>
struct TmaCfg {
  static constexpr int TY = TY_, R = R_, CTAS = CTAS_;
  static constexpr int BH = TY + 4;
  static constexpr int Field = kTmaBW * BH;  // doubles per field plane
  static constexpr int Slot = 5 * Field;     // doubles per slot
  static constexpr int Threads = 32 * (TY + 2);  // consumers + issuer + patcher
  static constexpr size_t Smem = static_cast<size_t>(R) * Slot * sizeof(double) + 3 * R * 8 + 5 * kDigits * 8;
  static_assert(Field * 8 % 128 == 0, "TMA destinations must stay 128-byte aligned");
  static_assert(R >= 5, "ring must hold planes k..k+2 plus prefetch");
};

struct TmaStepArgs {
  double* out;
  Geo g;
  cav_stencil_params sp;
  cav_box box;
  const IterScalars* sc;
  Acc* acc;
  unsigned long long* digits;
  int cx, cy, cz;
  long long n;
  int rank;
  int tiles_x, ntiles, chunk, nchunks;
  WallInfo walls;
  // single-rank fold (replaces k_scalar_sync when np == 1): the last CTA to
  // finish turns this iteration's maxima into dt_{n+1} and publishes pc_n
  int fold;
  unsigned* done;
  IterScalars* sc_next;
  Acc* acc_next;
  unsigned long long* err_sticky;
  double dx, dy, dz, cfl, nu, alpha;
  int rescale;
};

struct ItemGeom {
  int ti0, tj0, kb, ke;
};

template <int TY>
__device__ __forceinline__ ItemGeom item_geom(const TmaStepArgs& a, long long item) {
  const int chunk = static_cast<int>(item / a.ntiles);
  const int tile = static_cast<int>(item % a.ntiles);
  ItemGeom r;
  r.ti0 = a.box.lo[0] + (tile % a.tiles_x) * 32;
  r.tj0 = a.box.lo[1] + (tile / a.tiles_x) * TY;
  r.kb = a.box.lo[2] + chunk * a.chunk;
  r.ke = min(r.kb + a.chunk, a.box.hi[2]);
  return r;
}

// Consumer-side star accessor: in-plane neighbours from the ready slot,
// k-neighbours from the register window.
struct SmemAcc {
  const double *P, *U, *V, *W, *T;
  double pc_, pzm_, pzp_, pzm2_, pzp2_;
  double u_, uzm_, uzp_, v_, vzm_, vzp_, w_, wzm_, wzp_, t_, tzm_, tzp_;
  __device__ __forceinline__ double p() const { return pc_; }
  __device__ __forceinline__ double pxm() const { return P[-1]; }
  __device__ __forceinline__ double pxp() const { return P[1]; }
  __device__ __forceinline__ double pxm2() const { return P[-2]; }
  __device__ __forceinline__ double pxp2() const { return P[2]; }
  __device__ __forceinline__ double pym() const { return P[-kTmaBW]; }
  __device__ __forceinline__ double pyp() const { return P[kTmaBW]; }
  __device__ __forceinline__ double pym2() const { return P[-2 * kTmaBW]; }
  __device__ __forceinline__ double pyp2() const { return P[2 * kTmaBW]; }
  __device__ __forceinline__ double pzm() const { return pzm_; }
  __device__ __forceinline__ double pzp() const { return pzp_; }
  __device__ __forceinline__ double pzm2() const { return pzm2_; }
  __device__ __forceinline__ double pzp2() const { return pzp2_; }
#define CAV_Q(F, A)                                                                       \
  __device__ __forceinline__ double F() const { return F##_; }                           \
  __device__ __forceinline__ double F##xm() const { return A[-1]; }                      \
  __device__ __forceinline__ double F##xp() const { return A[1]; }                       \
  __device__ __forceinline__ double F##ym() const { return A[-kTmaBW]; }                 \
  __device__ __forceinline__ double F##yp() const { return A[kTmaBW]; }                  \
  __device__ __forceinline__ double F##zm() const { return F##zm_; }                     \
  __device__ __forceinline__ double F##zp() const { return F##zp_; }
  CAV_Q(u, U)
  CAV_Q(v, V)
  CAV_Q(w, W)
  CAV_Q(t, T)
#undef CAV_Q
};

// Producer: finalise one landed plane tile in shared memory (all 32 lanes).
template <int BH>
__device__ __forceinline__ void patch_plane(double* slot, const TmaStepArgs& a, const ItemGeom& it, int pl,
                                            double pc, int lane) {
  constexpr int kTmaBH = BH, kTmaField = kTmaBW * BH;
  const Geo& g = a.g;
  if (pl < 2 || pl >= g.nz + 2) return;  // ghost planes: read only as column values
  double* P = slot;
  const int i0 = it.ti0 - 2, j0 = it.tj0 - 2;
  // lazy rescale of interior pressure (rescale_pressure, src/solver.cpp:248-257),
  // two doubles per lane access; element (x, y) is cell (i0 + x, j0 + y)
  {
    constexpr int PAIRS = kTmaBW / 2;
    int row = lane / PAIRS, c = lane % PAIRS;
    for (int idx = lane; idx < kTmaBH * PAIRS; idx += 32) {
      const int j = j0 + row, i = i0 + 2 * c;
      if (j >= 2 && j < g.ny + 2) {
        double2* q = reinterpret_cast<double2*>(P + row * kTmaBW + 2 * c);
        double2 v = *q;
        if (i >= 2 && i < g.nx + 2) v.x = v.x - pc;
        if (i + 1 >= 2 && i + 1 < g.nx + 2) v.y = v.y - pc;
        *q = v;
      }
      c += 32 - PAIRS;  // idx += 32 in (row, c) coordinates
      row += 1;
      if (c >= PAIRS) {
        c -= PAIRS;
        row += 1;
      }
    }
  }
  __syncwarp();
  const WallInfo& w = a.walls;
  double* U = slot + kTmaField;
  double* V = U + kTmaField;
  double* W = V + kTmaField;
  double* T = W + kTmaField;
  // x walls: ghost columns for rows with interior j
  if (w.wall[0] && i0 == 0) {
    for (int y = lane; y < kTmaBH; y += 32) {
      const int j = j0 + y;
      if (j < 2 || j >= g.ny + 2) continue;
      const int r = y * kTmaBW;
      const double g0 = cubic_g0(P[r + 2], P[r + 3], P[r + 4]);
      P[r + 1] = g0;
      P[r] = cubic_g1(g0, P[r + 2], P[r + 3]);
      U[r + 1] = -U[r + 2];
      V[r + 1] = -V[r + 2];
      W[r + 1] = -W[r + 2];
      T[r + 1] = 2.0 * w.t_hot - T[r + 2];
    }
  }
  const int xg = g.nx + 2 - i0;  // tile column of the high x ghost g0
  if (w.wall[1] && xg >= 3 && xg < kTmaBW) {
    for (int y = lane; y < kTmaBH; y += 32) {
      const int j = j0 + y;
      if (j < 2 || j >= g.ny + 2) continue;
      const int r = y * kTmaBW;
      const double g0 = cubic_g0(P[r + xg - 1], P[r + xg - 2], P[r + xg - 3]);
      P[r + xg] = g0;
      if (xg + 1 < kTmaBW) P[r + xg + 1] = cubic_g1(g0, P[r + xg - 1], P[r + xg - 2]);
      U[r + xg] = -U[r + xg - 1];
      V[r + xg] = -V[r + xg - 1];
      W[r + xg] = -W[r + xg - 1];
      T[r + xg] = 2.0 * w.t_cold - T[r + xg - 1];
    }
  }
  // y walls: ghost rows for columns with interior i
  if (w.wall[2] && j0 == 0) {
    for (int x = lane; x < kTmaBW; x += 32) {
      const int i = i0 + x;
      if (i < 2 || i >= g.nx + 2) continue;
      const double g0 = cubic_g0(P[2 * kTmaBW + x], P[3 * kTmaBW + x], P[4 * kTmaBW + x]);
      P[kTmaBW + x] = g0;
      P[x] = cubic_g1(g0, P[2 * kTmaBW + x], P[3 * kTmaBW + x]);
      U[kTmaBW + x] = -U[2 * kTmaBW + x];
      V[kTmaBW + x] = -V[2 * kTmaBW + x];
      W[kTmaBW + x] = -W[2 * kTmaBW + x];
      T[kTmaBW + x] = T[2 * kTmaBW + x];
    }
  }
  const int yg = g.ny + 2 - j0;
  if (w.wall[3] && yg >= 3 && yg < kTmaBH) {
    for (int x = lane; x < kTmaBW; x += 32) {
      const int i = i0 + x;
      if (i < 2 || i >= g.nx + 2) continue;
      const double g0 = cubic_g0(P[(yg - 1) * kTmaBW + x], P[(yg - 2) * kTmaBW + x], P[(yg - 3) * kTmaBW + x]);
      P[yg * kTmaBW + x] = g0;
      if (yg + 1 < kTmaBH) P[(yg + 1) * kTmaBW + x] = cubic_g1(g0, P[(yg - 1) * kTmaBW + x], P[(yg - 2) * kTmaBW + x]);
      U[yg * kTmaBW + x] = -U[(yg - 1) * kTmaBW + x];
      V[yg * kTmaBW + x] = -V[(yg - 1) * kTmaBW + x];
      W[yg * kTmaBW + x] = -W[(yg - 1) * kTmaBW + x];
      T[yg * kTmaBW + x] = T[(yg - 1) * kTmaBW + x];
    }
  }
}

template <class Cfg, bool NORMS>
__global__ void __launch_bounds__(Cfg::Threads, Cfg::CTAS)
    k_step_tma(const __grid_constant__ CUtensorMap map, const TmaStepArgs a) {
  constexpr int C = Cfg::TY, R = Cfg::R, BW = kTmaBW;
  constexpr int kTmaField = Cfg::Field, kTmaSlot = Cfg::Slot, kTmaThreads = Cfg::Threads;
  extern __shared__ __align__(128) unsigned char smraw[];
  double* ring = reinterpret_cast<double*>(smraw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smraw + R * kTmaSlot * sizeof(double));
  uint64_t* ready = full + R;
  uint64_t* empty = ready + R;
  unsigned long long* sdig = reinterpret_cast<unsigned long long*>(empty + R);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < R; ++s) {
      tma::mbar_init(&full[s], 1);
      tma::mbar_init(&ready[s], 1);
      tma::mbar_init(&empty[s], C);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (NORMS)
    for (int x = threadIdx.x; x < 5 * kDigits; x += kTmaThreads) sdig[x] = 0;
  __syncthreads();

  const long long total = static_cast<long long>(a.ntiles) * a.nchunks;
  const long long G = gridDim.x;
  const double pc = a.sc->pc;

  if (warp == C) {
    // ---------------- TMA issuer (one lane) ----------------
    // A second cursor runs kPrefetch entries ahead and pulls those planes
    // into L2 (no smem), so the ring's own loads hit L2 instead of waiting
    // out DRAM latency with only R-3 slots in flight.
    if (lane != 0) return;
    int s = 0;
    uint32_t ph = 0, e = 0;  // slot / empty-barrier phase of entry e
    long long pf_item = blockIdx.x;
    ItemGeom pf{0, 0, 0, 0};
    int pf_pl = 0;
    if (pf_item < total) {
      pf = item_geom<C>(a, pf_item);
      pf_pl = pf.kb - 2;
    }
    auto prefetch_next = [&]() {
      if (pf_item >= total) return;
#pragma unroll
      for (int f = 0; f < 5; ++f) tma::prefetch_4d(&map, a.g.off + pf.ti0 - 2, pf.tj0 - 2, pf_pl, f);
      if (++pf_pl > pf.ke + 1) {
        pf_item += G;
        if (pf_item < total) {
          pf = item_geom<C>(a, pf_item);
          pf_pl = pf.kb - 2;
        }
      }
    };
    for (int q = 0; q < kPrefetch; ++q) prefetch_next();
    for (long long item = blockIdx.x; item < total; item += G) {
      const ItemGeom it = item_geom<C>(a, item);
      const int x0 = a.g.off + it.ti0 - 2, y0 = it.tj0 - 2;
      for (int pl = it.kb - 2; pl <= it.ke + 1; ++pl, ++e) {
        prefetch_next();
        if (e >= static_cast<uint32_t>(R)) tma::mbar_wait(&empty[s], ph ^ 1);
        tma::mbar_expect_tx(&full[s], kTmaSlot * sizeof(double));
        double* dst = ring + s * kTmaSlot;
#pragma unroll
        for (int f = 0; f < 5; ++f) tma::load_4d(dst + f * kTmaField, &map, x0, y0, pl, f, &full[s]);
        if (++s == R) {
          s = 0;
          ph ^= 1;
        }
      }
    }
    return;
  }
  if (warp == C + 1) {
    // ---------------- patcher (whole warp) ----------------
    int s = 0;
    uint32_t ph = 0;
    for (long long item = blockIdx.x; item < total; item += G) {
      const ItemGeom it = item_geom<C>(a, item);
      for (int pl = it.kb - 2; pl <= it.ke + 1; ++pl) {
        tma::mbar_wait(&full[s], ph);
        patch_plane<Cfg::BH>(ring + s * kTmaSlot, a, it, pl, pc, lane);
        tma::fence_proxy_async();  // generic writes before the slot's next TMA fill
        __syncwarp();
        if (lane == 0) tma::mbar_arrive(&ready[s]);
        if (++s == R) {
          s = 0;
          ph ^= 1;
        }
      }
    }
    return;
  }

  // ---------------- consumers ----------------
  // Each step computes two planes (k, k+1) of the thread's column: the
  // k-windows are shared (p: k-2..k+3, u,v,w,T: k-1..k+2), waits/releases and
  // loop control are paid once per two cells, and the two independent
  // residuals interleave.
  const int tx = lane, ty = warp;
  const Geo g = a.g;
  const double dt = a.sc->dt, u_ref = a.sp.u_ref;
  const long long fs = g.fstride;
  const long long plane = static_cast<long long>(g.pitch) * g.ypitch;
  const bool zlo = a.walls.wall[4], zhi = a.walls.wall[5];
  double m0 = 0.0, m1 = 0.0, m2 = 0.0;
  unsigned e_p = 0, e_u = 0, e_v = 0, e_w = 0, e_t = 0;  // max exponent field per variable
  unsigned nbad = 0;
  const double* ringc = ring + (ty + 2) * BW + tx + 2;  // own cell in slot 0, field 0
  int sw = 0;  // slot of the next entry to wait for, and its phase
  uint32_t phw = 0;
  auto advance = [&](int& sl, uint32_t& ph) {
    if (++sl == R) {
      sl = 0;
      ph ^= 1;
    }
  };
  auto wait_next = [&]() {
    const int sl = sw;
    tma::mbar_wait(&ready[sw], phw);
    advance(sw, phw);
    return sl;
  };
  auto release_slot = [&](int sl) {
    __syncwarp();
    if (lane == 0) tma::mbar_arrive(&empty[sl]);
  };
  auto slot = [&](int sl) { return ringc + sl * kTmaSlot; };

  // z-wall ghosts inside the register windows (apply_boundary_conditions for
  // the z walls). Two-plane step at k: P[0..5] = planes k-2..k+3,
  // Q[f][0..3] = planes k-1..k+2; one-plane step: P[0..4], Q[f][0..2].
  // Only compile-time indices, so the windows stay in registers.
  auto qmirror = [&](double (*Q)[4], int gi, int ii) {  // ghost gi from interior ii
    Q[0][gi] = -Q[0][ii];
    Q[1][gi] = -Q[1][ii];
    Q[2][gi] = -Q[2][ii];
    Q[3][gi] = Q[3][ii];
  };
  auto zwall2 = [&](double* P, double (*Q)[4], int k) {
    if (zlo && k == 2) {
      P[1] = cubic_g0(P[2], P[3], P[4]);
      P[0] = cubic_g1(P[1], P[2], P[3]);
      qmirror(Q, 0, 1);
    } else if (zlo && k == 3) {
      P[0] = cubic_g0(P[1], P[2], P[3]);
    }
    if (zhi && k == g.nz - 1) {
      P[5] = cubic_g0(P[4], P[3], P[2]);
    } else if (zhi && k == g.nz) {
      P[4] = cubic_g0(P[3], P[2], P[1]);
      P[5] = cubic_g1(P[4], P[3], P[2]);
      qmirror(Q, 3, 2);
    }
  };
  auto zwall1 = [&](double* P, double (*Q)[4], int k) {
    if (zlo && k == 2) {
      P[1] = cubic_g0(P[2], P[3], P[4]);
      P[0] = cubic_g1(P[1], P[2], P[3]);
      qmirror(Q, 0, 1);
    } else if (zlo && k == 3) {
      P[0] = cubic_g0(P[1], P[2], P[3]);
    }
    if (zhi && k == g.nz) {
      P[4] = cubic_g0(P[3], P[2], P[1]);
    } else if (zhi && k == g.nz + 1) {
      P[3] = cubic_g0(P[2], P[1], P[0]);
      P[4] = cubic_g1(P[3], P[2], P[1]);
      qmirror(Q, 2, 1);
    }
  };

  // one cell: residual + update + store + bookkeeping
  auto cell = [&](const double* B, double p0, double pzm, double pzp, double pzm2, double pzp2, const double* qc,
                  const double* qm, const double* qp, double* op, bool ccolk) {
    const SmemAcc sa{B, B + kTmaField, B + 2 * kTmaField, B + 3 * kTmaField, B + 4 * kTmaField,
                     p0, pzm, pzp, pzm2, pzp2, qc[0], qm[0], qp[0], qc[1], qm[1], qp[1], qc[2], qm[2], qp[2],
                     qc[3], qm[3], qp[3]};
    const Res r = residual_t(sa, a.sp);
    const double qpn = p0 + dt * r.p, qun = qc[0] + dt * r.u, qvn = qc[1] + dt * r.v, qwn = qc[2] + dt * r.w,
                 qtn = qc[3] + dt * r.t;
    // explicit global (streaming) stores: no possible aliasing with the
    // shared-memory ring, so the two cells of a step can interleave
    __stcs(op, qpn);
    __stcs(op + fs, qun);
    __stcs(op + 2 * fs, qvn);
    __stcs(op + 3 * fs, qwn);
    __stcs(op + 4 * fs, qtn);
    const Denoms d = cfl_denoms(qun, qvn, qwn, u_ref);
    m0 = dmax_d(m0, d.du);
    m1 = dmax_d(m1, d.dv);
    m2 = dmax_d(m2, d.dw);
    e_p = max(e_p, static_cast<unsigned>(__double2hiint(qpn)) & 0x7FF00000u);
    e_u = max(e_u, static_cast<unsigned>(__double2hiint(qun)) & 0x7FF00000u);
    e_v = max(e_v, static_cast<unsigned>(__double2hiint(qvn)) & 0x7FF00000u);
    e_w = max(e_w, static_cast<unsigned>(__double2hiint(qwn)) & 0x7FF00000u);
    e_t = max(e_t, static_cast<unsigned>(__double2hiint(qtn)) & 0x7FF00000u);
    if (ccolk) a.acc->pc_local = qpn;
    if (NORMS) {
      const double rr[5] = {r.p * r.p, r.u * r.u, r.v * r.v, r.w * r.w, r.t * r.t};
#pragma unroll
      for (int v = 0; v < 5; ++v) {
        if (nonfinite(rr[v])) nbad = 1;
        else add_term_digits(sdig + v * kDigits, rr[v]);
      }
    }
  };

  for (long long item = blockIdx.x; item < total; item += G) {
    const ItemGeom it = item_geom<C>(a, item);
    const int len = it.ke - it.kb;
    const int i = it.ti0 + tx, j = it.tj0 + ty;
    const bool active = i < a.box.hi[0] && j < a.box.hi[1];
    const bool ccol = i == a.cx && j == a.cy;
    // prologue: planes kb-2 .. kb+1
    const int s0 = wait_next(), s1 = wait_next(), s2 = wait_next(), s3 = wait_next();
    double P[6];     // p at planes k-2 .. k+3
    double Q[4][4];  // u,v,w,T at planes k-1 .. k+2
    P[0] = slot(s0)[0];
    P[1] = slot(s1)[0];
    P[2] = slot(s2)[0];
    P[3] = slot(s3)[0];
#pragma unroll
    for (int f = 0; f < 4; ++f) {
      Q[f][0] = slot(s1)[(f + 1) * kTmaField];
      Q[f][1] = slot(s2)[(f + 1) * kTmaField];
    }
    release_slot(s0);
    release_slot(s1);
    int sc0 = s2, sc1 = s3;  // slots of planes k, k+1
    double* op = a.out + g.idx(i, j, it.kb);
    int st = 0;
    for (; st + 1 < len; st += 2, op += 2 * plane) {
      const int k = it.kb + st;
      const int sc2 = wait_next(), sc3 = wait_next();  // planes k+2, k+3
      P[4] = slot(sc2)[0];
      P[5] = slot(sc3)[0];
#pragma unroll
      for (int f = 0; f < 4; ++f) {
        Q[f][2] = slot(sc1)[(f + 1) * kTmaField];
        Q[f][3] = slot(sc2)[(f + 1) * kTmaField];
      }
      if ((zlo && k <= 3) || (zhi && k + 3 >= g.nz + 2)) zwall2(P, Q, k);
      if (active) {
        const double qa[4] = {Q[0][1], Q[1][1], Q[2][1], Q[3][1]};
        const double qam[4] = {Q[0][0], Q[1][0], Q[2][0], Q[3][0]};
        const double qap[4] = {Q[0][2], Q[1][2], Q[2][2], Q[3][2]};
        const double qbp[4] = {Q[0][3], Q[1][3], Q[2][3], Q[3][3]};
        cell(slot(sc0), P[2], P[1], P[3], P[0], P[4], qa, qam, qap, op, ccol && k == a.cz);
        cell(slot(sc1), P[3], P[2], P[4], P[1], P[5], qap, qa, qbp, op + plane, ccol && k + 1 == a.cz);
      }
      release_slot(sc0);
      release_slot(sc1);
      sc0 = sc2;
      sc1 = sc3;
      P[0] = P[2];
      P[1] = P[3];
      P[2] = P[4];
      P[3] = P[5];
#pragma unroll
      for (int f = 0; f < 4; ++f) {
        Q[f][0] = Q[f][2];
        Q[f][1] = Q[f][3];
      }
    }
    if (st < len) {  // odd remainder: one plane
      const int k = it.kb + st;
      const int sc2 = wait_next();  // plane k+2
      P[4] = slot(sc2)[0];
#pragma unroll
      for (int f = 0; f < 4; ++f) Q[f][2] = slot(sc1)[(f + 1) * kTmaField];
      if ((zlo && k <= 3) || (zhi && k + 2 >= g.nz + 2)) zwall1(P, Q, k);
      if (active) {
        const double qa[4] = {Q[0][1], Q[1][1], Q[2][1], Q[3][1]};
        const double qam[4] = {Q[0][0], Q[1][0], Q[2][0], Q[3][0]};
        const double qap[4] = {Q[0][2], Q[1][2], Q[2][2], Q[3][2]};
        cell(slot(sc0), P[2], P[1], P[3], P[0], P[4], qa, qam, qap, op, ccol && k == a.cz);
      }
      release_slot(sc0);
      sc0 = sc1;
      sc1 = sc2;
      // remaining entries: plane k+1 (sc0 now) was waited; plane k+2 (sc1) waited
      release_slot(sc0);
      release_slot(sc1);
    } else {
      // planes ke, ke+1 (sc0, sc1) served only as column values
      release_slot(sc0);
      release_slot(sc1);
    }
  }
  constexpr unsigned EXP = 0x7FF00000u;
  unsigned bad = (e_p == EXP ? 1u : 0u) | (e_u == EXP ? 2u : 0u) | (e_v == EXP ? 4u : 0u) |
                 (e_w == EXP ? 8u : 0u) | (e_t == EXP ? 16u : 0u);

  // consumer-only reductions
  constexpr int NC = 32 * C;
  __shared__ double sred[3][C];
  __shared__ unsigned smask[C];
  for (int o = 16; o > 0; o >>= 1) {
    m0 = dmax_d(m0, __shfl_xor_sync(0xffffffffu, m0, o));
    m1 = dmax_d(m1, __shfl_xor_sync(0xffffffffu, m1, o));
    m2 = dmax_d(m2, __shfl_xor_sync(0xffffffffu, m2, o));
  }
  bad = __reduce_or_sync(0xffffffffu, bad);
  nbad = __reduce_or_sync(0xffffffffu, nbad);
  if (lane == 0) {
    sred[0][warp] = m0;
    sred[1][warp] = m1;
    sred[2][warp] = m2;
    smask[warp] = bad | (nbad << 8);
  }
  tma::named_sync(1, NC);
  if (threadIdx.x == 0) {
    unsigned mk = 0;
    for (int w = 0; w < C; ++w) {
      m0 = dmax_d(m0, sred[0][w]);
      m1 = dmax_d(m1, sred[1][w]);
      m2 = dmax_d(m2, sred[2][w]);
      mk |= smask[w];
    }
    acc_publish(a.acc, m0, m1, m2, mk & 0xFF, a.n + 1, a.rank);
    if (NORMS && (mk >> 8)) atomicMin(&a.acc->err, err_code(a.n, a.rank, 0));
    if (a.fold) {
      __threadfence();
      if (atomicAdd(a.done, 1u) == gridDim.x - 1) {  // every CTA has published
        __threadfence();
        volatile Acc* acc = a.acc;
        const unsigned long long dm[3] = {acc->dmax[0], acc->dmax[1], acc->dmax[2]};
        cav_fluid_params fl{};
        fl.nu = a.nu;
        fl.alpha = a.alpha;
        a.sc_next->dt = ops::dt_from_maxima(dm, a.dx, a.dy, a.dz, fl, a.cfl);
        a.sc_next->pc = a.rescale ? acc->pc_local : 0.0;
        const unsigned long long e = acc->err;
        if (e < *a.err_sticky) *a.err_sticky = e;
        Acc z{};
        z.err = ~0ull;
        *a.acc_next = z;
        *a.done = 0;
      }
    }
  }
  if (NORMS)
    for (int x = threadIdx.x; x < 5 * kDigits; x += NC)
      if (sdig[x]) atomicAdd(&a.digits[x], sdig[x]);
}

}  // namespace cav
