// step_tma.cuh — the fused pseudo-time step (K4) fed by TMA.
//
// One CTA = 1 producer warp + TY consumer warps (32 x TY cells per plane).
// The producer streams 36 x (TY+4) plane tiles of all five fields (the tile
// plus a 2-cell halo ring; corners ride along and are never read) into a ring
// of R shared-memory slots with cp.async.bulk.tensor, completion tracked by
// mbarrier transaction counts. Consumers keep their own column's k-window in
// registers (p: k-2..k+2, u,v,w,T: k-1..k+1), read in-plane neighbours from
// the slot of plane k, and release a slot through an `empty` mbarrier when no
// later step needs it. There is no CTA-wide barrier per plane.
//
// Work: the (tile, plane) space of the box is linearised tile-major and split
// evenly over a grid of exactly `ctas_per_sm x #SMs` CTAs; each CTA walks one
// or two contiguous segments (a segment restarts the k-window), so every SM
// gets the same number of cell updates (no wave tail).
//
// Arithmetic per cell is residual_of() from cell.cuh — identical to the
// pointwise kernels — so results are bitwise those of the reference.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include "device.cuh"

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
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
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
__device__ __forceinline__ void consumer_sync(int nthreads) {
  asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");
}

}  // namespace tma

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
  int tiles_x, tiles_y;
  long long total;  // tiles * depth
  WallInfo walls;   // wall ghosts are computed in-kernel (no BC pass)
};

constexpr int kTmaTY = 8;          // consumer warps per CTA / tile rows
constexpr int kTmaRing = 6;        // plane slots
constexpr int kTmaBW = 36;         // 32 + 2x2 halo
constexpr int kTmaBH = kTmaTY + 4;
constexpr int kTmaField = kTmaBW * kTmaBH;            // doubles per field plane
constexpr int kTmaSlot = 5 * kTmaField;               // doubles per slot
constexpr int kTmaThreads = 32 * (kTmaTY + 1);
constexpr size_t kTmaSmem = kTmaRing * kTmaSlot * sizeof(double) + 3 * kTmaRing * 8 + 5 * kDigits * 8 + 128;

template <bool NORMS>
__global__ void __maxnreg__(112)
    k_step_tma(const __grid_constant__ CUtensorMap map, const TmaStepArgs a) {
  constexpr int TY = kTmaTY, C = kTmaTY, R = kTmaRing, BW = kTmaBW;
  extern __shared__ __align__(128) unsigned char smraw[];
  double* ring = reinterpret_cast<double*>(smraw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smraw + R * kTmaSlot * sizeof(double));
  uint64_t* empty = full + R;
  unsigned long long* sdig = reinterpret_cast<unsigned long long*>(empty + 2 * R);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < R; ++s) {
      tma::mbar_init(&full[s], 1);
      tma::mbar_init(&empty[s], C);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (NORMS)
    for (int x = threadIdx.x; x < 5 * kDigits; x += kTmaThreads) sdig[x] = 0;
  __syncthreads();

  const int bd = a.box.hi[2] - a.box.lo[2];
  const long long u0 = a.total * blockIdx.x / gridDim.x;
  const long long u1 = a.total * (blockIdx.x + 1) / gridDim.x;

  if (warp == C) {
    // ---------------- producer ----------------
    if (lane == 0) {
      uint32_t e = 0;
      for (long long u = u0; u < u1;) {
        const int tile = static_cast<int>(u / bd);
        const int kb = a.box.lo[2] + static_cast<int>(u % bd);
        const long long rem_ = bd - u % bd;
        const int len = static_cast<int>(rem_ < u1 - u ? rem_ : u1 - u);
        const int ti0 = a.box.lo[0] + (tile % a.tiles_x) * 32;
        const int tj0 = a.box.lo[1] + (tile / a.tiles_x) * TY;
        for (int pl = kb - 2; pl <= kb + len + 1; ++pl, ++e) {
          const int s = e % R;
          if (e >= R) tma::mbar_wait(&empty[s], ((e / R) - 1) & 1);
          tma::mbar_expect_tx(&full[s], kTmaSlot * sizeof(double));
          double* dst = ring + s * kTmaSlot;
#pragma unroll
          for (int f = 0; f < 5; ++f) tma::load_4d(dst + f * kTmaField, &map, a.g.off + ti0 - 2, tj0 - 2, pl, f, &full[s]);
        }
        u += len;
      }
    }
    return;
  }

  // ---------------- consumers ----------------
  const int tx = lane, ty = warp;
  const Geo g = a.g;
  const double pc = a.sc->pc, dt = a.sc->dt, u_ref = a.sp.u_ref;
  const long long fs = g.fstride;
  const long long plane = static_cast<long long>(g.pitch) * g.ypitch;
  const int kzh = g.nz + 2;
  double m0 = 0.0, m1 = 0.0, m2 = 0.0;
  unsigned bad = 0, nbad = 0;
  uint32_t e = 0;
  const int cen = (ty + 2) * BW + tx + 2;  // own cell inside a field plane

  auto wait_full = [&](uint32_t idx) { tma::mbar_wait(&full[idx % R], (idx / R) & 1); };
  auto release = [&](uint32_t idx) {
    __syncwarp();
    if (lane == 0) tma::mbar_arrive(&empty[idx % R]);
  };
  auto fplane = [&](uint32_t idx, int f) -> const double* { return ring + (idx % R) * kTmaSlot + f * kTmaField; };

  for (long long u = u0; u < u1;) {
    const int tile = static_cast<int>(u / bd);
    const int kb = a.box.lo[2] + static_cast<int>(u % bd);
    const long long rem_ = bd - u % bd;
        const int len = static_cast<int>(rem_ < u1 - u ? rem_ : u1 - u);
    const int ti0 = a.box.lo[0] + (tile % a.tiles_x) * 32;
    const int tj0 = a.box.lo[1] + (tile / a.tiles_x) * TY;
    const int i = ti0 + tx, j = tj0 + ty;
    const bool active = i < a.box.hi[0] && j < a.box.hi[1];
    // in-plane pressure neighbours that are interior get the lazy shift
    const bool sxm = i - 1 >= 2, sxm2 = i - 2 >= 2, sxp = i + 1 < g.nx + 2, sxp2 = i + 2 < g.nx + 2;
    const bool sym = j - 1 >= 2, sym2 = j - 2 >= 2, syp = j + 1 < g.ny + 2, syp2 = j + 2 < g.ny + 2;
    const bool all_in = sxm && sxm2 && sxp && sxp2 && sym && sym2 && syp && syp2;
    auto pk = [&](double x, int k) { return x - (k >= 2 && k < kzh ? pc : 0.0); };

    // prologue: planes kb-2 .. kb+1 (sequence e .. e+3)
    wait_full(e);
    wait_full(e + 1);
    wait_full(e + 2);
    wait_full(e + 3);
    double pm2 = pk(fplane(e, 0)[cen], kb - 2);
    double pm1 = pk(fplane(e + 1, 0)[cen], kb - 1);
    double p0 = pk(fplane(e + 2, 0)[cen], kb);
    double pp1 = pk(fplane(e + 3, 0)[cen], kb + 1);
    double um1 = fplane(e + 1, 1)[cen], u0c = fplane(e + 2, 1)[cen];
    double vm1 = fplane(e + 1, 2)[cen], v0c = fplane(e + 2, 2)[cen];
    double wm1 = fplane(e + 1, 3)[cen], w0c = fplane(e + 2, 3)[cen];
    double tm1 = fplane(e + 1, 4)[cen], t0c = fplane(e + 2, 4)[cen];
    release(e);
    release(e + 1);

    for (int s = 0; s < len; ++s) {
      const int k = kb + s;
      const uint32_t q = e + 2 + s;  // sequence index of plane k
      wait_full(q + 2);
      const double pp2 = pk(fplane(q + 2, 0)[cen], k + 2);
      const double up1 = fplane(q + 1, 1)[cen], vp1 = fplane(q + 1, 2)[cen], wp1 = fplane(q + 1, 3)[cen],
                   tp1 = fplane(q + 1, 4)[cen];
      if (active) {
        const double* BP = fplane(q, 0) + cen;
        Star st;
        st.p = p0;
        st.pxm = BP[-1];
        st.pxp = BP[1];
        st.pxm2 = BP[-2];
        st.pxp2 = BP[2];
        st.pym = BP[-BW];
        st.pyp = BP[BW];
        st.pym2 = BP[-2 * BW];
        st.pyp2 = BP[2 * BW];
        if (all_in) {
          st.pxm -= pc;
          st.pxp -= pc;
          st.pxm2 -= pc;
          st.pxp2 -= pc;
          st.pym -= pc;
          st.pyp -= pc;
          st.pym2 -= pc;
          st.pyp2 -= pc;
        } else {
          st.pxm -= sxm ? pc : 0.0;
          st.pxp -= sxp ? pc : 0.0;
          st.pxm2 -= sxm2 ? pc : 0.0;
          st.pxp2 -= sxp2 ? pc : 0.0;
          st.pym -= sym ? pc : 0.0;
          st.pyp -= syp ? pc : 0.0;
          st.pym2 -= sym2 ? pc : 0.0;
          st.pyp2 -= syp2 ? pc : 0.0;
        }
        st.pzm = pm1;
        st.pzp = pp1;
        st.pzm2 = pm2;
        st.pzp2 = pp2;
        const double* BU = fplane(q, 1) + cen;
        st.u = u0c;
        st.uxm = BU[-1];
        st.uxp = BU[1];
        st.uym = BU[-BW];
        st.uyp = BU[BW];
        st.uzm = um1;
        st.uzp = up1;
        const double* BV = fplane(q, 2) + cen;
        st.v = v0c;
        st.vxm = BV[-1];
        st.vxp = BV[1];
        st.vym = BV[-BW];
        st.vyp = BV[BW];
        st.vzm = vm1;
        st.vzp = vp1;
        const double* BWp = fplane(q, 3) + cen;
        st.w = w0c;
        st.wxm = BWp[-1];
        st.wxp = BWp[1];
        st.wym = BWp[-BW];
        st.wyp = BWp[BW];
        st.wzm = wm1;
        st.wzp = wp1;
        const double* BT = fplane(q, 4) + cen;
        st.t = t0c;
        st.txm = BT[-1];
        st.txp = BT[1];
        st.tym = BT[-BW];
        st.typ = BT[BW];
        st.tzm = tm1;
        st.tzp = tp1;
        if (near_wall(a.walls, g, i, j, k)) apply_wall_ghosts(st, a.walls, g, i, j, k);
        const Res r = residual_of(st, a.sp);
        const double qp = p0 + dt * r.p, qu = u0c + dt * r.u, qv = v0c + dt * r.v, qw = w0c + dt * r.w,
                     qt = t0c + dt * r.t;
        const long long c = g.idx(i, j, k);
        a.out[c] = qp;
        a.out[fs + c] = qu;
        a.out[2 * fs + c] = qv;
        a.out[3 * fs + c] = qw;
        a.out[4 * fs + c] = qt;
        const Denoms d = cfl_denoms(qu, qv, qw, u_ref);
        m0 = dmax_d(m0, d.du);
        m1 = dmax_d(m1, d.dv);
        m2 = dmax_d(m2, d.dw);
        bad |= nonfinite(qp) | (nonfinite(qu) << 1) | (nonfinite(qv) << 2) | (nonfinite(qw) << 3) |
               (nonfinite(qt) << 4);
        if (i == a.cx && j == a.cy && k == a.cz) a.acc->pc_local = qp;
        if (NORMS) {
          const double rr[5] = {r.p * r.p, r.u * r.u, r.v * r.v, r.w * r.w, r.t * r.t};
#pragma unroll
          for (int v = 0; v < 5; ++v) {
            if (nonfinite(rr[v])) nbad = 1;
            else add_term_digits(sdig + v * kDigits, rr[v]);
          }
        }
      }
      release(q);  // plane k is never read again
      pm2 = pm1;
      pm1 = p0;
      p0 = pp1;
      pp1 = pp2;
      um1 = u0c;
      u0c = up1;
      vm1 = v0c;
      v0c = vp1;
      wm1 = w0c;
      w0c = wp1;
      tm1 = t0c;
      t0c = tp1;
    }
    release(e + len + 2);  // planes ke, ke+1 served only as column values
    release(e + len + 3);
    e += len + 4;
    u += len;
    (void)plane;
  }

  // consumer-only reductions (the producer warp has exited)
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
  tma::consumer_sync(NC);
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
  }
  if (NORMS)
    for (int x = threadIdx.x; x < 5 * kDigits; x += NC)
      if (sdig[x]) atomicAdd(&a.digits[x], sdig[x]);
}

}  // namespace cav
