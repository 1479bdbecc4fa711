// step_tma.cuh — the fused pseudo-time step (K4), TMA-fed and warp-specialised.
//
// Persistent CTAs (CTAS per SM): TY consumer warps (a 32 x TY tile of cells
// per plane, one column per consumer thread) and one TMA issuer warp.
//
// Issuer (one lane): streams each plane tile into a ring of R shared-memory
// slots with two cp.async.bulk.tensor.4d boxes — p as 36 x (TY+4) (2-cell
// halo ring) and u,v,w,T as 4 x 36 x (TY+2) (1-cell y ring), i.e. only the
// halo each variable's stencil reads (completion = the slot's `full` mbarrier
// transaction count); it only waits for a slot to be released (`empty`).
//
// Consumer warps wait on `full` directly and never write the ring: the x/y
// wall ghosts of apply_boundary_conditions (src/solver.cpp:158-191) are formed
// in registers by the warps whose cells touch a wall (the same
// apply_wall_ghosts the pointwise kernels use), like the z-wall ghosts in the
// k-window, or (G) already stored in the state. The ring is never patched:
// every block stores its rescaled pressure eagerly (fl(p' - pcs_n), see
// IterScalars), so landed tiles hold final values. (Measured: a dedicated
// patcher warp, or cooperative smem patches with a barrier per plane, cost
// 25% of the step on 256^3.)
//
// Each consumer keeps its column's p k-window in registers (k-2..k+3; z-wall
// ghosts are formed there) and reads u,v,w,T at k-1..k+1 from the slots it
// holds (planes k-1..k+3, five slots), and computes two planes per step:
// residual_t (cell.cuh, the reference's arithmetic), the Euler update, the
// next step's CFL maxima and the non-finite flags; it stores and releases the
// slots (`empty` mbarrier).
//
// Work: items are (k-chunk, tile) in chunk-major order; CTA c starts with item
// c, then takes the next unclaimed item from a global counter, so the ~G items
// in flight at any time are neighbouring tiles of the same chunk (their halo
// rows are L2 hits), slower items (wall tiles) do not unbalance the SMs, and
// each item restarts the k-window once. The last items in the order are
// short k-chunks, which shortens the tail where CTAs run out of work.
//
// Overlap (multi-rank blocks, src/runner.cpp:189-194): the item space is
// split into internal items, whose stencils never reach a joined face's halo,
// and shell items (the tile columns / rows and the 2-plane z chunks next to a
// joined face). One launch takes the internal items while the halo exchange
// is in flight, a second one the shell items after it landed; both are the
// same TMA kernel, so the shells run at full speed (the reference's shells
// of src/overlap.cpp:13-28 are a subset of these).
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
// Shared-window address forms: the consumer loop keeps the barrier arrays'
// shared addresses in registers instead of converting generic pointers
// (S2R of the CTA window + arithmetic) at every wait and release.
__device__ __forceinline__ void mbar_arrive_s(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait_s(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAITS:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n"
      "@!P1 bra WAITS;\n"
      "}\n" ::"r"(bar),
      "r"(parity), "r"(1000000u)
      : "memory");
}
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
#ifndef CAV_TMA_HINT  // variant builds: 1 = L2 evict_last, 2 = L2 evict_first on the tile loads
#define CAV_TMA_HINT 0
#endif
__device__ __forceinline__ void load_4d(void* dst, const CUtensorMap* map, int x, int y, int z, int f,
                                        uint64_t* bar) {
#if CAV_TMA_HINT
  uint64_t pol;
  if (CAV_TMA_HINT == 1)
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  else
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3, %4, %5}], "
      "[%6], %7;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(f), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
  return;
#endif
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
      "[%6];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(f), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void named_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

}  // namespace tma

// Plane tile of one slot: pressure with its 2-cell halo ring (36 x (TY+4))
// followed by u, v, w, T with their 1-cell y ring (4 x 36 x (TY+2)). Each part
// is one TMA box; corners are loaded but never read. The u..T rows also start
// at i0-2: a TMA box must start 16-byte aligned along x (probe:
// scripts/micro/tma_probe.cu), so an FP64 box cannot start at the odd i0-1.
constexpr int kPW = 36;            // 32 + 2x2 halo (p)
constexpr int kQW = 36;            // same x extent for u, v, w, T

// Tile height TY (= consumer warps), ring depth R and CTAs per SM.
template <int TY_, int R_, int CTAS_>
struct TmaCfg {
  static constexpr int TY = TY_, R = R_, CTAS = CTAS_;
  static constexpr int PH = TY + 4, QH = TY + 2;
  static constexpr int PHA = (PH + 3) / 4 * 4;  // p rows allotted: keeps the u..T box 128-byte aligned
  static constexpr int PField = kPW * PHA;      // doubles of the p part
  static constexpr int QField = kQW * QH;     // doubles per u/v/w/T part
  static constexpr int Slot = PField + 4 * QField;
  static constexpr int TxBytes = (kPW * PH + 4 * QField) * 8;  // bytes the two boxes deliver
  static constexpr int Threads = 32 * (TY + 1);  // consumers + issuer
  static constexpr int NC = 32 * TY;              // consumer threads
  static constexpr size_t Smem = static_cast<size_t>(R) * Slot * sizeof(double) + 3 * R * 8 + (5 * kDigits + 8) * 8;
  static_assert(PField * 8 % 128 == 0 && Slot * 8 % 128 == 0, "TMA destinations must stay 128-byte aligned");
  static_assert(R >= 5, "ring must hold planes k..k+3 plus one in flight");
};

// ---- scalars between ranks (np > 1) -----------------------------------------
// reduce_fixed_order(Min) of dt and the centre-pressure broadcast
// (src/transport.cpp:23-60, src/exchange.cpp:183-193), folded so that one
// exchange per iteration suffices and every block stores its rescaled
// pressure eagerly:
//   push (the last CTA of iteration n's last step launch; k_push for n = 0):
//     this rank's CFL maxima and error code, plus the values of S_n it owns
//     among the centre cell's stencil (the 13-point p star and the u, v, w
//     values R_p reads), into slot[rank][n&1] of every rank's arena, then a
//     release of the slot's stamp;
//   fold (every CTA of iteration n+1's step launches, after the stream waited
//     for every stamp): dt_{n+1} from the global maxima (the exact max
//     rewrite of compute_dt) and pcs_{n+1} = p'(centre) of step n+1 from the
//     gathered star — the residual and update of that one cell with the
//     step's own arithmetic — so the step stores fl(p' - pcs_{n+1}) exactly as
//     rescale_pressure (src/solver.cpp:248-257) would leave it.
// Star order: p, p-x, p+x, p-2x, p+2x, p-y, p+y, p-2y, p+2y, p-z, p+z, p-2z,
// p+2z, u, u-x, u+x, v, v-y, v+y, w, w-z, w+z.
constexpr int kStar = 22;
struct Slot {
  unsigned long long d[3];
  unsigned long long err;
  unsigned long long stamp;
  unsigned long long pad[3];
  double star[24];
};
static_assert(sizeof(Slot) == 256, "slot size");

struct StarCells {       // this rank's share of the centre star
  int n;
  int slot[kStar];
  int var[kStar];
  long long idx[kStar];  // storage index within the field
};

// Halo of one joined face, sent by the step kernel itself (X): every
// output cell within the face's send layers (p: 2, u,v,w,T: 1 — what the
// neighbour's stencils read; exchange_begin/copy_box_to's face_interior_box,
// src/exchange.cpp:115-145, src/slab.cpp:33-52) is stored straight into the
// neighbour's state — the ghost cell of the same global position — over
// NVLink / peer memory. base[s] is the neighbour's state s (ranks swap
// states in lockstep); shift maps our coordinate along the face axis to the
// neighbour's.
struct FaceSend {
  double* base[2];
  long long fstride;
  int pitch, ypitch, off, shift;
  int dq;  // u, v, w, T layers the plan sends on this face (1: V3 / V2 i-faces, else 2); p: always 2
};

// Halo bits of a cell in layer L (1 = next to the face, 2 = behind it, 0 =
// neither) of a face whose u..T depth is dq: bit 0 p, bit 1 u, v, w, T.
__device__ __forceinline__ int halo_bits(int L, int dq) { return L == 1 ? 3 : (L == 2 ? (dq == 2 ? 3 : 1) : 0); }

// Per-block constants of the cross-rank scalars, in device memory (written
// once when the block connects), so the kernels pass one pointer.
struct XDesc {
  FaceSend face[6];
  int xmask;                // joined faces whose halos the step sends (X)
  const Slot* slots;        // this rank's arena: Slot[np][2]
  Slot* const* peer_slots;  // every rank's Slot array
  int np, rank, rescale;
  const int* abort;          // set by a transport timeout: stop waiting
  signed char owner[kStar];  // rank holding each star value
  StarCells mine;
  cav_stencil_params sp;
  BetaFast bf;
  double dx, dy, dz, cfl, nu, alpha;
};

// dt_n and pcs_n from every rank's slot of iteration n-1 (parity par), by
// one warp (all 32 lanes): lane r reads rank r's maxima and error code, lane q
// the q-th star value; lane 0 folds. The stream waited for every stamp
// before the launch, so plain L2 loads see the pushed values (a stamp below
// `stamp` only remains after an abort released the wait: skipped).
__device__ __noinline__ void fold_scalars_warp(const XDesc* x, int par, unsigned long long stamp, double* sstar,
                                               double* out_dt, double* out_pcs, unsigned long long* out_err,
                                               uint64_t* gate) {
  const int lane = threadIdx.x & 31;
  unsigned long long d0 = 0, d1 = 0, d2 = 0, e = ~0ull;
  for (int r = lane; r < x->np; r += 32) {
    const Slot* s = x->slots + (r * 2 + par);
    // the stream waited for the stamp; the acquire orders the reads below after
    // the pusher's release (a lagging view waits here; an abort releases it)
    bool ok = true;
    while (ld_acquire_sys(&s->stamp) < stamp)
      if (*reinterpret_cast<const volatile int*>(x->abort)) {
        ok = false;
        break;
      }
    if (!ok) continue;
    d0 = max(d0, __ldcg(&s->d[0]));
    d1 = max(d1, __ldcg(&s->d[1]));
    d2 = max(d2, __ldcg(&s->d[2]));
    e = min(e, __ldcg(&s->err));
  }
  if (x->rescale && lane < kStar) sstar[lane] = __ldcg(&x->slots[x->owner[lane] * 2 + par].star[lane]);
  for (int o = 16; o > 0; o >>= 1) {
    d0 = max(d0, __shfl_xor_sync(0xffffffffu, d0, o));
    d1 = max(d1, __shfl_xor_sync(0xffffffffu, d1, o));
    d2 = max(d2, __shfl_xor_sync(0xffffffffu, d2, o));
    e = min(e, __shfl_xor_sync(0xffffffffu, e, o));
  }
  __syncwarp();
  if (gate && lane == 0) tma::mbar_arrive(gate);  // every stamp acquired: the issuer may load this state
  if (lane != 0) return;
  const unsigned long long dm[3] = {d0, d1, d2};
  cav_fluid_params fl{};
  fl.nu = x->nu;
  fl.alpha = x->alpha;
  const double dt = ops::dt_from_maxima(dm, x->dx, x->dy, x->dz, fl, x->cfl);
  double pcs = 0.0;
  if (x->rescale) {
    const double* v = sstar;
    Star s{};
    s.p = v[0];
    s.pxm = v[1];
    s.pxp = v[2];
    s.pxm2 = v[3];
    s.pxp2 = v[4];
    s.pym = v[5];
    s.pyp = v[6];
    s.pym2 = v[7];
    s.pyp2 = v[8];
    s.pzm = v[9];
    s.pzp = v[10];
    s.pzm2 = v[11];
    s.pzp2 = v[12];
    s.u = v[13];
    s.uxm = v[14];
    s.uxp = v[15];
    s.v = v[16];
    s.vym = v[17];
    s.vyp = v[18];
    s.w = v[19];
    s.wzm = v[20];
    s.wzp = v[21];
    // center_p_update's arithmetic (R_p reads only these values)
    pcs = s.p + dt * residual_of(s, x->sp, x->bf).p;
  }
  *out_dt = dt;
  *out_pcs = pcs;
  *out_err = e;
}

// This rank's scalars of iteration n (parity par) and its share of S_n's
// centre stencil into every rank's slot, then a release of the stamp; by one
// warp (lane r serves ranks r, r+32, ...).
__device__ __noinline__ void push_scalars_warp(const XDesc* x, int par, unsigned long long stamp,
                                               const volatile Acc* acc, const double* state, long long fs) {
  const int lane = threadIdx.x & 31;
  double st[kStar];
  for (int q = 0; q < kStar; ++q) st[q] = 0.0;
  for (int t = 0; t < x->mine.n; ++t) st[x->mine.slot[t]] = __ldcg(state + x->mine.var[t] * fs + x->mine.idx[t]);
  const unsigned long long d0 = acc->dmax[0], d1 = acc->dmax[1], d2 = acc->dmax[2], err = acc->err;
  for (int r = lane; r < x->np; r += 32) {
    Slot* s = x->peer_slots[r] + (x->rank * 2 + par);
    s->d[0] = d0;
    s->d[1] = d1;
    s->d[2] = d2;
    s->err = err;
    for (int q = 0; q < kStar; ++q) s->star[q] = st[q];
    __threadfence_system();
    st_release_sys(&s->stamp, stamp);
  }
}

// One output cell's halo contributions (X): m holds two bits per face (2f:
// within the face's two p layers, 2f+1: within its u..T layer).
__device__ __forceinline__ void send_cell(const XDesc* x, int par, int i, int j, int k, int m, double p, double u,
                                       double v, double w, double t) {
  for (int f = 0; f < 6; ++f) {
    const int bits = (m >> (2 * f)) & 3;
    if (!bits) continue;
    const FaceSend& fs = x->face[f];
    const int ax = f >> 1, sh = fs.shift;  // no indexed local array: selects keep it in registers
    const int c0 = i + (ax == 0 ? sh : 0), c1 = j + (ax == 1 ? sh : 0), c2 = k + (ax == 2 ? sh : 0);
    const long long q = fs.off + c0 + static_cast<long long>(fs.pitch) * (c1 + static_cast<long long>(fs.ypitch) * c2);
    double* b = fs.base[par];
    b[q] = p;
    if (bits & 2) {
      b[q + fs.fstride] = u;
      b[q + 2 * fs.fstride] = v;
      b[q + 3 * fs.fstride] = w;
      b[q + 4 * fs.fstride] = t;
    }
  }
}

struct TmaStepArgs {
  double* out;
  Geo g;
  cav_stencil_params sp;
  BetaFast bf;  // beta shortcuts (host::beta_fast)
  unsigned* work;  // dynamic item counter (items >= gridDim.x), reset by the last CTA
  const int* stop;  // set once converged (single rank) or aborted (timeout): later steps do nothing (or null)
  cav_box box;
  IterScalars* sc;
  Acc* acc;
  unsigned long long* digits;
  int cx, cy, cz;
  long long n;
  // one rank: the iteration number lives in device memory (advanced by the
  // last CTA), so a captured CUDA graph of steps can be replayed at any n
  long long* n_dev;
  int rank;
  int tiles_x, ntiles, chunk, nchunks;
  // chunks [0, nbig) have `chunk` planes from box.lo[2] (the last one may be
  // shorter, ending at bigend); chunks >= nbig have `chunk_tail` planes from
  // bigend: the items claimed last are short, which shortens the tail where
  // CTAs run out of work at different times
  int nbig, chunk_tail, bigend;
  // z chunks: zl (0/1) two-plane shell chunks at box.lo[2] and zh at
  // box.hi[2] (joined z faces), the rest from mlo = box.lo[2] + 2 zl as above
  int zl, zh, mlo;
  // item subset: 0 all, 1 internal only, 2 shell only; a tile is a shell
  // tile unless sx0 <= tile_x < sx1 and sy0 <= tile_y < sy1 (tile columns /
  // rows holding the two cell layers next to a joined face)
  int part, sx0, sx1, sy0, sy1;
  WallInfo walls;
  // single-rank fold (np == 1; many ranks fold in k_fold): the last CTA to
  // finish turns this iteration's maxima into dt_{n+1} and pcs_{n+1}
  int fold;
  unsigned* done;
  IterScalars* sc_next;
  Acc* acc_next;
  unsigned long long* err_sticky;
  double dx, dy, dz, cfl, nu, alpha;
  int rescale;
  // stored-ghost step (G): the lanes next to an x wall also store the x-wall
  // ghosts of the output state, from their neighbours' new values (shuffles;
  // the three interior layers lie in one warp: checked on the host); k_ghosts_yz
  // writes the y and z faces. 0: k_bc writes every face (block.cu).
  int gw;
  // many ranks: every CTA folds dt/pcs from the slots (xfold; write_sc: CTA 0
  // also stores them to sc and folds the peers' error codes); the last CTA of
  // the iteration's last launch pushes (xpush) and resets acc_next
  const XDesc* xd;
  int xfold, write_sc, xpush;
  int out_par;  // index of the output state (cur ^ 1): the neighbours' state the halos go to (X)
  int fold_par, push_par;
  unsigned long long fold_stamp, push_stamp;
  // G norm iterations: the residuals go to this scratch state (same layout)
  // and k_norm_runs sums their squares after the step (the step's own digit
  // runs need 5 x 4 more live registers and spill at 96)
  double* rs;
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
  const int m = chunk - a.zl;
  if (m < 0) {
    r.kb = a.box.lo[2];
    r.ke = r.kb + 2;
  } else if (chunk >= a.nchunks - a.zh) {
    r.ke = a.box.hi[2];
    r.kb = r.ke - 2;
  } else if (m < a.nbig) {
    r.kb = a.mlo + m * a.chunk;
    r.ke = min(r.kb + a.chunk, a.bigend);
  } else {
    r.kb = a.bigend + (m - a.nbig) * a.chunk_tail;
    r.ke = min(r.kb + a.chunk_tail, a.box.hi[2] - 2 * a.zh);
  }
  return r;
}

// Whether `item` belongs to this launch's subset (TmaStepArgs::part).
__device__ __forceinline__ bool item_wanted(const TmaStepArgs& a, long long item) {
  if (a.part == 0) return true;
  const int chunk = static_cast<int>(item / a.ntiles);
  const int tile = static_cast<int>(item % a.ntiles);
  const int tx = tile % a.tiles_x, ty = tile / a.tiles_x;
  const bool shell = chunk < a.zl || chunk >= a.nchunks - a.zh || tx < a.sx0 || tx >= a.sx1 || ty < a.sy0 ||
                     ty >= a.sy1;
  return shell == (a.part == 2);
}

// Consumer-side star accessor: p's in-plane neighbours from the landed slot
// of plane k, its k-neighbours from the register window; u, v, w, T entirely
// from the slots of planes k-1, k, k+1 (v, w, T follow u at multiples of QF).
// With W, the values
// of cells next to an x or y wall that lie in the ghost layers are the wall
// ghosts of apply_boundary_conditions (src/solver.cpp:158-191), formed in
// registers with exactly device.cuh's apply_wall_ghosts expressions: p by
// cubic extrapolation, u,v,w antisymmetric, T isothermal 2*t_wall - T on x
// walls and mirrored on y walls. Nothing is written to the ring.
constexpr int kXlo2 = 1, kXlo3 = 2, kXhi1 = 4, kXhi0 = 8;       // i == 2, 3, nx+1, nx
constexpr int kYlo2 = 16, kYlo3 = 32, kYhi1 = 64, kYhi0 = 128;  // j == 2, 3, ny+1, ny
constexpr int kZlo2 = 256, kZhi1 = 512;                         // k == 2, nz+1 (u,v,w,T only)

template <int QF, bool WX, bool WYZ>
struct SmemAcc {
  const double *P, *Um, *U, *Up;  // own cell: p in slot k; u part in slots k-1, k, k+1
  double pc_, pzm_, pzp_, pzm2_, pzp2_;
  int fl;
  double thot, tcold;
  // WX: x-wall flags may be set; WYZ: y- or z-wall flags may be set
  __device__ __forceinline__ bool on(int bit) const {
    return ((bit < kYlo2) ? WX : WYZ) && (fl & bit);
  }
  __device__ __forceinline__ double p() const { return pc_; }
  // stencil row along one axis (stride S): m2 m1 [p] p1 p2
  template <int S, int LO2, int LO3, int HI1, int HI0>
  __device__ __forceinline__ double m1() const {
    if (on(LO2)) return cubic_g0(pc_, P[S], P[2 * S]);
    return P[-S];
  }
  template <int S, int LO2, int LO3, int HI1, int HI0>
  __device__ __forceinline__ double p1() const {
    if (on(HI1)) return cubic_g0(pc_, P[-S], P[-2 * S]);
    return P[S];
  }
  template <int S, int LO2, int LO3, int HI1, int HI0>
  __device__ __forceinline__ double m2() const {
    if (on(LO2)) return cubic_g1(cubic_g0(pc_, P[S], P[2 * S]), pc_, P[S]);
    if (on(LO3)) return cubic_g0(P[-S], pc_, P[S]);
    return P[-2 * S];
  }
  template <int S, int LO2, int LO3, int HI1, int HI0>
  __device__ __forceinline__ double p2() const {
    if (on(HI1)) return cubic_g1(cubic_g0(pc_, P[-S], P[-2 * S]), pc_, P[-S]);
    if (on(HI0)) return cubic_g0(P[S], pc_, P[-S]);
    return P[2 * S];
  }
  __device__ __forceinline__ double pxm() const { return m1<1, kXlo2, kXlo3, kXhi1, kXhi0>(); }
  __device__ __forceinline__ double pxp() const { return p1<1, kXlo2, kXlo3, kXhi1, kXhi0>(); }
  __device__ __forceinline__ double pxm2() const { return m2<1, kXlo2, kXlo3, kXhi1, kXhi0>(); }
  __device__ __forceinline__ double pxp2() const { return p2<1, kXlo2, kXlo3, kXhi1, kXhi0>(); }
  __device__ __forceinline__ double pym() const { return m1<kPW, kYlo2, kYlo3, kYhi1, kYhi0>(); }
  __device__ __forceinline__ double pyp() const { return p1<kPW, kYlo2, kYlo3, kYhi1, kYhi0>(); }
  __device__ __forceinline__ double pym2() const { return m2<kPW, kYlo2, kYlo3, kYhi1, kYhi0>(); }
  __device__ __forceinline__ double pyp2() const { return p2<kPW, kYlo2, kYlo3, kYhi1, kYhi0>(); }
  __device__ __forceinline__ double pzm() const { return pzm_; }
  __device__ __forceinline__ double pzp() const { return pzp_; }
  __device__ __forceinline__ double pzm2() const { return pzm2_; }
  __device__ __forceinline__ double pzp2() const { return pzp2_; }
  // velocity ghosts (antisymmetric on every wall)
#define CAV_Q(F, N)                                                                                   \
  __device__ __forceinline__ double F() const { return U[N * QF]; }                                  \
  __device__ __forceinline__ double F##xm() const { return on(kXlo2) ? -F() : U[N * QF - 1]; }      \
  __device__ __forceinline__ double F##xp() const { return on(kXhi1) ? -F() : U[N * QF + 1]; }      \
  __device__ __forceinline__ double F##ym() const { return on(kYlo2) ? -F() : U[N * QF - kQW]; }    \
  __device__ __forceinline__ double F##yp() const { return on(kYhi1) ? -F() : U[N * QF + kQW]; }    \
  __device__ __forceinline__ double F##zm() const { return on(kZlo2) ? -F() : Um[N * QF]; }         \
  __device__ __forceinline__ double F##zp() const { return on(kZhi1) ? -F() : Up[N * QF]; }
  CAV_Q(u, 0)
  CAV_Q(v, 1)
  CAV_Q(w, 2)
#undef CAV_Q
  // temperature: isothermal x walls, adiabatic (mirror) y and z walls
  __device__ __forceinline__ double t() const { return U[3 * QF]; }
  __device__ __forceinline__ double txm() const { return on(kXlo2) ? 2.0 * thot - t() : U[3 * QF - 1]; }
  __device__ __forceinline__ double txp() const { return on(kXhi1) ? 2.0 * tcold - t() : U[3 * QF + 1]; }
  __device__ __forceinline__ double tym() const { return on(kYlo2) ? t() : U[3 * QF - kQW]; }
  __device__ __forceinline__ double typ() const { return on(kYhi1) ? t() : U[3 * QF + kQW]; }
  __device__ __forceinline__ double tzm() const { return on(kZlo2) ? t() : Um[3 * QF]; }
  __device__ __forceinline__ double tzp() const { return on(kZhi1) ? t() : Up[3 * QF]; }
};

// TMA issue cursor of the issuer warp (lane 0). (Measured: folding it into
// consumer warp 0 to free a warp slot was 16% slower — the ring is only fed
// when that warp reaches a wait.) Items:
// blockIdx.x first, then dynamically from a.work (wall tiles and the odd
// item out make a static round-robin uneven). Each entry's item id goes to
// sitem[] before the slot's arrive, which releases it to the consumers'
// acquire on `full`; after the last item one sentinel entry (-1) is issued.
struct Issuer {
  long long item;
  ItemGeom it;
  int pl;
  int s;
  uint32_t ph, e;  // slot, its empty-barrier phase, entries issued
  bool done, fin;
};

// Issues the next entry once its slot is free; false after the sentinel.
template <class Cfg>
__device__ __forceinline__ bool issue_one(Issuer& q, const CUtensorMap* mP, const CUtensorMap* mQ,
                                          const TmaStepArgs& a, double* ring, uint64_t* full, uint64_t* empty,
                                          long long* sitem, long long total) {
  constexpr int R = Cfg::R;
  if (q.fin) return false;
  if (q.e >= static_cast<uint32_t>(R)) tma::mbar_wait(&empty[q.s], q.ph ^ 1);
  if (q.done) {
    sitem[q.s] = -1;
    tma::mbar_arrive(&full[q.s]);
    q.fin = true;
  } else {
    sitem[q.s] = q.item;
    tma::mbar_expect_tx(&full[q.s], Cfg::TxBytes);
    double* dst = ring + q.s * Cfg::Slot;
    const int x0 = a.g.off + q.it.ti0 - 2, y0 = q.it.tj0 - 2;
    tma::load_4d(dst, mP, x0, y0, q.pl, 0, &full[q.s]);
    tma::load_4d(dst + Cfg::PField, mQ, x0, y0 + 1, q.pl, 0, &full[q.s]);
    if (++q.pl > q.it.ke + 1) {
      do {
        q.item = gridDim.x + atomicAdd(a.work, 1u);
      } while (q.item < total && !item_wanted(a, q.item));
      if (q.item >= total) {
        q.done = true;
      } else {
        q.it = item_geom<Cfg::TY>(a, q.item);
        q.pl = q.it.kb - 2;
      }
    }
  }
  if (++q.s == R) {
    q.s = 0;
    q.ph ^= 1;
  }
  ++q.e;
  return true;
}

// Per-thread run of exact norm terms that start at the same digit: the
// shifted mantissas (m << (off & 31), < 2^85) are summed in 96 bits and
// flushed to the CTA's carry-save digit words when a term starts at a
// different digit (neighbouring cells of a column mostly share a binade), at
// the end of each item and at the end. Each shifted mantissa is below 2^84,
// so 96 bits hold 2^12 = 4096 terms: the step's runs are bounded by one
// item's k-chunk (checked on the host), k_norm_runs' by its segment
// (kNormRunSeg, static_assert there). The digit words are carry-save, so any grouping
// gives the same words as ReproSum::add term by term (measured: a 256^3 check
// iteration 1.7 -> 1.4 ms against warp-aggregated atomics per term; 96 rather
// than 128 bits frees 5 registers).
struct DigitRun {
  int d;                // first digit of the run, -1 = empty
  unsigned w0, w1, w2;  // 96-bit sum
};
__device__ __forceinline__ void digit_run_flush(DigitRun& r, unsigned long long* dig) {
  if (r.d < 0) return;
  if (r.w0) atomicAdd(&dig[r.d], static_cast<unsigned long long>(r.w0));
  if (r.w1) atomicAdd(&dig[r.d + 1], static_cast<unsigned long long>(r.w1));
  if (r.w2) atomicAdd(&dig[r.d + 2], static_cast<unsigned long long>(r.w2));
  r.d = -1;
  r.w0 = r.w1 = r.w2 = 0u;
}
__device__ __forceinline__ void digit_run_add(DigitRun& r, unsigned long long* dig, double x) {
  if (x == 0.0) return;
  const unsigned long long bits = static_cast<unsigned long long>(__double_as_longlong(x));
  const int e = static_cast<int>((bits >> 52) & 0x7FF);
  unsigned long long m = bits & ((1ull << 52) - 1);
  int off = 66;  // ReproSum::add: bit offset e + 65 (normal), 66 (subnormal)
  if (e != 0) {
    m |= 1ull << 52;
    off = e + 65;
  }
  const int d = off >> 5, sh = off & 31;
  if (d != r.d) {
    digit_run_flush(r, dig);
    r.d = d;
  }
  const unsigned long long lo = m << sh;
  const unsigned hi = sh ? static_cast<unsigned>(m >> (64 - sh)) : 0u;
  asm("add.cc.u32 %0, %0, %3;\n\taddc.cc.u32 %1, %1, %4;\n\taddc.u32 %2, %2, %5;"
      : "+r"(r.w0), "+r"(r.w1), "+r"(r.w2)
      : "r"(static_cast<unsigned>(lo)), "r"(static_cast<unsigned>(lo >> 32)), "r"(hi));
}

// G (stored wall ghosts, single rank): every wall ghost the step reads is
// already in the input state (x walls: stored by the previous step's wall
// lanes, a.gw; y/z walls: k_ghosts_yz after it), so the consumers take the plain
// accessor everywhere. Without G they are formed in registers (x/y:
// SmemAcc<.., true>, z: the p window rules below); the three accessor
// instances cost 16% at 256^3 even though few warps take the wall paths.
// F: the box is a whole number of tiles (nx % 32 == 0, ny % TY == 0), so
// every consumer lane is live and the per-cell live tests compile away.
template <class Cfg, bool NORMS, bool G, bool X, bool F = false>
__global__ void __launch_bounds__(Cfg::Threads, Cfg::CTAS)
    k_step_tma(const __grid_constant__ CUtensorMap mapP, const __grid_constant__ CUtensorMap mapQ,
               const TmaStepArgs a) {
  constexpr int C = Cfg::TY, R = Cfg::R;
  constexpr int kTmaSlot = Cfg::Slot, kTmaThreads = Cfg::Threads, QF = Cfg::QField;
  extern __shared__ __align__(128) unsigned char smraw[];
  double* ring = reinterpret_cast<double*>(smraw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smraw + R * kTmaSlot * sizeof(double));
  uint64_t* empty = full + R;
  long long* sitem = reinterpret_cast<long long*>(empty + R);  // item of each slot's entry (-1 = end)
  unsigned long long* sdig = reinterpret_cast<unsigned long long*>(sitem + R);

  // the run converged at an earlier check (device decision): march no
  // further; many ranks still advance the scalar stamps their peers wait for
  if (a.stop && *reinterpret_cast<const volatile int*>(a.stop)) {
    if (a.xpush && blockIdx.x == 0 && threadIdx.x < 32)
      for (int r = threadIdx.x; r < a.xd->np; r += 32)
        st_release_sys(&(a.xd->peer_slots[r] + (a.xd->rank * 2 + a.push_par))->stamp, a.push_stamp);
    return;
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // X: the issuer's first TMA waits until warp 0's fold has acquired every
  // rank's stamp (the peers' halo stores into this state precede them)
  __shared__ uint64_t sgate;
  if (threadIdx.x == 0) {
    for (int s = 0; s < R; ++s) {
      tma::mbar_init(&full[s], 1);
      tma::mbar_init(&empty[s], C);
    }
    if (X) tma::mbar_init(&sgate, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (NORMS)
    for (int x = threadIdx.x; x < 5 * kDigits + 5; x += kTmaThreads) sdig[x] = 0;  // digits, then 5 L-inf maxima
  __syncthreads();

  const long long total = static_cast<long long>(a.ntiles) * a.nchunks;

  if (warp == C) {
    // ---------------- TMA issuer (one lane) ----------------
    if (lane != 0) return;
    if (X && a.xfold) {
      tma::mbar_wait(&sgate, 0);
      asm volatile("fence.proxy.async.global;" ::: "memory");  // generic-proxy acquire -> TMA reads
    }
    Issuer iq{};
    iq.item = blockIdx.x;
    while (iq.item < total && !item_wanted(a, iq.item)) iq.item = gridDim.x + atomicAdd(a.work, 1u);
    iq.done = iq.item >= total;
    if (!iq.done) {
      iq.it = item_geom<C>(a, iq.item);
      iq.pl = iq.it.kb - 2;
    }
    while (issue_one<Cfg>(iq, &mapP, &mapQ, a, ring, full, empty, sitem, total)) {
    }
    return;
  }
  // ---------------- consumers ----------------
  // Each step computes two planes (k, k+1) of the thread's column: the p
  // k-window (k-2..k+3) is shared, and the slot bookkeeping and loop control
  // are paid once per two cells.
  const int tx = lane, ty = warp;
  const Geo g = a.g;
  double dt, pcs;
  if (a.xfold) {
    __shared__ double sfold[2], sstar[kStar];
    if (warp == 0) {
      unsigned long long e;
      fold_scalars_warp(a.xd, a.fold_par, a.fold_stamp, sstar, &sfold[0], &sfold[1], &e, X ? &sgate : nullptr);
      if (lane == 0 && a.write_sc && blockIdx.x == 0) {
        a.sc->dt = sfold[0];
        a.sc->pc = 0.0;
        a.sc->pcs = sfold[1];
        if (e != ~0ull) atomicMin(a.err_sticky, e);
      }
    }
    tma::named_sync(2, 32 * C);
    dt = sfold[0];
    pcs = sfold[1];
  } else {
    dt = a.sc->dt;
    pcs = a.sc->pcs;
  }
  const double u_ref = a.sp.u_ref;
  const long long fs = g.fstride;
  const long long plane = static_cast<long long>(g.pitch) * g.ypitch;
  const bool zlo = a.walls.wall[4], zhi = a.walls.wall[5];
  double m0 = 0.0, m1 = 0.0, m2 = 0.0;
  unsigned e_p = 0, e_u = 0, e_v = 0, e_w = 0, e_t = 0;  // max exponent field per variable
  unsigned nbad = 0;
  DigitRun runs[NORMS && !G ? 5 : 1];
  unsigned long long lmax[NORMS && !G ? 5 : 1] = {};  // L-inf: bits of max |R_v|
  const long long rdelta = NORMS && G ? a.rs - a.out : 0;
  for (auto& r : runs) r = DigitRun{-1, 0u, 0u, 0u};
  const double* ringc = ring + (ty + 2) * kPW + tx + 2;                 // own p cell in slot 0
  const double* ringq = ring + Cfg::PField + (ty + 1) * kQW + tx + 2;  // own u cell in slot 0
  const uint32_t full_s = tma::smem_u32(full), empty_s = tma::smem_u32(empty);
  int sw = 0;  // slot of the next entry to wait for, and its phase
  uint32_t phw = 0;
  auto advance = [&](int& sl, uint32_t& ph) {
    if (++sl == R) {
      sl = 0;
      ph ^= 1;
    }
  };
  // Wait for the next 1 or 2 entries to land.
  int wfl = 0;         // wall flags of this thread's column (kXlo2 ... kYhi0)
  bool wx = false, wyz = false;  // some lane of this warp has an x / y wall flag (warp-uniform)
  // G: this lane's column lies inside the box. Lanes outside it (ragged
  // tiles) compute on whatever the slot holds there, without storing or reducing, so
  // the cell is not under a branch (1.4% faster at 256^3).
  bool live = true;
  // X, per item (two registers on the hot path): xs = this lane's x/y halo
  // bits (0-7) | some lane of the warp has x/y halo cells (8) | the item
  // reaches a joined z face's halo planes (9); xij = i | j << 16
  int xs = 0, xij = 0;
  auto wait_planes = [&](int count, int* sl) {
    for (int q = 0; q < count; ++q) {
      sl[q] = sw;
      tma::mbar_wait_s(full_s + 8u * sw, phw);
      advance(sw, phw);
    }
  };
  auto release_slot = [&](int sl) {
    __syncwarp();
    if (lane == 0) tma::mbar_arrive_s(empty_s + 8u * sl);
  };
  auto slot = [&](int sl) { return ringc + sl * kTmaSlot; };
  auto qslot = [&](int sl) { return ringq + sl * kTmaSlot; };

  // z-wall ghosts of p inside the register window (apply_boundary_conditions
  // for the z walls; u,v,w,T z ghosts are the accessor's kZlo2/kZhi1).
  // Two-plane step at k: P[0..5] = planes k-2..k+3; one-plane step: P[0..4].
  // Only compile-time indices, so the window stays in registers.
  auto zwall2 = [&](double* P, int k) {
    if (zlo && k == 2) {
      P[1] = cubic_g0(P[2], P[3], P[4]);
      P[0] = cubic_g1(P[1], P[2], P[3]);
    } else if (zlo && k == 3) {
      P[0] = cubic_g0(P[1], P[2], P[3]);
    }
    if (zhi && k == g.nz - 1) {
      P[5] = cubic_g0(P[4], P[3], P[2]);
    } else if (zhi && k == g.nz) {
      P[4] = cubic_g0(P[3], P[2], P[1]);
      P[5] = cubic_g1(P[4], P[3], P[2]);
    }
  };
  auto zwall1 = [&](double* P, int k) {
    if (zlo && k == 2) {
      P[1] = cubic_g0(P[2], P[3], P[4]);
      P[0] = cubic_g1(P[1], P[2], P[3]);
    } else if (zlo && k == 3) {
      P[0] = cubic_g0(P[1], P[2], P[3]);
    }
    if (zhi && k == g.nz) {
      P[4] = cubic_g0(P[3], P[2], P[1]);
    } else if (zhi && k == g.nz + 1) {
      P[3] = cubic_g0(P[2], P[1], P[0]);
      P[4] = cubic_g1(P[3], P[2], P[1]);
    }
  };

  // one cell at plane kk: residual + update + store + bookkeeping. Slots
  // slm, slk, slp hold planes kk-1, kk, kk+1.
  auto cell = [&](int slm, int slk, int slp, int kk, double p0, double pzm, double pzp, double pzm2, double pzp2,
                  double* op) {
    const int zf = G ? 0 : (zlo && kk == 2 ? kZlo2 : 0) | (zhi && kk == g.nz + 1 ? kZhi1 : 0);
    Res r;
    double uc, vc, wc, tc;
    // warp-uniform path choice: plain, x walls only (the x-wall tile columns),
    // or any wall (y-wall rows, z-wall planes)
#define CAV_RES(WX, WYZ)                                                                                    \
  {                                                                                                         \
    const SmemAcc<QF, WX, WYZ> sa{slot(slk), qslot(slm), qslot(slk), qslot(slp), p0, pzm, pzp, pzm2, pzp2, \
                                  wfl | zf, a.walls.t_hot, a.walls.t_cold};                                 \
    r = residual_t(sa, a.sp, a.bf);                                                                       \
    uc = sa.u();                                                                                            \
    vc = sa.v();                                                                                            \
    wc = sa.w();                                                                                            \
    tc = sa.t();                                                                                            \
  }
    if (!G && (wyz || zf)) CAV_RES(true, true)
    else if (!G && wx) CAV_RES(true, false)
    else CAV_RES(false, false)
#undef CAV_RES
    const double qpp = p0 + dt * r.p, qpn = qpp - pcs, qun = uc + dt * r.u, qvn = vc + dt * r.v, qwn = wc + dt * r.w,
                 qtn = tc + dt * r.t;
    // explicit global (streaming) stores: no possible aliasing with the
    // shared-memory ring, so the two cells of a step can interleave
    if (!G || live) {
      __stcs(op, qpn);
      __stcs(op + fs, qun);
      __stcs(op + 2 * fs, qvn);
      __stcs(op + 3 * fs, qwn);
      __stcs(op + 4 * fs, qtn);
    }
    if (G && (wfl & 4)) {  // x-wall ghosts of the output (k_bc's expressions), from the neighbours' p
      const unsigned am = __activemask();
      const bool h = (wfl & 2) != 0;
      const int sg = h ? 1 : -1;  // towards the wall
      const double q1 = __shfl_sync(am, qpn, tx - sg), q2 = __shfl_sync(am, qpn, tx - 2 * sg);
      if (wfl & 3) {
        const double pg0 = cubic_g0(qpn, q1, q2);
        // explicit global stores (see above)
        __stcs(op + sg, pg0);
        __stcs(op + 2 * sg, cubic_g1(pg0, qpn, q1));
        __stcs(op + fs + sg, -qun);
        __stcs(op + 2 * fs + sg, -qvn);
        __stcs(op + 3 * fs + sg, -qwn);
        __stcs(op + 4 * fs + sg, 2.0 * (h ? a.walls.t_cold : a.walls.t_hot) - qtn);
      }
    }
    if (X && (xs & 0x300)) {  // halo cells of joined faces: straight into the neighbours' states
      int m = xs & 0xFF;
      if ((xs & 0x200) && live) {
        const int xm = a.xd->xmask;
        if (xm & 16) m |= halo_bits(kk == 2 ? 1 : (kk == 3 ? 2 : 0), a.xd->face[4].dq) << 8;
        if (xm & 32) m |= halo_bits(kk == g.nz + 1 ? 1 : (kk == g.nz ? 2 : 0), a.xd->face[5].dq) << 10;
      }
      if (m) send_cell(a.xd, a.out_par, xij & 0xFFFF, xij >> 16, kk, m, qpn, qun, qvn, qwn, qtn);
    }
    if (!G || live) {
      const Denoms d = cfl_denoms(qun, qvn, qwn, u_ref, a.bf);
      m0 = dmax_d(m0, d.du);
      m1 = dmax_d(m1, d.dv);
      m2 = dmax_d(m2, d.dw);
      e_p = max(e_p, static_cast<unsigned>(__double2hiint(qpn)) & 0x7FF00000u);
      e_u = max(e_u, static_cast<unsigned>(__double2hiint(qun)) & 0x7FF00000u);
      e_v = max(e_v, static_cast<unsigned>(__double2hiint(qvn)) & 0x7FF00000u);
      e_w = max(e_w, static_cast<unsigned>(__double2hiint(qwn)) & 0x7FF00000u);
      e_t = max(e_t, static_cast<unsigned>(__double2hiint(qtn)) & 0x7FF00000u);
    }
    if (NORMS && G && live) {
      double* rp = op + rdelta;
      __stcs(rp, r.p);
      __stcs(rp + fs, r.u);
      __stcs(rp + 2 * fs, r.v);
      __stcs(rp + 3 * fs, r.w);
      __stcs(rp + 4 * fs, r.t);
    }
    if (NORMS && !G) {
      const double rv[5] = {r.p, r.u, r.v, r.w, r.t};
#pragma unroll
      for (int v = 0; v < 5; ++v) {
        lmax[v] = max(lmax[v], abs_bits(rv[v]));
        const double rr = rv[v] * rv[v];
        if (nonfinite(rr)) nbad = 1;
        else digit_run_add(runs[v], sdig + v * kDigits, rr);
      }
    }
  };

  for (;;) {
    tma::mbar_wait_s(full_s + 8u * sw, phw);  // the next entry's item (re-waited below: completed phase)
    const long long item = sitem[sw];
    if (item < 0) break;
    const ItemGeom it = item_geom<C>(a, item);
    const int len = it.ke - it.kb;
    const int i = it.ti0 + tx, j = it.tj0 + ty;
    const bool active = i < a.box.hi[0] && j < a.box.hi[1];
    live = F || active;
    if (X) {  // this column's x/y halo layers (fused send)
      const int xm = a.xd->xmask;
      int mm = 0;
      if (xm & 1) mm |= halo_bits(i == 2 ? 1 : (i == 3 ? 2 : 0), a.xd->face[0].dq);
      if (xm & 2) mm |= halo_bits(i == g.nx + 1 ? 1 : (i == g.nx ? 2 : 0), a.xd->face[1].dq) << 2;
      if (xm & 4) mm |= halo_bits(j == 2 ? 1 : (j == 3 ? 2 : 0), a.xd->face[2].dq) << 4;
      if (xm & 8) mm |= halo_bits(j == g.ny + 1 ? 1 : (j == g.ny ? 2 : 0), a.xd->face[3].dq) << 6;
      mm = active ? mm : 0;
      const bool zitem = ((xm & 16) && it.kb <= 3) || ((xm & 32) && it.ke > g.nz);
      xs = mm | (__any_sync(0xffffffffu, mm != 0) ? 0x100 : 0) | (zitem ? 0x200 : 0);
      xij = i | (j << 16);
    }
    // x/y walls next to this thread's column: register ghosts (SmemAcc<.., true>)
    if (G && a.gw) {  // wfl (G): 1 = i == 2 at the low x wall, 2 = i == nx+1 at the high one, 4 = in this warp
      const int xl = a.walls.wall[0] && i == 2, xh = a.walls.wall[1] && i == g.nx + 1;
      wfl = active ? (xl | (xh << 1)) : 0;
      if (__any_sync(0xffffffffu, wfl != 0)) wfl |= 4;
    }
    if (!G) {
      const WallInfo& w = a.walls;
      wfl = (w.wall[0] && i == 2 ? kXlo2 : 0) | (w.wall[0] && i == 3 ? kXlo3 : 0) |
            (w.wall[1] && i == g.nx + 1 ? kXhi1 : 0) | (w.wall[1] && i == g.nx ? kXhi0 : 0) |
            (w.wall[2] && j == 2 ? kYlo2 : 0) | (w.wall[2] && j == 3 ? kYlo3 : 0) |
            (w.wall[3] && j == g.ny + 1 ? kYhi1 : 0) | (w.wall[3] && j == g.ny ? kYhi0 : 0);
      if (!active) wfl = 0;
      wx = __any_sync(0xffffffffu, (wfl & (kYlo2 - 1)) != 0);
      wyz = __any_sync(0xffffffffu, (wfl & ~(kYlo2 - 1)) != 0);
    }
    // prologue: planes kb-2 .. kb+1; p window from all four, the slots of
    // kb-1 .. kb+1 stay held for u,v,w,T
    int sa[2], sb[2];
    wait_planes(2, sa);
    wait_planes(2, sb);
    double P[6];  // p at planes k-2 .. k+3
    P[0] = slot(sa[0])[0];
    P[1] = slot(sa[1])[0];
    P[2] = slot(sb[0])[0];
    P[3] = slot(sb[1])[0];
    release_slot(sa[0]);
    int skm = sa[1], sk0 = sb[0], sk1 = sb[1];  // slots of planes k-1, k, k+1
    double* op = a.out + g.idx(i, j, it.kb);
    int st = 0;
    for (; st + 1 < len; st += 2, op += 2 * plane) {
      const int k = it.kb + st;
      // plane k+3 is awaited only after cell k is done: cell k needs planes
      // k-1..k+2, cell k+1 also k+3, so the later plane gets a cell's worth
      // of extra time to land. The z-wall rules read P[0..4] only; a ghost
      // P[5] they form (k+3 >= nz+2) is not overwritten by the slot.
      int sn[2];
      wait_planes(1, sn);
      P[4] = slot(sn[0])[0];
      const bool zh5 = !G && zhi && k + 3 >= g.nz + 2;
      if (!G && ((zlo && k <= 3) || zh5)) zwall2(P, k);
      if (G || active) cell(skm, sk0, sk1, k, P[2], P[1], P[3], P[0], P[4], op);
      wait_planes(1, sn + 1);
      if (!zh5) P[5] = slot(sn[1])[0];
      if (G || active) cell(sk0, sk1, sn[0], k + 1, P[3], P[2], P[4], P[1], P[5], op + plane);
      release_slot(skm);
      release_slot(sk0);
      skm = sk1;
      sk0 = sn[0];
      sk1 = sn[1];
      P[0] = P[2];
      P[1] = P[3];
      P[2] = P[4];
      P[3] = P[5];
    }
    if (st < len) {  // odd remainder: one plane
      const int k = it.kb + st;
      int sn[2];
      wait_planes(1, sn);  // plane k+2
      P[4] = slot(sn[0])[0];
      if (!G && ((zlo && k <= 3) || (zhi && k + 2 >= g.nz + 2))) zwall1(P, k);
      if (G || active) cell(skm, sk0, sk1, k, P[2], P[1], P[3], P[0], P[4], op);
      release_slot(sn[0]);
    }
    // planes ke-1 .. ke+1 (odd: plus ke+2 above) served only as neighbours
    release_slot(skm);
    release_slot(sk0);
    release_slot(sk1);
    if (NORMS && !G)  // bounds every run to one item's planes (96-bit sums)
#pragma unroll
      for (int v = 0; v < 5; ++v) digit_run_flush(runs[v], sdig + v * kDigits);
  }
  constexpr unsigned EXP = 0x7FF00000u;
  unsigned bad = (e_p == EXP ? 1u : 0u) | (e_u == EXP ? 2u : 0u) | (e_v == EXP ? 4u : 0u) |
                 (e_w == EXP ? 8u : 0u) | (e_t == EXP ? 16u : 0u);

  if (NORMS && !G)
#pragma unroll
    for (int v = 0; v < 5; ++v) {
      digit_run_flush(runs[v], sdig + v * kDigits);
      const unsigned long long m = warp_max_u64(lmax[v]);
      if (lane == 0 && m) atomicMax(&sdig[5 * kDigits + v], m);
    }
  if (X) __threadfence_system();  // this thread's halo stores, before the flag/stamp release of the last CTA
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
  bool last = false;
  if (threadIdx.x == 0) {
    unsigned mk = 0;
    for (int w = 0; w < C; ++w) {
      m0 = dmax_d(m0, sred[0][w]);
      m1 = dmax_d(m1, sred[1][w]);
      m2 = dmax_d(m2, sred[2][w]);
      mk |= smask[w];
    }
    const long long nn = a.n_dev ? *reinterpret_cast<volatile long long*>(a.n_dev) : a.n;
    acc_publish(a.acc, m0, m1, m2, mk & 0xFF, nn + 1, a.rank);
    if (NORMS && (mk >> 8)) atomicMin(&a.acc->err, err_code(nn, a.rank, 0));
    __threadfence();
    last = atomicAdd(a.done, 1u) == gridDim.x - 1;
    if (X && last) __threadfence_system();
    if (last) {  // every CTA has published
      *a.work = 0;
      __threadfence();
      if (a.fold) {
        volatile Acc* acc = a.acc;
        const unsigned long long dm[3] = {acc->dmax[0], acc->dmax[1], acc->dmax[2]};
        cav_fluid_params fl{};
        fl.nu = a.nu;
        fl.alpha = a.alpha;
        const double dtn = ops::dt_from_maxima(dm, a.dx, a.dy, a.dz, fl, a.cfl);
        a.sc_next->dt = dtn;
        // this iteration's output is final; pcs_{n+1} = p'(centre) of the
        // next step, from the same inputs and arithmetic as that step
        a.sc_next->pcs = a.rescale ? center_p_update(a.out, a.g, a.walls, a.sp, a.bf, dtn, 0.0, a.cx, a.cy, a.cz)
                                   : 0.0;
        const unsigned long long e = acc->err;
        if (e < *a.err_sticky) *a.err_sticky = e;
        Acc z{};
        z.err = ~0ull;
        *a.acc_next = z;
      }
      if (a.n_dev) *a.n_dev = nn + 1;
      *a.done = 0;
    }
  }
  if (a.xpush && warp == 0 && __shfl_sync(0xffffffffu, last, 0)) {
    // many ranks: this iteration's scalars and centre-stencil share to every rank
    push_scalars_warp(a.xd, a.push_par, a.push_stamp, a.acc, a.out, a.g.fstride);
    if (lane == 0) {
      Acc z{};
      z.err = ~0ull;
      *a.acc_next = z;
    }
  }
  if (NORMS && !G) {
    for (int x = threadIdx.x; x < 5 * kDigits; x += NC)
      if (sdig[x]) atomicAdd(&a.digits[x], sdig[x]);
    if (threadIdx.x < 5 && sdig[5 * kDigits + threadIdx.x])
      atomicMax(&a.digits[5 * kDigits + threadIdx.x], sdig[5 * kDigits + threadIdx.x]);
  }
}

}  // namespace cav
