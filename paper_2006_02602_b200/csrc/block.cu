// block.cu — one rank's device-resident state and its per-iteration pipeline:
// the B200-native replacement of rank_main's loop body
// (/root/reference/proj/src/runner.cpp:184-235).
//
// Iteration n on rank r (stream s0), fused halos (the default):
//   fold     stream wait on every rank's scalar slot of n-1; one warp of
//            every step CTA then acquires the stamps and folds dt_n
//            (reduce_fixed_order(Min), src/transport.cpp:23-60, as the exact
//            max rewrite) and pcs_n = p'(centre) of step n from the gathered
//            centre stencil (center_pressure_broadcast)
//   step     k_step_tma: BC (register or stored wall ghosts) + residual +
//            [exact norm digits] + Euler update + eager rescale fl(p'-pcs_n)
//            + next-step CFL maxima + non-finite flags; every output cell in
//            a joined face's halo layers is also stored straight into the
//            neighbour's state over NVLink / peer memory (exchange_begin +
//            exchange_finish, src/exchange.cpp:115-176, fused into the step)
//   push     the step's last CTA (k_push before iteration 1): this rank's
//            maxima, error code and its share of S_n's centre stencil into
//            every rank's slot, release stamp (after the halo stores)
//   ghosts   k_ghosts_yz2 (k_ghosts_yz for odd nx): y/z wall ghosts of S_n (stored-ghost blocks)
// Slab exchange (CAV_FUSED_HALO=0, the corrupt-exchange hook): k_pack pushes
// plan entries of S_{n-1} into the neighbours' receive slabs with a release
// flag per entry; the receiver's stream waits for the flags and k_unpack
// scatters them into the join ghosts; with overlap this runs on stream s1
// while the step takes the internal items, the shell items follow
// (src/runner.cpp:189-194).
// One rank: the step kernel's last CTA folds dt and pcs itself (no fold or
// push). Every cross-rank wait is enqueued only after the launch that
// produces its value has been enqueued (HostProgress below).
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstring>
#include <map>
#include <mutex>
#include <memory>
#include <string>
#include <vector>

#include <cudaTypedefs.h>

#include <chrono>
#include <cstddef>
#include <thread>

#include <cstdlib>

#include "device.cuh"
#include "host.hpp"
#include "ops.hpp"
#include "status.hpp"
#include "step_tma.cuh"

namespace cav {

// ---------------------------------------------------------------------------
// Halo exchange: one descriptor per plan entry (= one reference message).
struct MsgDesc {
  int face;
  int nvars;
  int var[5];
  long long voff[6];  // payload offset of each variable's box (copy_box_to order)
  cav_box box[5];     // pack: face_interior_box; unpack: face_ghost_box
  long long scalars;
  double* slab;               // pack: receiver's slab (parity 0); unpack: own slab (2 parities)
  unsigned long long* flag;   // pack: receiver's flag; unpack: own flag
  unsigned* counter;          // pack: CTA completion counter
  int peer;
};

// Cross-rank values carry a generation in their high bits (one per run from
// iteration 1, i.e. per upload/initialize), so a flag or stamp left by an
// earlier run never satisfies a wait of the current one.
constexpr int kGenShift = 40;

struct XArgs {
  double* state;
  Geo g;
  const MsgDesc* msg;
  long long n;              // iteration (slab parity)
  unsigned long long val;   // flag value of this iteration (generation | n)
  int corrupt;
  const int* abort;
  const int* stop;  // set once the run converged (device decision) or aborted
};

constexpr int kXThreads = 256, kXItems = 4;

// payload element q of entry m -> (variable, storage cell); box volumes are
// far below 2^31, so 32-bit index arithmetic suffices
__device__ __forceinline__ void msg_locate(const MsgDesc& m, int q, int& v, int& i, int& j, int& k) {
  int s = 0;
  while (s + 1 < m.nvars && q >= m.voff[s + 1]) ++s;
  const cav_box& b = m.box[s];
  const int e = q - static_cast<int>(m.voff[s]);
  const int w = b.hi[0] - b.lo[0], h = b.hi[1] - b.lo[1];
  const int row = e / w;
  i = b.lo[0] + (e - row * w);
  const int k0 = row / h;
  j = b.lo[1] + (row - k0 * h);
  k = b.lo[2] + k0;
  v = m.var[s];
}

// exchange_begin (src/exchange.cpp:115-145): every plan entry's payload, in
// copy_box_to order (src/slab.cpp:33-52), stored straight into the
// neighbour's receive slab over NVLink / peer memory; the CTA that completes
// an entry last releases the neighbour's flag (system scope).
__global__ void __launch_bounds__(kXThreads) k_pack(const XArgs a) {
  if (*reinterpret_cast<const volatile int*>(a.abort)) return;
  const MsgDesc& m = a.msg[blockIdx.y];
  if (*reinterpret_cast<const volatile int*>(a.stop)) {  // converged: no payload, the flag still advances
    if (blockIdx.x == 0 && threadIdx.x == 0) st_release_sys(m.flag, a.val);
    return;
  }
  double* dst = m.slab + (a.n & 1) * m.scalars;
  const int base = static_cast<int>(blockIdx.x) * kXThreads * kXItems;
  if (base < m.scalars) {
#pragma unroll
    for (int it = 0; it < kXItems; ++it) {
      const int q = base + it * kXThreads + static_cast<int>(threadIdx.x);
      if (q < m.scalars) {
        int v, i, j, k;
        msg_locate(m, q, v, i, j, k);
        dst[q] = a.state[v * a.g.fstride + a.g.idx(i, j, k)];  // remote store into the neighbour's slab
      }
    }
  }
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned done = atomicAdd(m.counter, 1u);
    if (done == gridDim.x - 1) {
      *m.counter = 0;
      __threadfence_system();
      st_release_sys(m.flag, a.val);
    }
  }
}

// exchange_finish (src/exchange.cpp:147-176): the stream has waited for the
// flags (cuStreamWaitValue64, no resident spinning); the acquire below orders
// the slab reads after the peer's release, then copy_box_from
// (src/slab.cpp:54-71) into the join ghosts.
__global__ void __launch_bounds__(kXThreads) k_unpack(const XArgs a) {
  if (*reinterpret_cast<const volatile int*>(a.abort) || *reinterpret_cast<const volatile int*>(a.stop)) return;
  const MsgDesc& m = a.msg[blockIdx.y];
  const int base = static_cast<int>(blockIdx.x) * kXThreads * kXItems;
  if (base >= m.scalars) return;
  // the stream waited for the flag; the acquire also orders this CTA's slab
  // reads after the sender's release (a lagging view waits here, an abort
  // releases it)
  while (ld_acquire_sys(m.flag) < a.val)
    if (*reinterpret_cast<const volatile int*>(a.abort)) return;
  const double* src = m.slab + (a.n & 1) * m.scalars;
#pragma unroll
  for (int it = 0; it < kXItems; ++it) {
    const int q = base + it * kXThreads + static_cast<int>(threadIdx.x);
    if (q < m.scalars) {
      int v, i, j, k;
      msg_locate(m, q, v, i, j, k);
      double x = __ldcg(src + q);
      if (a.corrupt && blockIdx.y == 0 && q == 0) x += 1e-3;  // exchange_finish's corrupt_first hook
      a.state[v * a.g.fstride + a.g.idx(i, j, k)] = x;
    }
  }
}

// ---------------------------------------------------------------------------
// Scalars between ranks: see step_tma.cuh (fold_scalars_warp / push_scalars_warp).
// Iteration 0's push (the initial state's maxima and centre stencil) has no
// step kernel to ride on, so it is this one-thread kernel.
// Release `v` into up to six peer words (the prologue's "my state is in
// place" signal to each joined neighbour, fused halos).
struct PeerWords {
  unsigned long long* w[6];
  int n;
};
__global__ void k_signal(const PeerWords p, unsigned long long v) {
  if (threadIdx.x < p.n) {
    __threadfence_system();
    st_release_sys(p.w[threadIdx.x], v);
  }
}

// The initial state's halo layers of one joined face (one layer kind) into
// the neighbour's state (fused halos: the step kernel sends every later
// state's halos itself): p and, for the first layer, u, v, w, T.
__global__ void __launch_bounds__(256) k_face_send(const double* st, Geo g, const XDesc* x, int par, cav_box b,
                                                   int m) {
  const int w = b.hi[0] - b.lo[0], h = b.hi[1] - b.lo[1];
  const long long nb = static_cast<long long>(w) * h * (b.hi[2] - b.lo[2]);
  for (long long q = blockIdx.x * 256LL + threadIdx.x; q < nb; q += gridDim.x * 256LL) {
    const int i = b.lo[0] + static_cast<int>(q % w), j = b.lo[1] + static_cast<int>((q / w) % h),
              k = b.lo[2] + static_cast<int>(q / (static_cast<long long>(w) * h));
    const long long c = g.idx(i, j, k), fs = g.fstride;
    send_cell(x, par, i, j, k, m, st[c], st[c + fs], st[c + 2 * fs], st[c + 3 * fs], st[c + 4 * fs]);
  }
  __threadfence_system();
}

__global__ void __launch_bounds__(32) k_push(const XDesc* x, int par, unsigned long long stamp, const Acc* acc,
                                             const double* state, long long fs, const int* abort) {
  if (*reinterpret_cast<const volatile int*>(abort)) return;
  push_scalars_warp(x, par, stamp, acc, state, fs);
}

// Device convergence across ranks (the rule of src/runner.cpp:210-220 on
// global_norms' exact sums, :81-104): after each check iteration every rank
// pushes its exact norm digits into every rank's norm slot (parity of the
// check count) and releases a stamp; every rank's stream waits for all
// stamps, then k_conv_merge adds the np carry-save digit arrays word by word
// (each word stays below 2^64: pieces are 32-bit and a global sum has far
// fewer than 2^32 of them per digit) and applies the rule exactly as
// k_conv_check does on one rank, so every rank takes the same decision.
struct NormSlot {
  unsigned long long w[CAV_NORM_WORDS];
  unsigned long long stamp;
  unsigned long long pad[7];
};

__global__ void __launch_bounds__(256) k_push_norms(const unsigned long long* dig, NormSlot* const* peers, int np,
                                                    int rank, int par, unsigned long long stamp, const int* stop) {
  const bool skip = *reinterpret_cast<const volatile int*>(stop) != 0;  // converged: stamps only
  for (int r = blockIdx.x; r < np; r += gridDim.x) {
    NormSlot* s = peers[r] + (rank * 2 + par);
    if (!skip)
      for (int q = threadIdx.x; q < CAV_NORM_WORDS; q += blockDim.x) s->w[q] = __ldcg(dig + q);
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) st_release_sys(&s->stamp, stamp);
  }
}

// Whole-storage export in the reference Field3 layout: interior from `cur`
// with the pending shift, every ghost from `prev` (the last input state, whose
// ghosts are exactly what the reference's storage holds after the loop).
__global__ void k_export(const double* cur, const double* prev, Geo g, double pc, double* out) {
  const long long X = g.nx + 4, Y = g.ny + 4, Z = g.nz + 4, S = X * Y * Z;
  const long long q = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (q >= 5 * S) return;
  const int v = static_cast<int>(q / S);
  const long long e = q % S;
  const int i = static_cast<int>(e % X), j = static_cast<int>((e / X) % Y), k = static_cast<int>(e / (X * Y));
  const long long c = v * g.fstride + g.idx(i, j, k);
  double x;
  if (g.interior(i, j, k)) {
    x = cur[c];
    if (v == 0) x = x - pc;
  } else {
    x = prev[c];
  }
  out[q] = x;
}

// Host Field3 layout (contiguous, i-fastest, 5 fields) -> both padded states.
__global__ void k_import(const double* in, double* s0, double* s1, Geo g) {
  const long long X = g.nx + 4, Y = g.ny + 4, Z = g.nz + 4, S = X * Y * Z;
  const long long q = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (q >= 5 * S) return;
  const int v = static_cast<int>(q / S);
  const long long e = q % S;
  const int i = static_cast<int>(e % X), j = static_cast<int>((e / X) % Y), k = static_cast<int>(e / (X * Y));
  const long long c = v * g.fstride + g.idx(i, j, k);
  const double x = in[q];
  s0[c] = x;
  s1[c] = x;
}

__global__ void k_fill_ic(double* s0, double* s1, Geo g, double t_inf) {
  const long long X = g.nx + 4, Y = g.ny + 4, Z = g.nz + 4, S = X * Y * Z;
  const long long q = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (q >= 5 * S) return;
  const int v = static_cast<int>(q / S);
  const long long e = q % S;
  const int i = static_cast<int>(e % X), j = static_cast<int>((e / X) % Y), k = static_cast<int>(e / (X * Y));
  const long long c = v * g.fstride + g.idx(i, j, k);
  const double x = v == 4 ? t_inf : 0.0;  // initialize_fields (src/solver.cpp:292-298)
  s0[c] = x;
  s1[c] = x;
}

// ---------------------------------------------------------------------------
// Host side of a block.
namespace {

constexpr size_t kFlagBytes = 64 * sizeof(unsigned long long);

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

struct ArenaLayout {
  size_t slots = 0;                 // offset of Slot[np][2]
  size_t norms = 0;                 // offset of NormSlot[np][2]
  std::vector<size_t> slab;         // per plan entry (receiver side)
  size_t bytes = 0;
};

ArenaLayout arena_layout(const std::vector<cav_plan_entry>& plan, int np) {
  ArenaLayout L;
  L.slots = kFlagBytes;
  L.norms = align_up(L.slots + static_cast<size_t>(np) * 2 * sizeof(Slot), 256);
  size_t off = align_up(L.norms + static_cast<size_t>(np) * 2 * sizeof(NormSlot), 256);
  for (const auto& e : plan) {
    L.slab.push_back(off);
    off = align_up(off + 2 * static_cast<size_t>(e.scalars) * sizeof(double), 256);
  }
  L.bytes = off;
  return L;
}

int find_entry(const std::vector<cav_plan_entry>& plan, int face, const cav_plan_entry& like) {
  for (size_t n = 0; n < plan.size(); ++n)
    if (plan[n].face == face && plan[n].nvars == like.nvars && plan[n].var[0] == like.var[0])
      return static_cast<int>(n);
  throw std::logic_error("exchange: no matching receive entry on the neighbour");
}

// Device geometry of a block of interior n: interior rows start 128-byte
// aligned (off 14 -> i = 2 at 16 doubles), field stride a multiple of 32
// doubles (TMA strides).
Geo geo_of(const std::array<int, 3>& n) {
  Geo g{};
  g.nx = n[0];
  g.ny = n[1];
  g.nz = n[2];
  g.off = 14;
  g.pitch = static_cast<int>(align_up(static_cast<size_t>(g.off + n[0] + 4), 16));
  g.ypitch = n[1] + 4;
  g.fstride = static_cast<long long>(align_up(static_cast<size_t>(g.pitch) * g.ypitch * (n[2] + 4), 32));
  return g;
}

// A block's device memory is ONE allocation [arena | state 0 | state 1], so
// one pointer (in-process) or one CUDA IPC handle gives a peer both the
// exchange arena and the states its step kernel writes halos into. Every
// rank can compute any rank's layout from the decomposition.
struct BlockSpan {
  Geo g;
  ArenaLayout lay;
  size_t state_off = 0, state_bytes = 0, total = 0;
};
BlockSpan block_span(const std::array<int, 3>& n, const std::array<int, 6>& rank_at, int strategy, int np) {
  BlockSpan b;
  b.g = geo_of(n);
  b.lay = arena_layout(host::build_plan(n, rank_at, strategy), np);
  b.state_off = align_up(b.lay.bytes, 4096);
  b.state_bytes = align_up(5 * static_cast<size_t>(b.g.fstride) * sizeof(double), 4096);
  b.total = b.state_off + 2 * b.state_bytes;
  return b;
}

cudaEvent_t make_event() {
  cudaEvent_t e;
  CAV_CUDA(cudaEventCreate(&e));
  return e;
}

}  // namespace

// Device-side convergence decision (single-rank blocks): the rule of
// src/runner.cpp:210-220 — per-variable peaks of the L2 residual norms, stop
// at the first check where max_v |R_v| / peak_v <= conv_tol — evaluated on the
// exact norm digits right after each check iteration, so a solve runs without
// a host round trip per check. Later step kernels see `stop` and return.
struct ConvState {
  int stop;
  int pad;
  long long it;
  double peaks[5];
};

// Exact residual-norm digits of a stored-ghost norm iteration: the squares of
// the residuals k_step_tma<.., NORMS, G> left in the scratch state, summed into
// the iteration's carry-save digits as the step's own digit runs would
// (ReproSum, inc/util/repro_sum.hpp; residual_norm_partials,
// src/solver.cpp:259-274). Each thread walks one k-segment of one (i,j)
// column (coalesced across a warp), so its consecutive terms are z-neighbours
// and the runs stay long, as in the step kernel. It also takes the L-inf
// norm, max |R_v| over the interior: an exact, order-free maximum of the
// magnitudes' bit patterns.
constexpr int kNormRunThreads = 256, kNormRunSeg = 128;
static_assert(kNormRunSeg <= 4096, "a digit run of up to kNormRunSeg terms must fit its 96 bits");
// One variable per thread (blockIdx.y = variable): a 96-bit run and a
// running maximum are all the state a thread keeps; measured 2% faster per
// norm iteration than five per thread. A: planes loaded per batch before
// their terms are summed (the digit runs' shared atomics keep the compiler
// from hoisting later loads, so A = 1 has one load in flight per thread and
// is latency-bound: ncu at 256^3, 220 us and 3.0 TB/s for A = 1, 124 us and
// 5.4 TB/s for A = 8, 48 registers; CAV_NORM_AHEAD=1 selects the former).
template <int A>
__global__ void __launch_bounds__(kNormRunThreads) k_norm_runs(const double* rs, Geo g, cav_box b,
                                                               unsigned long long* dig,
                                                               unsigned long long* err_sticky, long long n,
                                                               int rank, const int* stop) {
  if (stop && *reinterpret_cast<const volatile int*>(stop)) return;
  const int v = static_cast<int>(blockIdx.y);
  __shared__ unsigned long long sd[kDigits], smx;
  for (int x = threadIdx.x; x < kDigits; x += kNormRunThreads) sd[x] = 0;
  if (threadIdx.x == 0) smx = 0;
  __syncthreads();
  const int bw = b.hi[0] - b.lo[0], bh = b.hi[1] - b.lo[1];
  const long long col = static_cast<long long>(blockIdx.x) * kNormRunThreads + threadIdx.x;
  const int i = b.lo[0] + static_cast<int>(col % bw), j = b.lo[1] + static_cast<int>((col / bw) % bh);
  const int k0 = b.lo[2] + static_cast<int>(col / (static_cast<long long>(bw) * bh)) * kNormRunSeg;
  unsigned nf = 0;
  unsigned long long mx = 0;
  if (col < static_cast<long long>(bw) * bh * ((b.hi[2] - b.lo[2] + kNormRunSeg - 1) / kNormRunSeg)) {
    DigitRun run{-1, 0u, 0u, 0u};
    const long long plane = static_cast<long long>(g.pitch) * g.ypitch;
    const int k1 = min(k0 + kNormRunSeg, b.hi[2]);
    const double* q = rs + v * g.fstride + g.idx(i, j, k0);
    for (int k = k0; k < k1; k += A, q += A * plane) {
      double x[A];
#pragma unroll
      for (int u = 0; u < A; ++u) x[u] = k + u < k1 ? __ldcs(q + u * plane) : 0.0;  // 0: no term
#pragma unroll
      for (int u = 0; u < A; ++u) {
        mx = max(mx, abs_bits(x[u]));
        const double x2 = x[u] * x[u];
        if (nonfinite(x2)) nf = 1;
        else digit_run_add(run, sd, x2);
      }
    }
    digit_run_flush(run, sd);
  }
  // warp collectives with every lane present (the last block's tail lanes
  // have no column: a full-mask shuffle inside the branch would wait forever)
  mx = warp_max_u64(mx);
  if ((threadIdx.x & 31) == 0 && mx) atomicMax(&smx, mx);
  __syncthreads();
  for (int x = threadIdx.x; x < kDigits; x += kNormRunThreads)
    if (sd[x]) atomicAdd(&dig[v * kDigits + x], sd[x]);
  if (threadIdx.x == 0 && smx) atomicMax(&dig[5 * kDigits + v], smx);
  if (nf) atomicMin(err_sticky, err_code(n, rank, 0));  // the step kernel's non-finite norm error
}

int getenv_int(const char* name, int dflt);

int norm_ahead() {
  static const int a = getenv_int("CAV_NORM_AHEAD", 8);
  return a;
}

void launch_norm_runs(const double* rs, const Geo& g, const cav_box& b, unsigned long long* dig,
                      unsigned long long* err, long long n, int rank, const int* stop, cudaStream_t st) {
  const long long cols = static_cast<long long>(b.hi[0] - b.lo[0]) * (b.hi[1] - b.lo[1]) *
                         ((b.hi[2] - b.lo[2] + kNormRunSeg - 1) / kNormRunSeg);
  const dim3 grid(static_cast<unsigned>((cols + kNormRunThreads - 1) / kNormRunThreads), 5);
  switch (norm_ahead()) {
    case 1: k_norm_runs<1><<<grid, kNormRunThreads, 0, st>>>(rs, g, b, dig, err, n, rank, stop); break;
    default: k_norm_runs<8><<<grid, kNormRunThreads, 0, st>>>(rs, g, b, dig, err, n, rank, stop); break;
  }
  CAV_CUDA(cudaGetLastError());
}

// The y and z wall ghosts a stored-ghost step reads (p both layers, u,v,w,T
// the first), of a state after a step whose wall lanes stored the x ghosts
// (joined faces are skipped; their ghosts come from the exchange): k_bc's expressions (apply_boundary_conditions, src/solver.cpp:
// 158-191) with no pending shift. One block row per (face, transverse index),
// threads along i: coalesced rows, no face search or 64-bit division.
constexpr int kGhostThreads = 128;
__global__ void __launch_bounds__(kGhostThreads) k_ghosts_yz(double* s, Geo g, WallInfo w, const int* stop) {
  if (stop && *reinterpret_cast<const volatile int*>(stop)) return;
  const int face = 2 + static_cast<int>(blockIdx.z);
  if (!w.wall[face]) return;
  const int ax = face >> 1, hi = face & 1;
  const int nn = ax == 1 ? g.ny : g.nz, nt = ax == 1 ? g.nz : g.ny;
  if (static_cast<int>(blockIdx.y) >= nt) return;
  const int t = 2 + static_cast<int>(blockIdx.y);  // k on a y face, j on a z face
  const int c0 = hi ? nn + 1 : 2, c1 = hi ? nn : 3, c2 = hi ? nn - 1 : 4, g0 = hi ? nn + 2 : 1, g1 = hi ? nn + 3 : 0;
  const long long fs = g.fstride;
  for (int i = 2 + static_cast<int>(blockIdx.x) * kGhostThreads + static_cast<int>(threadIdx.x); i < g.nx + 2;
       i += static_cast<int>(gridDim.x) * kGhostThreads) {
    auto at = [&](int nrm) { return ax == 1 ? g.idx(i, nrm, t) : g.idx(i, t, nrm); };
    const long long e0 = at(c0), q0 = at(g0);
    const double p0 = s[e0], p1 = s[at(c1)], p2 = s[at(c2)];
    const double u = s[fs + e0], v = s[2 * fs + e0], wv = s[3 * fs + e0], tt = s[4 * fs + e0];
    const double pg0 = cubic_g0(p0, p1, p2);
    s[q0] = pg0;
    s[at(g1)] = cubic_g1(pg0, p0, p1);
    s[fs + q0] = -u;  // no-slip: antisymmetric velocity
    s[2 * fs + q0] = -v;
    s[3 * fs + q0] = -wv;
    s[4 * fs + q0] = tt;  // adiabatic
  }
}

// Even nx: a 2 x 2 patch per thread — two neighbouring columns (16-byte loads
// and stores; rows start 128-byte aligned at i = 2) of two neighbouring rows
// — with all fourteen loads in flight before the stop flag is checked; the
// same expressions as k_ghosts_yz (measured: 10.4 -> 6.9 us at 256^3 under
// ncu, -1.2% per iteration, profiles/r02q_ghost_rows.txt).
__global__ void __launch_bounds__(kGhostThreads) k_ghosts_yz2(double* s, Geo g, WallInfo w, const int* stop) {
  const int face = 2 + static_cast<int>(blockIdx.z);
  if (!w.wall[face]) return;
  const int ax = face >> 1, hi = face & 1;
  const int nn = ax == 1 ? g.ny : g.nz, nt = ax == 1 ? g.nz : g.ny;
  const int t0 = 2 + 2 * static_cast<int>(blockIdx.y);
  if (t0 >= nt + 2) return;
  const bool two = t0 + 1 < nt + 2;
  const int c0 = hi ? nn + 1 : 2, c1 = hi ? nn : 3, c2 = hi ? nn - 1 : 4, g0 = hi ? nn + 2 : 1, g1 = hi ? nn + 3 : 0;
  const long long fs = g.fstride;
  const int i = 2 + 2 * (static_cast<int>(blockIdx.x) * kGhostThreads + static_cast<int>(threadIdx.x));
  if (i >= g.nx + 2) return;
  auto ld = [&](long long e) { return *reinterpret_cast<const double2*>(s + e); };
  auto st2 = [&](long long e, double a, double b) { *reinterpret_cast<double2*>(s + e) = make_double2(a, b); };
  double2 P0[2], P1[2], P2[2], U[2], V[2], W[2], T[2];
  long long E0[2], Q0[2], Q1[2];
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int t = t0 + (two ? r : 0);
    auto at = [&](int nrm) { return ax == 1 ? g.idx(i, nrm, t) : g.idx(i, t, nrm); };
    E0[r] = at(c0);
    Q0[r] = at(g0);
    Q1[r] = at(g1);
    P0[r] = ld(E0[r]);
    P1[r] = ld(at(c1));
    P2[r] = ld(at(c2));
    U[r] = ld(fs + E0[r]);
    V[r] = ld(2 * fs + E0[r]);
    W[r] = ld(3 * fs + E0[r]);
    T[r] = ld(4 * fs + E0[r]);
  }
  if (stop && *reinterpret_cast<const volatile int*>(stop)) return;
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    if (r == 1 && !two) break;
    const double ga = cubic_g0(P0[r].x, P1[r].x, P2[r].x), gb = cubic_g0(P0[r].y, P1[r].y, P2[r].y);
    st2(Q0[r], ga, gb);
    st2(Q1[r], cubic_g1(ga, P0[r].x, P1[r].x), cubic_g1(gb, P0[r].y, P1[r].y));
    st2(fs + Q0[r], -U[r].x, -U[r].y);
    st2(2 * fs + Q0[r], -V[r].x, -V[r].y);
    st2(3 * fs + Q0[r], -W[r].x, -W[r].y);
    st2(4 * fs + Q0[r], T[r].x, T[r].y);
  }
}

__global__ void k_conv_check(const unsigned long long* dig, ConvState* c, long long it, double tol, double nglobal,
                             const NormSlot* merge, int np, int par, unsigned long long stamp, const int* abort) {
  if (c->stop) return;
  __shared__ unsigned long long md[5 * kDigits];
  if (merge) {  // many ranks: every rank's digits of this check, summed word by word
    for (int r = threadIdx.x; r < np; r += blockDim.x)
      while (ld_acquire_sys(&merge[r * 2 + par].stamp) < stamp)
        if (*reinterpret_cast<const volatile int*>(abort)) break;
    __syncthreads();
    for (int q = threadIdx.x; q < 5 * kDigits; q += blockDim.x) {
      unsigned long long w = 0;
      for (int r = 0; r < np; ++r) w += __ldcg(&merge[r * 2 + par].w[q]);
      md[q] = w;
    }
    __syncthreads();
    dig = md;
  }
  if (threadIdx.x != 0) return;
  double worst = 0.0;
  for (int v = 0; v < 5; ++v) {
    const double l2 = sqrt_rn(repro_value_from_digits(dig + v * kDigits) / nglobal);  // norms_from_partials
    c->peaks[v] = smax(c->peaks[v], l2);
    if (c->peaks[v] > 0.0) worst = smax(worst, l2 / c->peaks[v]);
  }
  if (worst <= tol) {
    c->stop = 1;
    c->it = it;
  }
}

// Scalars of iteration 1 on a single-rank block (later ones are folded by the
// step kernel's last CTA): dt_1 from the initial state's scan maxima
// (acc[0]), pcs_1 = p'(centre) of the first step, acc[1] reset.
__global__ void k_center_pcs(const double* state, Geo g, WallInfo w, cav_stencil_params sp, BetaFast bf, Acc* acc,
                             IterScalars* sc, double dx, double dy, double dz, double cfl, cav_fluid_params fl,
                             int rescale, unsigned long long* err_sticky, int cx, int cy, int cz) {
  if (threadIdx.x != 0) return;
  const unsigned long long dm[3] = {acc[0].dmax[0], acc[0].dmax[1], acc[0].dmax[2]};
  const double dt = ops::dt_from_maxima(dm, dx, dy, dz, fl, cfl);
  sc->dt = dt;
  sc->pc = 0.0;
  sc->pcs = rescale ? center_p_update(state, g, w, sp, bf, dt, 0.0, cx, cy, cz) : 0.0;
  if (acc[0].err < *err_sticky) *err_sticky = acc[0].err;
  Acc z{};
  z.err = ~0ull;
  acc[1] = z;
}

int getenv_int(const char* name, int dflt) {
  const char* v = std::getenv(name);
  return v ? std::atoi(v) : dflt;
}

PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    CAV_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || !p) throw CudaError("cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// 4-D views (x = padded row, y, z, field) of one 5-field state for TMA:
// `p` = field 0 with a 36 x (TY+4) box, `q` = fields 1..4 (u, v, w, T) with a
// 34 x (TY+2) x 1 x 4 box (one TMA per plane for all four).
CUtensorMap make_state_map(const double* base, const Geo& g, int nfields, int bw, int bh) {
  // L2 sector promotion of the TMA reads (CAV_L2_PROMO: 0 none, 1 64 B, 2 128 B, 3 256 B)
  static const int promo = getenv_int("CAV_L2_PROMO", 3);
  static const CUtensorMapL2promotion kPromo[4] = {CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_64B,
                                                   CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                                                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B};
  CUtensorMap m;
  const cuuint64_t dims[4] = {static_cast<cuuint64_t>(g.pitch), static_cast<cuuint64_t>(g.ypitch),
                              static_cast<cuuint64_t>(g.nz + 4), static_cast<cuuint64_t>(nfields)};
  const cuuint64_t strides[3] = {static_cast<cuuint64_t>(g.pitch) * 8,
                                 static_cast<cuuint64_t>(g.pitch) * g.ypitch * 8,
                                 static_cast<cuuint64_t>(g.fstride) * 8};
  const cuuint32_t box[4] = {static_cast<cuuint32_t>(bw), static_cast<cuuint32_t>(bh), 1,
                             static_cast<cuuint32_t>(nfields)};
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  const CUresult r = tensor_map_encoder()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<double*>(base), dims,
                                          strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                          CU_TENSOR_MAP_SWIZZLE_NONE, kPromo[promo & 3],
                                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled failed: " + std::to_string(static_cast<int>(r)));
  return m;
}

// The step configuration: 32 x 8 tiles (8 consumer warps + 1 TMA issuer warp),
// a 7-slot ring, 2 CTAs per SM. The measured alternatives (other tile
// heights, ring depths, 1 CTA per SM) are listed in DESIGN.md §3.
#ifndef CAV_TMA_TY  // variant builds (scripts/build_variant.sh): -DCAV_TMA_TY=.. -DCAV_TMA_R=.. -DCAV_TMA_CTAS=..
#define CAV_TMA_TY 8
#endif
#ifndef CAV_TMA_R
#define CAV_TMA_R 7
#endif
#ifndef CAV_TMA_CTAS
#define CAV_TMA_CTAS 2
#endif
using TmaV0 = TmaCfg<CAV_TMA_TY, CAV_TMA_R, CAV_TMA_CTAS>;
constexpr int kTY = TmaV0::TY;

template <class Cfg, bool NORMS, bool G, bool X>
void tma_attrs() {
  CAV_CUDA(cudaFuncSetAttribute(k_step_tma<Cfg, NORMS, G, X>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(Cfg::Smem)));
  CAV_CUDA(cudaFuncSetAttribute(k_step_tma<Cfg, NORMS, G, X>, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
  cudaFuncAttributes fa;
  CAV_CUDA(cudaFuncGetAttributes(&fa, k_step_tma<Cfg, NORMS, G, X>));
}

template <class Cfg>
void tma_attrs_full() {
  CAV_CUDA(cudaFuncSetAttribute(k_step_tma<Cfg, false, true, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(Cfg::Smem)));
  CAV_CUDA(cudaFuncSetAttribute(k_step_tma<Cfg, false, true, false, true>,
                                cudaFuncAttributePreferredSharedMemoryCarveout, 100));
}

template <class Cfg>
int tma_setup(int device) {
  tma_attrs_full<Cfg>();
  tma_attrs<Cfg, false, false, false>();
  tma_attrs<Cfg, true, false, false>();
  tma_attrs<Cfg, false, true, false>();
  tma_attrs<Cfg, true, true, false>();
  tma_attrs<Cfg, false, false, true>();
  tma_attrs<Cfg, true, false, true>();
  tma_attrs<Cfg, false, true, true>();
  tma_attrs<Cfg, true, true, true>();
  int per_sm = 0, sms = 0;
  CAV_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_step_tma<Cfg, false, false, false>, Cfg::Threads,
                                                         Cfg::Smem));
  CAV_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  return std::max(1, std::min(per_sm, Cfg::CTAS)) * sms;
}

template <class Cfg, bool X>
void tma_launch_x(const CUtensorMap* m, const TmaStepArgs& a, bool check, bool ghosts, int grid, cudaStream_t st) {
  if (ghosts) {
    if (check) k_step_tma<Cfg, true, true, X><<<grid, Cfg::Threads, Cfg::Smem, st>>>(m[0], m[1], a);
    else k_step_tma<Cfg, false, true, X><<<grid, Cfg::Threads, Cfg::Smem, st>>>(m[0], m[1], a);
  } else {
    if (check) k_step_tma<Cfg, true, false, X><<<grid, Cfg::Threads, Cfg::Smem, st>>>(m[0], m[1], a);
    else k_step_tma<Cfg, false, false, X><<<grid, Cfg::Threads, Cfg::Smem, st>>>(m[0], m[1], a);
  }
  CAV_CUDA(cudaGetLastError());
}

template <class Cfg>
void tma_launch(const CUtensorMap* m, const TmaStepArgs& a, bool check, bool ghosts, bool send, bool full, int grid,
                cudaStream_t st) {
  if (full && ghosts && !check && !send) {  // the production plain step on whole tiles
    k_step_tma<Cfg, false, true, false, true><<<grid, Cfg::Threads, Cfg::Smem, st>>>(m[0], m[1], a);
    CAV_CUDA(cudaGetLastError());
  } else if (send) {
    tma_launch_x<Cfg, true>(m, a, check, ghosts, grid, st);
  } else {
    tma_launch_x<Cfg, false>(m, a, check, ghosts, grid, st);
  }
}

// Stream memory operations (driver API): a stream waits for a 64-bit value in
// device memory to reach a target without occupying any SM, so cross-rank
// waits survive kernel serialisation (profilers, sanitizers, ranks sharing a
// GPU) and can sit on a second stream next to the compute stream.
PFN_cuStreamBatchMemOp_v11070 batch_memop() {
  static PFN_cuStreamBatchMemOp_v11070 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    CAV_CUDA(cudaGetDriverEntryPointByVersion("cuStreamBatchMemOp", &p, 11070, cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || !p) throw CudaError("cuStreamBatchMemOp unavailable");
    fn = reinterpret_cast<PFN_cuStreamBatchMemOp_v11070>(p);
  }
  return fn;
}

// Waits on `st` until every address holds a value >= its target.
void stream_wait_geq(cudaStream_t st, const std::vector<std::pair<const unsigned long long*, unsigned long long>>& w,
                     unsigned flags) {
  if (w.empty()) return;
  std::vector<CUstreamBatchMemOpParams> ops(w.size());
  for (size_t q = 0; q < w.size(); ++q) {
    std::memset(&ops[q], 0, sizeof ops[q]);
    ops[q].waitValue.operation = CU_STREAM_MEM_OP_WAIT_VALUE_64;
    ops[q].waitValue.address = reinterpret_cast<CUdeviceptr>(w[q].first);
    ops[q].waitValue.value64 = w[q].second;
    ops[q].waitValue.flags = CU_STREAM_WAIT_VALUE_GEQ | flags;
  }
  for (size_t q = 0; q < ops.size(); q += 256) {  // the driver's per-call limit
    const unsigned cnt = static_cast<unsigned>(std::min<size_t>(256, ops.size() - q));
    const CUresult r = batch_memop()(reinterpret_cast<CUstream>(st), cnt, ops.data() + q, 0);
    if (r != CUDA_SUCCESS) throw CudaError("cuStreamBatchMemOp failed: " + std::to_string(static_cast<int>(r)));
  }
}

// counters[] words
constexpr int kCtrAbort = 60, kCtrWork = 62, kCtrDone = 63;

// Host-side enqueue progress of a block, shared with the blocks of the same
// process that connect to it (in-process ranks: cav_run_case's threads, or
// several capi.Block objects). A stream wait is only enqueued after every
// launch that produces its value has been enqueued: CUDA multiplexes streams
// onto a fixed set of hardware queues, and a wait that sits in a queue ahead
// of the work it waits for (another rank's stream mapped to the same queue)
// would never be satisfied. With producers always enqueued first, every wait
// finds its producer ahead of it in any queue they share, so the FIFO order
// cannot deadlock. Peers in other processes (other contexts) need no such
// ordering. Values carry the run generation like the device flags.
struct HostProgress {
  std::atomic<unsigned long long> push{0};  // base | it: push(it) enqueued (push(0) = +0 after prologue)
  std::atomic<unsigned long long> pack{0};  // base | it: pack(it) enqueued
  std::atomic<unsigned long long> norm{0};  // base | c: the norm push of check c (0-based) enqueued
  std::atomic<unsigned long long> ready{0};  // base: this run's state is in place (fused halos may land)
};

// arena words: [0, 32) halo flags of the plan entries (slab exchange),
// [40, 46) per face: the neighbour there has initialised its run (fused halos)
constexpr int kReadyWord = 40;

std::mutex g_reg_mu;
std::map<const void*, std::shared_ptr<HostProgress>>& registry() {
  static std::map<const void*, std::shared_ptr<HostProgress>> m;
  return m;
}

struct Block {
  cav_block_desc d{};
  std::array<int, 3> gn{}, dims{}, n{};
  std::vector<host::Extent> ext;
  std::array<int, 6> rank_at{};
  int walls[6]{};
  int owner = 0;
  int cx = -1, cy = -1, cz = -1;
  double dx = 0, dy = 0, dz = 0;
  cav_stencil_params sp{};
  Geo g{};
  double* state[2]{};
  double* staging = nullptr;   // 5 * S doubles in the host Field3 layout (upload / download)
  double* rscratch = nullptr;  // stored-ghost norm iterations: residuals (state layout)
  bool step_used_scratch = false;  // the last step kernel left its residuals in rscratch
  int cur = 0;
  std::vector<cav_plan_entry> plan;
  ArenaLayout lay;
  unsigned char* arena = nullptr;
  std::vector<unsigned char*> peer_arena;
  std::vector<bool> peer_ipc;
  std::shared_ptr<HostProgress> prog = std::make_shared<HostProgress>();
  std::vector<std::shared_ptr<HostProgress>> host_peer;  // in-process peers (else null)
  // device bookkeeping
  Acc* acc = nullptr;            // [2]
  IterScalars* sc = nullptr;     // [2]
  unsigned long long* err = nullptr;      // sticky min error code
  unsigned* counters = nullptr;  // [0, 32) pack entry counters; kCtrAbort, kCtrWork, kCtrDone
  int* abort_flag = nullptr;     // set (host) when a transport timeout aborts the block
  MsgDesc* d_pack = nullptr;
  MsgDesc* d_unpack = nullptr;
  Slot** d_peer_slots = nullptr;
  XDesc* d_xd = nullptr;         // cross-rank scalar constants (step_tma.cuh)
  long long* iter_dev = nullptr;  // one rank: the iteration the next step computes (TmaStepArgs::n_dev)
  // one rank: CUDA graphs of two plain iterations, keyed by (cur, it & 1)
  cudaGraphExec_t gexec[4]{};
  bool use_graphs = false;
  NormSlot** d_peer_norms = nullptr;  // every rank's NormSlot array (device convergence, np > 1)
  long long chk_count = 0;        // check iterations since the prologue (norm slot parity)
  unsigned long long* digits = nullptr;
  ConvState* conv = nullptr;              // device convergence state (single rank)
  const int* stop_flag = nullptr;         // = &conv->stop while a device-converging run is active
  long long digits_cap = 0;
  bool ready = false;
  long long next_n = 1;
  bool primed = false;
  unsigned long long gen = 0;   // run generation (kGenShift)
  bool dead = false;            // aborted by a transport timeout
  unsigned wait_flags = 0;      // CU_STREAM_WAIT_VALUE_FLUSH where supported
  cudaStream_t s0 = nullptr, s1 = nullptr, saux = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr, ev_a = nullptr, ev_b = nullptr;
  // host-side progress window (np > 1): at most kWindow iterations in flight,
  // iteration q's completion event at win[q % kWindow]
  static constexpr int kWindow = 12;
  cudaEvent_t win[kWindow]{};
  long long win_it[kWindow]{};
  // bench timing per iteration: e[0], e[1] around the wait for the peers'
  // scalars; e[2..] pairs around the step launches; e_join after the halo join
  struct IterTiming {
    cudaEvent_t e[7];
  };
  std::vector<IterTiming> timing;
  size_t timing_used = 0;
  CUtensorMap tmap[2][2];  // [state][p, uvwT]
  BetaFast bf{-1.0, 0u};
  bool ghosts = false;           // stored wall ghosts (see launch_step)
  bool fused = false;            // np > 1: the step kernel sends the halos itself (no pack/unpack)
  bool ghost_writes = true;      // CAV_GHOST_WRITES=0: always k_bc
  bool step_wrote_ghosts = false;  // the last step kernel wrote its output's x-wall ghosts itself
  int tail_chunks = -1;          // CAV_TAIL_CHUNKS: short chunks at the end (-1 = two waves)
  int tma_chunk = 0;             // CAV_TMA_CHUNK: fixed k-chunk (0 = balanced choice)
  WallInfo winfo{};
  int tma_grid = 0;      // persistent step grid: CTAs per SM x SMs
  int shell[4] = {0, 0, 0, 0};   // internal tile range sx0, sx1, sy0, sy1
  int zsh[2] = {0, 0};           // joined low / high z faces
  StarCells star_mine{};
  int star_owner[kStar]{};
  double host_marks[6] = {};  // diagnostics: host timestamps inside the first run (s)

  explicit Block(const cav_block_desc& desc);
  ~Block();
  double* field(int s, int v) const { return state[s] + v * g.fstride; }
  unsigned long long base() const { return gen << kGenShift; }
  void ensure_ready();
  void prologue();
  void iteration(long long it, bool check, unsigned long long* dig, IterTiming* tm);
  // returns the launch's item count; dry: only count
  long long launch_step(int part, long long it, bool check, unsigned long long* dig, bool xfold, bool write_sc,
                        bool push, bool dry);
  void wait_scalars(long long it);
  void launch_push(long long it);
  void launch_ghosts();
  void update_ledger(cav_ledger& l) const;
  // one rank: iterations it and it+1 (no norms) as one CUDA graph launch
  void iteration_pair_graph(long long it);
  // np > 1: keeps at most kWindow iterations in flight; polls with the
  // transport timeout (a missing peer raises TransportTimeout, not a hang)
  void window_mark(long long it);
  void window_drain();
  void wait_event(cudaEvent_t e);
  // in-process peers: returns once `word` of peer r's progress reaches `want`
  void wait_host(int r, const std::atomic<unsigned long long> HostProgress::*word, unsigned long long want,
                 long long it);
  [[noreturn]] void on_timeout(long long hint = 0);
};

Block::Block(const cav_block_desc& desc) : d(desc) {
  host::validate_params(d.fluid);
  gn = {d.gnx, d.gny, d.gnz};
  dims = {d.dims[0], d.dims[1], d.dims[2]};
  if (dims[0] * dims[1] * dims[2] != d.np) throw std::invalid_argument("block: dims do not multiply to np");
  if (d.rank < 0 || d.rank >= d.np) throw std::invalid_argument("rank out of range");
  const auto h = host::cavity_spacing(gn[0], gn[1], gn[2], d.fluid.length, d.fluid.length, d.fluid.length);
  dx = h[0];
  dy = h[1];
  dz = h[2];
  ext = host::partition(gn, dims);
  const host::Extent& e = ext[d.rank];
  n = {e.size(0), e.size(1), e.size(2)};
  host::validate_grid(n[0], n[1], n[2], dx, dy, dz);
  rank_at = host::neighbors(dims, d.rank);
  for (int f = 0; f < 6; ++f) walls[f] = rank_at[f] == CAV_WALL;
  for (int f = 0; f < 6; ++f) winfo.wall[f] = walls[f] ? 1 : 0;
  winfo.t_hot = d.fluid.t_hot;
  winfo.t_cold = d.fluid.t_cold;
  const auto c = host::center_node(gn);
  owner = host::owner_of(ext, c);
  if (owner == d.rank) {
    cx = c[0] - e.lo[0] + 2;
    cy = c[1] - e.lo[1] + 2;
    cz = c[2] - e.lo[2] + 2;
  }
  sp = host::stencil_params(dx, dy, dz, d.fluid);
  bf = host::beta_fast(sp.u_ref);
  plan = host::build_plan(n, rank_at, d.strategy);
  lay = arena_layout(plan, d.np);

  CAV_CUDA(cudaSetDevice(d.device));
  CAV_CUDA(cudaStreamCreateWithFlags(&s0, cudaStreamNonBlocking));
  CAV_CUDA(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking));
  CAV_CUDA(cudaStreamCreateWithFlags(&saux, cudaStreamNonBlocking));
  const BlockSpan span = block_span(n, rank_at, d.strategy, d.np);
  g = span.g;

  // the centre cell's stencil values this rank owns (k_push) and the owner of
  // each (k_fold); the centre of a valid grid (>= 5 nodes per axis) is at
  // least two nodes from every wall, so its stencil has no wall ghosts
  {
    static const int off[kStar][4] = {{0, 0, 0, 0},  {0, -1, 0, 0}, {0, 1, 0, 0},  {0, -2, 0, 0}, {0, 2, 0, 0},
                                      {0, 0, -1, 0}, {0, 0, 1, 0},  {0, 0, -2, 0}, {0, 0, 2, 0},  {0, 0, 0, -1},
                                      {0, 0, 0, 1},  {0, 0, 0, -2}, {0, 0, 0, 2},  {1, 0, 0, 0},  {1, -1, 0, 0},
                                      {1, 1, 0, 0},  {2, 0, 0, 0},  {2, 0, -1, 0}, {2, 0, 1, 0},  {3, 0, 0, 0},
                                      {3, 0, 0, -1}, {3, 0, 0, 1}};
    for (int q = 0; q < kStar; ++q) {
      const std::array<int, 3> cell{c[0] + off[q][1], c[1] + off[q][2], c[2] + off[q][3]};
      for (int a = 0; a < 3; ++a)
        if (cell[a] < 0 || cell[a] >= gn[a]) throw std::invalid_argument("block: centre stencil reaches a wall");
      star_owner[q] = host::owner_of(ext, cell);
      if (star_owner[q] == d.rank) {
        const int m = star_mine.n++;
        star_mine.slot[m] = q;
        star_mine.var[m] = off[q][0];
        star_mine.idx[m] = g.idx(cell[0] - e.lo[0] + 2, cell[1] - e.lo[1] + 2, cell[2] - e.lo[2] + 2);
      }
    }
  }

  CAV_CUDA(cudaMalloc(&arena, span.total));
  // Stream-ordered and completed before any peer can see this allocation.
  CAV_CUDA(cudaMemsetAsync(arena, 0, span.total, s0));
  for (int s = 0; s < 2; ++s) state[s] = reinterpret_cast<double*>(arena + span.state_off + s * span.state_bytes);
  // staging for upload/download, allocated once (a per-call allocation of
  // this size sat inside the e2e timed region)
  CAV_CUDA(cudaMalloc(&staging, 5 * static_cast<size_t>(n[0] + 4) * (n[1] + 4) * (n[2] + 4) * sizeof(double)));
  {  // load every kernel module now (see ops::preload_kernels)
    ops::preload_kernels();
    cudaFuncAttributes fa;
    CAV_CUDA(cudaFuncGetAttributes(&fa, k_pack));
    CAV_CUDA(cudaFuncGetAttributes(&fa, k_unpack));
    CAV_CUDA(cudaFuncGetAttributes(&fa, k_push));
    CAV_CUDA(cudaFuncGetAttributes(&fa, k_export));
    CAV_CUDA(cudaFuncGetAttributes(&fa, k_fill_ic));
    CAV_CUDA(cudaFuncGetAttributes(&fa, k_import));
    CAV_CUDA(cudaFuncGetAttributes(&fa, k_center_pcs));
    CAV_CUDA(cudaFuncGetAttributes(&fa, k_conv_check));
    CAV_CUDA(cudaFuncGetAttributes(&fa, k_norm_runs<8>));
    CAV_CUDA(cudaFuncGetAttributes(&fa, k_ghosts_yz));
  }
  {
    tail_chunks = getenv_int("CAV_TAIL_CHUNKS", -1);
    tma_chunk = getenv_int("CAV_TMA_CHUNK", 0);
    // stored ghosts pay from about 150^3 (measured per iteration: 32^3 14.6
    // vs 10.3 us, 128^3 62.1 vs 60.7 us, 256^3 321 vs 335 us): below that the
    // extra ghost-kernel launch costs more than the single accessor saves
    const int sg = getenv_int("CAV_STORED_GHOSTS", -1);
    ghosts = sg == 1 || (sg < 0 && static_cast<long long>(n[0]) * n[1] * n[2] >= 3000000LL);
    ghost_writes = getenv_int("CAV_GHOST_WRITES", 1) != 0;
    // fused halos unless the corrupt-exchange hook (a receive-side test of
    // exchange_finish) or CAV_FUSED_HALO=0 asks for the slab exchange
    fused = d.np > 1 && !d.corrupt_exchange && getenv_int("CAV_FUSED_HALO", 1) != 0;
    tma_grid = tma_setup<TmaV0>(d.device);
    for (int s = 0; s < 2; ++s) {
      tmap[s][0] = make_state_map(state[s], g, 1, kPW, kTY + 4);
      tmap[s][1] = make_state_map(state[s] + g.fstride, g, 4, kQW, kTY + 2);
    }
    // internal / shell tiles (overlap): a tile is internal unless it holds
    // one of the two cell layers next to a joined face
    const int tx = (n[0] + 31) / 32, ty = (n[1] + kTY - 1) / kTY;
    shell[0] = walls[0] ? 0 : 1;
    shell[1] = walls[1] ? tx : (n[0] - 2) / 32;
    shell[2] = walls[2] ? 0 : 1;
    shell[3] = walls[3] ? ty : (n[1] - 2) / kTY;
    if (shell[1] < shell[0]) shell[1] = shell[0];
    if (shell[3] < shell[2]) shell[3] = shell[2];
    zsh[0] = walls[4] ? 0 : 1;
    zsh[1] = walls[5] ? 0 : 1;
  }
  if (ghosts) {  // residual scratch of norm iterations, allocated up front (not inside the loop)
    CAV_CUDA(cudaMalloc(&rscratch, 5 * static_cast<size_t>(g.fstride) * sizeof(double)));
  }
  if (d.np > 1) {
    int dev = 0;
    CAV_CUDA(cudaGetDevice(&dev));
    int ok64 = 0, flush = 0;
    CAV_CUDA(cudaDeviceGetAttribute(&ok64, static_cast<cudaDeviceAttr>(CU_DEVICE_ATTRIBUTE_CAN_USE_64_BIT_STREAM_MEM_OPS),
                                    dev));
    if (!ok64) throw CudaError("block: the device does not support 64-bit stream memory operations");
    CAV_CUDA(cudaDeviceGetAttribute(&flush, static_cast<cudaDeviceAttr>(CU_DEVICE_ATTRIBUTE_CAN_FLUSH_REMOTE_WRITES),
                                    dev));
    wait_flags = flush ? CU_STREAM_WAIT_VALUE_FLUSH : 0;
    batch_memop();
  }
  CAV_CUDA(cudaMalloc(&acc, 2 * sizeof(Acc)));
  CAV_CUDA(cudaMalloc(&sc, 2 * sizeof(IterScalars)));
  CAV_CUDA(cudaMalloc(&err, 2 * sizeof(unsigned long long)));
  CAV_CUDA(cudaMalloc(&counters, 64 * sizeof(unsigned)));
  abort_flag = reinterpret_cast<int*>(counters + kCtrAbort);
  CAV_CUDA(cudaMalloc(&conv, sizeof(ConvState)));
  CAV_CUDA(cudaMemsetAsync(conv, 0, sizeof(ConvState), s0));
  CAV_CUDA(cudaMemsetAsync(counters, 0, 64 * sizeof(unsigned), s0));
  CAV_CUDA(cudaMalloc(&d_peer_slots, d.np * sizeof(Slot*)));
  CAV_CUDA(cudaMalloc(&d_xd, sizeof(XDesc)));
  CAV_CUDA(cudaMalloc(&iter_dev, sizeof(long long)));
  use_graphs = d.np == 1 && getenv_int("CAV_GRAPHS", 1) != 0;
  CAV_CUDA(cudaMalloc(&d_peer_norms, d.np * sizeof(NormSlot*)));
  if (!plan.empty()) {
    CAV_CUDA(cudaMalloc(&d_pack, plan.size() * sizeof(MsgDesc)));
    CAV_CUDA(cudaMalloc(&d_unpack, plan.size() * sizeof(MsgDesc)));
  }
  CAV_CUDA(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming));
  CAV_CUDA(cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming));
  for (auto& w : win) CAV_CUDA(cudaEventCreateWithFlags(&w, cudaEventDisableTiming));
  ev_a = make_event();
  ev_b = make_event();
  CAV_CUDA(cudaStreamSynchronize(s0));
  peer_arena.assign(d.np, nullptr);
  peer_ipc.assign(d.np, false);
  peer_arena[d.rank] = arena;
  host_peer.assign(d.np, nullptr);
  std::lock_guard<std::mutex> lk(g_reg_mu);
  registry()[arena] = prog;
}

Block::~Block() {
  {
    std::lock_guard<std::mutex> lk(g_reg_mu);
    registry().erase(arena);
  }
  cudaSetDevice(d.device);
  if (s0) cudaStreamSynchronize(s0);
  if (s1) cudaStreamSynchronize(s1);
  for (int r = 0; r < d.np; ++r)
    if (peer_ipc[r] && peer_arena[r]) cudaIpcCloseMemHandle(peer_arena[r]);
  for (auto& t : timing)
    for (auto e : t.e) cudaEventDestroy(e);
  for (auto w : win)
    if (w) cudaEventDestroy(w);
  cudaFree(staging);
  cudaFree(rscratch);
  cudaFree(arena);
  cudaFree(acc);
  cudaFree(sc);
  cudaFree(err);
  cudaFree(counters);
  cudaFree(conv);
  cudaFree(d_peer_slots);
  cudaFree(d_xd);
  cudaFree(iter_dev);
  for (auto& ge : gexec)
    if (ge) cudaGraphExecDestroy(ge);
  cudaFree(d_peer_norms);
  cudaFree(d_pack);
  cudaFree(d_unpack);
  if (digits) cudaFreeAsync(digits, s0);
  if (s0) cudaStreamSynchronize(s0);
  if (ev_fork) cudaEventDestroy(ev_fork);
  if (ev_join) cudaEventDestroy(ev_join);
  if (ev_a) cudaEventDestroy(ev_a);
  if (ev_b) cudaEventDestroy(ev_b);
  if (s0) cudaStreamDestroy(s0);
  if (s1) cudaStreamDestroy(s1);
  if (saux) cudaStreamDestroy(saux);
}

void Block::ensure_ready() {
  if (dead) throw std::logic_error("block: aborted by an earlier transport timeout");
  if (ready) return;
  for (int r = 0; r < d.np; ++r)
    if (!peer_arena[r])
      throw std::logic_error("block: rank " + std::to_string(r) + " not connected (cav_block_connect)");
  std::vector<Slot*> ps(d.np);
  for (int r = 0; r < d.np; ++r) ps[r] = reinterpret_cast<Slot*>(peer_arena[r] + lay.slots);
  CAV_CUDA(cudaMemcpyAsync(d_peer_slots, ps.data(), d.np * sizeof(Slot*), cudaMemcpyHostToDevice, s0));
  std::vector<NormSlot*> pn(d.np);
  for (int r = 0; r < d.np; ++r) pn[r] = reinterpret_cast<NormSlot*>(peer_arena[r] + lay.norms);
  CAV_CUDA(cudaMemcpyAsync(d_peer_norms, pn.data(), d.np * sizeof(NormSlot*), cudaMemcpyHostToDevice, s0));
  XDesc xd{};
  xd.slots = reinterpret_cast<const Slot*>(arena + lay.slots);
  xd.peer_slots = d_peer_slots;
  xd.np = d.np;
  xd.rank = d.rank;
  xd.rescale = d.rescale;
  xd.abort = abort_flag;
  for (int q = 0; q < kStar; ++q) xd.owner[q] = static_cast<signed char>(star_owner[q]);
  xd.mine = star_mine;
  if (fused) {
    for (int f = 0; f < 6; ++f) {
      const int nb = rank_at[f];
      if (nb < 0) continue;  // a wall
      const host::Extent& ne = ext[nb];
      const std::array<int, 3> nn{ne.size(0), ne.size(1), ne.size(2)};
      const BlockSpan sp_nb = block_span(nn, host::neighbors(dims, nb), d.strategy, d.np);
      FaceSend& fsd = xd.face[f];
      for (int q = 0; q < 2; ++q)
        fsd.base[q] = reinterpret_cast<double*>(peer_arena[nb] + sp_nb.state_off + q * sp_nb.state_bytes);
      fsd.fstride = sp_nb.g.fstride;
      fsd.pitch = sp_nb.g.pitch;
      fsd.ypitch = sp_nb.g.ypitch;
      fsd.off = sp_nb.g.off;
      const int ax = f >> 1;
      fsd.shift = (f & 1) ? -n[ax] : nn[ax];  // our halo layers -> the neighbour's ghost layers
      fsd.dq = 1;
      for (const auto& e : plan)  // the plan's u..T depth on this face (exchange parity of the ghost storage)
        if (e.face == f)
          for (int v = 0; v < e.nvars; ++v)
            if (e.var[v] != 0) fsd.dq = std::max(fsd.dq, e.depth[v]);
      xd.xmask |= 1 << f;
    }
  }
  xd.sp = sp;
  xd.bf = bf;
  xd.dx = dx;
  xd.dy = dy;
  xd.dz = dz;
  xd.cfl = d.cfl;
  xd.nu = d.fluid.nu;
  xd.alpha = d.fluid.alpha;
  CAV_CUDA(cudaMemcpyAsync(d_xd, &xd, sizeof xd, cudaMemcpyHostToDevice, s0));
  std::vector<MsgDesc> pk(plan.size()), up(plan.size());
  for (size_t m = 0; m < plan.size(); ++m) {
    const cav_plan_entry& e = plan[m];
    MsgDesc a{};
    a.face = e.face;
    a.nvars = e.nvars;
    a.scalars = e.scalars;
    a.peer = e.neighbor;
    long long off = 0;
    for (int v = 0; v < e.nvars; ++v) a.var[v] = e.var[v];
    MsgDesc b = a;
    for (int v = 0; v < e.nvars; ++v) {
      a.voff[v] = off;
      b.voff[v] = off;
      a.box[v] = host::face_box(n, e.face, e.depth[v], false);
      b.box[v] = host::face_box(n, e.face, e.depth[v], true);
      off += host::box_volume(a.box[v]);
    }
    a.voff[e.nvars] = b.voff[e.nvars] = off;
    // the neighbour receives on the opposite face into its own plan's entry
    const host::Extent& ne = ext[e.neighbor];
    const std::array<int, 3> nn{ne.size(0), ne.size(1), ne.size(2)};
    const auto nplan = host::build_plan(nn, host::neighbors(dims, e.neighbor), d.strategy);
    const ArenaLayout nl = arena_layout(nplan, d.np);
    const int ri = find_entry(nplan, e.face ^ 1, e);
    a.slab = reinterpret_cast<double*>(peer_arena[e.neighbor] + nl.slab[ri]);
    a.flag = reinterpret_cast<unsigned long long*>(peer_arena[e.neighbor]) + ri;
    a.counter = counters + m;
    b.slab = reinterpret_cast<double*>(arena + lay.slab[m]);
    b.flag = reinterpret_cast<unsigned long long*>(arena) + m;
    pk[m] = a;
    up[m] = b;
  }
  if (!plan.empty()) {
    CAV_CUDA(cudaMemcpyAsync(d_pack, pk.data(), pk.size() * sizeof(MsgDesc), cudaMemcpyHostToDevice, s0));
    CAV_CUDA(cudaMemcpyAsync(d_unpack, up.data(), up.size() * sizeof(MsgDesc), cudaMemcpyHostToDevice, s0));
  }
  CAV_CUDA(cudaStreamSynchronize(s0));
  ready = true;
}

void Block::prologue() {
  ++gen;
  chk_count = 0;
  Acc z[2] = {};
  z[0].err = z[1].err = ~0ull;
  CAV_CUDA(cudaMemcpyAsync(acc, z, sizeof z, cudaMemcpyHostToDevice, s0));
  CAV_CUDA(cudaMemsetAsync(sc, 0, 2 * sizeof(IterScalars), s0));
  const unsigned long long e0[2] = {~0ull, ~0ull};
  CAV_CUDA(cudaMemcpyAsync(err, e0, sizeof e0, cudaMemcpyHostToDevice, s0));
  const cav_field_ptrs f{field(cur, 0), field(cur, 1), field(cur, 2), field(cur, 3), field(cur, 4)};
  const cav_box ib{{2, 2, 2}, {n[0] + 2, n[1] + 2, n[2] + 2}};
  ops::launch_dt_scan(f, g, ib, sp.u_ref, acc, 1, d.rank, s0);  // dt_1 from the initial state
  if (ghosts) {  // the first input state's wall ghosts (stored-ghost step)
    double* fc[5] = {field(cur, 0), field(cur, 1), field(cur, 2), field(cur, 3), field(cur, 4)};
    ops::launch_bc(fc, g, walls, d.fluid, nullptr, s0);
  }
  if (d.np == 1) {
    // scalars of iteration 1 directly: dt_1 (the fold of the scan's maxima)
    // and pcs_1 = p'(centre) of the first step
    k_center_pcs<<<1, 32, 0, s0>>>(state[cur], g, winfo, sp, bf, acc, sc + 1, dx, dy, dz, d.cfl, d.fluid,
                                   d.rescale, err, cx, cy, cz);
    CAV_CUDA(cudaGetLastError());
  } else {
    if (fused) {
      // 1. tell every joined neighbour our state is in place (it may write
      //    halos into it from now on), 2. wait until theirs are, 3. send the
      //    initial state's halos; push(0) below then releases them with the
      //    scalars (every later state's halos ride on the step kernel)
      PeerWords pw{};
      for (int f = 0; f < 6; ++f)
        if (rank_at[f] >= 0)
          pw.w[pw.n++] = reinterpret_cast<unsigned long long*>(peer_arena[rank_at[f]]) + kReadyWord + (f ^ 1);
      k_signal<<<1, 32, 0, s0>>>(pw, base());
      CAV_CUDA(cudaGetLastError());
      prog->ready.store(base(), std::memory_order_release);
      std::vector<std::pair<const unsigned long long*, unsigned long long>> w;
      for (int f = 0; f < 6; ++f)
        if (rank_at[f] >= 0) {
          wait_host(rank_at[f], &HostProgress::ready, base(), 1);
          w.emplace_back(reinterpret_cast<unsigned long long*>(arena) + kReadyWord + f, base());
        }
      stream_wait_geq(s0, w, wait_flags);
      for (int f = 0; f < 6; ++f) {
        if (rank_at[f] < 0) continue;
        const int ax = f >> 1;
        for (int layer = 0; layer < 2; ++layer) {  // layer 0: p, u, v, w, T; layer 1: p (+ u..T at depth 2)
          cav_box b{{2, 2, 2}, {n[0] + 2, n[1] + 2, n[2] + 2}};
          b.lo[ax] = (f & 1) ? n[ax] + 1 - layer : 2 + layer;
          b.hi[ax] = b.lo[ax] + 1;
          int dq = 1;
          for (const auto& e : plan)
            if (e.face == f)
              for (int v = 0; v < e.nvars; ++v)
                if (e.var[v] != 0) dq = std::max(dq, e.depth[v]);
          const int bits = layer == 0 ? 3 : (dq == 2 ? 3 : 1);
          k_face_send<<<296, 256, 0, s0>>>(state[cur], g, d_xd, cur, b, bits << (2 * f));
          CAV_CUDA(cudaGetLastError());
        }
      }
    }
    launch_push(0);  // iteration 0's maxima (the scan) and the initial state's centre star
  }
  primed = true;
}

void Block::wait_scalars(long long it) {
  // every rank's push of iteration it-1: enqueued (in-process peers), then
  // landed (stream wait on the stamps, no SM held)
  const Slot* slots = reinterpret_cast<const Slot*>(arena + lay.slots);
  const int par = static_cast<int>((it - 1) & 1);
  std::vector<std::pair<const unsigned long long*, unsigned long long>> w;
  for (int r = 0; r < d.np; ++r) {
    wait_host(r, &HostProgress::push, base() + static_cast<unsigned long long>(it - 1), it);
    w.emplace_back(&slots[r * 2 + par].stamp, base() + static_cast<unsigned long long>(it));
  }
  stream_wait_geq(s0, w, wait_flags);
}

void Block::launch_push(long long it) {  // iteration 0 only (later pushes ride on the step kernel)
  k_push<<<1, 32, 0, s0>>>(d_xd, static_cast<int>(it & 1), base() + static_cast<unsigned long long>(it) + 1,
                           acc + (it & 1), state[cur], g.fstride, abort_flag);
  CAV_CUDA(cudaGetLastError());
  prog->push.store(base() + static_cast<unsigned long long>(it), std::memory_order_release);
}

long long Block::launch_step(int part, long long it, bool check, unsigned long long* dig, bool xfold, bool write_sc,
                              bool push, bool dry) {
  if (!dry) step_used_scratch = false;
  TmaStepArgs a{};
  a.out = state[cur ^ 1];
  a.g = g;
  a.sp = sp;
  a.bf = bf;
  a.work = counters + kCtrWork;
  a.stop = d.np == 1 ? &conv->stop : (stop_flag ? stop_flag : abort_flag);
  a.n_dev = d.np == 1 ? iter_dev : nullptr;
  a.box = cav_box{{2, 2, 2}, {n[0] + 2, n[1] + 2, n[2] + 2}};
  a.sc = sc + (it & 1);
  a.acc = acc + (it & 1);
  a.digits = dig;
  a.cx = cx;
  a.cy = cy;
  a.cz = cz;
  a.n = it;
  a.rank = d.rank;
  const int bw = n[0], bh = n[1], bd = n[2];
  a.tiles_x = (bw + 31) / 32;
  a.ntiles = a.tiles_x * ((bh + kTY - 1) / kTY);
  // z chunks: two-plane shell chunks next to joined z faces (overlap), the
  // middle in k-chunks. Long items amortise the per-item window restart (4
  // extra planes); the dynamic counter balances them and the short tail
  // chunks below trim the end (measured at 256^3: 48 best of 24..96, +0.6%
  // over 32). Small boxes get shorter chunks so that there are items for
  // every CTA (a 32^3 block has 4 tiles: 48-plane items would leave 292 CTAs idle).
  const bool split = d.np > 1 && d.overlap && !fused;
  a.zl = split ? zsh[0] : 0;
  a.zh = split ? zsh[1] : 0;
  a.mlo = a.box.lo[2] + 2 * a.zl;
  const int bm = bd - 2 * (a.zl + a.zh);  // planes in the middle chunks (>= 1: validate_grid needs 5)
  a.chunk = static_cast<int>(std::max<long long>(
      1, std::min<long long>(48, static_cast<long long>(bm) * a.ntiles / tma_grid)));
  a.chunk = std::min(a.chunk, bm);
  if (tma_chunk > 0) a.chunk = std::min(bm, tma_chunk);  // CAV_TMA_CHUNK (experiments)
  if (a.chunk > 4096) throw std::invalid_argument("block: k-chunk above 4096 planes (96-bit digit runs)");
  {  // tail: about two waves' worth of short items at the end of the order
    const int ls = std::max(4, a.chunk / 4);
    int nsmall = tail_chunks >= 0 ? tail_chunks : static_cast<int>((2LL * tma_grid + a.ntiles - 1) / a.ntiles);
    nsmall = std::min(nsmall, (bm / 2) / ls);  // keep most of the box in long items
    if (a.chunk <= ls) nsmall = 0;
    const int bigext = bm - nsmall * ls;
    a.nbig = (bigext + a.chunk - 1) / a.chunk;
    a.bigend = a.mlo + bigext;
    a.chunk_tail = ls;
    a.nchunks = a.zl + a.nbig + nsmall + a.zh;
  }
  a.part = split ? part : 0;
  a.sx0 = shell[0];
  a.sx1 = shell[1];
  a.sy0 = shell[2];
  a.sy1 = shell[3];
  a.walls = winfo;
  a.fold = d.np == 1 ? 1 : 0;
  a.done = counters + kCtrDone;
  a.sc_next = sc + ((it + 1) & 1);
  a.acc_next = acc + ((it + 1) & 1);
  a.err_sticky = err;
  a.dx = dx;
  a.dy = dy;
  a.dz = dz;
  a.cfl = d.cfl;
  a.nu = d.fluid.nu;
  a.alpha = d.fluid.alpha;
  a.rescale = d.rescale;
  // stored ghosts: the step writes its output's x-wall ghosts when the
  // three interior layers next to each x wall lie in one warp (one 32-wide
  // tile row); k_ghosts_yz writes the y and z faces after it (k_bc all faces otherwise)
  a.gw = ghosts && ghost_writes && bw >= 3 && (bw % 32 == 0 || bw % 32 >= 3) ? 1 : 0;
  const long long total = static_cast<long long>(a.ntiles) * a.nchunks;
  long long wanted = total;
  if (a.part != 0) {
    const long long internal = static_cast<long long>(a.nchunks - a.zl - a.zh) * (a.sx1 - a.sx0) * (a.sy1 - a.sy0);
    wanted = a.part == 1 ? internal : total - internal;
  }
  if (dry || wanted <= 0) return wanted;
  if (ghosts && check) {  // norm iteration: residuals to the scratch state, summed by k_norm_runs
    a.rs = rscratch;
    step_used_scratch = true;
  }
  step_wrote_ghosts = a.gw != 0;
  if (xfold) {  // many ranks: dt/pcs folded in the kernel, scalars pushed by its last CTA
    a.xd = d_xd;
    a.xfold = 1;
    a.write_sc = write_sc ? 1 : 0;
    a.fold_par = static_cast<int>((it - 1) & 1);
    a.fold_stamp = base() + static_cast<unsigned long long>(it);
    a.xpush = push ? 1 : 0;
    a.push_par = static_cast<int>(it & 1);
    a.push_stamp = base() + static_cast<unsigned long long>(it) + 1;
    a.out_par = cur ^ 1;
  }
  const int grid = static_cast<int>(std::min<long long>(tma_grid, wanted));
  tma_launch<TmaV0>(tmap[cur], a, check, ghosts, fused && xfold, bw % 32 == 0 && bh % kTY == 0, grid, s0);
  if (push) prog->push.store(base() + static_cast<unsigned long long>(it), std::memory_order_release);
  return wanted;
}

void Block::launch_ghosts() {
  if (!ghosts) return;
  // wall ghosts of the output state for the next step (no pending shift)
  if (step_wrote_ghosts) {
    if (!(walls[2] || walls[3] || walls[4] || walls[5])) return;
    const int* stp = d.np == 1 ? &conv->stop : (stop_flag ? stop_flag : abort_flag);
    static const bool pairs = getenv_int("CAV_GHOST_PAIRS", 1) != 0;
    if (pairs && n[0] % 2 == 0) {
      const dim3 grid((n[0] / 2 + kGhostThreads - 1) / kGhostThreads, (std::max(n[1], n[2]) + 1) / 2, 4);
      k_ghosts_yz2<<<grid, kGhostThreads, 0, s0>>>(state[cur ^ 1], g, winfo, stp);
    } else {
      const dim3 grid((n[0] + kGhostThreads - 1) / kGhostThreads, std::max(n[1], n[2]), 4);
      k_ghosts_yz<<<grid, kGhostThreads, 0, s0>>>(state[cur ^ 1], g, winfo, stp);
    }
    CAV_CUDA(cudaGetLastError());
  } else {
    double* fo[5] = {field(cur ^ 1, 0), field(cur ^ 1, 1), field(cur ^ 1, 2), field(cur ^ 1, 3), field(cur ^ 1, 4)};
    ops::launch_bc(fo, g, walls, d.fluid, nullptr, s0, true);
  }
}

void Block::iteration(long long it, bool check, unsigned long long* dig, IterTiming* tm) {
  const cav_box ib{{2, 2, 2}, {n[0] + 2, n[1] + 2, n[2] + 2}};
  auto mark = [&](int q, cudaStream_t st) {
    if (tm) CAV_CUDA(cudaEventRecord(tm->e[q], st));
  };
  if (d.np == 1) {  // the step kernel's last CTA folds the scalars (timing: e[2], e[3] only)
    mark(2, s0);
    launch_step(0, it, check, dig, false, false, false, false);
    mark(3, s0);
    if (step_used_scratch) launch_norm_runs(rscratch, g, ib, dig, err, it, d.rank, stop_flag, s0);
    launch_ghosts();
    cur ^= 1;
    return;
  }
  if (fused) {
    // halos travelled inside every rank's previous step (their last CTA
    // released the scalar stamps after them), so the scalar wait covers both
    mark(0, s0);
    wait_scalars(it);
    mark(1, s0);
    mark(2, s0);
    launch_step(0, it, check, dig, true, true, true, false);
    mark(3, s0);
    mark(4, s0);
    mark(5, s0);
    if (step_used_scratch) launch_norm_runs(rscratch, g, ib, dig, err, it, d.rank, stop_flag ? stop_flag : abort_flag, s0);
    launch_ghosts();
    mark(6, s0);
    cur ^= 1;
    return;
  }
  XArgs x{};
  x.state = state[cur];
  x.g = g;
  x.n = it;
  x.val = base() + static_cast<unsigned long long>(it);
  x.corrupt = d.corrupt_exchange;
  x.abort = abort_flag;
  x.stop = stop_flag ? stop_flag : abort_flag;
  long long maxs = 0;
  for (const auto& e : plan) maxs = std::max(maxs, e.scalars);
  const dim3 xgrid(static_cast<unsigned>((maxs + kXThreads * kXItems - 1) / (kXThreads * kXItems)),
                   static_cast<unsigned>(plan.size()));
  std::vector<std::pair<const unsigned long long*, unsigned long long>> fw;
  for (size_t m = 0; m < plan.size(); ++m)
    fw.emplace_back(reinterpret_cast<unsigned long long*>(arena) + m, x.val);
  // exchange_begin / exchange_finish on stream xs: the pack reads the input
  // state (complete in s0's order here) and the neighbours' slabs are free
  // (they passed our scalars of iteration it-2, so they unpacked it-2).
  const bool ov = d.overlap != 0;
  cudaStream_t xs = ov ? s1 : s0;
  if (ov) {
    CAV_CUDA(cudaEventRecord(ev_fork, s0));
    CAV_CUDA(cudaStreamWaitEvent(s1, ev_fork, 0));
  }
  auto exchange = [&] {
    if (plan.empty()) return;
    x.msg = d_pack;
    k_pack<<<xgrid, kXThreads, 0, xs>>>(x);
    CAV_CUDA(cudaGetLastError());
    prog->pack.store(x.val, std::memory_order_release);
    for (const auto& e : plan) wait_host(e.neighbor, &HostProgress::pack, x.val, it);
    stream_wait_geq(xs, fw, wait_flags);
    x.msg = d_unpack;
    k_unpack<<<xgrid, kXThreads, 0, xs>>>(x);
    CAV_CUDA(cudaGetLastError());
  };
  if (ov) exchange();  // on s1, concurrent with the internal items
  mark(0, s0);
  wait_scalars(it);  // every rank's scalars of iteration it-1
  mark(1, s0);
  if (ov) {
    CAV_CUDA(cudaEventRecord(ev_join, s1));
    // overlap (src/runner.cpp:189-194): internal items while the halos
    // travel, then the shell items once they landed. The first launch with
    // items stores the folded scalars, the last one pushes.
    const bool has1 = launch_step(1, it, check, dig, true, false, false, true) > 0;
    const bool has2 = launch_step(2, it, check, dig, true, false, false, true) > 0;
    mark(2, s0);
    if (has1) launch_step(1, it, check, dig, true, true, !has2, false);
    mark(3, s0);
    CAV_CUDA(cudaStreamWaitEvent(s0, ev_join, 0));
    mark(4, s0);
    if (has2) launch_step(2, it, check, dig, true, !has1, true, false);
    mark(5, s0);
  } else {
    exchange();
    mark(2, s0);
    launch_step(0, it, check, dig, true, true, true, false);
    mark(3, s0);
    mark(4, s0);
    mark(5, s0);
  }
  if (step_used_scratch) launch_norm_runs(rscratch, g, ib, dig, err, it, d.rank, stop_flag ? stop_flag : abort_flag, s0);
  launch_ghosts();
  mark(6, s0);
  cur ^= 1;
}

void Block::iteration_pair_graph(long long it) {
  const int key = (cur << 1) | static_cast<int>(it & 1);
  if (!gexec[key]) {  // capture once: the launches' arguments depend only on (cur, it & 1)
    cudaGraph_t gr = nullptr;
    CAV_CUDA(cudaStreamBeginCapture(s0, cudaStreamCaptureModeThreadLocal));
    try {
      iteration(it, false, nullptr, nullptr);
      iteration(it + 1, false, nullptr, nullptr);
    } catch (...) {  // leave the stream out of capture mode before reporting
      cudaStreamEndCapture(s0, &gr);
      if (gr) cudaGraphDestroy(gr);
      cudaGetLastError();
      throw;
    }
    CAV_CUDA(cudaStreamEndCapture(s0, &gr));
    const cudaError_t e = cudaGraphInstantiate(&gexec[key], gr, 0);
    cudaGraphDestroy(gr);
    CAV_CUDA(e);
    CAV_CUDA(cudaGraphLaunch(gexec[key], s0));
    return;  // the capture swapped cur twice: unchanged
  }
  CAV_CUDA(cudaGraphLaunch(gexec[key], s0));
}

void Block::update_ledger(cav_ledger& l) const {
  // exchange_begin/record_send (src/exchange.cpp:30-42, :115-145): one
  // begin_exchange per iteration, one record per plan entry
  ++l.exchanges;
  for (auto& b : l.last_face_bytes) b = 0;
  for (const auto& e : plan) {
    const uint64_t bytes = static_cast<uint64_t>(e.scalars) * sizeof(double);
    l.face_bytes[e.face] += bytes;
    l.last_face_bytes[e.face] += bytes;
    l.face_messages[e.face] += 1;
    l.bytes_sent += bytes;
    l.messages_sent += 1;
  }
}

void Block::wait_event(cudaEvent_t e) {
  const auto t0 = std::chrono::steady_clock::now();
  const double lim = d.timeout_ms > 0 ? d.timeout_ms : 20000.0;
  for (int spin = 0;; ++spin) {
    const cudaError_t r = cudaEventQuery(e);
    if (r == cudaSuccess) return;
    if (r != cudaErrorNotReady) CAV_CUDA(r);
    if (std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count() > lim) on_timeout();
    if (spin > 64) std::this_thread::sleep_for(std::chrono::microseconds(20));
    else std::this_thread::yield();
  }
}

void Block::wait_host(int r, const std::atomic<unsigned long long> HostProgress::*word, unsigned long long want,
                      long long it) {
  const HostProgress* p = host_peer[r].get();
  if (!p || r == d.rank || (p->*word).load(std::memory_order_acquire) >= want) return;
  const auto t0 = std::chrono::steady_clock::now();
  const double lim = d.timeout_ms > 0 ? d.timeout_ms : 20000.0;
  for (int spin = 0; (p->*word).load(std::memory_order_acquire) < want; ++spin) {
    if (std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count() > lim)
      on_timeout(it);
    if (spin > 64) std::this_thread::sleep_for(std::chrono::microseconds(5));
    else std::this_thread::yield();
  }
}

void Block::window_mark(long long it) {
  if (d.np == 1) return;
  const int q = static_cast<int>(it % kWindow);
  if (win_it[q] > 0) wait_event(win[q]);  // iteration it - kWindow is complete
  CAV_CUDA(cudaEventRecord(win[q], s0));
  win_it[q] = it;
}

void Block::window_drain() {
  if (d.np == 1) return;
  long long last = 0;
  int lq = -1;
  for (int q = 0; q < kWindow; ++q)
    if (win_it[q] > last) {
      last = win_it[q];
      lq = q;
    }
  if (lq >= 0) wait_event(win[lq]);
  for (auto& w : win_it) w = 0;
}

void Block::on_timeout(long long hint) {
  // the first iteration that has not completed is the stuck one
  long long stuck = 0;
  for (int q = 0; q < kWindow; ++q)
    if (win_it[q] > 0 && cudaEventQuery(win[q]) != cudaSuccess && (stuck == 0 || win_it[q] < stuck))
      stuck = win_it[q];
  cudaGetLastError();
  if (stuck == 0) stuck = hint > 0 ? hint : next_n;
  // what this rank still waits for, read from its arena on the side stream
  std::vector<unsigned long long> flags(64);
  std::vector<Slot> slots(2 * d.np);
  CAV_CUDA(cudaMemcpyAsync(flags.data(), arena, 64 * 8, cudaMemcpyDeviceToHost, saux));
  CAV_CUDA(cudaMemcpyAsync(slots.data(), arena + lay.slots, slots.size() * sizeof(Slot), cudaMemcpyDeviceToHost, saux));
  CAV_CUDA(cudaStreamSynchronize(saux));
  const unsigned long long want = base() + static_cast<unsigned long long>(stuck);
  std::string out;
  auto add = [&](int src, int tag) {
    out += (out.empty() ? "" : ", ");
    out += "(src=" + std::to_string(src) + ", tag=" + std::to_string(tag) + ")";
  };
  auto stamp_missing = [&](int r) { return slots[r * 2 + ((stuck - 1) & 1)].stamp < want; };
  for (size_t m = 0; m < plan.size(); ++m)  // fused halos arrive with the neighbour's scalars
    if (fused ? stamp_missing(plan[m].neighbor) : flags[m] < want) add(plan[m].neighbor, plan[m].recv_tag);
  for (int r = 0; r < d.np; ++r)
    if (r != d.rank && slots[r * 2 + ((stuck - 1) & 1)].stamp < want) add(r, 1001);  // kReduceTag
  // abort: later kernels return at once; release every wait so the streams drain
  const int one = 1;
  CAV_CUDA(cudaMemcpyAsync(abort_flag, &one, sizeof one, cudaMemcpyHostToDevice, saux));
  if (stop_flag) CAV_CUDA(cudaMemcpyAsync(&conv->stop, &one, sizeof one, cudaMemcpyHostToDevice, saux));
  const unsigned long long big = ~0ull >> 1;
  std::vector<unsigned long long> fl(64, big);  // plan-entry flags and the ready words
  CAV_CUDA(cudaMemcpyAsync(arena, fl.data(), fl.size() * 8, cudaMemcpyHostToDevice, saux));
  for (auto& s : slots) s.stamp = big;
  for (int r = 0; r < d.np; ++r)
    for (int p = 0; p < 2; ++p)
      CAV_CUDA(cudaMemcpyAsync(arena + lay.slots + (r * 2 + p) * sizeof(Slot) + offsetof(Slot, stamp), &big, 8,
                               cudaMemcpyHostToDevice, saux));
  CAV_CUDA(cudaStreamSynchronize(saux));
  cudaStreamSynchronize(s1);
  cudaStreamSynchronize(s0);
  cudaGetLastError();
  dead = true;
  for (auto& w : win_it) w = 0;
  throw Timeout("rank " + std::to_string(d.rank) + ": receive timed out at iteration " + std::to_string(stuck) +
                "; outstanding: " + out);
}

namespace {
const char* kVar[5] = {"p", "u", "v", "w", "T"};

std::string error_message(unsigned long long code) {
  const long long it = static_cast<long long>(code >> 24);
  const int kind = static_cast<int>(code & 15);
  if (kind == 0) return "iteration " + std::to_string(it) + ": repro_sum: non-finite term";
  return "iteration " + std::to_string(it) + ": compute_dt: non-finite value in field " + kVar[kind - 1];
}
}  // namespace

}  // namespace cav

using namespace cav;

struct cav_block {
  std::unique_ptr<Block> b;
};

extern "C" {

const char* cav_version(void) {
#ifdef CAV_FMAD
  return "cavity_b200 sm_100a fmad=true (tolerance build)";
#else
  return "cavity_b200 sm_100a fmad=false (bitwise build)";
#endif
}

int cav_block_create(const cav_block_desc* desc, cav_block** out) {
  return guarded([&] {
    auto h = std::make_unique<cav_block>();
    h->b = std::make_unique<Block>(*desc);
    *out = h.release();
  });
}

int cav_block_destroy(cav_block* b) {
  return guarded([&] { delete b; });
}

int cav_block_arena(cav_block* b, void** ptr, size_t* bytes) {
  return guarded([&] {
    *ptr = b->b->arena;
    *bytes = b->b->lay.bytes;
  });
}

int cav_block_arena_ipc(cav_block* b, unsigned char handle[64]) {
  return guarded([&] {
    CAV_CUDA(cudaSetDevice(b->b->d.device));
    cudaIpcMemHandle_t h;
    CAV_CUDA(cudaIpcGetMemHandle(&h, b->b->arena));
    static_assert(sizeof h == 64, "ipc handle size");
    std::memcpy(handle, &h, 64);
  });
}

int cav_block_connect(cav_block* bh, int r, void* ptr, const unsigned char* ipc) {
  return guarded([&] {
    Block& b = *bh->b;
    if (r < 0 || r >= b.d.np) throw std::invalid_argument("connect: rank out of range");
    if ((ptr == nullptr) == (ipc == nullptr)) throw std::invalid_argument("connect: pass exactly one of ptr/ipc");
    CAV_CUDA(cudaSetDevice(b.d.device));
    if (r == b.d.rank) return;  // own arena is always connected
    if (ptr) {
      cudaPointerAttributes at{};
      CAV_CUDA(cudaPointerGetAttributes(&at, ptr));
      if (at.device != b.d.device) {
        int ok = 0;
        CAV_CUDA(cudaDeviceCanAccessPeer(&ok, b.d.device, at.device));
        if (!ok) throw std::runtime_error("connect: no peer access from device " + std::to_string(b.d.device) +
                                          " to " + std::to_string(at.device));
        const cudaError_t e = cudaDeviceEnablePeerAccess(at.device, 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) CAV_CUDA(e);
        cudaGetLastError();
      }
      b.peer_arena[r] = static_cast<unsigned char*>(ptr);
      std::lock_guard<std::mutex> lk(g_reg_mu);
      const auto f = registry().find(ptr);
      b.host_peer[r] = f == registry().end() ? nullptr : f->second;  // same process: order the waits
    } else {
      cudaIpcMemHandle_t h;
      std::memcpy(&h, ipc, 64);
      void* p = nullptr;
      CAV_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
      b.peer_arena[r] = static_cast<unsigned char*>(p);
      b.peer_ipc[r] = true;
    }
    b.ready = false;
  });
}

int cav_block_upload(cav_block* bh, const double* host5) {
  return guarded([&] {
    Block& b = *bh->b;
    CAV_CUDA(cudaSetDevice(b.d.device));
    // one contiguous host->device copy (full PCIe rate, no 2-D row DMA), then
    // a device scatter into both padded states
    const long long S = static_cast<long long>(b.n[0] + 4) * (b.n[1] + 4) * (b.n[2] + 4);
    CAV_CUDA(cudaMemcpyAsync(b.staging, host5, 5 * S * sizeof(double), cudaMemcpyHostToDevice, b.s0));
    k_import<<<static_cast<unsigned>((5 * S + 255) / 256), 256, 0, b.s0>>>(b.staging, b.state[0], b.state[1], b.g);
    CAV_CUDA(cudaGetLastError());
    CAV_CUDA(cudaStreamSynchronize(b.s0));  // ordered with this block's non-blocking streams
    b.cur = 0;
    b.next_n = 1;
    b.primed = false;
  });
}

int cav_block_initialize(cav_block* bh) {
  return guarded([&] {
    Block& b = *bh->b;
    CAV_CUDA(cudaSetDevice(b.d.device));
    const long long S = static_cast<long long>(b.n[0] + 4) * (b.n[1] + 4) * (b.n[2] + 4);
    k_fill_ic<<<static_cast<unsigned>((5 * S + 255) / 256), 256, 0, b.s0>>>(b.state[0], b.state[1], b.g,
                                                                            b.d.fluid.t_inf);
    CAV_CUDA(cudaGetLastError());
    CAV_CUDA(cudaStreamSynchronize(b.s0));
    b.cur = 0;
    b.next_n = 1;
    b.primed = false;
  });
}

int cav_block_download(cav_block* bh, double* host5) {
  return guarded([&] {
    Block& b = *bh->b;
    CAV_CUDA(cudaSetDevice(b.d.device));
    const long long S = static_cast<long long>(b.n[0] + 4) * (b.n[1] + 4) * (b.n[2] + 4);
    if (b.primed && b.next_n > 1) {
      // wall ghosts the reference's BC stored at the last iteration: those of
      // the last input state (stored states are final, nothing is pending)
      double* fp[5] = {b.field(b.cur ^ 1, 0), b.field(b.cur ^ 1, 1), b.field(b.cur ^ 1, 2), b.field(b.cur ^ 1, 3),
                       b.field(b.cur ^ 1, 4)};
      ops::launch_bc(fp, b.g, b.walls, b.d.fluid, nullptr, b.s0);
    }
    k_export<<<static_cast<unsigned>((5 * S + 255) / 256), 256, 0, b.s0>>>(b.state[b.cur], b.state[b.cur ^ 1],
                                                                           b.g, 0.0, b.staging);
    CAV_CUDA(cudaGetLastError());
    CAV_CUDA(cudaMemcpyAsync(host5, b.staging, 5 * S * sizeof(double), cudaMemcpyDeviceToHost, b.s0));
    CAV_CUDA(cudaStreamSynchronize(b.s0));
  });
}

static double host_now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

// seeded pauses between iterations (cav_block_desc.jitter_seed): perturbs the
// relative timing of ranks; results must not depend on it
static void jitter(unsigned long long& st) {
  if (!st) return;
  st ^= st << 13;
  st ^= st >> 7;
  st ^= st << 17;
  if ((st & 3) == 0) std::this_thread::sleep_for(std::chrono::microseconds(static_cast<int>((st >> 8) % 400)));
}

int cav_block_run(cav_block* bh, cav_run_io* io) {
  return guarded([&] {
    Block& b = *bh->b;
    const bool mark = io->first_it == 1;
    if (mark) b.host_marks[0] = host_now();
    CAV_CUDA(cudaSetDevice(b.d.device));
    if (io->first_it != b.next_n)
      throw std::logic_error("block_run: iterations must continue at " + std::to_string(b.next_n));
    if (!(b.d.cfl > 0.0) || !std::isfinite(b.d.cfl))
      throw std::runtime_error("iteration " + std::to_string(io->first_it) + ": compute_dt: cfl must be positive, got " +
                               host::fmt_double_f(b.d.cfl));
    b.ensure_ready();
    if (mark) b.host_marks[1] = host_now();
    const long long first = io->first_it, last = io->first_it + io->n_its - 1;
    const int cadence = std::max(1, io->check_every);
    auto is_check = [&](long long it) { return io->want_norms && (it == 1 || it % cadence == 0); };
    long long nchk = 0;
    for (long long it = first; it <= last; ++it) nchk += is_check(it);
    if (nchk > b.digits_cap) {
      // stream-ordered (no device-wide synchronisation while peers run)
      if (b.digits) CAV_CUDA(cudaFreeAsync(b.digits, b.s0));
      CAV_CUDA(cudaMallocAsync(&b.digits, nchk * kNormWords * sizeof(unsigned long long), b.s0));
      b.digits_cap = nchk;
    }
    if (nchk) CAV_CUDA(cudaMemsetAsync(b.digits, 0, nchk * kNormWords * sizeof(unsigned long long), b.s0));
    if (!b.primed) b.prologue();
    if (mark) b.host_marks[2] = host_now();
    // device convergence (many ranks: every rank's digits merged on every
    // device after each check, see k_push_norms / k_conv_check)
    const bool dconv = io->device_conv && io->want_norms;
    io->device_conv = dconv ? 1 : 0;
    const int cur0 = b.cur;
    if (dconv) {
      ConvState c{};
      for (int v = 0; v < 5; ++v) c.peaks[v] = io->conv_peaks[v];
      CAV_CUDA(cudaMemcpyAsync(b.conv, &c, sizeof c, cudaMemcpyHostToDevice, b.s0));
      b.stop_flag = &b.conv->stop;
    }
    const double nglobal = static_cast<double>(b.gn[0]) * b.gn[1] * b.gn[2];
    bool started = false;
    if (first != 1) {
      CAV_CUDA(cudaEventRecord(b.ev_a, b.s0));
      started = true;
    }
    const cav_ledger ledger0 = io->ledger;
    unsigned long long js = b.d.jitter_seed ? b.d.jitter_seed * 0x9E3779B97F4A7C15ull + b.d.rank + 1 : 0;
    long long ci = 0;
    // one rank: the device iteration counter starts where this call starts
    if (b.d.np == 1) {
      CAV_CUDA(cudaMemcpyAsync(b.iter_dev, &first, sizeof first, cudaMemcpyHostToDevice, b.s0));
      if (!dconv) CAV_CUDA(cudaMemsetAsync(&b.conv->stop, 0, sizeof(int), b.s0));
    }
    for (long long it = first; it <= last; ++it) {
      const bool chk = is_check(it);
      // two plain iterations after the warm-up one: one graph launch
      if (b.use_graphs && it > 1 && it + 1 <= last && !chk && !is_check(it + 1)) {
        b.iteration_pair_graph(it);
        b.update_ledger(io->ledger);
        b.update_ledger(io->ledger);
        ++it;
        continue;
      }
      unsigned long long* dig = chk ? b.digits + ci * kNormWords : nullptr;
      if (chk && io->check_iters) io->check_iters[ci] = it;
      ci += chk;
      b.iteration(it, chk, dig, nullptr);
      if (dconv && chk) {
        const NormSlot* merge = nullptr;
        int par = 0;
        if (b.d.np > 1) {  // every rank's digits of this check into every rank's norm slot, then wait for all
          const long long c = b.chk_count++;
          par = static_cast<int>(c & 1);
          const unsigned long long stamp = b.base() + static_cast<unsigned long long>(c) + 1;
          k_push_norms<<<std::min(b.d.np, 8), 256, 0, b.s0>>>(dig, b.d_peer_norms, b.d.np, b.d.rank, par, stamp,
                                                               b.stop_flag);
          CAV_CUDA(cudaGetLastError());
          b.prog->norm.store(b.base() + static_cast<unsigned long long>(c), std::memory_order_release);
          merge = reinterpret_cast<const NormSlot*>(b.arena + b.lay.norms);
          std::vector<std::pair<const unsigned long long*, unsigned long long>> w;
          for (int r = 0; r < b.d.np; ++r) {
            b.wait_host(r, &HostProgress::norm, b.base() + static_cast<unsigned long long>(c), it);
            w.emplace_back(&merge[r * 2 + par].stamp, stamp);
          }
          stream_wait_geq(b.s0, w, b.wait_flags);
        }
        k_conv_check<<<1, 128, 0, b.s0>>>(dig, b.conv, it, io->conv_tol, nglobal, merge, b.d.np, par,
                                          b.base() + static_cast<unsigned long long>(b.chk_count), b.abort_flag);
        CAV_CUDA(cudaGetLastError());
      }
      if (mark && it == 1) b.host_marks[3] = host_now();
      b.update_ledger(io->ledger);
      if (it == 1) {  // iteration 1 is warm-up (src/runner.cpp:186)
        CAV_CUDA(cudaEventRecord(b.ev_a, b.s0));
        started = true;
      }
      b.window_mark(it);
      jitter(js);
    }
    CAV_CUDA(cudaEventRecord(b.ev_b, b.s0));
    if (mark) b.host_marks[4] = host_now();
    b.window_drain();
    CAV_CUDA(cudaStreamSynchronize(b.s0));
    if (mark) b.host_marks[5] = host_now();
    float ms = 0.f;
    if (started && io->n_its > 0) CAV_CUDA(cudaEventElapsedTime(&ms, b.ev_a, b.ev_b));
    io->seconds = ms * 1e-3;
    b.next_n = last + 1;
    io->n_checks = nchk;
    io->conv_iter = 0;
    if (dconv) {
      b.stop_flag = nullptr;
      ConvState c{};
      CAV_CUDA(cudaMemcpy(&c, b.conv, sizeof c, cudaMemcpyDeviceToHost));
      for (int v = 0; v < 5; ++v) io->conv_peaks[v] = c.peaks[v];
      if (c.stop) {  // iterations after c.it returned at once: rewind the host's view
        io->conv_iter = c.it;
        b.next_n = c.it + 1;
        b.cur = cur0 ^ static_cast<int>((c.it - first + 1) & 1);
        long long kept = 0;
        for (long long q = first; q <= c.it; ++q) kept += is_check(q);
        io->n_checks = nchk = kept;
        // the reference leaves its loop at the converged iteration: one
        // exchange per marched iteration, and the timed region ends there
        // (the no-op tail after it is a few microseconds per iteration)
        io->ledger = ledger0;
        for (long long q = first; q <= c.it; ++q) b.update_ledger(io->ledger);
        if (c.it == 1) io->seconds = 0.0;
      }
    }
    if (nchk && io->norm_digits)
      CAV_CUDA(cudaMemcpyAsync(io->norm_digits, b.digits, nchk * kNormWords * sizeof(unsigned long long),
                               cudaMemcpyDeviceToHost, b.s0));
    unsigned long long codes[2];
    CAV_CUDA(cudaMemcpyAsync(codes, b.err, sizeof codes, cudaMemcpyDeviceToHost, b.s0));
    CAV_CUDA(cudaStreamSynchronize(b.s0));
    io->err_iteration = 0;
    io->err_kind = 0;
    if (codes[0] != ~0ull && static_cast<long long>(codes[0] >> 24) <= last) {
      io->err_iteration = static_cast<long long>(codes[0] >> 24);
      io->err_kind = static_cast<int>(codes[0] & 15);
      throw std::runtime_error(error_message(codes[0]));
    }
  });
}

int cav_block_debug(cav_block* bh, uint64_t* out, int cap) {
  return guarded([&] {
    Block& b = *bh->b;
    CAV_CUDA(cudaSetDevice(b.d.device));
    // arena flags (64), then per slot (np x 2) its stamp, then the two error codes
    std::vector<uint64_t> v(64 + 2 * b.d.np + 2);
    CAV_CUDA(cudaMemcpyAsync(v.data(), b.arena, 64 * 8, cudaMemcpyDeviceToHost, b.saux));
    std::vector<Slot> sl(2 * b.d.np);
    CAV_CUDA(cudaMemcpyAsync(sl.data(), b.arena + b.lay.slots, sl.size() * sizeof(Slot), cudaMemcpyDeviceToHost,
                             b.saux));
    CAV_CUDA(cudaMemcpyAsync(v.data() + 64 + 2 * b.d.np, b.err, 16, cudaMemcpyDeviceToHost, b.saux));
    CAV_CUDA(cudaStreamSynchronize(b.saux));
    for (int q = 0; q < 2 * b.d.np; ++q) v[64 + q] = sl[q].stamp;
    for (size_t q = 0; q < v.size() && static_cast<int>(q) < cap; ++q) out[q] = v[q];
  });
}

int cav_block_launches_per_iteration(cav_block* bh, int check) {
  Block& b = *bh->b;
  int walls = 0;
  for (int f = 0; f < 6; ++f) walls += b.walls[f];
  const bool yz = b.walls[2] || b.walls[3] || b.walls[4] || b.walls[5];
  // step (two launches when overlapping), [ghosts after a stored-ghost step], [k_norm_runs]
  int n = (b.d.np > 1 && b.d.overlap ? 2 : 1) + (b.ghosts && (yz || !b.ghost_writes) && walls ? 1 : 0) +
          (check && b.ghosts ? 1 : 0);
  if (b.fused) n = 1 + (b.ghosts && (yz || !b.ghost_writes) && walls ? 1 : 0) + (check && b.ghosts ? 1 : 0);
  else if (b.d.np > 1) n += b.plan.empty() ? 0 : 2;  // pack, unpack (fold and push ride on the step kernel)
  return n;
}

int cav_block_scalars(cav_block* bh, double* dt, double* pc) {
  return guarded([&] {
    Block& b = *bh->b;
    CAV_CUDA(cudaSetDevice(b.d.device));
    IterScalars s{};
    CAV_CUDA(cudaMemcpyAsync(&s, b.sc + ((b.next_n - 1) & 1), sizeof s, cudaMemcpyDeviceToHost, b.s0));
    CAV_CUDA(cudaStreamSynchronize(b.s0));
    *dt = s.dt;
    *pc = s.pcs;
  });
}

int cav_block_bench(cav_block* bh, long long n_its, double out[3]) {
  return guarded([&] {
    Block& b = *bh->b;
    CAV_CUDA(cudaSetDevice(b.d.device));
    b.ensure_ready();
    if (!b.primed) b.prologue();
    while (b.timing.size() < static_cast<size_t>(n_its)) {
      Block::IterTiming t;
      for (auto& e : t.e) e = make_event();
      b.timing.push_back(t);
    }
    if (b.d.np == 1) {  // the device iteration counter and a cleared convergence stop
      const long long first = b.next_n;
      CAV_CUDA(cudaMemcpyAsync(b.iter_dev, &first, sizeof first, cudaMemcpyHostToDevice, b.s0));
      CAV_CUDA(cudaMemsetAsync(&b.conv->stop, 0, sizeof(int), b.s0));
    }
    CAV_CUDA(cudaEventRecord(b.ev_a, b.s0));
    for (long long k = 0; k < n_its; ++k) {
      b.iteration(b.next_n + k, false, nullptr, &b.timing[k]);
      b.window_mark(b.next_n + k);
    }
    CAV_CUDA(cudaEventRecord(b.ev_b, b.s0));
    b.window_drain();
    CAV_CUDA(cudaStreamSynchronize(b.s0));
    b.next_n += n_its;
    float ms = 0.f;
    CAV_CUDA(cudaEventElapsedTime(&ms, b.ev_a, b.ev_b));
    double ks = 0.0, wait = 0.0;
    for (long long k = 0; k < n_its; ++k) {
      const auto& e = b.timing[k].e;
      float t = 0.f;
      CAV_CUDA(cudaEventElapsedTime(&t, e[2], e[3]));
      ks += t;
      if (b.d.np == 1) continue;  // one launch, no peers
      CAV_CUDA(cudaEventElapsedTime(&t, e[4], e[5]));
      ks += t;
      CAV_CUDA(cudaEventElapsedTime(&t, e[0], e[1]));  // scalar wait (+ the 1-thread fold)
      wait += t;
      CAV_CUDA(cudaEventElapsedTime(&t, e[3], e[4]));  // halo join after the internal items
      wait += t;
    }
    out[0] = ms;
    out[1] = n_its ? ks / static_cast<double>(n_its) : 0.0;
    out[2] = n_its ? wait / static_cast<double>(n_its) : 0.0;
  });
}

}  // extern "C"
