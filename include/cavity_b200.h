/*
 * cavity_b200.h — C ABI of the B200-native buoyancy-driven-cavity hot path.
 *
 * Everything here is plain C: pointers, sizes, ints and doubles. No torch and
 * no C++ types cross this boundary, and no exception crosses it either: every
 * entry point returns an int status (CAV_OK on success) and leaves a
 * thread-local message readable through cav_last_error(). The C++ wrapper
 * (cavity_b200.hpp) rethrows the same exception types and messages the
 * reference throws; the Python wrapper maps them to ValueError/RuntimeError.
 *
 * Reference interfaces each group replaces (paths relative to
 * /root/reference/proj):
 *   op level     include/cavity/kernels.hpp:42-46   kernels::residual_box / update_box
 *                src/solver.cpp:158-285             BC, compute_dt, euler_step,
 *                                                   rescale_pressure, norm partials
 *                src/slab.cpp:33-71                 face boxes + copy_box_to/from
 *   host logic   src/decomp.cpp:67-255              choose_dims, partition, neighbors,
 *                                                   center_node/owner_of, grow_grid
 *                src/exchange.cpp:71-113            build_plan (+ ByteLedger)
 *                src/overlap.cpp:7-31               compute_overlap_regions
 *   block level  src/runner.cpp:150-251             rank_main (one rank = one block
 *                                                   on one GPU; the iteration loop
 *                                                   body is cav_block_run)
 *   case level   include/cavity/runner.hpp:36-52    run_case / compare_fields /
 *                                                   verify_against_serial
 *
 * Device pointers passed to op-level entry points must live on the current
 * CUDA device. `stream` is a cudaStream_t (NULL = legacy default stream);
 * op-level calls are asynchronous unless stated otherwise.
 */
#ifndef CAVITY_B200_H
#define CAVITY_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Words per check iteration in cav_run_io.norm_digits: 5 x 70 carry-save
 * digit words (the exact L2 sums), then the 5 L-inf maxima
 * as bit patterns of max |R_v| (p,u,v,w,T), then padding. */
#define CAV_NORM_WORDS 360

/* ---- status codes (mirror the reference's exception taxonomy) ---------- */
enum {
  CAV_OK = 0,
  CAV_EINVAL = 1,   /* std::invalid_argument   */
  CAV_ERUNTIME = 2, /* std::runtime_error      */
  CAV_ELOGIC = 3,   /* std::logic_error        */
  CAV_ELENGTH = 4,  /* std::length_error       */
  CAV_ECUDA = 5,    /* CUDA runtime failure (no reference analogue) */
  CAV_ETIMEOUT = 6  /* transport::TransportTimeout (inc/transport.hpp:17-25) */
};

/* Thread-local message of the last failing call on this thread. */
const char* cav_last_error(void);
/* Library build identity: "cavity_b200 sm_100a <fmad mode>". */
const char* cav_version(void);

/* ---- mesh vocabulary (include/cavity/grid.hpp:8-88) --------------------- */
/* Half-open storage-coordinate box; first interior node is index 2. */
typedef struct { int lo[3]; int hi[3]; } cav_box;

/* kernels::StencilParams, same field order (include/cavity/kernels.hpp:11-21). */
typedef struct {
  double inv2dx, inv2dy, inv2dz;
  double invdx2, invdy2, invdz2;
  double invdx4, invdy4, invdz4;
  double kdx3, kdy3, kdz3;
  double u_ref;
  double nu, alpha;
  double rho, inv_rho;
  double sigma, t_inf;
  double gx, gy, gz;
} cav_stencil_params;

/* FluidParams (include/cavity/solver.hpp:18-38). */
typedef struct {
  double rho, nu, alpha, sigma;
  double gravity[3];
  double u_ref, kappa, t_hot, t_cold, t_inf, length;
} cav_fluid_params;

typedef struct { const double *p, *u, *v, *w, *t; } cav_field_ptrs;
typedef struct { double *p, *u, *v, *w, *t; } cav_residual_ptrs;

/* FluidParams::for_rayleigh (src/solver.cpp:20-25). */
void cav_fluid_for_rayleigh(double ra, cav_fluid_params* out);
int cav_validate_params(const cav_fluid_params* p);
/* make_cavity_grid spacing + validate_grid (src/grid.cpp:17-47). */
int cav_make_cavity_grid(int nx, int ny, int nz, double lx, double ly, double lz,
                         double spacing_out[3]);
/* make_stencil_params (src/solver.cpp:77-103), computed on the host. */
void cav_make_stencil_params(double dx, double dy, double dz, const cav_fluid_params* prm,
                             cav_stencil_params* out);

/* ---- op level: the kernels:: backend seam, Cuda backend ----------------- */
/* Field3 layout: idx = i + X*(j + Y*k), X = nx+4, Y = ny+4, on the device. */

/* kernels::residual_box (include/cavity/kernels.hpp:42-43). */
int cav_residual_box(const cav_field_ptrs* in, const cav_residual_ptrs* out, int X, int Y,
                     const cav_box* box, const cav_stencil_params* sp, void* stream);
/* kernels::update_box (include/cavity/kernels.hpp:46): q += dt*r over box. */
int cav_update_box(double* q, const double* r, double dt, int X, int Y, const cav_box* box,
                   void* stream);
/* apply_boundary_conditions (src/solver.cpp:158-191) on a block with
 * interior nx,ny,nz; walls[f] != 0 marks face id f (2*axis+side) a wall. */
int cav_apply_boundary_conditions(const cav_residual_ptrs* fields, int nx, int ny, int nz,
                                  const int walls[6], const cav_fluid_params* prm, void* stream);
/* compute_dt (src/solver.cpp:193-232). Synchronous. Returns CAV_EINVAL for a
 * bad cfl and CAV_ERUNTIME naming the first non-finite field, exactly as the
 * reference's messages. */
int cav_compute_dt(const cav_field_ptrs* f, int nx, int ny, int nz, double dx, double dy,
                   double dz, const cav_fluid_params* prm, double cfl, double* dt_out,
                   void* stream);
/* rescale_pressure (src/solver.cpp:248-257). */
int cav_rescale_pressure(double* p, int nx, int ny, int nz, double p_center, void* stream);
/* residual_norm_partials (src/solver.cpp:259-274): exact sums of fl(r*r)
 * over the interior, returned as ReproSum limbs (inc/util/repro_sum.hpp:79-88
 * serialisation: 35 positive then 35 negative u64 limbs) per variable,
 * out = 5*70 u64. Synchronous. CAV_EINVAL "repro_sum: non-finite term". */
int cav_residual_norm_partials(const cav_field_ptrs* r, int nx, int ny, int nz,
                               uint64_t* limbs_out, void* stream);
/* ReproSum::value (inc/util/repro_sum.hpp:48-77) of serialised limbs. */
double cav_repro_value(const uint64_t* limbs70);
/* ReproSum::merge of b into a (both serialised, 70 words). */
void cav_repro_merge(uint64_t* a70, const uint64_t* b70);

/* face_interior_box / face_ghost_box (src/slab.cpp:33-49). face = 2*axis+side. */
int cav_face_interior_box(int nx, int ny, int nz, int face, int depth, cav_box* out);
int cav_face_ghost_box(int nx, int ny, int nz, int face, int depth, cav_box* out);
/* copy_box_to / copy_box_from (src/slab.cpp:51-71) on device data. */
int cav_copy_box_to(const double* f, int X, int Y, const cav_box* box, double* out, void* stream);
int cav_copy_box_from(double* f, int X, int Y, const cav_box* box, const double* in, void* stream);

/* ---- host logic (C++ inside the library, no GPU needed) ----------------- */
enum { CAV_MODE_1D_I = 0, CAV_MODE_1D_J = 1, CAV_MODE_1D_K = 2, CAV_MODE_2D = 3, CAV_MODE_3D = 4 };
enum { CAV_BASELINE = 0, CAV_V1 = 1, CAV_V2 = 2, CAV_V3 = 3 };
enum { CAV_WALL = -1 };

/* choose_dims (src/decomp.cpp:67-98). */
int cav_choose_dims(int np, int mode, int dims_out[3]);
/* partition (src/decomp.cpp:100-150): extents_out[r*6 + {lo0,lo1,lo2,hi0,hi1,hi2}]. */
int cav_partition(int nx, int ny, int nz, const int dims[3], int* extents_out);
/* neighbors (src/decomp.cpp:161-175): rank_at[6], CAV_WALL for walls. */
int cav_neighbors(const int dims[3], int rank, int rank_at[6]);
/* BlockMap::center_node + owner_of (src/decomp.cpp:193-205). */
int cav_center_owner(int nx, int ny, int nz, const int dims[3], int node_out[3], int* owner_out);
/* grow_grid (src/decomp.cpp:227-255). */
int cav_grow_grid(int nx, int ny, int nz, int np, int mode, int growth_type, int out[3]);

/* One message of build_plan (include/cavity/exchange.hpp:26-38). */
typedef struct {
  int face;         /* our face id; neighbour receives on the opposite one */
  int neighbor;
  int nvars;        /* 1 (per-variable message) or 5 (packed) */
  int var[5];       /* packing order within the payload */
  int depth[5];
  long long scalars;  /* payload length in doubles */
  int send_tag, recv_tag;
} cav_plan_entry;
/* build_plan (src/exchange.cpp:71-113). entries_out may be NULL to query
 * the count; capacity 30 always suffices. */
int cav_build_plan(int nx, int ny, int nz, const int rank_at[6], int strategy,
                   cav_plan_entry* entries_out, int capacity, int* count_out);
/* compute_overlap_regions (src/overlap.cpp:7-31): internal box + up to 6
 * external shells in face-id order. */
int cav_overlap_regions(int nx, int ny, int nz, const int rank_at[6], cav_box* internal_out,
                        cav_box external_out[6], int* n_external_out);

/* ---- run level: RunConfig / CaseOptions / CaseResult --------------------- */
/* RunConfig (include/cavity/util/config.hpp:15-34) + SolverConfig. */
typedef struct {
  int nx, ny, nz;
  int np;
  int mode;
  int dims[3];          /* {0,0,0} = choose_dims */
  int strategy;
  int overlap;
  long long steps;      /* >= 0 fixed; -1 run to convergence */
  cav_fluid_params fluid;
  double cfl;
  long long max_steps;
  double conv_tol;
  int rescale;
  int check_every;
  uint64_t seed;        /* != 0: randomized rank timing (the InprocBus shuffle,
                           src/inproc.cpp:92-114): rank threads start in a seeded
                           order and each enqueues its iterations with seeded
                           random pauses; results must not change */
  double timeout_ms;
  int monitor_every;
  double verify_tol;
  /* B200 extensions (no reference analogue) */
  int devices[8];       /* device of rank r is devices[r % 8]; default all 0 */
} cav_run_config;

/* RunConfig defaults (Ra = 1e5, v3, 32^3, converge). */
void cav_run_config_default(cav_run_config* out);

typedef struct {
  int collect_fields;
  int collect_history;
  int corrupt_exchange;
} cav_case_options;

/* ByteLedger (include/cavity/exchange.hpp:56-67), flattened. */
typedef struct {
  uint64_t face_bytes[6];
  uint64_t face_messages[6];
  uint64_t last_face_bytes[6];
  uint64_t bytes_sent;
  uint64_t messages_sent;
  uint64_t exchanges;
} cav_ledger;

/* CaseResult (include/cavity/runner.hpp:20-29). Buffers are caller-owned:
 * fields (5 * nx*ny*nz doubles, p,u,v,w,T each i-fastest over the global
 * interior) may be NULL; history arrays hold hist_capacity samples;
 * ledgers holds ledger_capacity ranks. */
typedef struct {
  long long steps_marched;
  long long steps_timed;
  int converged;
  int np;
  int dims[3];
  double wall_time_s;   /* timed iterations 2..N, max over ranks */
  double ssspnt;        /* metrics::ssspnt, NaN when nothing was timed */
  uint64_t bytes_sent;
  double* fields;
  long long hist_capacity;
  long long hist_count;
  long long* hist_iter;
  double* hist_l2;      /* 5 per sample */
  int ledger_capacity;
  cav_ledger* ledgers;
  double* hist_linf;    /* 5 per sample (max |R_v| over the global interior), or NULL */
} cav_case_result;

/* run_case (src/runner.cpp:259-338): one host thread per rank, one block per
 * rank on cfg->devices[rank % 8]; bitwise-equal to the reference. */
int cav_run_case(const cav_run_config* cfg, const cav_case_options* opt, cav_case_result* out);

/* ---- block level: one rank's device-resident state ---------------------- */
typedef struct cav_block cav_block;

/* Everything rank_main derives before its loop (src/runner.cpp:150-182):
 * the block's extent, neighbours, plan, overlap regions and centre owner are
 * computed from the global grid, the block dims and the rank, exactly as
 * make_block_map/partition/neighbors do. Local grids keep the global spacing
 * (src/runner.cpp:19-25). */
typedef struct {
  int rank, np;
  int gnx, gny, gnz;        /* global interior */
  int dims[3];              /* block counts (choose_dims or explicit) */
  int strategy, overlap;
  cav_fluid_params fluid;
  double cfl;
  int rescale;
  int corrupt_exchange;     /* ExchangePlan.corrupt_first hook */
  int device;
  double timeout_ms;        /* limit on waiting for a peer (TransportTimeout) */
  uint64_t jitter_seed;     /* != 0: seeded random host pauses between iterations (tests) */
} cav_block_desc;

int cav_block_create(const cav_block_desc* desc, cav_block** out);
int cav_block_destroy(cav_block* b);
/* This block's device memory as peers see it: ONE allocation holding the
 * exchange arena (flags, scalar and norm slots, receive slabs) followed by the
 * two states the neighbours' step kernels store halos into (fused halos).
 * Raw device pointer for in-process peers, CUDA IPC handle (64 bytes) for
 * peers in other processes; bytes_out is the arena part. */
int cav_block_arena(cav_block* b, void** dev_ptr_out, size_t* bytes_out);
int cav_block_arena_ipc(cav_block* b, unsigned char handle_out[64]);
/* Connect rank r's arena: exactly one of dev_ptr / ipc_handle is non-NULL. */
int cav_block_connect(cav_block* b, int peer_rank, void* dev_ptr, const unsigned char* ipc_handle);
/* Host <-> device, whole storage in the reference Field3 layout, 5 fields
 * p,u,v,w,T, each (nx+4)(ny+4)(nz+4) doubles. download applies the pending
 * centre-pressure shift so it returns exactly the reference's storage. */
int cav_block_upload(cav_block* b, const double* host5);
int cav_block_download(cav_block* b, double* host5);
/* Sets the quiescent initial condition (initialize_fields, src/solver.cpp:292). */
int cav_block_initialize(cav_block* b);

/* Per-run outputs of cav_block_run. norm_digits: per check iteration,
 * CAV_NORM_WORDS u64 words (5*70 carry-save digits of the exact L2 sums, see
 * DESIGN.md "exact norms", then 5 L-inf bit patterns), this rank's partial. */
typedef struct {
  long long first_it;       /* iteration number of the first step (1-based) */
  long long n_its;
  int check_every;
  int want_norms;
  uint64_t* norm_digits;    /* n_checks * CAV_NORM_WORDS, or NULL */
  long long* check_iters;   /* n_checks, or NULL */
  long long n_checks;       /* out */
  long long err_iteration;  /* out: 0 = no error */
  int err_kind;             /* out: 0 repro_sum non-finite, 1..5 compute_dt field p,u,v,w,T */
  double seconds;           /* out: device time of iterations first_it+1.. (iteration 1 excluded when first_it==1) */
  cav_ledger ledger;        /* in/out: accumulated */
  /* Device-side convergence: with device_conv and want_norms, the run stops
   * on the device after the first check iteration where
   * max_v |R_v| / peak_v <= conv_tol (the rule of src/runner.cpp:210-220);
   * no iteration after it is marched. With several ranks every rank pushes
   * its exact digits to every rank after each check and all decide on the
   * merged sums, so every rank must pass the same device_conv, check_every
   * and iteration range. */
  int device_conv;          /* in: request; out: 1 if this block honoured it (else all n_its were marched) */
  double conv_tol;          /* in */
  double conv_peaks[5];     /* in/out: per-variable peak norms carried across calls */
  long long conv_iter;      /* out: the converged iteration, 0 = not converged */
} cav_run_io;

/* Marches n_its iterations of rank_main's loop body (src/runner.cpp:184-235)
 * on the device: BC, exchange (plan per strategy; the step kernel stores the
 * halos into the neighbours' states, or the slab exchange with optional
 * overlap), fused residual + [norms] + dt + Euler update + centre-pressure
 * rescale. One-rank runs replay pairs of plain iterations as CUDA graphs.
 * Synchronous. */
int cav_block_run(cav_block* b, cav_run_io* io);
/* Number of launches of this library's kernels per iteration (bench claim). */
int cav_block_launches_per_iteration(cav_block* b, int check_iteration);
/* Diagnostics: arena flags (64), scalar slots (np*2*8 words), error codes
 * (2) and pack counters (64), as u64 words. */
int cav_block_debug(cav_block* b, uint64_t* out, int cap);
/* Last dt used and the current centre pressure shift (diagnostics). */
int cav_block_scalars(cav_block* b, double* dt_out, double* pc_out);

/* Bench hook: time n_its iterations with CUDA events on the block's compute
 * stream. out[0] total ms; out[1] fused-step kernel ms per iteration (both
 * launches when the slab exchange overlaps); out[2] ms per iteration the
 * compute stream spent waiting for peers (their scalars, and with the slab
 * exchange the halo join): the exposed communication. */
int cav_block_bench(cav_block* b, long long n_its, double out[3]);

#ifdef __cplusplus
}
#endif
#endif /* CAVITY_B200_H */
