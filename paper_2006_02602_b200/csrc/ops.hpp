// ops.hpp — host-side launchers shared between the op-level ABI (ops.cu) and
// the block pipeline (block.cu).
#pragma once

#include <cuda_runtime.h>

#include "device.cuh"

namespace cav::ops {

void residual_box(const cav_field_ptrs& in, const cav_residual_ptrs& out, int X, int Y,
                  const cav_box& box, const cav_stencil_params& sp, cudaStream_t st);
void update_box(double* q, const double* r, double dt, int X, int Y, const cav_box& box,
                cudaStream_t st);

// apply_boundary_conditions (src/solver.cpp:158-191) on layout g. When sc is
// non-null the interior pressure read by the cubic extrapolation gets the
// pending shift fl(p - sc->pc) (the lazy rescale).
void launch_bc(double* const fields[5], const Geo& g, const int walls[6], const cav_fluid_params& prm,
               const IterScalars* sc, cudaStream_t st, bool step_only = false);

// compute_dt's scans (src/solver.cpp:200-227) over `box` of layout g in one
// pass: CFL-denominator maxima and the non-finite mask, published into *acc
// with error iteration it_no.
void launch_dt_scan(const cav_field_ptrs& f, const Geo& g, const cav_box& box, double u_ref, Acc* acc,
                    long long it_no, int rank, cudaStream_t st);

// Forces every op-level kernel's module to load now. CUDA lazy loading would
// otherwise load a kernel at its first launch, which needs a context-wide
// synchronisation that can deadlock against a peer rank's spinning kernel on
// the same GPU.
void preload_kernels();

// dt = cfl * min(min(dx/Du, dy/Dv, dz/Dw), visc, therm) from the exact maxima
// of the CFL denominators (src/solver.cpp:215-231 with the max rewrite).
__host__ __device__ inline double dt_from_maxima(const unsigned long long dmax[3], double dx, double dy,
                                                 double dz, const cav_fluid_params& prm, double cfl) {
  double d[3];
  for (int a = 0; a < 3; ++a) {
#ifdef __CUDA_ARCH__
    d[a] = __longlong_as_double(static_cast<long long>(dmax[a]));
#else
    __builtin_memcpy(&d[a], &dmax[a], sizeof(double));
#endif
  }
  const double conv = smin(smin(dx / d[0], dy / d[1]), dz / d[2]);
  const double dmin = smin(smin(dx, dy), dz);
  const double visc = dmin * dmin / (6.0 * prm.nu);
  const double therm = dmin * dmin / (6.0 * prm.alpha);
  return cfl * smin(smin(conv, visc), therm);
}

}  // namespace cav::ops
