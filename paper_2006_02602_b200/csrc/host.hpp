// host.hpp — host-side C++ mirror of the reference's driver vocabulary:
// decomposition, exchange plan, overlap regions, parameter validation and the
// exact-sum finalisation. Fresh code; semantics (and exception messages)
// follow the reference lines cited at each declaration.
#pragma once

#include <array>
#include <cstdint>
#include <string>
#include <vector>

#include "cavity_b200.h"
#include "cell.cuh"

namespace cav::host {

struct Extent {
  std::array<int, 3> lo{}, hi{};
  int size(int a) const { return hi[a] - lo[a]; }
};

// validate_grid (src/grid.cpp:17-32).
void validate_grid(int nx, int ny, int nz, double dx, double dy, double dz);
// make_cavity_grid spacing (src/grid.cpp:34-47).
std::array<double, 3> cavity_spacing(int nx, int ny, int nz, double lx, double ly, double lz);
// validate_params (src/solver.cpp:27-51).
void validate_params(const cav_fluid_params& p);
// FluidParams::for_rayleigh (src/solver.cpp:20-25).
cav_fluid_params for_rayleigh(double ra);
// make_stencil_params (src/solver.cpp:77-103).
cav_stencil_params stencil_params(double dx, double dy, double dz, const cav_fluid_params& p);
// Largest double s with sqrt(s) < u_ref (correctly rounded), so that
// max(sqrt(s'), u_ref) == u_ref for every s' <= s; -1 when u_ref is not a
// positive finite number (the device then always takes the full sqrt).
double beta_fast_s2(double u_ref);
// BetaFast shortcuts for u_ref: {beta_fast_s2, high word of u_ref/2} (cell.cuh).
BetaFast beta_fast(double u_ref);

// choose_dims (src/decomp.cpp:67-98).
std::array<int, 3> choose_dims(int np, int mode);
// make_decomp_spec (src/decomp.cpp:177-191).
std::array<int, 3> decomp_dims(int np, int mode, const int dims_override[3]);
// partition (src/decomp.cpp:100-150), rank-ordered.
std::vector<Extent> partition(std::array<int, 3> n, std::array<int, 3> dims);
// neighbors (src/decomp.cpp:161-175).
std::array<int, 6> neighbors(std::array<int, 3> dims, int rank);
// center_node / owner_of (src/decomp.cpp:193-205).
std::array<int, 3> center_node(std::array<int, 3> n);
int owner_of(const std::vector<Extent>& ext, std::array<int, 3> node);
// grow_grid (src/decomp.cpp:227-255).
std::array<int, 3> grow_grid(std::array<int, 3> base, int np, int mode, int type);

// build_plan (src/exchange.cpp:71-113).
std::vector<cav_plan_entry> build_plan(std::array<int, 3> n, const std::array<int, 6>& rank_at,
                                       int strategy);
// face_interior_box / face_ghost_box (src/slab.cpp:33-49).
cav_box face_box(std::array<int, 3> n, int face, int depth, bool ghost);
long long box_volume(const cav_box& b);
// compute_overlap_regions (src/overlap.cpp:7-31).
void overlap_regions(std::array<int, 3> n, const std::array<int, 6>& rank_at, cav_box* internal,
                     std::vector<cav_box>& external);

// Exact sums: 70 carry-save radix-2^32 digits (u64 words) -> ReproSum's 35
// positive limbs (inc/util/repro_sum.hpp:16-22); merge; value (:48-77).
void digits_to_limbs(const uint64_t* digits70, uint64_t* limbs70);
void repro_merge(uint64_t* a70, const uint64_t* b70);
double repro_value(const uint64_t* limbs70);

std::string fmt_double_f(double v);  // std::to_string(double) format

}  // namespace cav::host
