/* cavity_oracle.h — TEST INFRASTRUCTURE ONLY: plain-C restatement of the
 * reference hot path (see cavity_oracle.c for the file:line each function
 * follows). Host pointers, Field3 layout idx = i + X*(j + Y*k). */
#ifndef CAVITY_ORACLE_H
#define CAVITY_ORACLE_H
#include <stdint.h>

#include "../include/cavity_b200.h"

const char* oc_last_error(void);
void oc_run_config_default(cav_run_config* c);
void oc_make_stencil_params(double dx, double dy, double dz, const cav_fluid_params* prm,
                            cav_stencil_params* sp);
void oc_residual_box(const cav_field_ptrs* in, const cav_residual_ptrs* out, int X, int Y,
                     const cav_box* box, const cav_stencil_params* sp);
void oc_update_box(double* q, const double* r, double dt, int X, int Y, const cav_box* box);
void oc_apply_bc(const cav_residual_ptrs* f, int nx, int ny, int nz, const int walls[6],
                 const cav_fluid_params* prm);
int oc_compute_dt(const cav_field_ptrs* f, int nx, int ny, int nz, double dx, double dy,
                  double dz, const cav_fluid_params* prm, double cfl, double* dt_out);
void oc_rescale(double* p, int nx, int ny, int nz, double pc);
int oc_norm_partials(const cav_field_ptrs* r, int nx, int ny, int nz, uint64_t* limbs350);
double oc_repro_value(const uint64_t* limbs70);
int oc_face_box(int nx, int ny, int nz, int face, int depth, int ghost, cav_box* out);
void oc_copy_box_to(const double* f, int X, int Y, const cav_box* b, double* out);
void oc_copy_box_from(double* f, int X, int Y, const cav_box* b, const double* in);
int oc_run_serial(const cav_run_config* cfg, const cav_case_options* opt, cav_case_result* out);

#endif
