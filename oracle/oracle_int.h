/*
 * TEST INFRASTRUCTURE ONLY -- private header shared by the CPU oracle's
 * translation units (reach_oracle.c: DT / MPC, ct_oracle.c: continuous-time
 * closed loop).  Never included by the product.
 */
#ifndef REACH_ORACLE_INT_H
#define REACH_ORACLE_INT_H

#include "reach_b200.h"

typedef struct { double lo, hi; } iv;

typedef struct {
  int rows, cols, act;
  const double* w; /* row-major rows x cols */
  const double* b;
} layer_t;

typedef struct {
  int n_layers;
  layer_t* layers;
} net_t;

/* Bridges into reach_oracle.c (see the static functions they wrap). */
net_t orc_i_net_from_desc(const reach_net_desc* d);
int orc_i_mat_solve(int n, int m, const double* A, const double* B, double* X);
int orc_i_certify_tm_input(const net_t* net, int n_i, int nz, const double* c, const double* A, const iv* ig,
                           double* out_c, double* out_A, iv* rem);

#endif
