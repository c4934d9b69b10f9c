// Batched damped Newton for the nonlinear (Brauer iron) model -- see
// newton_host.inc for the control flow (problems.py:201-244).
#pragma once
#include "common.cuh"

struct NewtonWork {
    double* u;        // current Newton iterate      [B][n]
    double* delta;    // Newton step                 [B][n]
    double* rhs;      // c M u_prev + f              [B][n]
    double* res;      // F(u)                        [B][n]
    double* ucur;     // trial iterate               [B][n]
    double* dinv;     // Jacobi of J(u)              [B][n]
    double* scale;    // max(|rhs|, 1e-300)          [B]
    double* rnorm;    // |F(u)|                      [B]
    double* tnorm;    // |F(trial)|                  [B]
    double* alpha;    // damping factor              [B]
    int* state;       // per-column Newton state     [B]
    int* nit;         // Newton iterations           [B]
    int* halv;        // halvings done               [B]
    double* zero;     // [B] zeros (inv_dt stand-in) 
};
