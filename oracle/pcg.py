"""Batched Jacobi-preconditioned CG (oracle) -- TEST INFRASTRUCTURE ONLY.

BASELINE config 5 names "Jacobi-PCG to 1e-10" for the isolated batched-Phi
microbenchmark.  The reference has no iterative solver (its Phi is the
banded direct solve, /root/reference/pkg/src/pintmg/problems.py:130-146), so
this restates the textbook algorithm with the product's conventions
(paper_1912_03106_b200/csrc/pcg_dia.cuh, k_dia_setup / k_sdir / k_supd):
x0 = u_prev, b = (1/dt) M u_prev + f, r0 = b - A x0, z = D^-1 r, stop a
column when its recursively updated ||r||^2 <= rtol^2 ||b||^2.  Parity for
config 5 is anchored on the direct solve of the same operator (the iterate
must be as accurate as this oracle's); this module gives the CPU the same
algorithm to compare iteration counts and accuracy with.
"""

import numpy as np


def jacobi_pcg(A, rhs, x0, rtol, max_iters=20000):
    """Solve A x = rhs for every row of rhs ([B][n]); returns (x, iterations
    per column).  A: scipy CSR, symmetric positive definite."""
    X = np.array(x0, dtype=np.float64, copy=True)
    Bv = np.asarray(rhs, dtype=np.float64)
    dinv = 1.0 / A.diagonal()
    R = Bv - (A @ X.T).T
    bb = np.einsum("ij,ij->i", Bv, Bv)
    tol2 = rtol * rtol * bb
    rr = np.einsum("ij,ij->i", R, R)
    active = ~((rr <= tol2) | (rr == 0.0))
    Z = R * dinv
    P = Z.copy()
    rz = np.einsum("ij,ij->i", R, Z)
    its = np.zeros(X.shape[0], dtype=np.int64)
    for _ in range(max_iters):
        idx = np.nonzero(active)[0]
        if idx.size == 0:
            break
        Pa = P[idx]
        Q = (A @ Pa.T).T
        alpha = rz[idx] / np.einsum("ij,ij->i", Pa, Q)
        X[idx] += alpha[:, None] * Pa
        R[idx] -= alpha[:, None] * Q
        its[idx] += 1
        rr_a = np.einsum("ij,ij->i", R[idx], R[idx])
        Za = R[idx] * dinv
        rz_new = np.einsum("ij,ij->i", R[idx], Za)
        beta = rz_new / rz[idx]
        P[idx] = Za + beta[:, None] * Pa
        rz[idx] = rz_new
        done = (rr_a <= tol2[idx]) | (rr_a == 0.0)
        active[idx[done]] = False
    return X, its
