// common.cuh -- shared definitions of the B200 block-MINRES hot path.
//
// Paper: Soodhalter, arXiv:1301.2102.  "P:L" = PAPER.md line L.
// Block form of one block step k (iterations j = (k-1)p+1 .. kp; DESIGN.md
// "Block form"):  A U_k = U_{k-1} C_{k-1}^T + U_k G_s + U_{k+1} C_k, i.e. the
// paper's banded recurrence (eqn.block-Lanczos-recurr) with the
// operator applied to p vectors every p iterations and the known
// coefficients reused by symmetry.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace bmr {

constexpr int MAXP = 32;      // largest compiled block size
constexpr int MAXQ = 8;       // largest replacement pool
constexpr int NB_MAX = 1024;  // largest grid of the reducing kernels

// Panel-row mapping of a warp: a row of p doubles is split over LANES lanes,
// VEC contiguous doubles (16 B when VEC = 2) each; RPW rows per warp.
template <int P>
struct PC {
    static constexpr int VEC = (P % 2 == 0) ? 2 : 1;
    static constexpr int LANES = P / VEC;
    static constexpr int LP = LANES <= 1 ? 1 : LANES <= 2 ? 2 : LANES <= 4 ? 4 : LANES <= 8 ? 8 : LANES <= 16 ? 16 : 32;
    static constexpr int RPW = 32 / LP;
};

// Mapped (pinned, host-visible) flags the small-QR kernel publishes each block step.
struct HostFlags {
    volatile int run;
    volatile int status;
    volatile int need_slow;
    volatile int pad;
    volatile long long k;
    volatile long long j_done;
};

// Device-resident solver state (one per handle).  Small dense p x p matrices
// are row-major [a*MAXP + b] with leading dimension MAXP.
struct DevState {
    // control
    int run;           // 1: block steps proceed; 0: every kernel of a step is a no-op
    int k4_pending;    // the small QR ended the solve; the update kernel still applies this step
    int need_slow;     // breakdown or Cholesky cancellation: host runs the column path
    int slow_given;    // host provided C_k and wrote U_{k+1} (normalised) into W
    int status;        // BMINRES_* code (1 = MAXIT while running)
    int q_first;       // first live pool vector
    int q_live;        // number of live pool vectors
    int pool_cap;      // pool panel row stride
    int stop_after;    // >0: the small QR stops after block column stop_after-1 (pool exhausted)
    int pad0;
    long long k;       // current block index (1-based)
    long long j_done;  // completed iterations
    long long maxit;
    long long hist_cap;
    double tol, tau;
    unsigned int cnt1, cnt2, cnt3, cnt4;   // last-CTA tickets
    // reductions (written by the last CTA of K1 / K2)
    double G[MAXP * MAXP];       // G(a,m) = u_{(k-1)p+a}^T w_m   (K1, after the known subtraction)
    double om2[MAXP];            // ||A u_j||^2, raw candidate norms (C14)
    double Gram2[MAXP * MAXP];   // W'^T W'
    double pdot[MAXQ * MAXP];    // pdot(q,m) = r_q^T w'_m
    // small dense state
    double Cprev[MAXP * MAXP];   // C_{k-1}: W'_{k-1} = U_k C_{k-1}, upper triangular
    double Ck[MAXP * MAXP];      // C_k (from Cholesky, or from the host column path)
    double Cinv[MAXP * MAXP];    // C_k^{-1}
    double coef[MAXP * MAXQ];    // coef(a,q) = u_{kp+a}^T r_q
    double T[MAXP * MAXP];       // tail of \bar Z (rows j..j+p-1), T(r,c)
    double Z[MAXP * MAXP];       // Z_k: row m = z_{(k-1)p+m+1}^T (rows past the stop are 0)
    double Ainv[MAXP * MAXP];    // R_kk^{-1}
    double B1[MAXP * MAXP];      // R_{k-1,k} R_kk^{-1}
    double B2[MAXP * MAXP];      // R_{k-2,k} R_kk^{-1}
    double rv[(2 * MAXP + 1) * (MAXP + 1)];   // Householder ring, slot = i mod (2p+1)
    double rtau[2 * MAXP + 1];
    double beta[MAXP];           // ||b_i||
    double res[MAXP];            // latest computed relative residuals
    double* hist;                // (hist_cap) x p computed relative residuals, or null
    HostFlags* hflags;           // device alias of the mapped host flags
};

}  // namespace bmr
