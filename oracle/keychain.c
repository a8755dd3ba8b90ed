/*
 * oracle/keychain.c -- TEST INFRASTRUCTURE ONLY (never linked into the
 * product; only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline
 * leg load it).
 *
 * CPU restatement of the FP64 "key chain" of sarsplat.geometry.project_all
 * (/root/reference/pkg/src/sarsplat/geometry.py:233-305) and the footprint
 * test of forward._footprint_pairs (forward.py:60-109): every quantity that
 * decides which (cell, Gaussian) pairs exist and in which depth order.
 *
 * Op order = the reference's, as measured on its host:
 *   x_r   = fma(p2,R2,fma(p1,R1,p0*R0)) + T      OpenBLAS dgemm, geometry.py:249
 *   Sigma = M M^T, same FMA chain, M = R(q) diag(e^s)  scene.py:92-97
 *   Sigma2 = sum_{b,c} (m[a,b]*Sigma[b,c])*m[d,c], sequential, no FMA
 *                                                 np.einsum, geometry.py:271-272
 *   q = a00*dx^2 + (2*a01)*dx*dy + a11*dy^2       forward.py:101-105
 * Compiled with -ffp-contract=off; fma() is the correctly rounded libm fma.
 * exp() of the log-scales is either libm-free `sdgr_exp` (bit-identical to
 * the device's, paper_2506_21633_b200/csrc/common.cuh) or caller-supplied
 * scales (numpy's exp, to reproduce the reference bit-for-bit on its host).
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

double oracle_exp(double x) {
  if (x != x) return x;
  if (x > 709.782712893384) return INFINITY;
  if (x < -745.1332191019412) return 0.0;
  const double kInvLn2 = 1.4426950408889634;
  const double kLn2Hi = 6.93147180369123816490e-01;
  const double kLn2Lo = 1.90821492927058770002e-10;
  double n = nearbyint(x * kInvLn2);
  double r = fma(-n, kLn2Hi, x);
  r = fma(-n, kLn2Lo, r);
  double p = 1.0 / 6227020800.0;
  p = fma(p, r, 1.0 / 479001600.0);
  p = fma(p, r, 1.0 / 39916800.0);
  p = fma(p, r, 1.0 / 3628800.0);
  p = fma(p, r, 1.0 / 362880.0);
  p = fma(p, r, 1.0 / 40320.0);
  p = fma(p, r, 1.0 / 5040.0);
  p = fma(p, r, 1.0 / 720.0);
  p = fma(p, r, 1.0 / 120.0);
  p = fma(p, r, 1.0 / 24.0);
  p = fma(p, r, 1.0 / 6.0);
  p = fma(p, r, 0.5);
  double r2 = r * r;
  double t = fma(r2, p, r);
  double e = 1.0 + t;
  return scalbn(e, (int)n);
}

/* View constants, same layout as sdgr_view's FP64 prefix. */
typedef struct {
  double R[9], T[3], mc[6], mi[6];
  double den_u, den_v, off_vi, cov_reg, cutoff;
  int32_t n_u, n_v, n_az, n_rg;
} oracle_view;

/*
 * Per Gaussian: out_uv (n,4) = uc, vc, ui, vi; out_depth (n); out_cc (n,3),
 * out_ci (n,3) regularised plane covariances (c00, c01, c11); out_flags (n):
 * bit0 ok (finite, det>0), bit1 inside (comp-plane 3-sigma cull).
 * scales: NULL -> oracle_exp(log_scales), else caller's e^s (n,3).
 */
void oracle_keychain(int64_t n, const double* pos, const double* rot, const double* logs,
                     const double* scales, const oracle_view* v, double* out_uv,
                     double* out_depth, double* out_cc, double* out_ci, uint8_t* out_flags) {
  for (int64_t g = 0; g < n; ++g) {
    const double p0 = pos[3 * g], p1 = pos[3 * g + 1], p2 = pos[3 * g + 2];
    double xr[3];
    for (int i = 0; i < 3; ++i)
      xr[i] = fma(p2, v->R[3 * i + 2], fma(p1, v->R[3 * i + 1], p0 * v->R[3 * i])) + v->T[i];
    const double undc = (2.0 * xr[0]) / v->den_u;
    const double vcndc = (2.0 * xr[1]) / v->den_v;
    const double vindc = (2.0 * xr[2]) / v->den_v - v->off_vi;
    out_uv[4 * g + 0] = ((undc + 1.0) * 0.5) * (double)v->n_u - 0.5;
    out_uv[4 * g + 1] = ((vcndc + 1.0) * 0.5) * (double)v->n_v - 0.5;
    out_uv[4 * g + 2] = ((undc + 1.0) * 0.5) * (double)v->n_az - 0.5;
    out_uv[4 * g + 3] = ((vindc + 1.0) * 0.5) * (double)v->n_rg - 0.5;
    out_depth[g] = xr[2];

    const double* q = rot + 4 * g;
    const double nrm = sqrt(((q[0] * q[0] + q[1] * q[1]) + q[2] * q[2]) + q[3] * q[3]);
    const double w = q[0] / nrm, x = q[1] / nrm, y = q[2] / nrm, z = q[3] / nrm;
    double Rq[9];
    Rq[0] = 1.0 - 2.0 * (y * y + z * z);
    Rq[1] = 2.0 * (x * y - w * z);
    Rq[2] = 2.0 * (x * z + w * y);
    Rq[3] = 2.0 * (x * y + w * z);
    Rq[4] = 1.0 - 2.0 * (x * x + z * z);
    Rq[5] = 2.0 * (y * z - w * x);
    Rq[6] = 2.0 * (x * z - w * y);
    Rq[7] = 2.0 * (y * z + w * x);
    Rq[8] = 1.0 - 2.0 * (x * x + y * y);
    double s[3];
    for (int j = 0; j < 3; ++j) s[j] = scales ? scales[3 * g + j] : oracle_exp(logs[3 * g + j]);
    double M[9], Cv[9];
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) M[3 * i + j] = Rq[3 * i + j] * s[j];
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j)
        Cv[3 * i + j] = fma(M[3 * i + 2], M[3 * j + 2], fma(M[3 * i + 1], M[3 * j + 1], M[3 * i] * M[3 * j]));
    double cc[4], ci[4];
    for (int a = 0; a < 2; ++a)
      for (int d = 0; d < 2; ++d) {
        double sc = 0.0, si = 0.0;
        int first = 1;
        for (int b = 0; b < 3; ++b)
          for (int c = 0; c < 3; ++c) {
            const double tc = (v->mc[3 * a + b] * Cv[3 * b + c]) * v->mc[3 * d + c];
            const double ti = (v->mi[3 * a + b] * Cv[3 * b + c]) * v->mi[3 * d + c];
            sc = first ? tc : sc + tc;
            si = first ? ti : si + ti;
            first = 0;
          }
        cc[2 * a + d] = sc;
        ci[2 * a + d] = si;
      }
    const double c00 = cc[0] + v->cov_reg, c11 = cc[3] + v->cov_reg, c01 = 0.5 * (cc[1] + cc[2]);
    const double i00 = ci[0] + v->cov_reg, i11 = ci[3] + v->cov_reg, i01 = 0.5 * (ci[1] + ci[2]);
    out_cc[3 * g] = c00; out_cc[3 * g + 1] = c01; out_cc[3 * g + 2] = c11;
    out_ci[3 * g] = i00; out_ci[3 * g + 1] = i01; out_ci[3 * g + 2] = i11;
    const double detc = c00 * c11 - c01 * c01, deti = i00 * i11 - i01 * i01;
    const double* uv = out_uv + 4 * g;
    const int finite = isfinite(uv[0]) && isfinite(uv[1]) && isfinite(uv[2]) && isfinite(uv[3]) &&
                       isfinite(xr[2]) && isfinite(detc) && isfinite(deti);
    const int ok = finite && detc > 0.0 && deti > 0.0;
    int inside = 1;
    if (isfinite(v->cutoff)) {
      const double ru = v->cutoff * sqrt(c00 >= 0.0 || c00 != c00 ? c00 : 0.0);
      const double rv = v->cutoff * sqrt(c11 >= 0.0 || c11 != c11 ? c11 : 0.0);
      inside = (uv[0] + ru >= 0.0) && (uv[0] - ru <= (double)v->n_u - 1.0) && (uv[1] + rv >= 0.0) &&
               (uv[1] - rv <= (double)v->n_v - 1.0);
    }
    out_flags[g] = (uint8_t)((ok ? 1 : 0) | (inside ? 2 : 0));
  }
}
