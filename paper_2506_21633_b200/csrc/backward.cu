// backward.cu — K8 (imaging-plane backward) and K10 (per-Gaussian epilogue).
//
// K8 replaces grad_image_stage (backward.py:86-104).  The imaging splat is an
// unordered sum, so its adjoint is a gather: one thread per Gaussian visits
// its own member pixels (cell bit-window from K1) and accumulates dL/dI, the
// quadratic-form gradient and the center gradient in FP64 registers.  No
// atomics, no pair lists, deterministic.
//
// K10 replaces grad_geometry_stage + grad_sh_stage + the scatter/activation
// epilogue of backward() (backward.py:151-290): inverse chain
// dSigma2 = -A G A, the two projection sandwiches, the covariance
// factorisation (log-scales, quaternion with the normalisation projector),
// the position terms (two planes + phase-function look direction), SH
// coefficients, softplus' and the densification statistic.
#include "common.cuh"

namespace sdgr {

template <typename T>
__device__ __forceinline__ double ldv(const void* p, int64_t i) {
  return (double)__ldg(static_cast<const T*>(p) + i);
}

__global__ void __launch_bounds__(256, SDGR_MINB_GRAD_IMAGE) k_grad_image(sdgr_view view, sdgr_plane pl, const uint8_t* flags,
                                                    const double* intensity, const double* dLdS,
                                                    double* acc, int64_t n) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= n) return;
  double dI = 0, g00 = 0, g01 = 0, g11 = 0, gu = 0, gv = 0;
  // every row is loaded before the visibility test (coalesced, in bounds;
  // unused for invisible Gaussians): one memory round trip instead of two
  const uint8_t fl = flags[g];
  const double2 uv = reinterpret_cast<const double2*>(pl.uv)[g];
  const double4 A = reinterpret_cast<const double4*>(pl.inv_cov)[g];
  const short4 bb = reinterpret_cast<const short4*>(pl.bbox)[g];
  const double I = intensity[g];
  const uint64_t cm0 = pl.cell_mask[g];
  if (fl & SDGR_FLAG_VISIBLE) {
    const bool dense = !isfinite(view.cutoff);
    const double cut2 = dmul(view.cutoff, view.cutoff);
    auto visit = [&](int iu, int iv, double dx, double dy, double q) {
      const double G = __ldg(dLdS + (int64_t)iv * view.n_az + iu);
      const double w = nexp(-q);
      dI += G * w;
      const double dq = -(G * I) * w;
      g00 += dq * dx * dx;
      g01 += dq * dx * dy;
      g11 += dq * dy * dy;
      gu += -2.0 * dq * (A.x * dx + A.y * dy);
      gv += -2.0 * dq * (A.y * dx + A.z * dy);
    };
    if (bb.x <= bb.y && bb.z <= bb.w) {
      if ((bb.y - bb.x) < 8 && (bb.w - bb.z) < 8) {
        uint64_t cm = cm0;
        while (cm) {
          const int b = __ffsll((long long)cm) - 1;
          cm &= cm - 1;
          const int iu = bb.x + (b & 7), iv = bb.z + (b >> 3);
          const double dx = dsub((double)iu, uv.x), dy = dsub((double)iv, uv.y);
          visit(iu, iv, dx, dy, quadform(A.x, A.y, A.z, dx, dy));
        }
      } else {
        for (int iv = bb.z; iv <= bb.w; ++iv)
          for (int iu = bb.x; iu <= bb.y; ++iu) {
            const double dx = dsub((double)iu, uv.x), dy = dsub((double)iv, uv.y);
            const double q = quadform(A.x, A.y, A.z, dx, dy);
            if (dense || q <= cut2) visit(iu, iv, dx, dy, q);
          }
      }
    }
  }
  acc[g] = dI;
  acc[n + g] = g00;
  acc[2 * n + g] = g01;
  acc[3 * n + g] = g11;
  acc[4 * n + g] = gu;
  acc[5 * n + g] = gv;
}

// d(basis)/d(dir) for the 16 real SH functions (sh.py:68-113), contracted
// with the coefficients: returns sum_k c_k grad Y_k.
__device__ __forceinline__ void sh_grad_contract(double x, double y, double z, const double* c,
                                                 double* out, double* basis) {
  const double C0 = 0.28209479177387814, C1 = 0.4886025119029199;
  const double C20 = 1.0925484305920792, C21 = 0.31539156525252005, C22 = 0.5462742152960396;
  const double C30 = 0.5900435899266435, C31 = 2.890611442640554, C32 = 0.4570457994644658,
               C33 = 0.3731763325901154, C34 = 1.445305721320277;
  const double xx = x * x, yy = y * y, zz = z * z;
  basis[0] = C0; basis[1] = C1 * y; basis[2] = C1 * z; basis[3] = C1 * x;
  basis[4] = C20 * x * y; basis[5] = C20 * y * z; basis[6] = C21 * (2.0 * zz - xx - yy);
  basis[7] = C20 * x * z; basis[8] = C22 * (xx - yy);
  basis[9] = C30 * y * (3.0 * xx - yy); basis[10] = C31 * x * y * z;
  basis[11] = C32 * y * (4.0 * zz - xx - yy); basis[12] = C33 * z * (2.0 * zz - 3.0 * xx - 3.0 * yy);
  basis[13] = C32 * x * (4.0 * zz - xx - yy); basis[14] = C34 * z * (xx - yy);
  basis[15] = C30 * x * (xx - 3.0 * yy);
  double gx = 0, gy = 0, gz = 0;
  gy += c[1] * C1;
  gz += c[2] * C1;
  gx += c[3] * C1;
  gx += c[4] * C20 * y;            gy += c[4] * C20 * x;
  gy += c[5] * C20 * z;            gz += c[5] * C20 * y;
  gx += c[6] * (-2.0 * C21 * x);   gy += c[6] * (-2.0 * C21 * y);  gz += c[6] * (4.0 * C21 * z);
  gx += c[7] * C20 * z;            gz += c[7] * C20 * x;
  gx += c[8] * (2.0 * C22 * x);    gy += c[8] * (-2.0 * C22 * y);
  gx += c[9] * (C30 * 6.0 * x * y); gy += c[9] * (C30 * (3.0 * xx - 3.0 * yy));
  gx += c[10] * (C31 * y * z);     gy += c[10] * (C31 * x * z);    gz += c[10] * (C31 * x * y);
  gx += c[11] * (C32 * (-2.0 * x * y));
  gy += c[11] * (C32 * (4.0 * zz - xx - 3.0 * yy));
  gz += c[11] * (C32 * 8.0 * y * z);
  gx += c[12] * (C33 * (-6.0 * x * z));
  gy += c[12] * (C33 * (-6.0 * y * z));
  gz += c[12] * (C33 * (6.0 * zz - 3.0 * xx - 3.0 * yy));
  gx += c[13] * (C32 * (4.0 * zz - 3.0 * xx - yy));
  gy += c[13] * (C32 * (-2.0 * x * y));
  gz += c[13] * (C32 * 8.0 * x * z);
  gx += c[14] * (C34 * 2.0 * x * z); gy += c[14] * (-C34 * 2.0 * y * z); gz += c[14] * (C34 * (xx - yy));
  gx += c[15] * (C30 * (3.0 * xx - 3.0 * yy)); gy += c[15] * (C30 * (-6.0 * x * y));
  out[0] = gx; out[1] = gy; out[2] = gz;
}

// dL/dSigma2 = -A G A for symmetric 2x2 A = (a,b,c), G = (g0,g1,g2)
__device__ __forceinline__ void inverse_chain(double a, double b, double c, double g0, double g1,
                                              double g2, double* d) {
  const double p00 = a * g0 + b * g1, p01 = a * g1 + b * g2;
  const double p10 = b * g0 + c * g1, p11 = b * g1 + c * g2;
  d[0] = -(p00 * a + p01 * b);
  d[1] = -(p00 * b + p01 * c);
  d[2] = -(p10 * a + p11 * b);
  d[3] = -(p10 * b + p11 * c);
}

// Per-view inputs of the geometry epilogue.  A launch covers up to
// SDGR_MAX_BATCH views: every view-independent factor (scene loads, the
// covariance factorisation, the gradient read-modify-write) is paid once per
// batch, and the view terms are summed in FP64 registers.  All view terms of
// the covariance chain are linear in G3 = mc^T dSc mc + mi^T dSi mi, so the
// chain runs once on the summed G3.
struct GeoView {
  double mc[6], mi[6], cam[3];
  double half_u, half_v, half_az, half_rg;
  const uint8_t* flags;
  const double* inv_c;
  const double* inv_i;
  const int32_t* n_tiles;
  const double* phase_raw;
  const int32_t* pair_start;
  const double* acc;      // (6, n) imaging-plane sums
  const double* partial;  // (n_pairs, 8) computation-plane partial records
  int64_t cap;            // n_pairs: records beyond it were never written (overflowed step)
  const double* ex;       // explicit plane-space gradients (14, n) or NULL: dSigma_c (4), dSigma_i (4),
                          // duv_c (2), duv_i (2), dP, dkappa (grad_geometry_stage's arguments)
};
struct GeoBatch {
  int n_views;
  GeoView v[SDGR_MAX_BATCH];
};

// 5 CTAs/SM: the extra latency hiding beats the register spills it costs
// (measured 5.7 -> 5.0 ms/step on the c4 batch).
// T: scene parameter type; OT: gradient element type (sdgr_grads.dtype).
template <typename T, typename OT>
__global__ void __launch_bounds__(128, SDGR_MINB_GEOMETRY) k_grad_geometry(sdgr_scene sc, const __grid_constant__ GeoBatch B,
                                                       sdgr_grads out, int accumulate) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t n = sc.n;
  if (g >= n) return;
  auto put = [&](void* base_, int64_t i, double v) {
    OT* base = static_cast<OT*>(base_);
    base[i] = accumulate ? base[i] + (OT)v : (OT)v;
  };
  auto put_visible = [&](int n_vis) {
    if (out.visible_dtype) put(out.visible, g, (double)n_vis);
    else {
      int32_t* vis = static_cast<int32_t*>(out.visible);
      vis[g] = accumulate ? vis[g] + n_vis : n_vis;
    }
  };
  int n_vis = 0;
  for (int k = 0; k < B.n_views; ++k) n_vis += (B.v[k].flags[g] & SDGR_FLAG_VISIBLE) ? 1 : 0;
  if (n_vis == 0) {
    if (!accumulate) {
      for (int k = 0; k < 3; ++k) put(out.positions, 3 * g + k, 0.0);
      for (int k = 0; k < 4; ++k) put(out.rotations, 4 * g + k, 0.0);
      for (int k = 0; k < 3; ++k) put(out.log_scales, 3 * g + k, 0.0);
      for (int k = 0; k < 16; ++k) put(out.sh_coeffs, 16 * g + k, 0.0);
      put(out.ke_raw, 2 * g, 0.0);
      put(out.ke_raw, 2 * g + 1, 0.0);
      put(out.uv_grad_norm, g, 0.0);
      put_visible(0);
    }
    return;
  }
  const double p0 = ldv<T>(sc.positions, 3 * g), p1 = ldv<T>(sc.positions, 3 * g + 1),
               p2 = ldv<T>(sc.positions, 3 * g + 2);
  // the 16 SH-gradient accumulators live in this thread's shared-memory
  // column (only touched when the phase gate is open) and the SH coefficients
  // are re-read from L1 per view: keeps the view loop's state in registers
  __shared__ double s_dsh[16][128];
  const T* csh = static_cast<const T*>(sc.sh_coeffs) + 16 * g;
#pragma unroll
  for (int k = 0; k < 16; ++k) s_dsh[k][threadIdx.x] = 0.0;
  double G3[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  double dpos[3] = {0, 0, 0};
  double dk = 0.0, uvn = 0.0;
#pragma unroll 1
  for (int vi = 0; vi < B.n_views; ++vi) {
    const GeoView& V = B.v[vi];
    if (!(V.flags[g] & SDGR_FLAG_VISIBLE)) continue;
    double dSc[4], dSi[4], duc[2], dui[2], dP;
    if (V.ex) {
      // plane-space gradients given by the caller (backward.py:171-240 arguments)
#pragma unroll
      for (int i = 0; i < 4; ++i) { dSc[i] = V.ex[i * n + g]; dSi[i] = V.ex[(4 + i) * n + g]; }
      duc[0] = V.ex[8 * n + g]; duc[1] = V.ex[9 * n + g];
      dui[0] = V.ex[10 * n + g]; dui[1] = V.ex[11 * n + g];
      dP = V.ex[12 * n + g];
      dk += V.ex[13 * n + g];
    } else {
      // plane-space gradients
      const double4 Ac = reinterpret_cast<const double4*>(V.inv_c)[g];
      const double4 Ai = reinterpret_cast<const double4*>(V.inv_i)[g];
      // computation-plane partials: one record per member tile, fixed order
      double c7[7] = {0, 0, 0, 0, 0, 0, 0};
      {
        const int s0 = V.pair_start[g];
        const int64_t room = V.cap - s0 > 0 ? V.cap - s0 : 0;   // overflowed step: stay in bounds
        const int cnt = V.n_tiles[g] < room ? V.n_tiles[g] : (int)room;
        for (int k = 0; k < cnt; ++k) {
          const double4* rec = reinterpret_cast<const double4*>(V.partial + (int64_t)(s0 + k) * 8);
          const double4 r0 = rec[0], r1 = rec[1];
          c7[0] += r0.x; c7[1] += r0.y; c7[2] += r0.z; c7[3] += r0.w;
          c7[4] += r1.x; c7[5] += r1.y; c7[6] += r1.z;
        }
      }
      inverse_chain(Ac.x, Ac.y, Ac.z, c7[2], c7[3], c7[4], dSc);
      inverse_chain(Ai.x, Ai.y, Ai.z, V.acc[1 * n + g], V.acc[2 * n + g], V.acc[3 * n + g], dSi);
      duc[0] = c7[5]; duc[1] = c7[6];
      dui[0] = V.acc[4 * n + g]; dui[1] = V.acc[5 * n + g];
      dP = c7[0];
      dk += c7[1];
    }
    // G3 += mc^T dSc mc + mi^T dSi mi   (backward.py:191-193)
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        double s = 0.0;
#pragma unroll
        for (int b = 0; b < 2; ++b)
#pragma unroll
          for (int e = 0; e < 2; ++e)
            s += V.mc[3 * b + a] * dSc[2 * b + e] * V.mc[3 * e + d] +
                 V.mi[3 * b + a] * dSi[2 * b + e] * V.mi[3 * e + d];
        G3[3 * a + d] += s;
      }
    // position: both affine plane projections + phase look direction
    double dp[3];
#pragma unroll
    for (int k = 0; k < 3; ++k)
      dp[k] = duc[0] * V.mc[k] + duc[1] * V.mc[3 + k] + dui[0] * V.mi[k] + dui[1] * V.mi[3 + k];
    const double r0 = p0 - V.cam[0], r1 = p1 - V.cam[1], r2 = p2 - V.cam[2];
    double dist = sqrt(r0 * r0 + r1 * r1 + r2 * r2);
    if (dist == 0.0) dist = 1.0;
    const double d0 = r0 / dist, d1 = r1 / dist, d2 = r2 / dist;
    if (V.phase_raw[g] > 0.0) {
      double cd[16], basis[16], gP[3];
#pragma unroll
      for (int k = 0; k < 16; ++k) cd[k] = (double)__ldg(csh + k);
      sh_grad_contract(d0, d1, d2, cd, gP, basis);
      const double proj_d = gP[0] * d0 + gP[1] * d1 + gP[2] * d2;
      dp[0] += dP * (gP[0] - proj_d * d0) / dist;
      dp[1] += dP * (gP[1] - proj_d * d1) / dist;
      dp[2] += dP * (gP[2] - proj_d * d2) / dist;
#pragma unroll
      for (int k = 0; k < 16; ++k) s_dsh[k][threadIdx.x] += dP * basis[k];
    }
#pragma unroll
    for (int k = 0; k < 3; ++k) dpos[k] += dp[k];
    // densification statistic in NDC units (backward.py:285-289)
    const double gx = duc[0] * V.half_u + dui[0] * V.half_az;
    const double gy = duc[1] * V.half_v + dui[1] * V.half_rg;
    uvn += sqrt(gx * gx + gy * gy);
  }
  // covariance factor M = R(q) diag(e^s)   (backward.py:195-213)
  double q[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) q[k] = ldv<T>(sc.rotations, 4 * g + k);
  const double nrm = sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
  const double w = q[0] / nrm, x = q[1] / nrm, y = q[2] / nrm, z = q[3] / nrm;
  const double Rq[9] = {1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y),
                        2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x),
                        2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)};
  double s[3];
#pragma unroll
  for (int j = 0; j < 3; ++j) s[j] = exp(ldv<T>(sc.log_scales, 3 * g + j));
  double M[9];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) M[3 * i + j] = Rq[3 * i + j] * s[j];
  double dM[9];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      dM[3 * i + j] = 2.0 * (G3[3 * i] * M[j] + G3[3 * i + 1] * M[3 + j] + G3[3 * i + 2] * M[6 + j]);
  double dR[9];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) dR[3 * i + j] = dM[3 * i + j] * s[j];
  // dR/dq-hat partials (backward.py:151-168)
  const double dqw = 2.0 * (-z * dR[1] + y * dR[2] + z * dR[3] - x * dR[5] - y * dR[6] + x * dR[7]);
  const double dqx = 2.0 * (y * dR[1] + z * dR[2] + y * dR[3] - 2 * x * dR[4] - w * dR[5] + z * dR[6] +
                            w * dR[7] - 2 * x * dR[8]);
  const double dqy = 2.0 * (-2 * y * dR[0] + x * dR[1] + w * dR[2] + x * dR[3] + z * dR[5] - w * dR[6] +
                            z * dR[7] - 2 * y * dR[8]);
  const double dqz = 2.0 * (-2 * z * dR[0] - w * dR[1] + x * dR[2] + w * dR[3] - 2 * z * dR[4] + y * dR[5] +
                            x * dR[6] + y * dR[7]);
  const double dot = dqw * w + dqx * x + dqy * y + dqz * z;
  put(out.rotations, 4 * g + 0, (dqw - dot * w) / nrm);
  put(out.rotations, 4 * g + 1, (dqx - dot * x) / nrm);
  put(out.rotations, 4 * g + 2, (dqy - dot * y) / nrm);
  put(out.rotations, 4 * g + 3, (dqz - dot * z) / nrm);
#pragma unroll
  for (int j = 0; j < 3; ++j) put(out.log_scales, 3 * g + j, dM[j] * M[j] + dM[3 + j] * M[3 + j] + dM[6 + j] * M[6 + j]);
#pragma unroll
  for (int k = 0; k < 16; ++k) put(out.sh_coeffs, 16 * g + k, s_dsh[k][threadIdx.x]);
#pragma unroll
  for (int k = 0; k < 3; ++k) put(out.positions, 3 * g + k, dpos[k]);
  // softplus' = sigmoid (scene.py:36-39)
  const double k0 = ldv<T>(sc.ke_raw, 2 * g), k1 = ldv<T>(sc.ke_raw, 2 * g + 1);
  put(out.ke_raw, 2 * g, dk * 0.5 * (1.0 + tanh(0.5 * k0)));
  put(out.ke_raw, 2 * g + 1, dk * 0.5 * (1.0 + tanh(0.5 * k1)));
  put(out.uv_grad_norm, g, uvn);
  put_visible(n_vis);
}

int launch_grad_image(const sdgr_view& v, const sdgr_projection& p, const double* intensity,
                      const double* dLdS, double* acc, cudaStream_t st) {
  {
    KernelTimer kt(SDGR_K_GRAD_IMAGE, st);
    k_grad_image<<<(unsigned)((p.n + 255) / 256), 256, 0, st>>>(v, p.img, p.flags, intensity, dLdS, acc, p.n);
  }
  note_launch();
  return check_launch();
}

static void launch_geometry_batch(const sdgr_scene& sc, const GeoBatch& B, const sdgr_grads& out, int accumulate,
                                  cudaStream_t st);

int launch_grad_geometry_explicit(const sdgr_scene& sc, const sdgr_view& v, const sdgr_projection& p,
                                  const double* ex, const sdgr_grads& out, cudaStream_t st) {
  GeoBatch B;
  B.n_views = 1;
  GeoView& G = B.v[0];
  for (int i = 0; i < 6; ++i) { G.mc[i] = v.mc[i]; G.mi[i] = v.mi[i]; }
  for (int i = 0; i < 3; ++i) G.cam[i] = v.cam[i];
  G.half_u = v.n_u / 2.0; G.half_v = v.n_v / 2.0;
  G.half_az = v.n_az / 2.0; G.half_rg = v.n_rg / 2.0;
  G.flags = p.flags;
  G.inv_c = p.comp.inv_cov;
  G.inv_i = p.img.inv_cov;
  G.n_tiles = nullptr;
  G.phase_raw = p.phase_raw;
  G.pair_start = nullptr;
  G.acc = nullptr;
  G.partial = nullptr;
  G.cap = 0;
  G.ex = ex;
  launch_geometry_batch(sc, B, out, 0, st);
  note_launch();
  return check_launch();
}

int launch_grad_geometry(const sdgr_scene& sc, int n_views, const sdgr_view* views,
                         const sdgr_projection* projs, const sdgr_tiles* comps, const double* const* acc_imgs,
                         const double* const* partials, const sdgr_grads& out, int accumulate,
                         cudaStream_t st) {
  GeoBatch B;
  B.n_views = n_views;
  for (int k = 0; k < n_views; ++k) {
    const sdgr_view& v = views[k];
    GeoView& G = B.v[k];
    for (int i = 0; i < 6; ++i) { G.mc[i] = v.mc[i]; G.mi[i] = v.mi[i]; }
    for (int i = 0; i < 3; ++i) G.cam[i] = v.cam[i];
    G.half_u = v.n_u / 2.0; G.half_v = v.n_v / 2.0;
    G.half_az = v.n_az / 2.0; G.half_rg = v.n_rg / 2.0;
    G.flags = projs[k].flags;
    G.inv_c = projs[k].comp.inv_cov;
    G.inv_i = projs[k].img.inv_cov;
    G.n_tiles = projs[k].comp.n_tiles;
    G.phase_raw = projs[k].phase_raw;
    G.pair_start = comps[k].pair_start;
    G.acc = acc_imgs[k];
    G.partial = partials[k];
    G.cap = comps[k].n_pairs;
    G.ex = nullptr;
  }
  {
    KernelTimer kt(SDGR_K_GEOMETRY, st);
    launch_geometry_batch(sc, B, out, accumulate, st);
  }
  note_launch();
  return check_launch();
}

static void launch_geometry_batch(const sdgr_scene& sc, const GeoBatch& B, const sdgr_grads& out, int accumulate,
                                  cudaStream_t st) {
  const unsigned blocks = (unsigned)((sc.n + 127) / 128);
  {
    if (sc.dtype == 0 && out.dtype == 0)
      k_grad_geometry<float, float><<<blocks, 128, 0, st>>>(sc, B, out, accumulate);
    else if (sc.dtype == 0)
      k_grad_geometry<float, double><<<blocks, 128, 0, st>>>(sc, B, out, accumulate);
    else if (out.dtype == 0)
      k_grad_geometry<double, float><<<blocks, 128, 0, st>>>(sc, B, out, accumulate);
    else
      k_grad_geometry<double, double><<<blocks, 128, 0, st>>>(sc, B, out, accumulate);
  }
}

}  // namespace sdgr
