// preprocess.cu — K1: one thread per Gaussian projects it onto both planes.
//
// Replaces geometry.project_all (geometry.py:233-340) plus the per-Gaussian
// half of forward._footprint_pairs (forward.py:60-109): the clipped cell
// bbox, the exact membership test of every bbox cell (q <= cutoff^2) and the
// set of 16x16 tiles that hold at least one member cell.  Membership is
// decided once here, in FP64 with the reference's op order, and stored as an
// 8x8 cell bit-window so no later kernel repeats FP64 work for small
// footprints.
#include "common.cuh"

namespace sdgr {

// Real SH basis degrees 0-3 in the reference's (non-3DGS) ordering and
// signs (sh.py:15-65): Y1 = C1*(y, z, x).
__device__ __forceinline__ void sh_basis(double x, double y, double z, double* b) {
  const double C0 = 0.28209479177387814, C1 = 0.4886025119029199;
  const double C20 = 1.0925484305920792, C21 = 0.31539156525252005, C22 = 0.5462742152960396;
  const double C30 = 0.5900435899266435, C31 = 2.890611442640554, C32 = 0.4570457994644658,
               C33 = 0.3731763325901154, C34 = 1.445305721320277;
  double xx = x * x, yy = y * y, zz = z * z;
  b[0] = C0;
  b[1] = C1 * y;
  b[2] = C1 * z;
  b[3] = C1 * x;
  b[4] = C20 * x * y;
  b[5] = C20 * y * z;
  b[6] = C21 * (2.0 * zz - xx - yy);
  b[7] = C20 * x * z;
  b[8] = C22 * (xx - yy);
  b[9] = C30 * y * (3.0 * xx - yy);
  b[10] = C31 * x * y * z;
  b[11] = C32 * y * (4.0 * zz - xx - yy);
  b[12] = C33 * z * (2.0 * zz - 3.0 * xx - 3.0 * yy);
  b[13] = C32 * x * (4.0 * zz - xx - yy);
  b[14] = C34 * z * (xx - yy);
  b[15] = C30 * x * (xx - 3.0 * yy);
}

template <typename T>
__device__ __forceinline__ double ld(const T* p, int64_t i) { return (double)__ldg(p + i); }

// bbox as the short4 bit pattern (x0, x1, y0, y1) in one u64 (sdgr_plane.emit)
__device__ __forceinline__ unsigned long long emit_bbox(int x0, int x1, int y0, int y1) {
  return (unsigned long long)(uint16_t)x0 | ((unsigned long long)(uint16_t)x1 << 16) |
         ((unsigned long long)(uint16_t)y0 << 32) | ((unsigned long long)(uint16_t)y1 << 48);
}

// Footprint of one plane: inverse covariance, clipped bbox, member masks.
// Writes the plane records for Gaussian g.  (forward.py:33-42, 60-109)
// Returns an upper bound of the Gaussian's member cells on this plane (exact
// for footprints inside the 8x8 window, the bbox area otherwise).
// ru, rv = cutoff * sqrt(max(c00, 0)), cutoff * sqrt(max(c11, 0)) (forward.py:74-75),
// computed by the caller (the computation plane's are the cull's).
// SoA outputs other than inv_cov / n_tiles may be NULL (multi-view steps read
// the packed / emit rows instead).
__device__ int plane_footprint(const sdgr_plane& pl, int64_t g, double u, double v,
                                double c00, double c01, double c11, double ru, double rv, int nu, int nv,
                                double cutoff, bool dense, double4& rec_out) {
  // invert_cov2d (forward.py:33-42)
  double det = dsub(dmul(c00, c11), dmul(c01, c01));
  double a00 = ddiv(c11, det), a01 = ddiv(-c01, det), a11 = ddiv(c00, det);
  rec_out = make_double4(a00, a01, a11, 0.0);
  if (pl.uv) reinterpret_cast<double2*>(pl.uv)[g] = make_double2(u, v);
  reinterpret_cast<double4*>(pl.inv_cov)[g] = make_double4(a00, a01, a11, 0.0);
  if (pl.cov) reinterpret_cast<double4*>(pl.cov)[g] = make_double4(c00, c01, c11, 0.0);

  int x0, x1, y0, y1;
  if (!dense) {
    double fx0 = fmax(ceil(dsub(u, ru)), 0.0);
    double fx1 = fmin(floor(dadd(u, ru)), (double)nu - 1.0);
    double fy0 = fmax(ceil(dsub(v, rv)), 0.0);
    double fy1 = fmin(floor(dadd(v, rv)), (double)nv - 1.0);
    // visible Gaussians have finite u, r; clamp into int16 range safely
    fx0 = fmin(fx0, 32767.0); fy0 = fmin(fy0, 32767.0);
    fx1 = fmax(fx1, -32768.0); fy1 = fmax(fy1, -32768.0);
    x0 = (int)fx0; x1 = (int)fx1; y0 = (int)fy0; y1 = (int)fy1;
  } else {
    x0 = 0; x1 = nu - 1; y0 = 0; y1 = nv - 1;
  }
  uint64_t cmask = 0, tmask = 0;
  int ntiles = 0;
  if (x0 <= x1 && y0 <= y1) {
    const int tx0 = x0 >> 4, ty0 = y0 >> 4, tx1 = x1 >> 4, ty1 = y1 >> 4;
    const bool small = (x1 - x0) < 8 && (y1 - y0) < 8;
    const bool tsmall = (tx1 - tx0) < 8 && (ty1 - ty0) < 8;
    const double cut2 = dmul(cutoff, cutoff);
    if (small) {
      const double a01x2 = dmul(2.0, a01);
      const int ncol = x1 - x0 + 1;
      // cell centres as exact FP64 integers (fx0 + c has the same bits as
      // (double)(x0 + c)).  Columns go in fixed groups of 4 (one group for
      // the usual <= 4-column windows): every thread of a warp runs the same
      // straight-line code whether its window has 3 or 4 columns -- a
      // ncol-bounded loop split into an unrolled body and a remainder path
      // that mixed warps ran one after the other -- and the bits past the
      // window are masked off.
      const double fx0 = (double)x0;
      const uint32_t colmask = (1u << ncol) - 1u;
      double fy = (double)y0;
      for (int r = 0; r <= y1 - y0; ++r, fy += 1.0) {
        const double dy = dsub(fy, v);
        const double t3 = dmul(a11, dmul(dy, dy));
        uint32_t row = 0;   // this row's member bits (32-bit shifts, one 64-bit merge per row)
        double fxg = fx0;
        for (int c0 = 0; c0 < ncol; c0 += 4, fxg += 4.0) {
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const double dx = dsub(fxg + (double)c, u);
            const double q = dadd(dadd(dmul(a00, dmul(dx, dx)), dmul(dmul(a01x2, dx), dy)), t3);
            row |= (uint32_t)(q <= cut2) << (c0 + c);
          }
        }
        row = dense ? colmask : (row & colmask);
        cmask |= (uint64_t)row << (8 * r);
      }
      // member tiles of the (<= 2x2 tile) window from the cell bits: split the
      // window's columns / rows at the tile boundary
      const int csplit = min(8, kTile - (x0 & 15)), rsplit = min(8, kTile - (y0 & 15));
      const uint64_t col0 = 0x0101010101010101ull * ((1ull << csplit) - 1ull);
      const uint64_t row0 = rsplit >= 8 ? ~0ull : ((1ull << (8 * rsplit)) - 1ull);
      if (cmask & col0 & row0) tmask |= 1ull;
      if (cmask & ~col0 & row0) tmask |= 1ull << 1;
      if (cmask & col0 & ~row0) tmask |= 1ull << 8;
      if (cmask & ~col0 & ~row0) tmask |= 1ull << 9;
      ntiles = __popcll(tmask);
    } else if (dense) {
      ntiles = (tx1 - tx0 + 1) * (ty1 - ty0 + 1);
      if (tsmall)
        for (int ty = ty0; ty <= ty1; ++ty)
          for (int tx = tx0; tx <= tx1; ++tx) tmask |= 1ull << ((ty - ty0) * 8 + (tx - tx0));
    } else {
      // large footprint: per tile, stop at the first member cell
      const double a01x2 = dmul(2.0, a01);
      for (int ty = ty0; ty <= ty1; ++ty) {
        for (int tx = tx0; tx <= tx1; ++tx) {
          const int cx0 = max(x0, tx * kTile), cx1 = min(x1, tx * kTile + kTile - 1);
          const int cy0 = max(y0, ty * kTile), cy1 = min(y1, ty * kTile + kTile - 1);
          bool hit = false;
          for (int iv = cy0; iv <= cy1 && !hit; ++iv) {
            const double dy = dsub((double)iv, v);
            const double t3 = dmul(a11, dmul(dy, dy));
            for (int iu = cx0; iu <= cx1; ++iu) {
              const double dx = dsub((double)iu, u);
              const double q = dadd(dadd(dmul(a00, dmul(dx, dx)), dmul(dmul(a01x2, dx), dy)), t3);
              if (q <= cut2) { hit = true; break; }
            }
          }
          if (hit) {
            ++ntiles;
            if (tsmall) tmask |= 1ull << ((ty - ty0) * 8 + (tx - tx0));
          }
        }
      }
    }
  }
  if (pl.bbox) reinterpret_cast<short4*>(pl.bbox)[g] = make_short4((short)x0, (short)x1, (short)y0, (short)y1);
  if (pl.cell_mask) pl.cell_mask[g] = cmask;
  rec_out.w = __longlong_as_double((long long)cmask);
  if (pl.tile_mask) pl.tile_mask[g] = tmask;
  if (pl.emit)
    reinterpret_cast<ulonglong2*>(pl.emit)[g] =
        make_ulonglong2(emit_bbox(x0, x1, y0, y1), (unsigned long long)tmask);
  pl.n_tiles[g] = ntiles;
  if (x0 > x1 || y0 > y1) return 0;
  if ((x1 - x0) < 8 && (y1 - y0) < 8) return __popcll(cmask);
  return (x1 - x0 + 1) * (y1 - y0 + 1);
}

__device__ void plane_empty(const sdgr_plane& pl, int64_t g) {
  if (pl.bbox) reinterpret_cast<short4*>(pl.bbox)[g] = make_short4(1, 0, 1, 0);
  if (pl.emit) reinterpret_cast<ulonglong2*>(pl.emit)[g] = make_ulonglong2(emit_bbox(1, 0, 1, 0), 0ull);
  if (pl.cell_mask) pl.cell_mask[g] = 0;
  if (pl.tile_mask) pl.tile_mask[g] = 0;
  pl.n_tiles[g] = 0;
}

// View batch of K1: per-view constants and outputs, passed by value (the
// kernel parameter space holds up to SDGR_MAX_BATCH views).
struct ProjBatch {
  sdgr_view view[SDGR_MAX_BATCH];
  sdgr_projection proj[SDGR_MAX_BATCH];
  int nv;
  int zero_col2;   // every view has mc[0][2] == mi[0][2] == 0 (R[0][2] = 0, geometry.py:41-47)
};

// One plane's covariance sandwich m Sigma m^T (geometry.py:269-272): per
// entry (a, d) the sequential sum over (b, c) of (m[a,b] Sigma[b,c]) m[d,c]
// (np.einsum's order, no FMA).  kZero: row 0 of m has m[0][2] == 0, so the
// 22 terms with (a = 0, b = 2) or (d = 0, c = 2) are exactly +-0 (Sigma
// finite) and adding them changes no bit of a non-zero sum -- skipped.
template <bool kZero>
__device__ __forceinline__ void sandwich(const double* m, const double* Cm, double* out) {
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int d = 0; d < 2; ++d) {
      double acc = 0.0;
      bool first = true;
#pragma unroll
      for (int b = 0; b < 3; ++b)
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          if (kZero && ((a == 0 && b == 2) || (d == 0 && c == 2))) continue;
          const double t = dmul(dmul(m[3 * a + b], Cm[3 * b + c]), m[3 * d + c]);
          acc = first ? t : dadd(acc, t);
          first = false;
        }
      out[2 * a + d] = acc;
    }
}

// One thread per Gaussian, looping over the batch's views: the parameters
// are read once and the view-independent half of project_all -- quaternion
// normalisation, R(q), e^s, Sigma = M M^T (scene.py:49-97) and the softplus
// extinctions (geometry.py:317) -- is computed once per batch instead of once
// per view.  Per view: x_r, plane coordinates, the two covariance sandwiches,
// skip/cull, footprints, depth key and the SH phase (geometry.py:249-317).
template <typename T, bool kZero>
__global__ void __launch_bounds__(256, SDGR_MINB_PROJECT) k_project(sdgr_scene scene, const __grid_constant__ ProjBatch B) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool live = g < scene.n;
  const T* P = static_cast<const T*>(scene.positions);
  double p0 = 0.0, p1 = 0.0, p2 = 0.0;
  double C00 = 0.0, C01 = 0.0, C02 = 0.0, C11 = 0.0, C12 = 0.0, C22 = 0.0;
  double kf = 0.0, kb = 0.0;
  if (live) {
    const T* Q = static_cast<const T*>(scene.rotations);
    const T* L = static_cast<const T*>(scene.log_scales);
    p0 = ld(P, 3 * g); p1 = ld(P, 3 * g + 1); p2 = ld(P, 3 * g + 2);
    // covariance R(q) diag(e^s)^2 R(q)^T  (scene.py:49-97)
    double q[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) q[k] = ld(Q, 4 * g + k);
    const double nrm = dsqrt(dadd(dadd(dadd(dmul(q[0], q[0]), dmul(q[1], q[1])), dmul(q[2], q[2])),
                                  dmul(q[3], q[3])));
    const double w = ddiv(q[0], nrm), x = ddiv(q[1], nrm), y = ddiv(q[2], nrm), z = ddiv(q[3], nrm);
    double Rq[9];
    Rq[0] = dsub(1.0, dmul(2.0, dadd(dmul(y, y), dmul(z, z))));
    Rq[1] = dmul(2.0, dsub(dmul(x, y), dmul(w, z)));
    Rq[2] = dmul(2.0, dadd(dmul(x, z), dmul(w, y)));
    Rq[3] = dmul(2.0, dadd(dmul(x, y), dmul(w, z)));
    Rq[4] = dsub(1.0, dmul(2.0, dadd(dmul(x, x), dmul(z, z))));
    Rq[5] = dmul(2.0, dsub(dmul(y, z), dmul(w, x)));
    Rq[6] = dmul(2.0, dsub(dmul(x, z), dmul(w, y)));
    Rq[7] = dmul(2.0, dadd(dmul(y, z), dmul(w, x)));
    Rq[8] = dsub(1.0, dmul(2.0, dadd(dmul(x, x), dmul(y, y))));
    double s[3];
#pragma unroll
    for (int j = 0; j < 3; ++j) s[j] = sdgr_exp(ld(L, 3 * g + j));
    double M[9];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) M[3 * i + j] = dmul(Rq[3 * i + j], s[j]);
    // Sigma_ij = fma(M_i2, M_j2, fma(M_i1, M_j1, M_i0 M_j0)): symmetric bit for bit
    auto cij = [&](int i, int j) {
      return dfma(M[3 * i + 2], M[3 * j + 2], dfma(M[3 * i + 1], M[3 * j + 1], dmul(M[3 * i], M[3 * j])));
    };
    C00 = cij(0, 0); C01 = cij(0, 1); C02 = cij(0, 2);
    C11 = cij(1, 1); C12 = cij(1, 2); C22 = cij(2, 2);
    const T* K = static_cast<const T*>(scene.ke_raw);
    kf = softplus64(ld(K, 2 * g));
    kb = softplus64(ld(K, 2 * g + 1));
  }
  // view-independent state lives in shared memory across the view loop (keeps
  // the per-view FP64 chain inside 64 registers without spills); per-view
  // counters are block accumulators flushed once at the end
  __shared__ double s_state[11][256];
  // FP32 scenes: the block's SH coefficients, staged once with coalesced
  // loads (read every view; otherwise 16 strided global loads per view per
  // Gaussian).  FP64 scenes read them from global (the FP64 copy would not
  // fit next to s_state).
  constexpr bool kStageSh = sizeof(T) == 4;
  __shared__ float s_sh[16][256];
  const T* S = static_cast<const T*>(scene.sh_coeffs);
  if (kStageSh) {
    const int64_t g0 = (int64_t)blockIdx.x * blockDim.x;
    const int64_t lim = (scene.n - g0) * 16;   // valid coefficients of this block
    for (int e = threadIdx.x; e < 16 * 256; e += blockDim.x)
      s_sh[e & 15][e >> 4] = e < lim ? (float)__ldg(S + g0 * 16 + e) : 0.f;
  }
  // per-warp counter slots (plain stores; 64-bit shared atomics are CAS loops)
  __shared__ unsigned long long s_cnt[SDGR_MAX_BATCH][5][8];
  {
    const double st[11] = {p0, p1, p2, C00, C01, C02, C11, C12, C22, kf, kb};
#pragma unroll
    for (int j = 0; j < 11; ++j) s_state[j][threadIdx.x] = st[j];
    for (int i = threadIdx.x; i < SDGR_MAX_BATCH * 5 * 8; i += blockDim.x) (&s_cnt[0][0][0])[i] = 0ull;
  }
  __syncthreads();

  for (int k = 0; k < B.nv; ++k) {
    const sdgr_view& view = B.view[k];
    const sdgr_projection& proj = B.proj[k];
    int n_vis = 0, n_skip = 0, n_cull = 0;
    unsigned long long m_comp = 0, m_img = 0;
    if (live) {
      const double p0 = s_state[0][threadIdx.x], p1 = s_state[1][threadIdx.x], p2 = s_state[2][threadIdx.x];
      const double Cm[9] = {s_state[3][threadIdx.x], s_state[4][threadIdx.x], s_state[5][threadIdx.x],
                            s_state[4][threadIdx.x], s_state[6][threadIdx.x], s_state[7][threadIdx.x],
                            s_state[5][threadIdx.x], s_state[7][threadIdx.x], s_state[8][threadIdx.x]};
      const double* R = view.R;
      // x_r = positions @ R.T + T  (geometry.py:249; OpenBLAS FMA chain)
      double xr[3];
#pragma unroll
      for (int i = 0; i < 3; ++i)
        xr[i] = dadd(dfma(p2, R[3 * i + 2], dfma(p1, R[3 * i + 1], dmul(p0, R[3 * i]))), view.T[i]);
      // plane coordinates (geometry.py:78-105) and ndc_to_pixel (:73-75)
      const double undc = ddiv(dmul(2.0, xr[0]), view.den_u);
      const double vcndc = ddiv(dmul(2.0, xr[1]), view.den_v);
      const double vindc = dsub(ddiv(dmul(2.0, xr[2]), view.den_v), view.off_vi);
      const double uc = dsub(dmul(dmul(dadd(undc, 1.0), 0.5), (double)view.n_u), 0.5);
      const double vc = dsub(dmul(dmul(dadd(vcndc, 1.0), 0.5), (double)view.n_v), 0.5);
      const double ui = dsub(dmul(dmul(dadd(undc, 1.0), 0.5), (double)view.n_az), 0.5);
      const double vi = dsub(dmul(dmul(dadd(vindc, 1.0), 0.5), (double)view.n_rg), 0.5);
      const double depth = xr[2];

      // sandwich mc C mc^T (geometry.py:269-278): sequential over (b, c)
      double cc[4], ci[4];
      // kZero: a non-finite Sigma makes the reference's sandwich non-finite
      // (0 * inf = NaN in the skipped terms), i.e. the Gaussian is skipped
      const bool sig_fin = !kZero || (isfinite(Cm[0]) && isfinite(Cm[1]) && isfinite(Cm[2]) &&
                                      isfinite(Cm[4]) && isfinite(Cm[5]) && isfinite(Cm[8]));
      sandwich<kZero>(view.mc, Cm, cc);
      sandwich<kZero>(view.mi, Cm, ci);
      const double cc00 = dadd(cc[0], view.cov_reg), cc11 = dadd(cc[3], view.cov_reg);
      const double cc01 = dmul(0.5, dadd(cc[1], cc[2]));
      const double ci00 = dadd(ci[0], view.cov_reg), ci11 = dadd(ci[3], view.cov_reg);
      const double ci01 = dmul(0.5, dadd(ci[1], ci[2]));
      const double detc = dsub(dmul(cc00, cc11), dmul(cc01, cc01));
      const double deti = dsub(dmul(ci00, ci11), dmul(ci01, ci01));
      const bool finite = isfinite(uc) && isfinite(vc) && isfinite(ui) && isfinite(vi) &&
                          isfinite(depth) && isfinite(detc) && isfinite(deti);
      const bool ok = finite && sig_fin && detc > 0.0 && deti > 0.0;
      const bool dense = !isfinite(view.cutoff);
      bool inside = true;
      double ru = 0.0, rv = 0.0;
      if (!dense) {
        // frustum cull (geometry.py:293-305); the radii are the footprint's too
        ru = dmul(view.cutoff, dsqrt(np_max0(cc00)));
        rv = dmul(view.cutoff, dsqrt(np_max0(cc11)));
        inside = (dadd(uc, ru) >= 0.0) && (dsub(uc, ru) <= (double)view.n_u - 1.0) &&
                 (dadd(vc, rv) >= 0.0) && (dsub(vc, rv) <= (double)view.n_v - 1.0);
      }
      const bool vis = ok && inside;
      n_vis = vis; n_skip = !ok; n_cull = ok && !inside;
      proj.flags[g] = (uint8_t)((vis ? SDGR_FLAG_VISIBLE : 0) | (!ok ? SDGR_FLAG_SKIPPED : 0) |
                                ((ok && !inside) ? SDGR_FLAG_CULLED : 0));
      if (vis) {
        double4 rc, ri;
        m_comp = plane_footprint(proj.comp, g, uc, vc, cc00, cc01, cc11, ru, rv, view.n_u, view.n_v, view.cutoff,
                                 dense, rc);
        const double rui = dense ? 0.0 : dmul(view.cutoff, dsqrt(np_max0(ci00)));
        const double rvi = dense ? 0.0 : dmul(view.cutoff, dsqrt(np_max0(ci11)));
        m_img = plane_footprint(proj.img, g, ui, vi, ci00, ci01, ci11, rui, rvi, view.n_az, view.n_rg, view.cutoff,
                                dense, ri);
        proj.depth_key[g] = depth_key(depth);
        // phase function and extinction (geometry.py:308-317)
        const double r0 = p0 - view.cam[0], r1 = p1 - view.cam[1], r2 = p2 - view.cam[2];
        double dist = sqrt(r0 * r0 + r1 * r1 + r2 * r2);
        if (dist == 0.0) dist = 1.0;
        const double idist = 1.0 / dist;   // (not a key: one division instead of three)
        const double d0 = r0 * idist, d1 = r1 * idist, d2 = r2 * idist;
        double b[16];
        sh_basis(d0, d1, d2, b);
        double praw = 0.0;
#pragma unroll
        for (int j = 0; j < 16; ++j)
          praw += b[j] * (kStageSh ? (double)s_sh[j][threadIdx.x] : ld(S, 16 * g + j));
        const double ph = (praw == praw) ? fmax(praw, 0.0) : praw;  // NaN propagates (np.maximum)
        const double kfv = s_state[9][threadIdx.x], kbv = s_state[10][threadIdx.x], kappa_g = kfv + kbv;
        if (proj.kappa) proj.kappa[g] = kappa_g;
        if (proj.phase) proj.phase[g] = ph;
        if (proj.comp.packed) {
          double4* pk = reinterpret_cast<double4*>(proj.comp.packed) + 2 * g;
          pk[0] = make_double4(uc, vc, rc.x, rc.y);
          pk[1] = make_double4(rc.z, kappa_g, ph, rc.w);
        }
        proj.phase_raw[g] = praw;
        if (proj.ke_act) reinterpret_cast<double2*>(proj.ke_act)[g] = make_double2(kfv, kbv);
        if (proj.look) reinterpret_cast<double4*>(proj.look)[g] = make_double4(d0, d1, d2, dist);
      } else {
        plane_empty(proj.comp, g);
        plane_empty(proj.img, g);
        proj.depth_key[g] = ~0ull;
        if (proj.kappa) proj.kappa[g] = 0.0;
        if (proj.phase) proj.phase[g] = 0.0;
        proj.phase_raw[g] = 0.0;
        // accessor arrays keep the raw projection for non-visible rows too
        if (proj.comp.uv) reinterpret_cast<double2*>(proj.comp.uv)[g] = make_double2(uc, vc);
        if (proj.img.uv) reinterpret_cast<double2*>(proj.img.uv)[g] = make_double2(ui, vi);
        if (proj.comp.cov) reinterpret_cast<double4*>(proj.comp.cov)[g] = make_double4(cc00, cc01, cc11, 0.0);
        if (proj.img.cov) reinterpret_cast<double4*>(proj.img.cov)[g] = make_double4(ci00, ci01, ci11, 0.0);
      }
    }
    // warp-aggregated into the block's shared counters (no block barrier per view)
    const int cv = __popc(__ballot_sync(0xffffffffu, n_vis)), cs = __popc(__ballot_sync(0xffffffffu, n_skip)),
              cc = __popc(__ballot_sync(0xffffffffu, n_cull));
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      m_comp += __shfl_down_sync(0xffffffffu, m_comp, off);
      m_img += __shfl_down_sync(0xffffffffu, m_img, off);
    }
    if ((threadIdx.x & 31) == 0) {
      const int w = threadIdx.x >> 5;
      s_cnt[k][0][w] = (unsigned long long)cv;
      s_cnt[k][1][w] = (unsigned long long)cs;
      s_cnt[k][2][w] = (unsigned long long)cc;
      s_cnt[k][3][w] = m_comp;
      s_cnt[k][4][w] = m_img;
    }
  }
  __syncthreads();
  if (threadIdx.x < 5 * B.nv) {
    const int k = threadIdx.x / 5, j = threadIdx.x % 5;
    unsigned long long c = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) c += s_cnt[k][j][w];
    const sdgr_projection& proj = B.proj[k];
    if (c) {
      if (j < 3) atomicAdd(proj.counters + j, (int)c);
      else if (proj.member_pairs) atomicAdd(proj.member_pairs + (j - 3), c);
    }
  }
}

// zero every view's counters (one launch instead of 2 memsets per view)
__global__ void k_project_init(const __grid_constant__ ProjBatch B) {
  const int k = threadIdx.x >> 2, i = threadIdx.x & 3;
  if (k >= B.nv) return;
  B.proj[k].counters[i] = 0;
  if (i < 2 && B.proj[k].member_pairs) B.proj[k].member_pairs[i] = 0ull;
}

// Records of a projection given in plane space (the reference tests'
// hand-assembled Projection, tests/test_forward.py:43-59): every row is
// visible; footprints, depth keys and packed rows exactly as k_project would
// write them for the same plane-space values.
__global__ void __launch_bounds__(256) k_project_planes(sdgr_view view, int64_t n, const double* __restrict__ uv_c,
                                                        const double* __restrict__ uv_i,
                                                        const double* __restrict__ depth,
                                                        const double* __restrict__ cov_c,
                                                        const double* __restrict__ cov_i,
                                                        const double* __restrict__ praw,
                                                        const double* __restrict__ kappa, sdgr_projection proj) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long mc = 0, mi = 0;
  if (g < n) {
    const bool dense = !isfinite(view.cutoff);
    const double c00 = cov_c[3 * g], c01 = cov_c[3 * g + 1], c11 = cov_c[3 * g + 2];
    const double i00 = cov_i[3 * g], i01 = cov_i[3 * g + 1], i11 = cov_i[3 * g + 2];
    const double ru = dense ? 0.0 : dmul(view.cutoff, dsqrt(np_max0(c00)));
    const double rv = dense ? 0.0 : dmul(view.cutoff, dsqrt(np_max0(c11)));
    const double rui = dense ? 0.0 : dmul(view.cutoff, dsqrt(np_max0(i00)));
    const double rvi = dense ? 0.0 : dmul(view.cutoff, dsqrt(np_max0(i11)));
    double4 rc, ri;
    mc = plane_footprint(proj.comp, g, uv_c[2 * g], uv_c[2 * g + 1], c00, c01, c11, ru, rv, view.n_u, view.n_v,
                         view.cutoff, dense, rc);
    mi = plane_footprint(proj.img, g, uv_i[2 * g], uv_i[2 * g + 1], i00, i01, i11, rui, rvi, view.n_az, view.n_rg,
                         view.cutoff, dense, ri);
    proj.flags[g] = SDGR_FLAG_VISIBLE;
    proj.depth_key[g] = depth_key(depth[g]);
    const double pr = praw[g];
    const double ph = (pr == pr) ? fmax(pr, 0.0) : pr;
    if (proj.kappa) proj.kappa[g] = kappa[g];
    if (proj.phase) proj.phase[g] = ph;
    proj.phase_raw[g] = pr;
    if (proj.comp.packed) {
      double4* pk = reinterpret_cast<double4*>(proj.comp.packed) + 2 * g;
      pk[0] = make_double4(uv_c[2 * g], uv_c[2 * g + 1], rc.x, rc.y);
      pk[1] = make_double4(rc.z, kappa[g], ph, rc.w);
    }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    mc += __shfl_down_sync(0xffffffffu, mc, off);
    mi += __shfl_down_sync(0xffffffffu, mi, off);
  }
  const int nv = __popc(__ballot_sync(0xffffffffu, g < n));
  if ((threadIdx.x & 31) == 0) {
    if (nv) atomicAdd(proj.counters, nv);
    if (proj.member_pairs) {
      if (mc) atomicAdd(proj.member_pairs, mc);
      if (mi) atomicAdd(proj.member_pairs + 1, mi);
    }
  }
}

int launch_project_planes(const sdgr_view& view, int64_t n, const double* uv_c, const double* uv_i,
                          const double* depth, const double* cov_c, const double* cov_i, const double* praw,
                          const double* kappa, const sdgr_projection& proj, cudaStream_t st) {
  ProjBatch B;
  B.nv = 1;
  B.view[0] = view;
  B.proj[0] = proj;
  k_project_init<<<1, 4 * SDGR_MAX_BATCH, 0, st>>>(B);
  k_project_planes<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(view, n, uv_c, uv_i, depth, cov_c, cov_i, praw,
                                                                kappa, proj);
  note_launch(2);
  return check_launch();
}

int launch_project(const sdgr_scene& scene, int nv, const sdgr_view* views, sdgr_projection* projs,
                   cudaStream_t stream) {
  if (scene.n <= 0 || nv < 1 || nv > SDGR_MAX_BATCH) return SDGR_ERR_INVALID;
  ProjBatch B;
  B.nv = nv;
  B.zero_col2 = 1;
  for (int k = 0; k < nv; ++k) {
    B.view[k] = views[k];
    B.proj[k] = projs[k];
    if (views[k].mc[2] != 0.0 || views[k].mi[2] != 0.0) B.zero_col2 = 0;
  }
  k_project_init<<<1, 4 * SDGR_MAX_BATCH, 0, stream>>>(B);
  const int threads = 256;
  const unsigned blocks = (unsigned)((scene.n + threads - 1) / threads);
  {
    KernelTimer kt(SDGR_K_PROJECT, stream);
    if (scene.dtype == 0 && B.zero_col2)
      k_project<float, true><<<blocks, threads, 0, stream>>>(scene, B);
    else if (scene.dtype == 0)
      k_project<float, false><<<blocks, threads, 0, stream>>>(scene, B);
    else if (B.zero_col2)
      k_project<double, true><<<blocks, threads, 0, stream>>>(scene, B);
    else
      k_project<double, false><<<blocks, threads, 0, stream>>>(scene, B);
  }
  note_launch(2);
  return check_launch();
}

}  // namespace sdgr
