// stages.cu — the reference-shaped outputs of the hot path's stages.
//
// The fused hot path keeps per-Gaussian / per-(tile, Gaussian) state only.
// The reference's stage functions also expose per-(cell, Gaussian) pair
// arrays (forward.RayLists / SplatPairs / IntensityBuffer, forward.py:112-210)
// and per-stage plane-space gradients (backward.py:86-240); these kernels
// produce them on the device from the same records, for callers and tests
// that use the stage API:
//   k_cell_pairs      _footprint_pairs + the (cell, depth, index) lexsort +
//                     CSR offsets of build_ray_lists / _build_splat_pairs
//                     (forward.py:60-155, 213-224): one CTA per 16x16 tile
//                     walks the tile's key list in order, so each cell's
//                     members come out in list order (depth, index / index).
//   k_cell_intensities the per-pair recurrence of compute_intensities
//                     (forward.py:178-199): tau, trans, absorb, contrib.
//   k_stage_grads     per-Gaussian plane-space gradients of
//                     grad_image_stage / grad_intensity_stage (backward.py:86-148).
#include "common.cuh"

namespace sdgr {

struct PlaneSoA {
  const double* uv;
  const double* inv;
  const int16_t* bbox;
  const uint64_t* cmask;
  int nu, nv;
};

// kEmit = false: offsets[cell + 1] = member count of the cell.
// kEmit = true : pairs written at offsets[cell] onward, in tile-list order.
template <bool kEmit>
__global__ void __launch_bounds__(256) k_cell_pairs(PlaneSoA pl, const int32_t* __restrict__ tile_prim,
                                                    const int32_t* __restrict__ range, int tiles_x, double cutoff,
                                                    int64_t* offsets, int32_t* prim, double* delta, double* q,
                                                    double* w) {
  __shared__ uint32_t rows[8 * kRays];   // bit (j & 31) of word j >> 5: Gaussian j of the chunk covers cell r
  __shared__ double su[kChunk], sv[kChunk], sa0[kChunk], sa1[kChunk], sa2[kChunk];
  __shared__ int32_t sg[kChunk];
  const int t = blockIdx.x, tid = threadIdx.x;
  const int tx = t % tiles_x, ty = t / tiles_x;
  const int iu = tx * kTile + (tid & 15), iv = ty * kTile + (tid >> 4);
  const bool valid = iu < pl.nu && iv < pl.nv;
  const int64_t cell = (int64_t)iv * pl.nu + iu;
  int64_t cur = (kEmit && valid) ? offsets[cell] : 0;
  int64_t cnt = 0;
  const int s = range[2 * t], e = range[2 * t + 1];
  for (int c0 = s; c0 < e; c0 += kChunk) {
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 8; ++k) rows[k * kRays + tid] = 0u;
    const int nG = min(kChunk, e - c0);
    uint64_t m[4] = {0, 0, 0, 0};
    if (tid < nG) {
      const int g = tile_prim[c0 + tid];
      const double2 uv = reinterpret_cast<const double2*>(pl.uv)[g];
      const double4 A = reinterpret_cast<const double4*>(pl.inv)[g];
      const short4 bb = reinterpret_cast<const short4*>(pl.bbox)[g];
      member_mask(uv.x, uv.y, A.x, A.y, A.z, pl.cmask[g], bb.x, bb.y, bb.z, bb.w, tx, ty, cutoff, m);
      su[tid] = uv.x; sv[tid] = uv.y; sa0[tid] = A.x; sa1[tid] = A.y; sa2[tid] = A.z; sg[tid] = g;
    }
    __syncthreads();
    {
      const uint32_t bit = 1u << (tid & 31);
      uint32_t* col = rows + (tid >> 5) * kRays;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        uint64_t x = m[k];
        while (x) {
          const int b = __ffsll((long long)x) - 1;
          x &= x - 1;
          atomicOr(col + (k * 64 + b), bit);
        }
      }
    }
    __syncthreads();
    if (!valid) continue;
#pragma unroll 1
    for (int k = 0; k < 8; ++k) {
      uint32_t x = rows[k * kRays + tid];
      if constexpr (!kEmit) {
        cnt += __popc(x);
      } else {
      while (x) {
        const int j = k * 32 + __ffs(x) - 1;
        x &= x - 1;
        const double dx = dsub((double)iu, su[j]), dy = dsub((double)iv, sv[j]);
        const double qq = quadform(sa0[j], sa1[j], sa2[j], dx, dy);
        prim[cur] = sg[j];
        reinterpret_cast<double2*>(delta)[cur] = make_double2(dx, dy);
        q[cur] = qq;
        w[cur] = nexp(-qq);
        ++cur;
      }
      }
    }
  }
  if (!kEmit && valid) offsets[cell + 1] = cnt;
}

// offsets[0] = 0, offsets[1..n] <- inclusive prefix sums (one CTA).
__global__ void __launch_bounds__(1024) k_scan_offsets(int64_t* off, int64_t n) {
  __shared__ int64_t part[1024];
  const int t = threadIdx.x;
  const int64_t per = (n + 1023) / 1024;
  const int64_t b = 1 + t * per, e = min(b + per, n + 1);
  int64_t s = 0;
  for (int64_t i = b; i < e; ++i) s += off[i];
  part[t] = s;
  __syncthreads();
  for (int d = 1; d < 1024; d <<= 1) {   // Hillis-Steele inclusive scan
    const int64_t v = t >= d ? part[t - d] : 0;
    __syncthreads();
    part[t] += v;
    __syncthreads();
  }
  int64_t run = t > 0 ? part[t - 1] : 0;
  for (int64_t i = b; i < e; ++i) {
    run += off[i];
    off[i] = run;
  }
  if (t == 0) off[0] = 0;
}

// compute_intensities per pair (forward.py:178-199): one thread per cell walks
// its run in list order; S is the exclusive prefix of tau within the run.
__global__ void __launch_bounds__(256) k_cell_intensities(const int64_t* __restrict__ off, int64_t n_cells,
                                                          const int32_t* __restrict__ prim,
                                                          const double* __restrict__ w,
                                                          const double* __restrict__ kappa,
                                                          const double* __restrict__ phase, double* tau,
                                                          double* trans, double* absorb, double* contrib) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n_cells) return;
  double S = 0.0;
  for (int64_t p = off[c]; p < off[c + 1]; ++p) {
    const int g = prim[p];
    const double t = kappa[g] * w[p];
    const double T = nexp(-S);
    const double a = nexp(-t);
    tau[p] = t;
    trans[p] = T;
    absorb[p] = a;
    contrib[p] = T * (1.0 - a) * phase[g];
    S += t;
  }
}

// dL/dbeta per imaging pair (backward.py:99): dL/dS[pixel] * I[prim]
__global__ void __launch_bounds__(256) k_splat_pair_grads(int64_t n, const int32_t* __restrict__ pixel,
                                                          const int32_t* __restrict__ prim,
                                                          const double* __restrict__ dLdS,
                                                          const double* __restrict__ I, double* out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = dLdS[pixel[i]] * I[prim[i]];
}

// Plane-space gradients per Gaussian, (8, n) rows:
//   plane 0: dL/dP, dL/dkappa, dL/dSigma_c (4 entries, row-major), dL/du, dL/dv
//            from the per-(tile, Gaussian) partial records in pre-sort order;
//   plane 1: dL/dI, 0, dL/dSigma_i (4), dL/du, dL/dv from the imaging sums.
// dSigma = -A G A (_inverse_chain, backward.py:81-83).
__global__ void __launch_bounds__(256) k_stage_grads(int plane, const uint8_t* __restrict__ flags,
                                                     const double* __restrict__ inv,
                                                     const int32_t* __restrict__ pair_start,
                                                     const int32_t* __restrict__ n_tiles,
                                                     const double* __restrict__ src, int64_t cap, int64_t n,
                                                     double* out) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= n) return;
  double r[7] = {0, 0, 0, 0, 0, 0, 0};
  if (flags[g] & SDGR_FLAG_VISIBLE) {
    if (plane == 0) {
      const int s0 = pair_start[g];
      const int64_t room = cap - s0 > 0 ? cap - s0 : 0;
      const int cnt = n_tiles[g] < room ? n_tiles[g] : (int)room;
      for (int k = 0; k < cnt; ++k)
#pragma unroll
        for (int i = 0; i < 7; ++i) r[i] += src[(int64_t)(s0 + k) * 8 + i];
    } else {
      r[0] = src[g];
#pragma unroll
      for (int i = 1; i < 6; ++i) r[i + 1] = src[i * n + g];
    }
  }
  const double4 A = reinterpret_cast<const double4*>(inv)[g];
  const double a = A.x, b = A.y, c = A.z, g0 = r[2], g1 = r[3], g2 = r[4];
  const double p00 = a * g0 + b * g1, p01 = a * g1 + b * g2;
  const double p10 = b * g0 + c * g1, p11 = b * g1 + c * g2;
  const bool vis = flags[g] & SDGR_FLAG_VISIBLE;
  out[0 * n + g] = r[0];
  out[1 * n + g] = r[1];
  out[2 * n + g] = vis ? -(p00 * a + p01 * b) : 0.0;
  out[3 * n + g] = vis ? -(p00 * b + p01 * c) : 0.0;
  out[4 * n + g] = vis ? -(p10 * a + p11 * b) : 0.0;
  out[5 * n + g] = vis ? -(p10 * b + p11 * c) : 0.0;
  out[6 * n + g] = r[5];
  out[7 * n + g] = r[6];
}

static PlaneSoA plane_soa(const sdgr_plane& p, int nu, int nv) {
  return PlaneSoA{p.uv, p.inv_cov, p.bbox, p.cell_mask, nu, nv};
}

int launch_cell_pairs(const sdgr_projection& p, const sdgr_view& v, const sdgr_tiles& t, int64_t* offsets,
                      int32_t* prim, double* delta, double* q, double* w, cudaStream_t st) {
  const sdgr_plane& pl = t.plane == 0 ? p.comp : p.img;
  const int nu = t.plane == 0 ? v.n_u : v.n_az, nv = t.plane == 0 ? v.n_v : v.n_rg;
  const PlaneSoA ps = plane_soa(pl, nu, nv);
  if (!prim) {
    k_cell_pairs<false><<<t.n_tiles, 256, 0, st>>>(ps, t.pair_prim, t.tile_range, t.tiles_x, v.cutoff, offsets,
                                                    nullptr, nullptr, nullptr, nullptr);
    k_scan_offsets<<<1, 1024, 0, st>>>(offsets, (int64_t)nu * nv);
    note_launch(2);
  } else {
    k_cell_pairs<true><<<t.n_tiles, 256, 0, st>>>(ps, t.pair_prim, t.tile_range, t.tiles_x, v.cutoff, offsets,
                                                   prim, delta, q, w);
    note_launch();
  }
  return check_launch();
}

int launch_cell_intensities(const sdgr_projection& p, int64_t n_cells, const int64_t* off, const int32_t* prim,
                            const double* w, double* tau, double* trans, double* absorb, double* contrib,
                            cudaStream_t st) {
  k_cell_intensities<<<(unsigned)((n_cells + 255) / 256), 256, 0, st>>>(off, n_cells, prim, w, p.kappa, p.phase,
                                                                        tau, trans, absorb, contrib);
  note_launch();
  return check_launch();
}

__global__ void __launch_bounds__(256) k_exp_check(int64_t n, const double* __restrict__ x, double* __restrict__ y) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) y[i] = nexp(x[i]);
}

int launch_exp_check(int64_t n, const double* x, double* y, cudaStream_t st) {
  if (n > 0) k_exp_check<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(n, x, y);
  note_launch();
  return check_launch();
}

int launch_splat_pair_grads(int64_t n, const int32_t* pixel, const int32_t* prim, const double* dLdS,
                            const double* I, double* out, cudaStream_t st) {
  if (n == 0) return SDGR_OK;
  k_splat_pair_grads<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(n, pixel, prim, dLdS, I, out);
  note_launch();
  return check_launch();
}

int launch_stage_grads(const sdgr_projection& p, int plane, const sdgr_tiles* comp, const double* src,
                       double* out, cudaStream_t st) {
  const sdgr_plane& pl = plane == 0 ? p.comp : p.img;
  k_stage_grads<<<(unsigned)((p.n + 255) / 256), 256, 0, st>>>(
      plane, p.flags, pl.inv_cov, comp ? comp->pair_start : nullptr, pl.n_tiles, src, comp ? comp->n_pairs : 0,
      p.n, out);
  note_launch();
  return check_launch();
}

}  // namespace sdgr
