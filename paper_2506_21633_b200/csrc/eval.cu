// eval.cu — point-cloud evaluation on the device:
// nearest-neighbour distances for chamfer / precision-recall-F1 and DBSCAN
// labels (reference: metrics.py:140-183, which uses scipy's cKDTree and
// sklearn's DBSCAN).
//
// Both run on a uniform grid: points are keyed by cell, stably sorted by key
// (the library's onesweep radix sort) and copied into cell order, with a CSR
// of cell ranges.
//   NN:     one thread per query scans Chebyshev rings of cells around its
//           cell until the best squared distance is below the squared
//           distance to every unscanned cell (exact nearest neighbour).
//   DBSCAN: cell edge >= eps, so an eps-ball touches at most the 27
//           surrounding cells.  Core points (>= min_pts points within eps,
//           itself included, like sklearn's radius neighbours with <=) are
//           unioned with a lock-free min-root union-find, so every cluster's
//           root is its smallest core index -- the order in which sklearn's
//           index-order expansion discovers clusters.  A border point takes
//           the smallest root among its core neighbours (the first cluster
//           whose expansion reaches it); noise keeps -1.
// Distances are FP64: d2 = dx^2 + dy^2 + dz^2.
#include <cmath>

#include "common.cuh"

namespace sdgr {

size_t sort_u32_ws_bytes(int64_t n);
int sort_u32(const uint32_t* keys, int64_t n, int bits, uint32_t* keys_out, uint32_t* perm_out, void* ws,
             size_t ws_bytes, cudaStream_t st);

static size_t al(size_t x) { return (x + 255) & ~size_t(255); }

struct Grid {
  double lo[3];
  double h;
  int dims[3];
};

__device__ __forceinline__ int cell_coord(double x, double lo, double h, int dim) {
  double c = floor((x - lo) / h);
  c = fmin(fmax(c, 0.0), (double)(dim - 1));
  return (int)c;
}

__global__ void __launch_bounds__(256) k_cell_keys(const double* pts, int64_t n, Grid G, uint32_t* keys) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int cx = cell_coord(pts[3 * i], G.lo[0], G.h, G.dims[0]);
  const int cy = cell_coord(pts[3 * i + 1], G.lo[1], G.h, G.dims[1]);
  const int cz = cell_coord(pts[3 * i + 2], G.lo[2], G.h, G.dims[2]);
  keys[i] = (uint32_t)((cz * G.dims[1] + cy) * G.dims[0] + cx);
}

// sorted copy of the points and the cell ranges (cell_start preset to -1)
__global__ void __launch_bounds__(256) k_cell_fill(const double* pts, const uint32_t* skeys, const uint32_t* perm,
                                                   int64_t n, double* spts, int32_t* cell_start,
                                                   int32_t* cell_end) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t p = perm[i];
  spts[3 * i] = pts[3 * p];
  spts[3 * i + 1] = pts[3 * p + 1];
  spts[3 * i + 2] = pts[3 * p + 2];
  const uint32_t k = skeys[i];
  if (i == 0 || skeys[i - 1] != k) cell_start[k] = (int32_t)i;
  if (i == n - 1 || skeys[i + 1] != k) cell_end[k] = (int32_t)(i + 1);
}

struct GridWs {
  uint32_t* keys;
  uint32_t* skeys;
  uint32_t* perm;
  double* spts;
  int32_t* cell_start;
  int32_t* cell_end;
  int32_t* aux0;   // DBSCAN: core flags / roots
  int32_t* aux1;
  void* sort_ws;
  size_t sort_bytes;
};

static size_t grid_ws_bytes(int64_t n, int64_t cells) {
  return 3 * al(4 * (size_t)n) + al(24 * (size_t)n) + 2 * al(4 * (size_t)cells) + 2 * al(4 * (size_t)n) +
         sort_u32_ws_bytes(n);
}

static GridWs grid_layout(void* ws, int64_t n, int64_t cells) {
  GridWs w;
  char* p = static_cast<char*>(ws);
  w.keys = reinterpret_cast<uint32_t*>(p); p += al(4 * (size_t)n);
  w.skeys = reinterpret_cast<uint32_t*>(p); p += al(4 * (size_t)n);
  w.perm = reinterpret_cast<uint32_t*>(p); p += al(4 * (size_t)n);
  w.spts = reinterpret_cast<double*>(p); p += al(24 * (size_t)n);
  w.cell_start = reinterpret_cast<int32_t*>(p); p += al(4 * (size_t)cells);
  w.cell_end = reinterpret_cast<int32_t*>(p); p += al(4 * (size_t)cells);
  w.aux0 = reinterpret_cast<int32_t*>(p); p += al(4 * (size_t)n);
  w.aux1 = reinterpret_cast<int32_t*>(p); p += al(4 * (size_t)n);
  w.sort_ws = p;
  w.sort_bytes = sort_u32_ws_bytes(n);
  return w;
}

static int build_grid(const double* pts, int64_t n, const Grid& G, const GridWs& w, cudaStream_t st) {
  const int64_t cells = (int64_t)G.dims[0] * G.dims[1] * G.dims[2];
  int bits = 1;
  while ((int64_t(1) << bits) < cells) ++bits;
  if (cudaMemsetAsync(w.cell_start, 0xff, 4 * (size_t)cells, st) != cudaSuccess ||
      cudaMemsetAsync(w.cell_end, 0xff, 4 * (size_t)cells, st) != cudaSuccess)
    return SDGR_ERR_CUDA;
  const unsigned b = (unsigned)((n + 255) / 256);
  k_cell_keys<<<b, 256, 0, st>>>(pts, n, G, w.keys);
  note_launch();
  int rc = sort_u32(w.keys, n, bits, w.skeys, w.perm, w.sort_ws, w.sort_bytes, st);
  if (rc != SDGR_OK) return rc;
  k_cell_fill<<<b, 256, 0, st>>>(pts, w.skeys, w.perm, n, w.spts, w.cell_start, w.cell_end);
  note_launch();
  return check_launch();
}

__device__ __forceinline__ double sqd(double ax, double ay, double az, double bx, double by, double bz) {
  const double dx = ax - bx, dy = ay - by, dz = az - bz;
  return dx * dx + dy * dy + dz * dz;
}

// ---------------------------------------------------------------- NN ------
__global__ void __launch_bounds__(256) k_nn(const double* q, int64_t nq, Grid G, const double* spts,
                                            const int32_t* cell_start, const int32_t* cell_end, double* d2out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nq) return;
  const double x = q[3 * i], y = q[3 * i + 1], z = q[3 * i + 2];
  const int c[3] = {cell_coord(x, G.lo[0], G.h, G.dims[0]), cell_coord(y, G.lo[1], G.h, G.dims[1]),
                    cell_coord(z, G.lo[2], G.h, G.dims[2])};
  const double qc[3] = {x, y, z};
  double best = INFINITY;
  const int rmax = max(G.dims[0], max(G.dims[1], G.dims[2]));
  for (int r = 0; r <= rmax; ++r) {
    // cells at Chebyshev distance exactly r from c (clipped to the grid)
    const int z0 = max(c[2] - r, 0), z1 = min(c[2] + r, G.dims[2] - 1);
    const int y0 = max(c[1] - r, 0), y1 = min(c[1] + r, G.dims[1] - 1);
    const int x0 = max(c[0] - r, 0), x1 = min(c[0] + r, G.dims[0] - 1);
    for (int cz = z0; cz <= z1; ++cz)
      for (int cy = y0; cy <= y1; ++cy) {
        const bool zy_edge = (cz == c[2] - r || cz == c[2] + r || cy == c[1] - r || cy == c[1] + r);
        // rows inside the ring's z/y extent only contribute their two x ends
        const int step = (zy_edge || r == 0) ? 1 : 2 * r;
        for (int cx = zy_edge ? x0 : c[0] - r; cx <= x1; cx += step) {
          if (cx < x0) continue;
          const int cell = (cz * G.dims[1] + cy) * G.dims[0] + cx;
          const int s = cell_start[cell];
          if (s < 0) continue;
          const int e = cell_end[cell];
          for (int j = s; j < e; ++j) {
            const double d = sqd(x, y, z, spts[3 * j], spts[3 * j + 1], spts[3 * j + 2]);
            best = d < best ? d : best;
          }
        }
      }
    // lower bound on the distance to any cell outside the scanned block
    double bound = INFINITY;
    for (int a = 0; a < 3; ++a) {
      if (c[a] - r > 0) bound = fmin(bound, qc[a] - (G.lo[a] + (double)(c[a] - r) * G.h));
      if (c[a] + r < G.dims[a] - 1) bound = fmin(bound, G.lo[a] + (double)(c[a] + r + 1) * G.h - qc[a]);
    }
    if (bound == INFINITY) break;                       // the whole grid was scanned
    bound -= 1e-12 * (G.h + fabs(bound));               // cell assignment rounds by ~1 ulp
    if (bound > 0.0 && best <= bound * bound) break;
  }
  d2out[i] = best;
}

// ------------------------------------------------------------ DBSCAN ------
__global__ void __launch_bounds__(256) k_db_core(int64_t n, Grid G, const double* spts, const int32_t* cell_start,
                                                 const int32_t* cell_end, double eps2, int min_pts, int32_t* core) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;   // sorted order
  if (i >= n) return;
  const double x = spts[3 * i], y = spts[3 * i + 1], z = spts[3 * i + 2];
  const int cx = cell_coord(x, G.lo[0], G.h, G.dims[0]), cy = cell_coord(y, G.lo[1], G.h, G.dims[1]),
            cz = cell_coord(z, G.lo[2], G.h, G.dims[2]);
  int cnt = 0;
  for (int zz = max(cz - 1, 0); zz <= min(cz + 1, G.dims[2] - 1) && cnt < min_pts; ++zz)
    for (int yy = max(cy - 1, 0); yy <= min(cy + 1, G.dims[1] - 1) && cnt < min_pts; ++yy)
      for (int xx = max(cx - 1, 0); xx <= min(cx + 1, G.dims[0] - 1); ++xx) {
        const int cell = (zz * G.dims[1] + yy) * G.dims[0] + xx;
        const int s = cell_start[cell];
        if (s < 0) continue;
        const int e = cell_end[cell];
        for (int j = s; j < e; ++j) cnt += sqd(x, y, z, spts[3 * j], spts[3 * j + 1], spts[3 * j + 2]) <= eps2;
      }
  core[i] = cnt >= min_pts;
}

// parent pointers hold ORIGINAL indices (perm) so roots are minimum original
// core indices; parent[k] indexed by sorted position
__device__ int32_t find_root(int32_t* parent, const int32_t* pos_of, int32_t a) {
  // a: original index; walk via sorted positions with path halving (a benign
  // race: a node's parent only ever moves to one of its ancestors)
  while (true) {
    const int32_t p = parent[pos_of[a]];
    if (p == a) return a;
    const int32_t gp = parent[pos_of[p]];
    if (gp != p) parent[pos_of[a]] = gp;
    a = gp;
  }
}

__global__ void __launch_bounds__(256) k_db_init(int64_t n, const uint32_t* perm, const int32_t* core,
                                                 int32_t* parent, int32_t* pos_of) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  parent[i] = core[i] ? (int32_t)perm[i] : -1;
  pos_of[perm[i]] = (int32_t)i;
}

__global__ void __launch_bounds__(256) k_db_link(int64_t n, Grid G, const double* spts, const uint32_t* perm,
                                                 const int32_t* cell_start, const int32_t* cell_end, double eps2,
                                                 const int32_t* core, int32_t* parent, const int32_t* pos_of) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n || !core[i]) return;
  const int32_t me = (int32_t)perm[i];
  const double x = spts[3 * i], y = spts[3 * i + 1], z = spts[3 * i + 2];
  const int cx = cell_coord(x, G.lo[0], G.h, G.dims[0]), cy = cell_coord(y, G.lo[1], G.h, G.dims[1]),
            cz = cell_coord(z, G.lo[2], G.h, G.dims[2]);
  for (int zz = max(cz - 1, 0); zz <= min(cz + 1, G.dims[2] - 1); ++zz)
    for (int yy = max(cy - 1, 0); yy <= min(cy + 1, G.dims[1] - 1); ++yy)
      for (int xx = max(cx - 1, 0); xx <= min(cx + 1, G.dims[0] - 1); ++xx) {
        const int cell = (zz * G.dims[1] + yy) * G.dims[0] + xx;
        const int s = cell_start[cell];
        if (s < 0) continue;
        const int e = cell_end[cell];
        for (int j = s; j < e; ++j) {
          if (!core[j]) continue;
          const int32_t other = (int32_t)perm[j];
          if (other >= me) continue;   // each core-core edge once
          if (sqd(x, y, z, spts[3 * j], spts[3 * j + 1], spts[3 * j + 2]) > eps2) continue;
          // union by minimum root (lock-free: hook the larger root under the smaller)
          int32_t a = find_root(parent, pos_of, me), b = find_root(parent, pos_of, other);
          while (a != b) {
            if (a < b) { const int32_t t = a; a = b; b = t; }   // a > b: hook a under b
            const int32_t old = atomicCAS(&parent[pos_of[a]], a, b);
            if (old == a) break;
            a = find_root(parent, pos_of, old);
            b = find_root(parent, pos_of, b);
          }
        }
      }
}

// root (minimum core index of the cluster) per point in ORIGINAL order; border
// points: the smallest root among core neighbours; noise: -1
__global__ void __launch_bounds__(256) k_db_label(int64_t n, Grid G, const double* spts, const uint32_t* perm,
                                                  const int32_t* cell_start, const int32_t* cell_end, double eps2,
                                                  const int32_t* core, int32_t* parent, const int32_t* pos_of,
                                                  int32_t* root_out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int32_t me = (int32_t)perm[i];
  if (core[i]) {
    root_out[me] = find_root(parent, pos_of, me);
    return;
  }
  const double x = spts[3 * i], y = spts[3 * i + 1], z = spts[3 * i + 2];
  const int cx = cell_coord(x, G.lo[0], G.h, G.dims[0]), cy = cell_coord(y, G.lo[1], G.h, G.dims[1]),
            cz = cell_coord(z, G.lo[2], G.h, G.dims[2]);
  int32_t best = INT32_MAX;
  for (int zz = max(cz - 1, 0); zz <= min(cz + 1, G.dims[2] - 1); ++zz)
    for (int yy = max(cy - 1, 0); yy <= min(cy + 1, G.dims[1] - 1); ++yy)
      for (int xx = max(cx - 1, 0); xx <= min(cx + 1, G.dims[0] - 1); ++xx) {
        const int cell = (zz * G.dims[1] + yy) * G.dims[0] + xx;
        const int s = cell_start[cell];
        if (s < 0) continue;
        const int e = cell_end[cell];
        for (int j = s; j < e; ++j) {
          if (!core[j]) continue;
          if (sqd(x, y, z, spts[3 * j], spts[3 * j + 1], spts[3 * j + 2]) > eps2) continue;
          const int32_t r = find_root(parent, pos_of, (int32_t)perm[j]);
          best = r < best ? r : best;
        }
      }
  root_out[me] = best == INT32_MAX ? -1 : best;
}

static bool grid_ok(const double* lo, double h, const int32_t* dims, int64_t* cells) {
  if (!lo || !dims || !(h > 0.0) || !std::isfinite(h)) return false;
  int64_t c = 1;
  for (int a = 0; a < 3; ++a) {
    if (dims[a] < 1 || dims[a] > 4096 || !std::isfinite(lo[a])) return false;
    c *= dims[a];
  }
  if (c > (int64_t(1) << 24)) return false;
  *cells = c;
  return true;
}

static Grid make_grid(const double* lo, double h, const int32_t* dims) {
  Grid G;
  for (int a = 0; a < 3; ++a) { G.lo[a] = lo[a]; G.dims[a] = dims[a]; }
  G.h = h;
  return G;
}

}  // namespace sdgr

using namespace sdgr;

extern "C" {

size_t sdgr_grid_workspace_bytes(int64_t n, int64_t n_cells) {
  if (n < 1) n = 1;
  if (n_cells < 1) n_cells = 1;
  return grid_ws_bytes(n, n_cells);
}

int sdgr_nn_sqdist(const double* ref, int64_t n_ref, const double* query, int64_t n_query, const double* lo,
                   double h, const int32_t* dims, double* d2, void* ws, size_t ws_bytes, void* stream) {
  int64_t cells = 0;
  if (!ref || !query || !d2 || !ws || n_ref < 1 || n_query < 0 || !grid_ok(lo, h, dims, &cells))
    return SDGR_ERR_INVALID;
  if (n_ref > 0x7fffffffLL || n_query > 0x7fffffffLL) return SDGR_ERR_INVALID;
  if (ws_bytes < grid_ws_bytes(n_ref, cells)) return SDGR_ERR_CAPACITY;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const Grid G = make_grid(lo, h, dims);
  const GridWs w = grid_layout(ws, n_ref, cells);
  int rc = build_grid(ref, n_ref, G, w, st);
  if (rc != SDGR_OK || n_query == 0) return rc;
  k_nn<<<(unsigned)((n_query + 255) / 256), 256, 0, st>>>(query, n_query, G, w.spts, w.cell_start, w.cell_end, d2);
  note_launch();
  return check_launch();
}

int sdgr_dbscan(const double* pts, int64_t n, const double* lo, double h, const int32_t* dims, double eps,
                int32_t min_pts, int32_t* root, void* ws, size_t ws_bytes, void* stream) {
  int64_t cells = 0;
  if (!pts || !root || !ws || n < 1 || !grid_ok(lo, h, dims, &cells)) return SDGR_ERR_INVALID;
  if (!(eps > 0.0) || !std::isfinite(eps) || h < eps || min_pts < 1 || n > 0x7fffffffLL) return SDGR_ERR_INVALID;
  if (ws_bytes < grid_ws_bytes(n, cells)) return SDGR_ERR_CAPACITY;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const Grid G = make_grid(lo, h, dims);
  const GridWs w = grid_layout(ws, n, cells);
  int rc = build_grid(pts, n, G, w, st);
  if (rc != SDGR_OK) return rc;
  const double eps2 = eps * eps;
  const unsigned b = (unsigned)((n + 255) / 256);
  int32_t* core = w.aux0;
  int32_t* parent = w.aux1;
  int32_t* pos_of = reinterpret_cast<int32_t*>(w.keys);   // keys are dead after the sort
  k_db_core<<<b, 256, 0, st>>>(n, G, w.spts, w.cell_start, w.cell_end, eps2, min_pts, core);
  k_db_init<<<b, 256, 0, st>>>(n, w.perm, core, parent, pos_of);
  k_db_link<<<b, 256, 0, st>>>(n, G, w.spts, w.perm, w.cell_start, w.cell_end, eps2, core, parent, pos_of);
  k_db_label<<<b, 256, 0, st>>>(n, G, w.spts, w.perm, w.cell_start, w.cell_end, eps2, core, parent, pos_of, root);
  note_launch(4);
  return check_launch();
}

}  // extern "C"
