// ops.cuh — the reference's per-op kernel API (kernels/__init__.py:67-103)
// as standalone device kernels, plus the in-HBM problem generators.
#pragma once
#include "lines.cuh"

namespace spcg {

// y = A x over the tile table (same staging + line bodies as the CG kernel).
template <int FMT, bool WIDE = false>
__global__ void __launch_bounds__(kBlock, kStreamMinBlocks) spmv_kernel(const MatView M, const double* x,
                                                         double* y) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  Smem& sm = *reinterpret_cast<Smem*>(smem_raw);
  constexpr bool TWO = (FMT == K_SCSR_PRIV);
  smem_init(sm);
  Pipe P;
  pipe_start<TWO>(P, sm, M);
  SrcPlain src{x};
  for (int j = 0; j < P.m; ++j) {
    const int s = pipe_acquire(P, sm, j);
    if (WIDE && wide_tile<FMT>(sm, s)) {
      LineOut o2[2];
      bool act[2];
      int li[2];
      csr_line_pair(sm, s, src, o2, act, li, nullptr);
#pragma unroll
      for (int t = 0; t < 2; ++t)
        if (act[t]) y[li[t]] = o2[t].q;
    } else {
      bool active = false;
      int line = -1;
      const LineOut o = tile_line<FMT, false>(sm, s, M, src, y, active, line, sm.val[s]);
      if (active) finish_plain<FMT>(o, line, y);
    }
    pipe_release<TWO>(P, sm, M, s);
  }
  pipe_drain(P, sm);
}

// Deterministic dot, phase 1: fixed element->thread map, per-thread
// sequential FMA sums, fixed-order block sum -> part[blockIdx].
__global__ void __launch_bounds__(kBlock) dot_partial_kernel(long long n, const double* u,
                                                             const double* v, double* part) {
  __shared__ double red[32];
  double s = 0.0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    s = fma(u[i], v[i], s);
  s = warp_sum(s);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) red[w] = s;
  __syncthreads();
  if (w == 0) {
    double t = lane < (int)(blockDim.x >> 5) ? red[lane] : 0.0;
    t = warp_sum(t);
    if (lane == 0) part[blockIdx.x] = t;
  }
}

// Phase 2: one CTA sums the block partials in fixed order.
__global__ void __launch_bounds__(kBlock) dot_final_kernel(int nparts, const double* part,
                                                           double* out) {
  __shared__ double red[32];
  double s = 0.0;
  for (int i = threadIdx.x; i < nparts; i += blockDim.x) s += part[i];
  s = warp_sum(s);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) red[w] = s;
  __syncthreads();
  if (w == 0) {
    double t = lane < (int)(blockDim.x >> 5) ? red[lane] : 0.0;
    t = warp_sum(t);
    if (lane == 0) *out = t;
  }
}

// out = v + alpha*u (IEEE mul then add: bitwise equal to axpy_kernel).
__global__ void __launch_bounds__(kBlock) axpy_kernel(long long n, double alpha, const double* u,
                                                      const double* v, double* out) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    out[i] = mul_add_rn(v[i], alpha, u[i]);
}

// ---- generators -----------------------------------------------------------
// Stencil on an nx*ny*nz grid in natural order (node = ix + nx*(iy + ny*iz)).
// Neighbour offsets are visited in ascending linear order, which is the
// (row, col)-sorted order build_csr_from_triplets produces (core.py:190-200).
// kind 0: 5-point 2-D (nz = 1), diag 4 (genprob.poisson2d)
// kind 1: 7-point 3-D, diag 6 (genprob.poisson3d)
// kind 2: 27-point 3-D, diag 26, off-diagonal -1
// part 0: full, 1: lower incl. diagonal (L+D), 2: strictly upper (= CSR of L^T)
__device__ __forceinline__ int stencil_row(int kind, int part, long long i, int nx, int ny, int nz,
                                           int* cols, double* vals) {
  const int ix = (int)(i % nx);
  const int iy = (int)((i / nx) % ny);
  const int iz = (int)(i / ((long long)nx * ny));
  const long long nxy = (long long)nx * ny;
  int c = 0;
  const double diag = kind == 0 ? 4.0 : (kind == 1 ? 6.0 : 26.0);
  for (int dz = -1; dz <= 1; ++dz)
    for (int dy = -1; dy <= 1; ++dy)
      for (int dx = -1; dx <= 1; ++dx) {
        const int nnzoff = (dx != 0) + (dy != 0) + (dz != 0);
        if (kind == 0 && (dz != 0 || nnzoff > 1)) continue;
        if (kind == 1 && nnzoff > 1) continue;
        const int jx = ix + dx, jy = iy + dy, jz = iz + dz;
        if (jx < 0 || jx >= nx || jy < 0 || jy >= ny || jz < 0 || jz >= nz) continue;
        const long long j = i + dz * nxy + (long long)dy * nx + dx;
        if (part == 1 && j > i) continue;
        if (part == 2 && j <= i) continue;
        if (cols) {
          cols[c] = (int)j;
          vals[c] = (j == i) ? diag : -1.0;
        }
        ++c;
      }
  return c;
}

// Rows [row0, row0+nrows) of the global stencil (global column ids).
__global__ void stencil_count_kernel(int kind, int part, long long row0, long long nrows, int nx,
                                     int ny, int nz, int* counts) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < nrows; t += stride)
    counts[t] = stencil_row(kind, part, row0 + t, nx, ny, nz, nullptr, nullptr);
}

__global__ void stencil_fill_kernel(int kind, int part, long long row0, long long nrows, int nx,
                                    int ny, int nz, const int* ptr, int* idx, double* val) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < nrows; t += stride) {
    int cols[27];
    double vals[27];
    const int c = stencil_row(kind, part, row0 + t, nx, ny, nz, cols, vals);
    const int k0 = ptr[t];
    for (int u = 0; u < c; ++u) {
      idx[k0 + u] = cols[u];
      val[k0 + u] = vals[u];
    }
  }
}

// Per-tile column extent (max, min over both segments), one CTA per tile.
__global__ void tile_colext_kernel(const int4* tdesc, const int2* tdescB, int ntiles,
                                   const int* idxA, const int* idxB, int* colmax, int* colmin) {
  __shared__ int smax[32], smin[32];
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int4 d = tdesc[t];
    int mx = -1, mn = 0x7fffffff;
    for (int k = d.z + threadIdx.x; k < d.w; k += blockDim.x) {
      const int c = idxA[k];
      mx = max(mx, c);
      mn = min(mn, c);
    }
    if (tdescB) {
      const int2 e = tdescB[t];
      for (int k = e.x + threadIdx.x; k < e.y; k += blockDim.x) {
        const int c = idxB[k];
        mx = max(mx, c);
        mn = min(mn, c);
      }
    }
    for (int o = 16; o > 0; o >>= 1) {
      mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    }
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) {
      smax[w] = mx;
      smin[w] = mn;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int i = 1; i < (int)(blockDim.x >> 5); ++i) {
        mx = max(mx, smax[i]);
        mn = min(mn, smin[i]);
      }
      colmax[t] = mx;
      colmin[t] = mn;
    }
  }
}

// Leading-edge window of tile t: the columns beyond everything tile t-1
// touched (banded / stencil matrices: ~one tile's worth of new columns);
// empty when the tile brings nothing new or the window exceeds `cap`.
__global__ void tile_window_kernel(int ntiles, const int* colmax, const int* colmin, int cap,
                                   int2* twin) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= ntiles) return;
  const int hi = colmax[t];
  int lo = colmin[t];
  if (t > 0) lo = max(lo, colmax[t - 1] + 1);
  if (hi < 0 || hi - lo + 1 > cap) lo = hi + 1;
  twin[t] = make_int2(lo, hi);
}

// int64 -> int32 narrowing on the device (upload path).
__global__ void narrow_i64_kernel(long long n, const long long* src, int* dst) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    dst[i] = (int)src[i];
}

}  // namespace spcg
