// assemble.cuh — matrix assembly in HBM from coordinate data.
//
// Two users:
//  * the generators of genprob.random_spd / fem_mesh (genprob.py:96-129 of
//    spcg; the 30880-row F-mesh of SURVEY §8d): the host draws the random
//    pairs exactly as the reference does (numpy PCG64), the device mirrors
//    them, forms the diagonal and assembles CSR / SCSR (+ L^T) / CSC;
//  * the device upload of a .spcg container (matio.py:171-208): u64 offsets
//    and u32 indices converted and validated on the device.
//
// The diagonal of the generators is d_i = sum |v| over row i's entries in
// the order [I-occurrences in draw order, J-occurrences in draw order] +
// shift: np.bincount's sequential accumulation, reproduced by a STABLE radix
// sort of the entries by row followed by an in-order per-row sum, so the
// device matrix is bitwise the host generator's.
#pragma once
#include <cub/device/device_radix_sort.cuh>

namespace spcg {

enum : int {
  ASM_ERR_RANGE = 1,      // a pair outside 0 <= J < I < n
  ASM_ERR_DUPLICATE = 2,  // the same (row, col) twice
  ASM_ERR_OFFSETS = 4,    // offsets not 0 .. nnz non-decreasing
  ASM_ERR_INDEX = 8,      // index outside [0, n)
  ASM_ERR_DIAG = 16,      // SCSR row without a final diagonal entry
  ASM_ERR_UPPER = 32      // SCSR entry above the diagonal
};

// e in [0, 2m): the mirrored off-diagonal entries (row of entry e, its id)
__global__ void asm_rows_kernel(long long m, int n, const long long* I, const long long* J,
                                int* rows, int* ids, int* err) {
  const long long G = (long long)gridDim.x * blockDim.x;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < 2 * m; e += G) {
    const long long k = e < m ? e : e - m;
    const long long i = I[k], j = J[k];
    if (!(j >= 0 && j < i && i < n)) atomicOr(err, ASM_ERR_RANGE);
    rows[e] = (int)(e < m ? i : j);
    ids[e] = (int)e;
  }
}

// d_i = (entries of row i in array order) sum |v| + shift, like np.bincount
__global__ void asm_diag_kernel(int n, const int* seg, const int* ids, long long m, const double* v,
                                double shift, double* diag) {
  const int G = gridDim.x * blockDim.x;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += G) {
    double d = 0.0;
    for (int k = seg[i]; k < seg[i + 1]; ++k) {
      const long long e = ids[k];
      d = __dadd_rn(d, fabs(v[e < m ? e : e - m]));
    }
    diag[i] = __dadd_rn(d, shift);
  }
}

// per-row counts from sorted rows (segment offsets by a histogram)
__global__ void asm_hist_kernel(long long cnt, const int* rows, int* hist) {
  const long long G = (long long)gridDim.x * blockDim.x;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < cnt; e += G)
    atomicAdd(hist + rows[e], 1);
}

// keys (row << 32 | col) of every matrix entry: the 2m mirrored pairs (only
// the m lower ones when lower_only) and the n diagonal entries; vid: value id
// (e < 2m: pair value, 2m + i: diagonal i)
__global__ void asm_keys_kernel(long long m, int n, const long long* I, const long long* J,
                                int lower_only, unsigned long long* keys, int* vid) {
  const long long off = lower_only ? m : 2 * m;
  const long long total = off + n;
  const long long G = (long long)gridDim.x * blockDim.x;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += G) {
    unsigned long long r, c;
    int id;
    if (e < off) {
      const long long k = e < m ? e : e - m;
      r = (unsigned long long)(e < m ? I[k] : J[k]);
      c = (unsigned long long)(e < m ? J[k] : I[k]);
      id = (int)e;
    } else {
      r = c = (unsigned long long)(e - off);
      id = (int)(2 * m + (e - off));
    }
    keys[e] = (r << 32) | c;
    vid[e] = id;
  }
}

// rows of sorted keys: count entries with col <= row (A) and col > row (B,
// SCSR's L^T); flag duplicates
__global__ void asm_count_kernel(long long total, const unsigned long long* keys, int split,
                                 int* cntA, int* cntB, int* err) {
  const long long G = (long long)gridDim.x * blockDim.x;
  for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < total; k += G) {
    const unsigned long long key = keys[k];
    if (k > 0 && keys[k - 1] == key) atomicOr(err, ASM_ERR_DUPLICATE);
    const int r = (int)(key >> 32), c = (int)(key & 0xffffffffu);
    if (split && c > r) atomicAdd(cntB + r, 1);
    else atomicAdd(cntA + r, 1);
  }
}

// sorted key k -> its slot in A (row r: the first cntA[r] entries of the row's
// run) or B (the rest); value by id
__global__ void asm_scatter_kernel(long long total, const unsigned long long* keys, const int* vid,
                                   long long m, const double* v, const double* diag,
                                   const int* ptrA, const int* ptrB, int* idxA, double* valA,
                                   int* idxB, double* valB) {
  const long long G = (long long)gridDim.x * blockDim.x;
  for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < total; k += G) {
    const unsigned long long key = keys[k];
    const int r = (int)(key >> 32), c = (int)(key & 0xffffffffu);
    const long long id = vid[k];
    const double val = id < 2 * m ? v[id < m ? id : id - m] : diag[id - 2 * m];
    const long long start = (long long)ptrA[r] + (ptrB ? ptrB[r] : 0);
    const long long t = k - start;
    const long long na = ptrA[r + 1] - ptrA[r];
    if (t < na) {
      idxA[ptrA[r] + t] = c;
      valA[ptrA[r] + t] = val;
    } else {
      idxB[ptrB[r] + (t - na)] = c;
      valB[ptrB[r] + (t - na)] = val;
    }
  }
}

// ---- device upload of host / container arrays ------------------------------
// offsets (u64 / i64) -> int32 with the checks of core.py:117-131
template <class PT>
__global__ void conv_ptr_kernel(long long n, long long nnz, const PT* src, int* dst, int* err) {
  const long long G = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i <= n; i += G) {
    const long long v = (long long)src[i];
    bool bad = v < 0 || v > nnz || (i == 0 && v != 0) || (i == n && v != nnz);
    if (i > 0 && (long long)src[i - 1] > v) bad = true;
    if (bad) atomicOr(err, ASM_ERR_OFFSETS);
    dst[i] = (int)v;
  }
}

// indices -> int32 (range check); SCSR: col <= row and the diagonal last;
// also the strictly-lower keys (col << 32 | row) for the L^T sort
template <class IT>
__global__ void conv_idx_kernel(int n, int scsr, const int* ptr, const IT* src, int* dst,
                                int* err, unsigned long long* tkeys, int* tvid, int* tcount) {
  const int lane = threadIdx.x & 31;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  for (int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n; i += warps) {
    const int a = ptr[i], b = ptr[i + 1];
    for (int k = a + lane; k < b; k += 32) {
      const long long c = (long long)src[k];
      if (c < 0 || c >= n) atomicOr(err, ASM_ERR_INDEX);
      dst[k] = (int)c;
      if (scsr) {
        if (c > i) atomicOr(err, ASM_ERR_UPPER);
        if (c < i && tkeys) {
          const int slot = atomicAdd(tcount, 1);
          tkeys[slot] = ((unsigned long long)c << 32) | (unsigned long long)i;
          tvid[slot] = k;
        }
      }
    }
    if (scsr && lane == 0 && (b <= a || (long long)src[b - 1] != i)) atomicOr(err, ASM_ERR_DIAG);
  }
}

// L^T rows from the sorted (col << 32 | row) keys of the strict entries
__global__ void lt_scatter_kernel(long long cnt, const unsigned long long* keys, const int* vid,
                                  const double* val, int* idxB, double* valB) {
  const long long G = (long long)gridDim.x * blockDim.x;
  for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < cnt; k += G) {
    const unsigned long long key = keys[k];  // (row of L^T = column of L) << 32 | row of L
    idxB[k] = (int)(key & 0xffffffffu);
    valB[k] = val[vid[k]];
  }
}

__global__ void lt_hist_kernel(long long cnt, const unsigned long long* keys, int* hist) {
  const long long G = (long long)gridDim.x * blockDim.x;
  for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < cnt; k += G)
    atomicAdd(hist + (int)(keys[k] >> 32), 1);
}

}  // namespace spcg
