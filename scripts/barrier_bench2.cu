// barrier_bench2.cu — dev microbenchmark: grid all-reduce barrier cost vs
// participant count, and a cluster-hierarchical variant (DSMEM inside a
// cluster, global slot polling among clusters).
#include <cooperative_groups.h>
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

constexpr int kBlock = 512;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ void fence_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ void st_v2(unsigned long long* p, unsigned long long a, unsigned long long b) {
  asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b) : "memory");
}
__device__ __forceinline__ void ld_v2(const unsigned long long* p, unsigned long long& a, unsigned long long& b) {
  asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
}

struct Sm {
  double red[32];
  double bcast;
  double cpart;  // this CTA's block sum, read by the cluster over DSMEM
};

// CL = cluster size (1 = flat).  Slots: one per cluster.
template <int CL, int FENCE, bool PAR = false>
__global__ void __launch_bounds__(kBlock, 1) bar_kernel(unsigned long long* slots, int iters, double* out) {
  __shared__ Sm sm;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int nclu = gridDim.x / CL;
  double acc = 0.0;
  cg::cluster_group cl = cg::this_cluster();
  const int crank = CL > 1 ? (int)cl.block_rank() : 0;
  const int cid = blockIdx.x / CL;
  for (uint32_t epoch = 1; epoch <= (uint32_t)iters; ++epoch) {
    double v = (double)(blockIdx.x + threadIdx.x) * 1e-3 + epoch;
    v = warp_sum(v);
    if (lane == 0) sm.red[w] = v;
    __syncthreads();
    if (w == 0) {
      double bs = lane < 16 ? sm.red[lane] : 0.0;
      bs = warp_sum(bs);
      if (lane == 0) sm.cpart = bs;
    }
    double csum = 0.0;
    if (CL > 1) {
      cl.sync();  // release/acquire at cluster scope; publishes cpart
      if (w == 0) {
        double t = 0.0;
        if (lane < CL) t = *cl.map_shared_rank(&sm.cpart, lane);
        csum = warp_sum(t);  // same order in every CTA of the cluster
      }
    } else {
      csum = (w == 0) ? __shfl_sync(0xffffffffu, sm.cpart, 0) : 0.0;
    }
    if (w == 0) {
      unsigned long long* bank = slots + (size_t)(epoch & 1u) * nclu * 32;
      if (lane == 0 && crank == 0) {
        if (FENCE & 1) fence_gpu();
        const unsigned long long bits = (unsigned long long)__double_as_longlong(csum);
        st_v2(bank + (size_t)32 * cid, (bits & 0xffffffff00000000ull) | epoch, (bits << 32) | epoch);
      }
      double s = 0.0;
      if (PAR) {
        constexpr int P = 10;
        unsigned long long a[P], c[P];
        bool pend[P];
#pragma unroll
        for (int u = 0; u < P; ++u) pend[u] = lane + 32 * u < nclu;
        bool any = true;
        while (any) {
#pragma unroll
          for (int u = 0; u < P; ++u)
            if (pend[u]) ld_v2(bank + (size_t)32 * (lane + 32 * u), a[u], c[u]);
          any = false;
#pragma unroll
          for (int u = 0; u < P; ++u)
            if (pend[u]) {
              pend[u] = (uint32_t)a[u] != epoch || (uint32_t)c[u] != epoch;
              any |= pend[u];
            }
        }
#pragma unroll
        for (int u = 0; u < P; ++u)
          if (lane + 32 * u < nclu)
            s += __longlong_as_double((long long)((a[u] & 0xffffffff00000000ull) | (c[u] >> 32)));
      } else {
        for (int t = lane; t < nclu; t += 32) {
          unsigned long long a, c;
          do {
            ld_v2(bank + (size_t)32 * t, a, c);
          } while ((uint32_t)a != epoch || (uint32_t)c != epoch);
          s += __longlong_as_double((long long)((a & 0xffffffff00000000ull) | (c >> 32)));
        }
      }
      if (FENCE & 2) fence_gpu();
      s = warp_sum(s);
      if (lane == 0) sm.bcast = s;
    }
    if (CL > 1) cl.sync();  // cpart reuse + bcast
    else __syncthreads();
    acc += sm.bcast;
  }
  if (threadIdx.x == 0) out[blockIdx.x] = acc;
}

template <int CL, int FENCE, bool PAR = false>
void run(int G, int iters) {
  unsigned long long* slots;
  double* out;
  cudaMalloc(&slots, sizeof(unsigned long long) * 2 * 32 * 1024);
  cudaMalloc(&out, 8 * 1024);
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    cudaMemset(slots, 0, sizeof(unsigned long long) * 2 * 32 * 1024);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(G);
    cfg.blockDim = dim3(kBlock);
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    at[1].id = cudaLaunchAttributeClusterDimension;
    at[1].val.clusterDim.x = CL;
    at[1].val.clusterDim.y = 1;
    at[1].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    if (CL > 8) cudaFuncSetAttribute(bar_kernel<CL, FENCE, PAR>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    cudaError_t e = cudaLaunchKernelEx(&cfg, bar_kernel<CL, FENCE, PAR>, slots, iters, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaError_t e2 = cudaGetLastError();
    if (e != cudaSuccess || e2 != cudaSuccess) {
      printf("CL=%2d G=%4d fence=%d: failed %s / %s\n", CL, G, FENCE, cudaGetErrorString(e), cudaGetErrorString(e2));
      cudaDeviceReset();
      return;
    }
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  printf("CL=%2d G=%4d fence=%d par=%d  %.3f us/barrier\n", CL, G, FENCE, (int)PAR, best * 1e3f / iters);
  cudaFree(slots);
  cudaFree(out);
}

int main() {
  const int it = 20000;
  for (int G : {8, 32, 74, 148}) run<1, 3, true>(G, it);
  run<1, 0, true>(148, it);
  run<1, 1, true>(148, it);
  run<1, 2, true>(148, it);
  run<1, 3, false>(148, it);
  run<4, 3, true>(148, it);
  run<2, 3, true>(148, it);
  return 0;
}
