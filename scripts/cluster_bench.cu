// Dev microbenchmark (not product code): (1) per-SM L2 read bandwidth when
// G CTAs (one per SM) each re-read a private L2-resident region, by plain
// vector loads and by TMA bulk copies; (2) cluster barrier + DSMEM
// all-reduce latency for cluster sizes 8 and 16.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o cb scripts/cluster_bench.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>
#include <vector>
namespace cg = cooperative_groups;

__global__ void l2_ld(const double2* __restrict__ buf, size_t per_cta, int reps, double* out) {
  const double2* b = buf + blockIdx.x * (per_cta / 16);
  double acc = 0.0;
  for (int r = 0; r < reps; ++r)
    for (size_t i = threadIdx.x; i < per_cta / 16; i += blockDim.x) {
      double2 v = __ldcg(b + i);
      acc += v.x + v.y;
    }
  if (acc == 1.2345) out[0] = acc;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__global__ void l2_tma(const char* __restrict__ buf, size_t per_cta, int reps, double* out) {
  extern __shared__ __align__(128) char sm[];
  __shared__ __align__(8) uint64_t bar;
  const char* b = buf + blockIdx.x * per_cta;
  const int chunk = 32768;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  uint32_t phase = 0;
  double acc = 0.0;
  for (int r = 0; r < reps; ++r)
    for (size_t off = 0; off < per_cta; off += 4 * chunk) {
      if (threadIdx.x == 0) {
        const uint32_t bytes = (uint32_t)min((size_t)4 * chunk, per_cta - off);
        asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)),
                     "r"(bytes));
        for (uint32_t c = 0; c < bytes; c += chunk)
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                  smem_u32(sm + c)),
              "l"(b + off + c), "r"((uint32_t)min((uint32_t)chunk, bytes - c)), "r"(smem_u32(&bar))
              : "memory");
      }
      asm volatile(
          "{ .reg .pred p; W: mbarrier.try_wait.parity.shared.b64 p, [%0], %1; @!p bra W; }" ::"r"(
              smem_u32(&bar)),
          "r"(phase));
      phase ^= 1;
      acc += ((double*)sm)[threadIdx.x];
      __syncthreads();
    }
  if (acc == 1.2345) out[0] = acc;
}

// cluster all-reduce of one double per CTA: DSMEM writes into CTA 0's slots
// ... here: every CTA writes its value into every CTA's slot array, then one
// barrier.cluster; each CTA sums locally in fixed order.
__global__ void cl_allreduce(int iters, double* out) {
  __shared__ double slots[2][16];
  cg::cluster_group cl = cg::this_cluster();
  const int rank = cl.block_rank();
  const int cs = cl.num_blocks();
  double v = rank + 1.0, tot = 0.0;
  for (int it = 0; it < iters; ++it) {
    const int bank = it & 1;
    if (threadIdx.x < cs) {
      double* remote = cl.map_shared_rank(&slots[bank][0], threadIdx.x);
      remote[rank] = v;
    }
    asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
    asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
    double s = 0.0;
    for (int k = 0; k < cs; ++k) s += slots[bank][k];
    tot += s;
    v = s * 1e-3;
  }
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = tot;
}

// Two-level all-reduce: DSMEM + cluster barrier inside each cluster, then
// the cluster leaders exchange tagged 64-bit slots through global memory
// (one fence each side), then a second cluster barrier releases the
// cluster.  gslots: [2][K] words {hi|epoch, lo|epoch} x 2.
__global__ void cl2_allreduce(int iters, unsigned long long* gslots, double* out, int fence) {
  __shared__ double slots[2][16];
  __shared__ double tot_sh[2];
  cg::cluster_group cl = cg::this_cluster();
  const int rank = cl.block_rank();
  const int cs = cl.num_blocks();
  const int K = gridDim.x / cs;
  const int cid = blockIdx.x / cs;
  double v = blockIdx.x + 1.0, acc = 0.0;
  for (int it = 0; it < iters; ++it) {
    const int bank = it & 1;
    const unsigned epoch = (unsigned)it + 1;
    if (threadIdx.x < cs) {
      double* remote = cl.map_shared_rank(&slots[bank][0], threadIdx.x);
      remote[rank] = v;
    }
    asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
    asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
    if (rank == 0 && threadIdx.x < 32) {
      double s = 0.0;
      for (int k = 0; k < cs; ++k) s += slots[bank][k];
      unsigned long long* g = gslots + (size_t)bank * K * 2;
      if (threadIdx.x == 0) {
        if (fence) __threadfence();
        const unsigned long long u = (unsigned long long)__double_as_longlong(s);
        volatile unsigned long long* dst = g + 2 * cid;
        dst[0] = (u & 0xffffffff00000000ull) | epoch;
        dst[1] = (u << 32) | epoch;
      }
      __syncwarp();
      double t = 0.0;
      const int lane = threadIdx.x;
      if (lane < K) {
        volatile unsigned long long* src = g + 2 * lane;
        unsigned long long a, c;
        do {
          a = src[0];
          c = src[1];
        } while ((unsigned)a != epoch || (unsigned)c != epoch);
        t = __longlong_as_double((long long)((a & 0xffffffff00000000ull) | (c >> 32)));
      }
      for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
      if (fence) __threadfence();
      if (lane < cs) {
        double* remote = cl.map_shared_rank(&tot_sh[bank], lane);
        *remote = t;
      }
    }
    asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
    asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
    acc += tot_sh[bank];
    v = tot_sh[bank] * 1e-6;
  }
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = acc;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 64);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const size_t per = 288 * 1024;
  char* buf;
  cudaMalloc(&buf, per * 148);
  cudaMemset(buf, 0, per * 148);
  for (int G : {8, 16, 32, 74, 148}) {
    for (int thr : {512, 1024}) {
      const int reps = 20;
      l2_ld<<<G, thr>>>((const double2*)buf, per, 2, out);
      cudaEventRecord(e0);
      l2_ld<<<G, thr>>>((const double2*)buf, per, reps, out);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      printf("l2_ld  G=%3d thr=%4d  %.3f us per %zu KB pass  %.1f GB/s per SM  %.2f TB/s total\n", G,
             thr, ms * 1e3 / reps, per / 1024, per * reps / (ms * 1e-3) / 1e9,
             per * reps * (double)G / (ms * 1e-3) / 1e12);
    }
    cudaFuncSetAttribute(l2_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 32768);
    const int reps = 20;
    l2_tma<<<G, 256, 4 * 32768>>>(buf, per, 2, out);
    cudaEventRecord(e0);
    l2_tma<<<G, 256, 4 * 32768>>>(buf, per, reps, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("l2_tma G=%3d           %.3f us per %zu KB pass  %.1f GB/s per SM (%s)\n", G,
           ms * 1e3 / reps, per / 1024, per * reps / (ms * 1e-3) / 1e9,
           cudaGetErrorString(cudaGetLastError()));
  }
  cudaFuncSetAttribute(cl_allreduce, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int cs : {2, 4, 8, 16}) {
    for (int thr : {512, 1024}) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(cs);
      cfg.blockDim = dim3(thr);
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = cs;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      int ncl = -1;
      cudaOccupancyMaxActiveClusters(&ncl, cl_allreduce, &cfg);
      const int iters = 20000;
      cudaLaunchKernelEx(&cfg, cl_allreduce, 100, out);
      cudaEventRecord(e0);
      cudaError_t err = cudaLaunchKernelEx(&cfg, cl_allreduce, iters, out);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      printf("cluster=%2d thr=%4d maxActiveClusters=%d  %.3f us per all-reduce (%s)\n", cs, thr, ncl,
             ms * 1e3 / iters, cudaGetErrorString(err));
    }
  }
  // two-level: K clusters of 16 (cooperative cluster launch), 512 threads, big smem
  cudaFuncSetAttribute(cl2_allreduce, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  unsigned long long* gs;
  cudaMalloc(&gs, 2 * 64 * 2 * sizeof(unsigned long long));
  for (int cs : {8, 16}) {
    for (int fence : {0, 1}) {
      cudaLaunchConfig_t cfg = {};
      cfg.blockDim = dim3(512);
      cfg.dynamicSmemBytes = 200 * 1024;
      cudaFuncSetAttribute(cl2_allreduce, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      cudaLaunchAttribute at[2];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = cs;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      at[1].id = cudaLaunchAttributeCooperative;
      at[1].val.cooperative = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      cfg.gridDim = dim3(cs);
      int ncl = -1;
      cudaOccupancyMaxActiveClusters(&ncl, cl2_allreduce, &cfg);
      cfg.numAttrs = 2;
      for (int K : {1, 2, 4, ncl}) {
        if (K < 1 || K > ncl) continue;
        cfg.gridDim = dim3(cs * K);
        cudaMemset(gs, 0, 2 * 64 * 2 * sizeof(unsigned long long));
        const int iters = 20000;
        cudaError_t err = cudaLaunchKernelEx(&cfg, cl2_allreduce, 10, gs, out, fence);
        cudaDeviceSynchronize();
        cudaMemset(gs, 0, 2 * 64 * 2 * sizeof(unsigned long long));
        cudaEventRecord(e0);
        err = cudaLaunchKernelEx(&cfg, cl2_allreduce, iters, gs, out, fence);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("two-level cluster=%2d K=%2d (max %d) fence=%d  %.3f us per all-reduce (%s)\n", cs, K,
               ncl, fence, ms * 1e3 / iters, cudaGetErrorString(err));
      }
    }
  }
  return 0;
}
