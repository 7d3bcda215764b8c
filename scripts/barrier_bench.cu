// barrier_bench.cu — dev microbenchmark (not part of the product): cost of
// grid-wide all-reduce barrier variants in a cooperative kernel on B200.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/barrier_bench scripts/barrier_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int kBlock = 512;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ void fence_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ void st_rel_v2(unsigned long long* p, unsigned long long a, unsigned long long b) {
  asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b) : "memory");
}
__device__ __forceinline__ void ld_rel_v2(const unsigned long long* p, unsigned long long& a, unsigned long long& b) {
  asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acq(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_rlx(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void red_release_add(unsigned long long* p, unsigned long long v) {
  asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

struct Sm {
  double red[32];
  double bcast;
};

// VARIANT: 0 = slot all-to-all (256B slots, warp0 polls, fences)
//          1 = same without fences
//          2 = slots packed 16B
//          3 = counter barrier + slots read after
//          4 = 0 but polls with ld.acquire (no separate reader fence)
//          5 = only __syncthreads (baseline)
//          6 = slot all-to-all, value in slot + flag in separate word; writer st.release flag
template <int VARIANT>
__global__ void __launch_bounds__(kBlock, 1) bar_kernel(unsigned long long* slots, unsigned long long* counter,
                                                      int iters, double* out) {
  __shared__ Sm sm;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int G = gridDim.x;
  double acc = 0.0;
  for (uint32_t epoch = 1; epoch <= (uint32_t)iters; ++epoch) {
    double v = (double)(blockIdx.x + threadIdx.x) * 1e-3 + epoch;
    v = warp_sum(v);
    if (lane == 0) sm.red[w] = v;
    __syncthreads();
    if (VARIANT == 5) {
      if (w == 0) {
        double bs = lane < 16 ? sm.red[lane] : 0.0;
        bs = warp_sum(bs);
        if (lane == 0) sm.bcast = bs;
      }
      __syncthreads();
      acc += sm.bcast;
      continue;
    }
    if (w == 0) {
      double bs = lane < 16 ? sm.red[lane] : 0.0;
      bs = warp_sum(bs);
      const int stride = VARIANT == 2 ? 2 : 32;
      unsigned long long* bank = slots + (size_t)(epoch & 1u) * G * stride;
      const unsigned long long bits = (unsigned long long)__double_as_longlong(bs);
      double s = 0.0;
      if (VARIANT == 3) {
        if (lane == 0) {
          st_rel_v2(bank + (size_t)stride * blockIdx.x, (bits & 0xffffffff00000000ull) | epoch, (bits << 32) | epoch);
          red_release_add(counter, 1ull);
          const unsigned long long target = (unsigned long long)G * epoch;
          while (ld_acq(counter) < target) {}
        }
        __syncwarp();
        for (int t = lane; t < G; t += 32) {
          unsigned long long a, c;
          ld_rel_v2(bank + (size_t)stride * t, a, c);
          s += __longlong_as_double((long long)((a & 0xffffffff00000000ull) | (c >> 32)));
        }
        fence_gpu();
      } else if (VARIANT == 6) {
        // value words + separate flag word, release store of flag
        if (lane == 0) {
          bank[(size_t)stride * blockIdx.x] = bits;
          st_release(bank + (size_t)stride * blockIdx.x + 1, epoch);
        }
        for (int t = lane; t < G; t += 32) {
          while ((uint32_t)ld_acq(bank + (size_t)stride * t + 1) != epoch) {}
          s += __longlong_as_double((long long)ld_rlx(bank + (size_t)stride * t));
        }
      } else {
        if (lane == 0) {
          if (VARIANT != 1) fence_gpu();
          st_rel_v2(bank + (size_t)stride * blockIdx.x, (bits & 0xffffffff00000000ull) | epoch, (bits << 32) | epoch);
        }
        for (int t = lane; t < G; t += 32) {
          unsigned long long a, c;
          if (VARIANT == 4) {
            do {
              a = ld_acq(bank + (size_t)stride * t);
              c = ld_acq(bank + (size_t)stride * t + 1);
            } while ((uint32_t)a != epoch || (uint32_t)c != epoch);
          } else {
            do {
              ld_rel_v2(bank + (size_t)stride * t, a, c);
            } while ((uint32_t)a != epoch || (uint32_t)c != epoch);
          }
          s += __longlong_as_double((long long)((a & 0xffffffff00000000ull) | (c >> 32)));
        }
        if (VARIANT == 0 || VARIANT == 2) fence_gpu();
      }
      s = warp_sum(s);
      if (lane == 0) sm.bcast = s;
    }
    __syncthreads();
    acc += sm.bcast;
  }
  if (threadIdx.x == 0) out[blockIdx.x] = acc;
}

template <int V>
void run(const char* name, int G, int iters) {
  unsigned long long *slots, *counter;
  double* out;
  cudaMalloc(&slots, sizeof(unsigned long long) * 2 * 32 * 1024);
  cudaMalloc(&counter, 8);
  cudaMalloc(&out, 8 * 1024);
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    cudaMemset(slots, 0, sizeof(unsigned long long) * 2 * 32 * 1024);
    cudaMemset(counter, 0, 8);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    void* args[] = {&slots, &counter, &iters, &out};
    cudaEventRecord(a);
    cudaError_t e = cudaLaunchCooperativeKernel((void*)bar_kernel<V>, dim3(G), dim3(kBlock), args, 0, 0);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    if (e != cudaSuccess || cudaGetLastError() != cudaSuccess) {
      printf("%s: launch failed %s\n", name, cudaGetErrorString(e));
      return;
    }
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  printf("%-44s G=%4d  %.3f us/barrier\n", name, G, best * 1e3f / iters);
  cudaFree(slots);
  cudaFree(counter);
  cudaFree(out);
}

int main() {
  const int iters = 20000;
  for (int G : {148, 296}) {
    run<5>("syncthreads only", G, iters);
    run<0>("slots256 fence+relaxed, warp poll, fence", G, iters);
    run<1>("slots256 no fences", G, iters);
    run<2>("slots16 fence+relaxed", G, iters);
    run<3>("counter red.release + acquire poll", G, iters);
    run<4>("slots256 fence, acquire polls", G, iters);
    run<6>("slots256 value+release flag, acquire poll", G, iters);
  }
  return 0;
}
