// L2 round-trip latency from each SM to candidate lines (dev micro-benchmark):
// CTA b (one per SM) times 32 dependent relaxed.gpu loads of each of NL lines
// (4 KB apart) and writes the mean cycles per load; prints SM x line.
#include <cstdio>
#include <cuda_runtime.h>
constexpr int NL = 64;
__global__ void lat(unsigned long long* buf, float* out) {
  if (threadIdx.x != 0) return;
  unsigned smid;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  for (int l = 0; l < NL; ++l) {
    unsigned long long* p = buf + (size_t)l * 512;  // 4 KB apart
    unsigned long long v = 0;
    // warm (line in L2), then time dependent loads (address depends on value = 0)
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    long long t0 = clock64();
    for (int k = 0; k < 32; ++k) {
      unsigned long long* q = p + (v & 1);
      asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(q) : "memory");
    }
    long long t1 = clock64();
    out[(size_t)blockIdx.x * (NL + 1) + l] = (float)(t1 - t0) / 32.f + (float)(v & 1);
  }
  out[(size_t)blockIdx.x * (NL + 1) + NL] = (float)smid;
}
int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* buf;
  float* out;
  cudaMalloc(&buf, (size_t)NL * 4096);
  cudaMemset(buf, 0, (size_t)NL * 4096);
  cudaMalloc(&out, sizeof(float) * sms * (NL + 1));
  lat<<<sms, 32>>>(buf, out);
  cudaDeviceSynchronize();
  float* h = new float[(size_t)sms * (NL + 1)];
  cudaMemcpy(h, out, sizeof(float) * sms * (NL + 1), cudaMemcpyDeviceToHost);
  for (int b = 0; b < sms; ++b) {
    printf("%d", (int)h[(size_t)b * (NL + 1) + NL]);
    for (int l = 0; l < NL; ++l) printf(" %.0f", h[(size_t)b * (NL + 1) + l]);
    printf("\n");
  }
  return 0;
}
