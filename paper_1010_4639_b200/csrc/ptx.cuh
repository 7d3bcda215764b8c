// ptx.cuh — thin inline-PTX wrappers for sm_100a: mbarrier + 1-D bulk async
// copies (the TMA engine's non-tensor path), fp64 reductions to global
// memory, and the relaxed/acquire loads used by the grid all-reduce barrier.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace spcg {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ---- mbarrier -------------------------------------------------------------
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// Arrive once and add `bytes` to the expected transaction count.
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
// Bounded spins: a wait that cannot complete (a bug, never a slow GPU) traps
// instead of wedging the device; the host then sees a launch failure.
constexpr unsigned long long kSpinLimit = 1ull << 25;

__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n"
      "selp.u32 %0, 1, 0, P1;\n"
      "}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  unsigned long long spins = 0;
  while (!mbar_try_wait(bar, parity)) {
    if (++spins > kSpinLimit) asm volatile("trap;");
  }
}

// ---- cluster messages: DSMEM stores that complete on the receiver's mbarrier
// shared::cluster address of `p` (this CTA's shared memory) in cluster CTA `rank`
__device__ __forceinline__ uint32_t mapa_u32(const void* p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}
// st.async: the store and its byte count land on the receiver's mbarrier
// together (no fence, no cluster barrier); the receiver waits with
// mbar_wait_cluster
__device__ __forceinline__ void st_async_f64(uint32_t raddr, double v, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(raddr),
               "l"(__double_as_longlong(v)), "r"(rbar)
               : "memory");
}
__device__ __forceinline__ void st_async_v2f64(uint32_t raddr, double a, double b, uint32_t rbar) {
  asm volatile(
      "st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.b64 [%0], {%1, %2}, [%3];" ::"r"(raddr),
      "l"(__double_as_longlong(a)), "l"(__double_as_longlong(b)), "r"(rbar)
      : "memory");
}
// wait for a phase whose bytes came from other CTAs (acquire at cluster
// scope; the CTA-scope form measured 0.02 us faster per engine-6 iteration,
// not worth the memory-model doubt)
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  unsigned long long spins = 0;
  for (;;) {
    uint32_t ok;
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%1], %2;\n"
        "selp.u32 %0, 1, 0, P1;\n"
        "}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    if (ok) break;
    if (++spins > kSpinLimit) asm volatile("trap;");
  }
}

// 1-D bulk copy global -> shared, completion signalled on `bar` (complete_tx).
// dst/src 16-byte aligned, bytes a multiple of 16.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// Same with an L2 evict-first policy: streamed matrix bytes should not push
// the (reused) vectors out of L2.
#ifndef SPCG_MAT_EVICT_FIRST
#define SPCG_MAT_EVICT_FIRST 1
#endif
__device__ __forceinline__ void bulk_g2s_stream(void* dst, const void* src, uint32_t bytes,
                                                uint64_t* bar) {
#if SPCG_MAT_EVICT_FIRST
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], "
      "%2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
#else
  bulk_g2s(dst, src, bytes, bar);
#endif
}

// L2 prefetch of a contiguous global range (bulk, no registers, no completion).
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

// ---- global memory ----------------------------------------------------------
// fp64 reduction without return (SASS: RED.E.ADD.F64).
__device__ __forceinline__ void red_add_f64(double* addr, double v) {
  asm volatile("red.relaxed.gpu.global.add.f64 [%0], %1;" ::"l"(addr), "d"(v) : "memory");
}
// two's-complement 64-bit add (exact, order-independent): the fixed-point
// transposed contributions of K_SCSR_FIX
__device__ __forceinline__ void red_add_s64(unsigned long long* addr, long long v) {
  asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(addr), "l"(v) : "memory");
}
// 64-bit integer <-> fp64 conversions of the fixed-point SCSR.  Native
// I2F / F2I by default; SPCG_FIX_MAGIC=1 (A/B) builds them from fp64 adds and
// bit moves (the 1.5 * 2^52 trick on two 31-bit halves) -- measured slower in
// pass A (0.72 vs 0.68 ms on Q27) and equal in pass B, so off.
#ifndef SPCG_FIX_MAGIC
#define SPCG_FIX_MAGIC 0
#endif
constexpr double kMagic52 = 6755399441055744.0;           // 1.5 * 2^52
constexpr long long kMagic52Bits = 0x4338000000000000LL;  // its bit pattern
// correctly rounded (double)v, any v
__device__ __forceinline__ double s64_to_f64(long long v) {
#if SPCG_FIX_MAGIC
  const long long hi = v >> 31, lo = v & 0x7fffffffLL;
  const double dh = __dsub_rn(__longlong_as_double(hi + kMagic52Bits), kMagic52);
  const double dl = __dsub_rn(__longlong_as_double(lo + kMagic52Bits), kMagic52);
  return __dadd_rn(__dmul_rn(dh, 2147483648.0), dl);  // one rounding of the exact sum
#else
  return (double)v;
#endif
}
// rint(x) (round half to even) for |x| <= 2^62
__device__ __forceinline__ long long f64_to_s64_rn(double x) {
#if SPCG_FIX_MAGIC
  const double h = __dadd_rn(__dmul_rn(x, 4.656612873077392578125e-10), kMagic52);  // x / 2^31
  const long long hi = __double_as_longlong(h) - kMagic52Bits;
  const double rem = __dsub_rn(x, __dmul_rn(__dsub_rn(h, kMagic52), 2147483648.0));  // exact
  const long long lo = __double_as_longlong(__dadd_rn(rem, kMagic52)) - kMagic52Bits;
  return (hi << 31) + lo;
#else
  return __double2ll_rn(x);
#endif
}

// Scale of the fixed-point accumulation: 2^(62 - eM - ex) with 2^ex >= max|x|
// and 2^eM >= max_j sum_i |a_ij| (strict lower part), so every contribution
// and every row total stays below 2^62 in magnitude; a power of two, so the
// scaling itself is exact.
__device__ __forceinline__ double fix_scale(const unsigned long long* xmax_bits, int eM) {
  const double xmax = __longlong_as_double((long long)*xmax_bits);
  int ex = 0;
  if (xmax > 0.0) frexp(xmax, &ex);
  return ldexp(1.0, 62 - eM - ex);
}

// Streaming read-only loads of matrix data (not written during a kernel).
__device__ __forceinline__ double ld_stream_f64(const double* p) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ int ld_stream_s32(const int* p) {
  int v;
  asm volatile("ld.global.nc.L1::no_allocate.s32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}

// Barrier slot word pair: both 64-bit words carry the epoch in the low half,
// so a reader validates each single-copy-atomic word independently.
__device__ __forceinline__ void st_relaxed_v2_u64(unsigned long long* p, unsigned long long a,
                                                  unsigned long long b) {
  asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b)
               : "memory");
}
__device__ __forceinline__ void ld_relaxed_v2_u64(const unsigned long long* p,
                                                  unsigned long long& a,
                                                  unsigned long long& b) {
  asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];"
               : "=l"(a), "=l"(b)
               : "l"(p)
               : "memory");
}
// Slot accesses of the grid barriers (relaxed.gpu vector accesses: the
// volatile-scalar form that wins for the cluster exchange was slower here).
__device__ __forceinline__ void slot_st2(unsigned long long* p, unsigned long long a,
                                         unsigned long long b) {
  st_relaxed_v2_u64(p, a, b);
}
__device__ __forceinline__ void slot_ld2(const unsigned long long* p, unsigned long long& a,
                                         unsigned long long& b) {
  ld_relaxed_v2_u64(p, a, b);
}
__device__ __forceinline__ void ld_acquire_v2_u64(const unsigned long long* p,
                                                  unsigned long long& a,
                                                  unsigned long long& b) {
  asm volatile("ld.acquire.gpu.global.v2.u64 {%0, %1}, [%2];"
               : "=l"(a), "=l"(b)
               : "l"(p)
               : "memory");
}
__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void fence_acq_rel_gpu() {
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
}

// IEEE mul-then-add without contraction: reproduces the reference's compiled
// `acc + v*x` / `v + alpha*u` (x86-64 baseline, no FMA) bit for bit.
__device__ __forceinline__ double mul_add_rn(double acc, double a, double b) {
  return __dadd_rn(acc, __dmul_rn(a, b));
}

}  // namespace spcg
