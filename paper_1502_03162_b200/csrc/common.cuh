// Device-side building blocks shared by the renderer kernels (sm_100a only).
//
//  * TMEM (tensor memory) as a per-lane, dynamically indexable sliding window:
//    tcgen05.st writes a lane's window row, tcgen05.ld.32x32b.x16 reads 16
//    consecutive columns starting at a *runtime* column -- this is what lets a
//    sparse tap list (runtime offsets) feed FFMA without a shared-memory load
//    per multiply-accumulate.
//  * cp.async.bulk (TMA, non-tensor) stores from shared memory, so each warp's
//    output run leaves the SM as one contiguous bulk write.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "launch.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "paper_1502_03162_b200 kernels target sm_100a only"
#endif

namespace toep {


__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

// ---------------------------------------------------------------- TMEM ----
template <int COLS>
__device__ __forceinline__ void tmem_alloc(unsigned* dst_smem) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
               "n"(COLS)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
template <int COLS>
__device__ __forceinline__ void tmem_dealloc(unsigned base) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(base), "n"(COLS) : "memory");
}
__device__ __forceinline__ void tmem_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tmem_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ void tmem_ld16(float (&d)[16], unsigned ta) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=f"(d[0]), "=f"(d[1]), "=f"(d[2]), "=f"(d[3]), "=f"(d[4]), "=f"(d[5]), "=f"(d[6]), "=f"(d[7]),
        "=f"(d[8]), "=f"(d[9]), "=f"(d[10]), "=f"(d[11]), "=f"(d[12]), "=f"(d[13]), "=f"(d[14]), "=f"(d[15])
      : "r"(ta)
      : "memory");
}
__device__ __forceinline__ void tmem_st16(unsigned ta, const float (&d)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(ta),
      "f"(d[0]), "f"(d[1]), "f"(d[2]), "f"(d[3]), "f"(d[4]), "f"(d[5]), "f"(d[6]), "f"(d[7]), "f"(d[8]),
      "f"(d[9]), "f"(d[10]), "f"(d[11]), "f"(d[12]), "f"(d[13]), "f"(d[14]), "f"(d[15])
      : "memory");
}

// Same store without a compiler memory barrier: it reads registers only, so
// shared-memory loads that feed later stores may be hoisted above it (its
// order against other tcgen05 ops is that of the volatile asm statements).
__device__ __forceinline__ void tmem_st16_nb(unsigned ta, const float (&d)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(ta),
      "f"(d[0]), "f"(d[1]), "f"(d[2]), "f"(d[3]), "f"(d[4]), "f"(d[5]), "f"(d[6]), "f"(d[7]), "f"(d[8]),
      "f"(d[9]), "f"(d[10]), "f"(d[11]), "f"(d[12]), "f"(d[13]), "f"(d[14]), "f"(d[15]));
}

// One lane of the (converged) warp; lets ptxas issue uniform-datapath ops
// (UTMA*/UBLKCP) without a per-lane serialisation loop.
__device__ __forceinline__ bool elect_one() {
  unsigned pred;
  asm volatile(
      "{\n"
      ".reg .pred P;\n"
      "elect.sync _|P, 0xffffffff;\n"
      "selp.u32 %0, 1, 0, P;\n"
      "}\n"
      : "=r"(pred));
  return pred != 0;
}

// ------------------------------------------------------- bulk (TMA) ops ----
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void bulk_store(float* gdst, const float* ssrc, unsigned bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(smem_u32(ssrc)),
               "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// ------------------------------------------------------------ mbarrier ----
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred P;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 P, [%0], %1;\n"
      "@!P bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// Producer-side wait: lets the thread sleep in hardware between probes.
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred P;\n"
      "WAITS_%=:\n"
      "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 P, [%0], %1, %2;\n"
      "@!P bra WAITS_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity), "r"(100000)
      : "memory");
}
// 1-D bulk copy global -> shared, completion counted on `bar` (bytes % 16 == 0).
__device__ __forceinline__ void bulk_load(void* sdst, const void* gsrc, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(sdst)),
               "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// Padded shared-memory layout for signal tiles read as 16-float chunks by
// consecutive lanes: 4 pad words per 32 keeps LDS.128 conflict-free.
__device__ __forceinline__ int padi(int i) { return i + ((i >> 5) << 2); }
__host__ __device__ constexpr int padded_len(int n) { return n + ((n + 31) / 32) * 4; }

// Register-blocked dense FIR over a padded shared tile:
//   acc[r] += sum_{j<ntaps} h[j] * x[base + r - j],  r = 0..15
// `x` is the padded tile, `base` a logical index (multiple of 16) with at
// least ntaps_padded earlier samples available; `h` is zero-padded to a
// multiple of 16 in shared memory.  256 FFMA per 8+4 LDS.128.
// Packed fp32 pair arithmetic (sm_100 FFMA2 / FMUL2): {a0,a1} = {x0,x1} * v (+ {a0,a1}).
// Two correctly rounded fp32 FMAs per instruction -- bitwise the same as two fmaf,
// half the issue slots.  The ptxas form takes v as a broadcast scalar register.
__device__ __forceinline__ void ffma2(float& a0, float& a1, float x0, float x1, float v) {
  asm("{\n\t.reg .b64 a, x, v;\n\tmov.b64 a, {%0,%1};\n\tmov.b64 x, {%2,%3};\n\tmov.b64 v, {%4,%4};\n\t"
      "fma.rn.f32x2 a, x, v, a;\n\tmov.b64 {%0,%1}, a;\n}"
      : "+f"(a0), "+f"(a1)
      : "f"(x0), "f"(x1), "f"(v));
}
__device__ __forceinline__ void fadd2(float& a0, float& a1, float x0, float x1) {
  asm("{\n\t.reg .b64 a, x;\n\tmov.b64 a, {%0,%1};\n\tmov.b64 x, {%2,%3};\n\t"
      "add.rn.f32x2 a, a, x;\n\tmov.b64 {%0,%1}, a;\n}"
      : "+f"(a0), "+f"(a1)
      : "f"(x0), "f"(x1));
}
__device__ __forceinline__ void fmul2(float& a0, float& a1, float x0, float x1, float v) {
  asm("{\n\t.reg .b64 a, x, v;\n\tmov.b64 x, {%2,%3};\n\tmov.b64 v, {%4,%4};\n\t"
      "mul.rn.f32x2 a, x, v;\n\tmov.b64 {%0,%1}, a;\n}"
      : "=f"(a0), "=f"(a1)
      : "f"(x0), "f"(x1), "f"(v));
}

__device__ __forceinline__ void fir16_block(float (&acc)[16], const float* __restrict__ x, int base,
                                            const float* __restrict__ h, int ntaps_padded) {
  for (int j0 = 0; j0 < ntaps_padded; j0 += 16) {
    float w[32];
    const int a = base - j0 - 16;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const float4 v = *reinterpret_cast<const float4*>(&x[padi(a + 4 * q)]);
      w[4 * q] = v.x;
      w[4 * q + 1] = v.y;
      w[4 * q + 2] = v.z;
      w[4 * q + 3] = v.w;
    }
    float hh[16];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float4 v = *reinterpret_cast<const float4*>(&h[j0 + 4 * q]);
      hh[4 * q] = v.x;
      hh[4 * q + 1] = v.y;
      hh[4 * q + 2] = v.z;
      hh[4 * q + 3] = v.w;
    }
#pragma unroll
    for (int jj = 0; jj < 16; ++jj)
#pragma unroll
      for (int r = 0; r < 16; ++r) acc[r] = fmaf(hh[jj], w[16 + r - jj], acc[r]);
  }
}

}  // namespace toep
