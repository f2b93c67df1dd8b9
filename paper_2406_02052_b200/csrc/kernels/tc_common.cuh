// tc_common.cuh -- sm_100a building blocks: mbarriers, TMA, tcgen05 (UMMA + TMEM).
// Raw PTX; encodings follow the PTX ISA / CUTLASS cute::UMMA descriptor layouts.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <stdint.h>

#include "../kernels.h"

namespace petra {
namespace tc {

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ---------------------------------------------------------------- mbarrier
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  uint32_t a = smem_u32(bar);
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(a),
      "r"(parity)
      : "memory");
}

// wait for a phase of a pipeline barrier from a producer / MMA-issuer thread: the
// suspend-time hint lets the hardware park the thread until the phase completes
// instead of re-issuing try_wait (the polling loop otherwise takes issue slots from the
// epilogue warps sharing its SM sub-partition)
#ifndef PETRA_WAIT_HINT
#define PETRA_WAIT_HINT 0x100000u
#endif
__device__ __forceinline__ void mbar_wait_idle(uint64_t *bar, uint32_t parity) {
  if constexpr (PETRA_WAIT_HINT == 0u) {  // experiment switch: plain try_wait polling
    mbar_wait(bar, parity);
    return;
  }
  uint32_t a = smem_u32(bar);
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(a),
      "r"(parity), "r"(PETRA_WAIT_HINT)
      : "memory");
}

// register cap of the conv kernels (launch-time allocation decides which other
// stages' kernels can share an SM with a conv CTA)
#ifndef PETRA_CONV_MAXREG
#define PETRA_CONV_MAXREG 128
#endif

// division by a kernel-constant divisor as multiply-high + shift (round-up method,
// exact for dividends < 2^31); the magic numbers travel in the kernel parameters
struct FastDiv {
  uint32_t d, m;
  int s;  // -1: d == 1
};
inline FastDiv fastdiv_make(uint32_t d) {  // host: filled into the kernel parameters
  FastDiv f;
  f.d = d;
  if (d <= 1) {
    f.m = 0;
    f.s = -1;
  } else {
    const int l = 32 - __builtin_clz(d - 1);  // ceil(log2 d)
    f.m = (uint32_t)(((1ull << (31 + l)) + d - 1) / d);
    f.s = l - 1;
  }
  return f;
}
__device__ __forceinline__ int fdiv(int n, const FastDiv &f) {
  return f.s < 0 ? n : (int)(__umulhi((uint32_t)n, f.m) >> f.s);
}
__device__ __forceinline__ int fmod_(int n, int q, const FastDiv &f) { return n - q * (int)f.d; }

// 32-bit shared-window accesses (avoid generic 64-bit address arithmetic)
__device__ __forceinline__ uint32_t lds32(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ uint4 lds128(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
  return v;
}
__device__ __forceinline__ void sts128(uint32_t addr, const uint4 &v) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}

// ---------------------------------------------------------------- clusters (distributed shared memory)
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// every thread of every CTA of the cluster: release this CTA's smem writes, acquire the peers'
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// four floats of CTA `rank`'s shared memory at the (16-byte aligned) address `saddr` has in
// this CTA.  Volatile (kept after the cluster barrier); the caller issues all ranks' loads
// before the first add, so they are in flight together.
__device__ __forceinline__ float4 ld_dsmem_f32x4(uint32_t saddr, uint32_t rank) {
  uint32_t remote;
  float4 v;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(saddr), "r"(rank));
  asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(remote)
               : "memory");
  return v;
}

// the shared::cluster address of `saddr` (this CTA's) in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa(uint32_t saddr, uint32_t rank) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(saddr), "r"(rank));
  return remote;
}
// posted 16-byte store into a cluster peer's shared memory (address from mapa)
__device__ __forceinline__ void st_dsmem_f32x4(uint32_t raddr, float4 v) {
  asm volatile("st.shared::cluster.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(raddr), "f"(v.x), "f"(v.y), "f"(v.z),
               "f"(v.w)
               : "memory");
}

// generic-proxy smem writes (st.shared) made visible to the async proxy (tcgen05.mma)
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// ---------------------------------------------------------------- TMA (bulk tensor copies, zero-filled OOB)
__device__ __forceinline__ void tma_prefetch(const CUtensorMap *m) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(m)) : "memory");
}
__device__ __forceinline__ void tma_load_2d(void *dst, const CUtensorMap *m, uint64_t *bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::
          "r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void tma_load_4d(void *dst, const CUtensorMap *m, uint64_t *bar, int c0, int c1, int c2,
                                            int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], "
      "[%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}

__device__ __forceinline__ void tma_load_3d(void *dst, const CUtensorMap *m, uint64_t *bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::
          "r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
__device__ __forceinline__ void tma_load_5d(void *dst, const CUtensorMap *m, uint64_t *bar, int c0, int c1, int c2,
                                            int c3, int c4) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6, %7}], "
      "[%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4)
      : "memory");
}

// TMA stores (smem -> global, bulk-group completion; out-of-bounds elements are skipped)
__device__ __forceinline__ void tma_store_2d(const CUtensorMap *m, const void *src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(m)),
               "r"(smem_u32(src)), "r"(c0), "r"(c1)
               : "memory");
}
__device__ __forceinline__ void tma_store_4d(const CUtensorMap *m, const void *src, int c0, int c1, int c2, int c3) {
  asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(m)),
               "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// ---------------------------------------------------------------- tcgen05
// UMMA shared-memory descriptor, 128B-swizzled canonical layout (version 1 = sm100).
//   K-major : rows of 64 bf16 (128 B), 8-row atoms 1024 B apart (SBO), LBO unused (1)
//   MN-major: rows = K, 64 MN-elements per 128 B row; SBO = distance between 8-row (K)
//             groups, LBO = distance between 64-element MN blocks
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version
  d |= (uint64_t)2 << 61;  // SWIZZLE_128B
  return d;
}

// instruction descriptor: D fp32, A/B bf16, M x N, majors (0 = K, 1 = MN)
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N, int a_mn, int b_mn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
// one lane of a converged warp (the leader): tcgen05 ops are issued from warp-uniform
// code under this predicate, as CUTLASS does.  Issuing them from a lone diverged lane
// (if (lane == 0) { ... }) makes the compiler wrap every UTCHMMA in an
// ELECT / R2UR.BROADCAST / BRA.U.ANY waterfall -- measured ~133 cycles per MMA whatever
// its N (tools/micro/umma_rate.cu), 4x the 128x64x16 tensor-pipe time.
__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .b32 rx;\n\t.reg .pred px;\n\telect.sync rx|px, 0xffffffff;\n\t@px mov.s32 %0, 1;\n\t}"
      : "+r"(pred));
  return pred != 0;
}

__device__ __forceinline__ void umma_commit(uint64_t *bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tmem_alloc(uint32_t *dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
               "r"(ncols));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols));
}

// ---------------------------------------------------------------- CTA pairs (cta_group::2)
// Two CTAs of a cluster of 2 (one TPC) run one M = 256 UMMA: rank 0 (the leader) issues it;
// A rows 0-127 / 128-255 and B columns [0, N/2) / [N/2, N) come from the same shared-memory
// offsets of rank 0 / rank 1, and each CTA's TMEM holds its own 128 accumulator rows.
// Every tcgen05 alloc / dealloc / mma / commit of such a kernel uses cta_group::2.
__device__ __forceinline__ void tmem_alloc2(uint32_t *dst_smem, uint32_t ncols) {  // one warp of EACH CTA
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
               "r"(ncols));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
}
__device__ __forceinline__ void tmem_dealloc2(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols));
}
__device__ __forceinline__ void umma_bf16_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                               uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
// arrive (when the leader's issued MMAs complete) on the barrier at this smem offset in
// both CTAs of the pair
__device__ __forceinline__ void umma_commit_pair(uint64_t *bar) {
  asm volatile(
      "{\n\t.reg .b16 m;\n\tmov.b16 m, 3;\n\t"
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], m;\n\t}" ::"r"(
          smem_u32(bar))
      : "memory");
}
// arrive on the barrier at this smem offset in CTA `rank` of the cluster (release, cluster scope)
__device__ __forceinline__ void mbar_arrive_remote(uint64_t *bar, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(bar)), "r"(rank));
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(r) : "memory");
}
// TMA loads of a pair: the bytes land in THIS CTA's shared memory, the transaction count is
// credited to the barrier at `bar`'s offset in the leader CTA (rank 0), which expects both
// CTAs' bytes
__device__ __forceinline__ uint32_t leader_bar(uint64_t *bar) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(bar)), "r"(0));
  return r;
}
__device__ __forceinline__ void tma_load_3d_pair(void *dst, const CUtensorMap *m, uint32_t lbar, int c0, int c1,
                                                 int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, "
      "%5}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(lbar), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
__device__ __forceinline__ void tma_load_5d_pair(void *dst, const CUtensorMap *m, uint32_t lbar, int c0, int c1,
                                                 int c2, int c3, int c4) {
  asm volatile(
      "cp.async.bulk.tensor.5d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, "
      "%5, %6, %7}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(lbar), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4)
      : "memory");
}

// 32 lanes x 32 bit, 16 consecutive columns per thread
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// NC consecutive 16-column chunks with ONE wait: the tcgen05.ld's go out back to back
// and their latencies overlap.  Every chunk's registers are threaded through an empty asm
// that follows the (volatile) wait, so no use of them can be scheduled before it.
template <int NC>
__device__ __forceinline__ void tmem_ld16xN(uint32_t taddr, float *v) {
  uint32_t r[NC][16];
#pragma unroll
  for (int c = 0; c < NC; ++c)
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=r"(r[c][0]), "=r"(r[c][1]), "=r"(r[c][2]), "=r"(r[c][3]), "=r"(r[c][4]), "=r"(r[c][5]), "=r"(r[c][6]), "=r"(r[c][7]), "=r"(r[c][8]), "=r"(r[c][9]), "=r"(r[c][10]), "=r"(r[c][11]), "=r"(r[c][12]), "=r"(r[c][13]), "=r"(r[c][14]), "=r"(r[c][15])
                 : "r"(taddr + 16 * c));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    asm volatile("" : "+r"(r[c][0]), "+r"(r[c][1]), "+r"(r[c][2]), "+r"(r[c][3]), "+r"(r[c][4]), "+r"(r[c][5]), "+r"(r[c][6]), "+r"(r[c][7]), "+r"(r[c][8]), "+r"(r[c][9]), "+r"(r[c][10]), "+r"(r[c][11]), "+r"(r[c][12]), "+r"(r[c][13]), "+r"(r[c][14]), "+r"(r[c][15]));
#pragma unroll
    for (int i = 0; i < 16; ++i) v[16 * c + i] = __uint_as_float(r[c][i]);
  }
}

// Column sums of a 32-row x 16-column fragment held one row per lane: butterfly
// transpose-reduce (8+4+2+1+1 shuffles).  Afterwards lane L holds the sum over the
// 32 rows of column (L >> 1) in x[0] (lanes 2k, 2k+1 both).
__device__ __forceinline__ void colsum16(float (&x)[16], int lane) {
#pragma unroll
  for (int half = 8, off = 16; half >= 1; half >>= 1, off >>= 1) {
    const bool upper = lane & off;
#pragma unroll
    for (int k = 0; k < half; ++k) {
      float send = upper ? x[k] : x[k + half];
      float keep = upper ? x[k + half] : x[k];
      x[k] = keep + __shfl_xor_sync(0xffffffffu, send, off);
    }
  }
  x[0] += __shfl_xor_sync(0xffffffffu, x[0], 1);
}

// BN statistics of a warp's 32 staged output rows (each 128 bytes: 64 bf16 or 32 fp32
// values), read back from the epilogue staging buffer instead of reduced across lanes:
// lane L owns 4-byte word L of every row -- columns 2L, 2L+1 (bf16) or column L (fp32)
// -- and sums (z - k) and (z - k)^2 over the 32 rows, k = the lane's per-column shift
// (conflict-free: for a fixed row the lanes read 32 distinct banks).  Row r starts at
// buf + r * pitch; SWZ: 16-byte chunks in the 128B-swizzled order of a TMA box (chunk
// c of row r at (c ^ (r & 7)) * 16).
template <bool BF16, bool SWZ>
__device__ __forceinline__ void staged_colsums(const uint8_t *buf, int pitch, int lane, const float (&k)[2],
                                               float (&s)[2], float (&q)[2]) {
  if constexpr (BF16) {
    // packed fp32x2 adds / FMAs (sm_100 FADD2 / FFMA2), even and odd rows in separate
    // accumulators (two dependency chains); bf16 -> fp32 is a 16-bit shift
    float2 s0 = make_float2(0.f, 0.f), s1 = s0, q0 = s0, q1 = s0;
    const float2 nk = make_float2(-k[0], -k[1]);
    const uint32_t base = smem_u32(buf) + 4 * (lane & 3);
#pragma unroll
    for (int r = 0; r < 32; r += 2) {
      const int c0 = SWZ ? ((lane >> 2) ^ (r & 7)) : (lane >> 2);
      const int c1 = SWZ ? ((lane >> 2) ^ ((r + 1) & 7)) : (lane >> 2);
      const uint32_t w0 = lds32(base + r * pitch + c0 * 16);
      const uint32_t w1 = lds32(base + (r + 1) * pitch + c1 * 16);
      const float2 f0 = __fadd2_rn(make_float2(__uint_as_float(w0 << 16), __uint_as_float(w0 & 0xffff0000u)), nk);
      const float2 f1 = __fadd2_rn(make_float2(__uint_as_float(w1 << 16), __uint_as_float(w1 & 0xffff0000u)), nk);
      s0 = __fadd2_rn(s0, f0);
      q0 = __ffma2_rn(f0, f0, q0);
      s1 = __fadd2_rn(s1, f1);
      q1 = __ffma2_rn(f1, f1, q1);
    }
    s[0] = s0.x + s1.x;
    s[1] = s0.y + s1.y;
    q[0] = q0.x + q1.x;
    q[1] = q0.y + q1.y;
  } else {
    s[0] = s[1] = q[0] = q[1] = 0.f;
    const uint32_t base = smem_u32(buf) + 4 * (lane & 3);
#pragma unroll
    for (int r = 0; r < 32; ++r) {
      const int chunk = SWZ ? ((lane >> 2) ^ (r & 7)) : (lane >> 2);
      const float f = __uint_as_float(lds32(base + r * pitch + chunk * 16)) - k[0];
      s[0] += f;
      q[0] = fmaf(f, f, q[0]);
    }
  }
}

// BN batch statistics in the conv epilogues: every lane keeps, for
// its (up to two) columns, the shifted sums S = sum (z - k), Q = sum (z - k)^2 over the
// valid rows of the tiles it has seen, with k = the column's value in the first valid
// row it saw (the shifted-data algorithm: no cancellation between E[z^2] and mean^2 --
// a sample of the column is within a few standard deviations of its mean).  Padding
// rows are staged as exact zeros; their (0 - k) terms are removed.  At the end:
// n (warp-uniform), mean = k + S / n, M2 = Q - S^2 / n -- the (count, mean, M2) triple
// the CTA merges over its lane quarters and the finalize merges over CTAs.
struct ColStats {
  float k[2], s[2], q[2];
};
__device__ __forceinline__ void colstats_zero(ColStats &c) {
  c.k[0] = c.k[1] = c.s[0] = c.s[1] = c.q[0] = c.q[1] = 0.f;
}
// add one staged 32-row tile whose valid rows are the set bits of vmask (warp-uniform);
// n = valid rows seen so far
template <bool BF16, bool SWZ>
__device__ __forceinline__ void colstats_tile(const uint8_t *buf, int pitch, int lane, uint32_t vmask, int n,
                                              ColStats &c) {
  if (vmask == 0u) return;
  if (n == 0) {  // the shift: this lane's word in the first valid row
    const int r = __ffs(vmask) - 1;
    const int chunk = SWZ ? ((lane >> 2) ^ (r & 7)) : (lane >> 2);
    const uint32_t w = lds32(smem_u32(buf) + r * pitch + chunk * 16 + 4 * (lane & 3));
    if constexpr (BF16) {
      c.k[0] = __uint_as_float(w << 16);
      c.k[1] = __uint_as_float(w & 0xffff0000u);
    } else {
      c.k[0] = __uint_as_float(w);
    }
  }
  float s[2], q[2];
  staged_colsums<BF16, SWZ>(buf, pitch, lane, c.k, s, q);
  const float pad = (float)(32 - __popc(vmask));
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    c.s[j] += fmaf(pad, c.k[j], s[j]);
    c.q[j] += fmaf(-pad * c.k[j], c.k[j], q[j]);
  }
}
// (mean, M2) of column j after n valid rows
__device__ __forceinline__ float2 colstats_final(const ColStats &c, int j, int n) {
  if (n == 0) return make_float2(0.f, 0.f);
  const float inv = 1.f / (float)n;
  return make_float2(c.k[j] + c.s[j] * inv, fmaxf(fmaf(-c.s[j] * inv, c.s[j], c.q[j]), 0.f));
}
// Chan's merge of (nb, mb, M2b) into (n, m, M2)
template <typename T>
__device__ __forceinline__ void chan_merge(T &n, T &m, T &M2, T nb, T mb, T M2b) {
  if (nb <= T(0)) return;
  const T nn = n + nb, d = mb - m;
  m += d * (nb / nn);
  M2 += M2b + d * d * (n * nb / nn);
  n = nn;
}
// A CTA's partial statistics row from its NQ slots (4 lane quarters, or 8 epilogue warps
// when the warps split rows): sq[slot][BN][2] holds (mean, M2) per column, cnt[slot] the
// slot's valid-row count; merged in slot order and written as (mean, M2) to row[BN][2]
// (global), the count to *row_n.
template <int NQ = 4>
__device__ __forceinline__ void cta_stats_row(const float *sq, const int *cnt, int BN, int tid, int nthreads,
                                              float *row, float *row_n) {
  for (int c = tid; c < BN; c += nthreads) {
    float n = 0.f, m = 0.f, M2 = 0.f;
#pragma unroll
    for (int qq = 0; qq < NQ; ++qq)
      chan_merge(n, m, M2, (float)cnt[qq], sq[(qq * BN + c) * 2], sq[(qq * BN + c) * 2 + 1]);
    row[2 * c] = m;
    row[2 * c + 1] = M2;
  }
  if (tid == 0) {
    int t = 0;
#pragma unroll
    for (int qq = 0; qq < NQ; ++qq) t += cnt[qq];
    *row_n = (float)t;
  }
}

}  // namespace tc

// host: 2-D TMA map of a row-major bf16 matrix [rows][K], 128B swizzle, box (64 K, box_rows)
CUtensorMap kmajor_map_bf16(const __nv_bfloat16 *m, int rows, int K, int box_rows);
// host: any tiled TMA map with 128B swizzle (throws PetraError on failure)
CUtensorMap tma_map(const void *base, CUtensorMapDataType dt, int rank, const cuuint64_t *dims,
                    const cuuint64_t *strides_bytes, const cuuint32_t *box, const cuuint32_t *es);
// row-major [rows][cols] tensor map, no swizzle, box (box_cols, box_rows) (conv_tc.cu)
CUtensorMap plain_map_2d(const void *base, CUtensorMapDataType dt, int esize, int64_t rows, int cols, int box_cols,
                         int box_rows);
CUtensorMap plain_map_2d_strided(const void *base, CUtensorMapDataType dt, int esize, int64_t rows, int cols, int ld,
                                 int box_cols, int box_rows);

}  // namespace petra
