// conv_halo.cu -- 3x3 / stride-1 tcgen05 convolutions on a zero-bordered activation
// buffer, with ONE A load per 64-channel block instead of one per tap.
//
// The bf16 operand x (forward) or dz (stride-1 dgrad) is stored padded, [B][H+2][W+2][C]
// with zero borders (written so by its producer kernels).  GEMM rows are the padded
// positions p of that grid; tap (kh, kw) reads row p + (kh-1)*(W+2) + (kw-1).  A tile of
// 128 consecutive positions therefore needs the contiguous "halo" run of rows
// [m0 - (W+3), m0 + 127 + (W+3)] -- one 2-D TMA box per channel block -- and each tap's
// A operand is the same smem run viewed from a start shifted by whole 128-byte rows.
// (Measured, tools/umma_shift_probe.cu: the 128B swizzle of a tcgen05 K-major operand
// follows the absolute smem address, so row-shifted descriptor starts with base
// offset 0 read exactly the rows a TMA box wrote.)  Compared with the per-tap im2col
// boxes of conv_tc.cu this cuts the A bytes moved into shared memory 9x.
// Border positions are computed and dropped by the epilogue, which stages each warp's
// 32 rows in smem and writes them out coalesced (8 lanes per 128-byte pixel chunk).
#include <cudaTypedefs.h>

#include <cstdio>
#include <mutex>
#include <vector>

#include "../errors.h"
#include "../kernels.h"
#include "tc_common.cuh"

namespace petra {
namespace {

constexpr int kEpiWarps = 8;                     // two epilogue warps per TMEM lane quarter
constexpr int kThreads = (2 + kEpiWarps) * 32;
constexpr int kBoxMax = 256;                     // TMA box height limit (rows per halo load)
constexpr uint32_t kRowPitch = 144;              // epilogue staging row pitch (bank spread)
constexpr uint32_t kEpiWarp = 32 * kRowPitch;
constexpr int kMaxStatN = 512;
constexpr int kMaxBStages = 8;
constexpr size_t kSmemLimit = 232448;            // 227 KB opt-in per CTA

struct HaloParams {
  int Mp;                  // GEMM rows = B * Hp * Wp padded positions
  int N;                   // output channels
  int CB, Cred;            // 64-channel blocks / channels of the reduction operand
  int ntaps;
  int off[9], wk[9];       // A row offset and weight tap index of each tap
  int Hp, Wp, H, W, B;
  int lead, HR;            // halo rows before the tile group (Wp + 1); rows loaded per halo
  int box_rows;            // rows per TMA box (HR = boxes * box_rows, box_rows % 8 == 0)
  uint32_t a_stage;        // bytes per A stage (HR * 128)
  int bstages;             // B ring depth (resident: the CB * ntaps weight tiles, loaded once)
  int resident;            // 1: the whole weight matrix of the (single) N tile stays in smem
  const float *addend;     // nullable, fp32 output only
  void *out;               // [B][H][W][N] fp32 or bf16
  float *stats;            // nullable: one BN partial row per CTA [grid][N][2] (mean, M2) + float[grid] counts
  tc::FastDiv f_ghw, f_wp, f_nn;  // Hp * Wp, Wp, N / BN (set by launch)
  int rs;                  // epilogue row split allowed (PETRA_EPI_RS)
  unsigned long long *tl;  // nullable: per-CTA timeline (PETRA_TIMELINE=1 debug runs, kTl slots per CTA)
};
// timeline slots (clock64 per CTA): 0 entry, 1 setup done, 2 weights resident, 3 exit,
// 4 + 4i: item i MMA start (operands + accumulator ready), MMAs issued, epilogue (warp 2)
// start, epilogue end
constexpr int kTl = 64;
__device__ __forceinline__ void tl_mark(unsigned long long *tl, int slot) {
  if (tl && slot < kTl) tl[(size_t)blockIdx.x * kTl + slot] = clock64();
}

// T consecutive 128-row M tiles share every B (weight) stage: the MMA warp applies one
// (tap, channel block) weight tile to all T tiles before releasing it, so the weight
// bytes per output row drop T-fold; their accumulators sit side by side in TMEM.
template <int BN, int T, bool OUT16>
__global__ void __maxnreg__(PETRA_CONV_MAXREG)
conv_halo_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                 const __grid_constant__ HaloParams P) {
  pdl_wait_trigger();
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  constexpr uint32_t B_BYTES = BN * 128;
  constexpr int ASTAGES = 2;
  constexpr int ACC = T * BN;  // TMEM columns per accumulator set
  uint8_t *sA = smem;
  uint8_t *sB = sA + ASTAGES * P.a_stage;
  uint64_t *afull = reinterpret_cast<uint64_t *>(sB + P.bstages * B_BYTES);  // resident: bstages = CB*ntaps
  uint64_t *aempty = afull + ASTAGES;
  uint64_t *bfull = aempty + ASTAGES;
  uint64_t *bempty = bfull + kMaxBStages;
  uint64_t *tfull = bempty + kMaxBStages;
  uint64_t *tempty = tfull + 2;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tempty + 2);
  uint8_t *sepi = reinterpret_cast<uint8_t *>(afull) + 512;       // [8 warps][32 rows x 144 B]
  // Epilogue work split: two warps per TMEM lane quarter.  A row of BN outputs wider than
  // one 128-byte chunk is split by column chunks (hc = chunk parity); a row that fits in
  // one chunk (BN = 64, bf16 out) is not split -- the two warps take alternate tiles of the
  // item (T >= 2) or alternate items (T == 1, each its own TMEM accumulator), so all eight
  // warps work (RS: rows split).
  const bool RS = BN * (OUT16 ? 2 : 4) <= 128 && P.rs;  // (P.rs: PETRA_EPI_RS, default on)
  const bool RS_ITEMS = RS && T == 1;   // alternate items: 4 warps release each accumulator
  const int NSLOT = RS ? 8 : 4;          // statistics slots: per warp (RS) or per lane quarter
  float *sstat = reinterpret_cast<float *>(sepi + kEpiWarps * kEpiWarp);  // [NSLOT][BN][2] (mean, M2)
  int *scnt = reinterpret_cast<int *>(sstat + NSLOT * BN * 2);              // [NSLOT] valid rows

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_nt = P.N / BN;
  const int n_work = (int)cdiv(P.Mp, 128 * T) * n_nt;
  const int GHW = P.Hp * P.Wp;
  const tc::FastDiv &f_ghw = P.f_ghw, &f_wp = P.f_wp, &f_nn = P.f_nn;
  const int BS = P.resident ? 1 : P.bstages;  // resident: one barrier for the whole weight load
  if (threadIdx.x == 0) tl_mark(P.tl, 0);

  if (threadIdx.x == 0) {
    for (int s = 0; s < ASTAGES; ++s) {
      tc::mbar_init(&afull[s], 1);
      tc::mbar_init(&aempty[s], 1);
    }
    for (int s = 0; s < BS; ++s) {
      tc::mbar_init(&bfull[s], 1);
      tc::mbar_init(&bempty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      tc::mbar_init(&tfull[a], 1);
      tc::mbar_init(&tempty[a], RS_ITEMS ? kEpiWarps / 2 : kEpiWarps);
    }
    tc::fence_mbar_init();
    tc::tma_prefetch(&tmA);
    tc::tma_prefetch(&tmB);
  }
  if (warp == 1) tc::tmem_alloc(tmem_slot, 2 * ACC);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (threadIdx.x == 0) tl_mark(P.tl, 1);

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer: halo per channel block, B per (channel block, tap)
      int as = 0, bs = 0;
      uint32_t aph = 0, bph = 0;
      if (P.resident) {  // every (channel block, tap) weight tile once, on bfull[0]
        tc::mbar_arrive_expect_tx(&bfull[0], (uint32_t)P.CB * P.ntaps * B_BYTES);
        for (int cb = 0; cb < P.CB; ++cb)
          for (int t = 0; t < P.ntaps; ++t)
            tc::tma_load_2d(sB + (cb * P.ntaps + t) * B_BYTES, &tmB, &bfull[0], P.wk[t] * P.Cred + cb * 64, 0);
      }
      for (int w = blockIdx.x; w < n_work; w += gridDim.x) {
        const int mg = tc::fdiv(w, f_nn), nt = w - mg * n_nt;
        const int r0 = mg * 128 * T - P.lead;  // may be negative: TMA zero-fills
        for (int cb = 0; cb < P.CB; ++cb) {
          tc::mbar_wait_idle(&aempty[as], aph ^ 1);
          tc::mbar_arrive_expect_tx(&afull[as], P.HR * 128);
          for (int r = 0; r < P.HR; r += P.box_rows)  // equal boxes, 1 KB-aligned (swizzle-consistent)
            tc::tma_load_2d(sA + as * P.a_stage + r * 128, &tmA, &afull[as], cb * 64, r0 + r);
          if (++as == ASTAGES) { as = 0; aph ^= 1; }
          for (int t = 0; t < P.ntaps && !P.resident; ++t) {
            tc::mbar_wait_idle(&bempty[bs], bph ^ 1);
            tc::mbar_arrive_expect_tx(&bfull[bs], B_BYTES);
            tc::tma_load_2d(sB + bs * B_BYTES, &tmB, &bfull[bs], P.wk[t] * P.Cred + cb * 64, nt * BN);
            if (++bs == BS) { bs = 0; bph ^= 1; }
          }
        }
      }
    }
  } else if (warp == 1) {  // ---------------- MMA issuer: warp-uniform loop, elected lane issues
    constexpr uint32_t idesc = tc::idesc_bf16(128, BN, 0, 0);
    int as = 0, bs = 0;
    uint32_t aph = 0, bph = 0;
    int it = 0;
    if (P.resident) {
      tc::mbar_wait(&bfull[0], 0);
      tc::tc_fence_after();
    }
    if (lane == 0) tl_mark(P.tl, 2);
    for (int w = blockIdx.x; w < n_work; w += gridDim.x, ++it) {
      const int acc = it & 1;
      tc::mbar_wait_idle(&tempty[acc], ((it >> 1) & 1) ^ 1);
      tc::tc_fence_after();
      const uint32_t dtm = tmem_base + acc * ACC;
      for (int cb = 0; cb < P.CB; ++cb) {
        tc::mbar_wait(&afull[as], aph);
        tc::tc_fence_after();
        if (cb == 0 && lane == 0) tl_mark(P.tl, 4 + 4 * it);
        const uint32_t abase = tc::smem_u32(sA + as * P.a_stage) + P.lead * 128;
        for (int t = 0; t < P.ntaps; ++t) {
          if (!P.resident) {
            tc::mbar_wait(&bfull[bs], bph);
            tc::tc_fence_after();
          }
          const int bslot = P.resident ? cb * P.ntaps + t : bs;
          const uint64_t bd = tc::sw128_desc(tc::smem_u32(sB + bslot * B_BYTES), 16, 1024);
          uint64_t ad[T];
#pragma unroll
          for (int tt = 0; tt < T; ++tt) ad[tt] = tc::sw128_desc(abase + (tt * 128 + P.off[t]) * 128, 16, 1024);
          if (tc::elect_one()) {
#pragma unroll
            for (int k = 0; k < 4; ++k)
#pragma unroll
              for (int tt = 0; tt < T; ++tt)  // tiles innermost: independent accumulators back to back
                tc::umma_bf16(dtm + tt * BN, ad[tt] + 2 * k, bd + 2 * k, idesc, (cb > 0 || t > 0 || k > 0) ? 1u : 0u);
            if (!P.resident) tc::umma_commit(&bempty[bs]);
          }
          __syncwarp();
          if (!P.resident && ++bs == BS) { bs = 0; bph ^= 1; }
        }
        if (tc::elect_one()) tc::umma_commit(&aempty[as]);
        __syncwarp();
        if (++as == ASTAGES) { as = 0; aph ^= 1; }
      }
      if (tc::elect_one()) tc::umma_commit(&tfull[acc]);
      __syncwarp();
      if (lane == 0) tl_mark(P.tl, 5 + 4 * it);
    }
  } else {  // ---------------- epilogue warps 2..9 (two per TMEM lane quarter, alternating column chunks)
    const int q = warp & 3;
    const int hc = (warp - 2) >> 2;
    const int row = q * 32 + lane;
    const int slot = RS ? warp - 2 : q;
    float *my_stat = sstat + (size_t)slot * BN * 2;  // this CTA's N tile (fixed: grid % n_nt == 0)
    uint8_t *ebuf = sepi + (warp - 2) * kEpiWarp;
    constexpr int ES = OUT16 ? 2 : 4;
    constexpr int CW = 128 / ES;  // columns per 128-byte chunk
    // per-lane shifted statistics of this warp's columns in registers (tc::ColStats)
    constexpr int NCH = (BN + 2 * CW - 1) / (2 * CW);
    tc::ColStats cst[NCH];
#pragma unroll
    for (int k = 0; k < NCH; ++k) tc::colstats_zero(cst[k]);
    int nrows = 0;  // valid rows of this warp's tiles so far (warp-uniform)
    int it = 0;
    for (int w = blockIdx.x; w < n_work; w += gridDim.x, ++it) {
      const int mg = tc::fdiv(w, f_nn), nt = w - mg * n_nt;
      const int acc = it & 1;
      if (RS_ITEMS && acc != hc) continue;  // the other warp of this lane quarter takes it
      tc::mbar_wait(&tfull[acc], (it >> 1) & 1);
      tc::tc_fence_after();
      if (warp == 2 && lane == 0) tl_mark(P.tl, 6 + 4 * it);
#pragma unroll 1
      for (int tt = (RS && !RS_ITEMS) ? hc : 0; tt < T; tt += (RS && !RS_ITEMS) ? 2 : 1) {
        const uint32_t trow = tmem_base + ((uint32_t)(q * 32) << 16) + acc * ACC + tt * BN;
        const int m = (mg * T + tt) * 128 + row;
        const int b = tc::fdiv(m, f_ghw), r = m - b * GHW, hp = tc::fdiv(r, f_wp), wp = r - hp * P.Wp;
        const bool valid = b < P.B && hp >= 1 && hp <= P.H && wp >= 1 && wp <= P.W;
        const int64_t opix = valid ? ((int64_t)b * P.H + hp - 1) * P.W + wp - 1 : -1;
        const float *arow = (valid && P.addend) ? P.addend + opix * P.N + nt * BN : nullptr;
        const uint32_t vmask = __ballot_sync(0xffffffffu, valid);
#pragma unroll
        for (int k = 0; k < NCH; ++k) {
          const int c = RS ? 0 : CW * hc + 2 * CW * k;
          if (c >= BN) break;
          float v[CW];
#pragma unroll
          tc::tmem_ld16xN<CW / 16>(trow + c, v);
          if (arow) {
#pragma unroll
            for (int jj = 0; jj < CW; jj += 4) {
              const float4 a4 = *reinterpret_cast<const float4 *>(arow + c + jj);
              v[jj] += a4.x; v[jj + 1] += a4.y; v[jj + 2] += a4.z; v[jj + 3] += a4.w;
            }
          }
          if (!valid) {  // padding row: never stored, zero for the statistics
#pragma unroll
            for (int jj = 0; jj < CW; ++jj) v[jj] = 0.f;
          }
          // stage this lane's row (128 B) ...
          const uint32_t rp = tc::smem_u32(ebuf) + lane * kRowPitch;
#pragma unroll
          for (int ch = 0; ch < 8; ++ch) {
            uint4 u;
            if constexpr (OUT16) {
              uint32_t wv[4];
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                __nv_bfloat162 hb = __floats2bfloat162_rn(v[8 * ch + 2 * e], v[8 * ch + 2 * e + 1]);
                wv[e] = *reinterpret_cast<uint32_t *>(&hb);
                const float2 f = __bfloat1622float2(hb);  // statistics of the stored values (reading c24)
                v[8 * ch + 2 * e] = f.x;
                v[8 * ch + 2 * e + 1] = f.y;
              }
              u = make_uint4(wv[0], wv[1], wv[2], wv[3]);
            } else {
              u = make_uint4(__float_as_uint(v[4 * ch]), __float_as_uint(v[4 * ch + 1]),
                             __float_as_uint(v[4 * ch + 2]), __float_as_uint(v[4 * ch + 3]));
            }
            tc::sts128(rp + ch * 16, u);
          }
          __syncwarp();
          // ... and write the warp's 32 rows out: 8 lanes per 128-byte pixel chunk
#pragma unroll
          for (int pc = 0; pc < 8; ++pc) {
            const int idx = pc * 32 + lane, rr = idx >> 3, piece = idx & 7;
            const int64_t op = __shfl_sync(0xffffffffu, opix, rr);
            if (op >= 0) {
              const uint4 u = tc::lds128(tc::smem_u32(ebuf) + rr * kRowPitch + piece * 16);
              char *dst = static_cast<char *>(P.out) + (op * P.N + nt * BN + c) * ES + piece * 16;
              *reinterpret_cast<uint4 *>(dst) = u;
            }
          }
          if (P.stats)  // statistics of z as stored (reading c24), from the staged rows
            tc::colstats_tile<OUT16, false>(ebuf, kRowPitch, lane, vmask, nrows, cst[k]);
          __syncwarp();
        }
        nrows += __popc(vmask);
      }
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&tempty[acc]);
      if (warp == 2 && lane == 0) tl_mark(P.tl, 7 + 4 * it);
    }
    if (P.stats) {  // this CTA's partial row: the slots merged (Chan) in a fixed order
#pragma unroll
      for (int k = 0; k < NCH; ++k) {
        const int c = RS ? 0 : CW * hc + 2 * CW * k;
        if (c >= BN) break;
        const int col = c + (OUT16 ? 2 * lane : lane);  // column within the N tile
        const float2 a = tc::colstats_final(cst[k], 0, nrows);
        my_stat[2 * col] = a.x;
        my_stat[2 * col + 1] = a.y;
        if (OUT16) {
          const float2 b = tc::colstats_final(cst[k], 1, nrows);
          my_stat[2 * col + 2] = b.x;
          my_stat[2 * col + 3] = b.y;
        }
      }
      if ((RS || hc == 0) && lane == 0) scnt[slot] = nrows;
      asm volatile("bar.sync 1, %0;" ::"n"(kEpiWarps * 32) : "memory");
      if (RS)
        tc::cta_stats_row<8>(sstat, scnt, BN, (warp - 2) * 32 + lane, kEpiWarps * 32,
                          P.stats + ((size_t)blockIdx.x * P.N + (size_t)(blockIdx.x % n_nt) * BN) * 2,
                          P.stats + (size_t)gridDim.x * P.N * 2 + blockIdx.x);
      else
        tc::cta_stats_row<4>(sstat, scnt, BN, (warp - 2) * 32 + lane, kEpiWarps * 32,
                          P.stats + ((size_t)blockIdx.x * P.N + (size_t)(blockIdx.x % n_nt) * BN) * 2,
                          P.stats + (size_t)gridDim.x * P.N * 2 + blockIdx.x);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) tl_mark(P.tl, 3);
  if (warp == 1) {
    tc::tc_fence_after();
    tc::tmem_dealloc(tmem_base, 2 * ACC);
  }
}

size_t fixed_smem() { return 1024 + 512 + kEpiWarps * kEpiWarp + (size_t)256 * 32 + 64; }  // stats: BN*NSLOT <= 1024
// the halo of T tiles (128*T + 2*(W+3) rows) as equal TMA boxes of <= 256 rows, each a
// multiple of 8 rows so every box starts 1 KB-aligned
void halo_rows(int T, int W, int &box_rows, int &HR) {
  const int need = 128 * T + 2 * (W + 3);
  const int nbox = (int)cdiv(need, kBoxMax);
  box_rows = (int)cdiv(cdiv(need, nbox), 8) * 8;
  HR = nbox * box_rows;
}
uint32_t a_stage_bytes(int T, int W) {
  int br, HR;
  halo_rows(T, W, br, HR);
  return (uint32_t)HR * 128;
}

struct HaloPlan {
  int BN, T, bstages;
  bool ok, resident;
};
// Tile group T (weight reuse) and N tile: the largest T whose A halos fit next to >= 3
// weight stages while the work items still fill 3/4 of a wave (measured: the weight
// bytes per output row, not load/epilogue overlap, bound these kernels); grids whose
// zero border adds > 35% rows, or that fill under 3/4 of a wave, stay on the split-K
// path of conv_tc.cu.
HaloPlan halo_plan(int B, int H, int W, int Cred, int N) {
  HaloPlan p{0, 0, 0, false, false};
  if (Cred % 64 || N % 64) return p;
  const int64_t Mp = (int64_t)B * (H + 2) * (W + 2);
  static const int max_pad = env_int("PETRA_HALO_MAX_PAD", 135);  // padded rows, % of real rows
  static const int64_t min_work = env_int("PETRA_HALO_MIN_WORK", (kNumSMs * 3 + 3) / 4);
  if (Mp >= ((int64_t)1 << 31) || Mp * 100 > (int64_t)B * H * W * max_pad) return p;
  // Weight-resident plan: one N tile (BN = N <= 128) whose 9 * Cred x N weights stay in
  // smem for the whole persistent CTA, so only the halos stream from L2 (~42 B/clk per
  // SM on B200: the weight stream, not the MMA, bounds the streamed plan for C = 64).
  static const bool resident_ok = env_int("PETRA_HALO_RESIDENT", 0) != 0;  // 0 under the 40-CTA caps
  if (resident_ok && N <= 128) {
    const size_t wbytes = (size_t)9 * (Cred / 64) * N * 128;
    for (int T : {4, 2, 1}) {
      if (T * N * 2 > 512) continue;
      if (fixed_smem() + 2 * (size_t)a_stage_bytes(T, W) + wbytes > kSmemLimit) continue;
      if (cdiv(Mp, 128 * T) < min_work) continue;
      p.BN = N;
      p.T = T;
      p.bstages = 9 * (Cred / 64);
      p.ok = p.resident = true;
      return p;
    }
  }
  for (int pass = 0; pass < 1; ++pass) {
    for (int bn : {256, 128, 64}) {
      if (N % bn) continue;
      for (int T : {4, 2, 1}) {
        if (T * bn * 2 > 512) continue;  // two accumulator sets in TMEM
        const size_t base = fixed_smem() + 2 * (size_t)a_stage_bytes(T, W);
        if (base + 3 * (size_t)bn * 128 > kSmemLimit) continue;
        const int64_t work = cdiv(Mp, 128 * T) * (N / bn);
        if (work < min_work) continue;
        p.BN = bn;
        p.T = T;
        p.bstages = (int)std::min<size_t>(kMaxBStages, (kSmemLimit - base) / ((size_t)bn * 128));
        p.ok = true;
        return p;
      }
    }
  }
  return p;
}

// a multiple of the N-tile count: every CTA's work items share one N tile
int halo_grid(int work, int n_nt) {
  // PETRA_HALO_CTAS (default: the common conv cap)
  static const int hcap = env_int("PETRA_HALO_CTAS", 0);
  const int g = hcap > 0 ? std::max(1, std::min({work, hcap, kNumSMs})) : conv_grid(work);
  return std::max(n_nt, g / n_nt * n_nt);
}

template <int BN, int T, bool OUT16>
void launch(const CUtensorMap &ta, const CUtensorMap &tb, const HaloParams &P0, cudaStream_t st) {
  HaloParams P = P0;
  P.f_ghw = tc::fastdiv_make(P.Hp * P.Wp);
  P.f_wp = tc::fastdiv_make(P.Wp);
  P.f_nn = tc::fastdiv_make(P.N / BN);
  static const int rs_on = env_int("PETRA_EPI_RS", 1);
  P.rs = rs_on;
  const int work = (int)cdiv(P.Mp, 128 * T) * (P.N / BN);
  const size_t smem = fixed_smem() + 2 * (size_t)P.a_stage + (size_t)P.bstages * BN * 128;
  static const bool tl_on = env_int("PETRA_TIMELINE", 0) != 0;  // debug: per-CTA timeline to stderr
  const int grid = halo_grid(work, P.N / BN);
  static unsigned long long *tl_buf = nullptr;
  if (tl_on) {
    if (!tl_buf) PETRA_CUDA(cudaMalloc(&tl_buf, (size_t)kNumSMs * kTl * sizeof(unsigned long long)));
    PETRA_CUDA(cudaMemsetAsync(tl_buf, 0, (size_t)kNumSMs * kTl * sizeof(unsigned long long), st));
    P.tl = tl_buf;
  }
  launch_k(conv_halo_kernel<BN, T, OUT16>, grid, kThreads, smem, st, ta, tb, P);
  PETRA_LAUNCH_CHECK();
  if (tl_on) {
    std::vector<unsigned long long> h((size_t)grid * kTl);
    PETRA_CUDA(cudaStreamSynchronize(st));
    PETRA_CUDA(cudaMemcpy(h.data(), tl_buf, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
    fprintf(stderr, "timeline conv_halo_kernel<%d,%d,%d> grid %d work %d (cycles from CTA entry)\n", BN, T, (int)OUT16,
            grid, work);
    for (int c = 0; c < grid; ++c) {
      const unsigned long long *r = &h[(size_t)c * kTl], t0 = r[0];
      auto d = [&](int i) { return r[i] ? (long long)(r[i] - t0) : -1LL; };
      fprintf(stderr, "cta %3d setup %6lld wres %6lld exit %6lld |", c, d(1), d(2), d(3));
      for (int i = 0; 4 + 4 * i + 3 < kTl && r[4 + 4 * i]; ++i)
        fprintf(stderr, " [%lld %lld %lld %lld]", d(4 + 4 * i), d(5 + 4 * i), d(6 + 4 * i), d(7 + 4 * i));
      fprintf(stderr, "\n");
    }
  }
}

template <bool OUT16>
void dispatch(int BN, int T, const CUtensorMap &ta, const CUtensorMap &tb, const HaloParams &P, cudaStream_t st) {
  if (BN == 64 && T == 4) launch<64, 4, OUT16>(ta, tb, P, st);
  else if (BN == 64 && T == 2) launch<64, 2, OUT16>(ta, tb, P, st);
  else if (BN == 64) launch<64, 1, OUT16>(ta, tb, P, st);
  else if (BN == 128 && T == 2) launch<128, 2, OUT16>(ta, tb, P, st);
  else if (BN == 128) launch<128, 1, OUT16>(ta, tb, P, st);
  else launch<256, 1, OUT16>(ta, tb, P, st);
}


// ------------------------------------------------------------------ wgrad on the halo
// dW[co][tap][ci] = sum_p x_pad[p + off(tap)][ci] * dz_pad[p][co] over the padded grid
// positions p (border positions of dz_pad are zero, so they add nothing).  One CTA per
// (64-channel block of x, 64-channel block of dz, K split of pixel blocks) keeps ALL
// nine taps in TMEM: five accumulators of 128 rows x 64 columns, each M = 128 MMA
// pairing two taps as the two 64-element MN blocks of its A operand -- both are
// windows of ONE halo load of x (descriptor start = window of the first tap, LBO =
// row distance to the second tap's window; the fifth pair repeats tap 7 and its first
// half is discarded).  Per 64-pixel block the CTA loads the x halo once and the dz
// tile once instead of a tap box per (tap, 64-channel block) and a dz tile per M tile.
struct WHaloParams {
  int Ci, Co, CB, n_nt, KBtot, kb_per_split, splits;
  int lead, HR, box_rows;
  int pb;      // pixels per block (64 or 128): pb / 16 MMA K steps per accumulator
  int off[9];
  int Mr;      // 9 * Ci
  int cs;      // > 1: clusters of cs consecutive K splits of one item reduce their partials
               // through distributed shared memory (single pass: one work item per CTA)
  float *out;  // [splits / cs][Co][Mr]
};
// the cluster-reduction tile: accumulators 0-3 (taps 0-7, 128 rows) and the tap-8 half of
// accumulator 4, fp32 [acc][64 co][128 rows] (the last one rows 64..127 only)
constexpr int kWTileFloats = 4 * 64 * 128 + 64 * 64;
constexpr int kWStages = 4;
constexpr int kWThreads = 192;
__device__ __forceinline__ int tap_a(int i) { return i < 4 ? 2 * i : 7; }
__device__ __forceinline__ int tap_b(int i) { return i < 4 ? 2 * i + 1 : 8; }

__global__ void __launch_bounds__(kWThreads, 1)
wgrad_halo_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmDZ,
                  const __grid_constant__ WHaloParams P) {
  pdl_wait_trigger();
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t XB = (uint32_t)P.HR * 128, STAGE = XB + (uint32_t)P.pb * 128;
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + kWStages * STAGE);
  uint64_t *empty = full + kWStages;
  uint64_t *tfull = empty + kWStages;
  uint64_t *tempty = tfull + 1;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tempty + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_work = P.CB * P.n_nt * P.splits;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kWStages; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], 1);
    }
    tc::mbar_init(tfull, 1);
    tc::mbar_init(tempty, 4);
    tc::fence_mbar_init();
    tc::tma_prefetch(&tmX);
    tc::tma_prefetch(&tmDZ);
  }
  if (warp == 1) tc::tmem_alloc(tmem_slot, 512);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  auto decode = [&](int w, int &cb, int &nt, int &kb0, int &kb1) {
    const int sp = w % P.splits, r = w / P.splits;
    nt = r % P.n_nt;
    cb = r / P.n_nt;
    kb0 = sp * P.kb_per_split;
    kb1 = min(P.KBtot, kb0 + P.kb_per_split);
  };
  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer: x halo + dz tile per 64-pixel block
      int stage = 0;
      uint32_t phase = 0;
      for (int w = blockIdx.x; w < n_work; w += gridDim.x) {
        int cb, nt, kb0, kb1;
        decode(w, cb, nt, kb0, kb1);
        for (int kb = kb0; kb < kb1; ++kb) {
          tc::mbar_wait_idle(&empty[stage], phase ^ 1);
          uint8_t *sx = smem + stage * STAGE;
          tc::mbar_arrive_expect_tx(&full[stage], STAGE);
          const int p0 = kb * P.pb;
          for (int r = 0; r < P.HR; r += P.box_rows)
            tc::tma_load_2d(sx + r * 128, &tmX, &full[stage], cb * 64, p0 - P.lead + r);
          for (int r = 0; r < P.pb; r += 64) tc::tma_load_2d(sx + XB + r * 128, &tmDZ, &full[stage], nt * 64, p0 + r);
          if (++stage == kWStages) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {  // ---------------- MMA issuer (warp-uniform, elected lane)
    constexpr uint32_t idesc = tc::idesc_bf16(128, 64, 1, 1);
    int stage = 0;
    uint32_t phase = 0;
    int it = 0;
    for (int w = blockIdx.x; w < n_work; w += gridDim.x, ++it) {
      int cb, nt, kb0, kb1;
      decode(w, cb, nt, kb0, kb1);
      tc::mbar_wait_idle(tempty, (it & 1) ^ 1);
      tc::tc_fence_after();
      for (int kb = kb0; kb < kb1; ++kb) {
        tc::mbar_wait(&full[stage], phase);
        tc::tc_fence_after();
        const uint32_t sx = tc::smem_u32(smem + stage * STAGE);
        const uint64_t bd = tc::sw128_desc(sx + XB, 8192, 1024);
        const int nk = P.pb >> 4;
        if (tc::elect_one()) {
#pragma unroll
          for (int i = 0; i < 5; ++i) {
            const int ta = tap_a(i), tb = tap_b(i);
            const uint64_t ad = tc::sw128_desc(sx + (P.lead + P.off[ta]) * 128, (P.off[tb] - P.off[ta]) * 128, 1024);
#pragma unroll 1
            for (int k = 0; k < nk; ++k)  // 16 pixels = 16 rows x 128 B per step
              tc::umma_bf16(tmem_base + i * 64, ad + (uint64_t)(k * 2048 >> 4), bd + (uint64_t)(k * 2048 >> 4),
                            idesc, (kb > kb0 || k) ? 1u : 0u);
          }
          tc::umma_commit(&empty[stage]);
        }
        __syncwarp();
        if (++stage == kWStages) { stage = 0; phase ^= 1; }
      }
      if (tc::elect_one()) tc::umma_commit(tfull);
      __syncwarp();
    }
  } else {  // ---------------- epilogue warps 2..5: D rows (tap pair, ci) x 64 co -> out[split][co][tap*Ci + ci]
    const int q = warp & 3;
    const int row = q * 32 + lane, half = row >> 6, ci = row & 63;
    int it = 0;
    for (int w = blockIdx.x; w < n_work; w += gridDim.x, ++it) {
      int cb, nt, kb0, kb1;
      decode(w, cb, nt, kb0, kb1);
      const int sp = w % P.splits;
      tc::mbar_wait(tfull, it & 1);
      tc::tc_fence_after();
      if (P.cs > 1) {  // stage the partial in this CTA's (idle) operand ring for the cluster
        float *tile = reinterpret_cast<float *>(smem);
#pragma unroll 1
        for (int i = 0; i < 5; ++i) {
          if (i == 4 && half == 0) continue;  // the repeated tap 7
          float v[64];
          if (kb1 > kb0) {
            tc::tmem_ld16xN<4>(tmem_base + ((uint32_t)(q * 32) << 16) + i * 64, v);
          } else {  // an empty (padding) split: nothing was accumulated
#pragma unroll
            for (int j = 0; j < 64; ++j) v[j] = 0.f;
          }
          float *t = tile + (i < 4 ? (size_t)i * 64 * 128 : (size_t)4 * 64 * 128 - 64);  // i = 4: rows 64..127
#pragma unroll
          for (int j = 0; j < 64; ++j) t[(size_t)j * (i < 4 ? 128 : 64) + row] = v[j];
        }
        tc::tc_fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(tempty);
        continue;
      }
      float *o = P.out + ((size_t)sp * P.Co + nt * 64) * P.Mr;
#pragma unroll 1
      for (int i = 0; i < 5; ++i) {
        const int tap = half ? tap_b(i) : tap_a(i);
        const bool store = !(i == 4 && half == 0);  // the repeated tap 7
        const int r = tap * P.Ci + cb * 64 + ci;
        {
          float v[64];
          tc::tmem_ld16xN<4>(tmem_base + ((uint32_t)(q * 32) << 16) + i * 64, v);
          if (store) {
#pragma unroll
            for (int j = 0; j < 64; ++j) o[(size_t)j * P.Mr + r] = v[j];
          }
        }
      }
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(tempty);
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc::tc_fence_after();
    tc::tmem_dealloc(tmem_base, 512);
  }
  if (P.cs > 1) {
    // every CTA of the cluster staged its split's partial; CTA `rank` sums slice `rank` of
    // the tile over the cluster's CTAs in rank order (deterministic) and writes it to the
    // cluster's partial (or dw when one cluster covers all splits)
    tc::cluster_sync();
    const uint32_t rank = tc::cluster_ctarank();
    int cb, nt, kb0, kb1;
    decode(blockIdx.x, cb, nt, kb0, kb1);
    const int grp = (blockIdx.x % P.splits) / P.cs;
    float *o = P.out + ((size_t)grp * P.Co + nt * 64) * P.Mr;
    const uint32_t tbase = tc::smem_u32(smem);
    const int per = kWTileFloats / P.cs;  // a multiple of 4 for cs in {2, 4, 8}
    const int g0 = (int)rank * per / 4, g1 = g0 + per / 4;
    for (int gq = g0 + (int)threadIdx.x; gq < g1; gq += blockDim.x) {
      float4 part[8];
#pragma unroll
      for (int r = 0; r < 8; ++r)  // every rank's four floats in flight at once ...
        if (r < P.cs) part[r] = tc::ld_dsmem_f32x4(tbase + 16u * (uint32_t)gq, (uint32_t)r);
      float4 sum = part[0];
#pragma unroll
      for (int r = 1; r < 8; ++r)  // ... then added in rank order (deterministic)
        if (r < P.cs) {
          sum.x += part[r].x; sum.y += part[r].y; sum.z += part[r].z; sum.w += part[r].w;
        }
      const int e = 4 * gq;
      int i, c, rw;
      if (e < 4 * 64 * 128) {
        i = e >> 13;
        c = (e >> 7) & 63;
        rw = e & 127;
      } else {
        i = 4;
        c = (e - 4 * 64 * 128) >> 6;
        rw = 64 + ((e - 4 * 64 * 128) & 63);
      }
      const int hf = rw >> 6, tap = hf ? tap_b(i) : tap_a(i);  // four consecutive rows of one half
      *reinterpret_cast<float4 *>(o + (size_t)c * P.Mr + tap * P.Ci + cb * 64 + (rw & 63)) = sum;
    }
    tc::cluster_sync();  // the peers have read this CTA's tile
  }
}

struct WHaloPlan {
  int pb, HR, box_rows, splits, kb_per_split, KBtot, cs;
  size_t smem;
};
WHaloPlan whalo_plan(int B, int H, int W, int Ci, int Co, int ctas_override = 0) {
  WHaloPlan p{};
  static const int pb_env = env_int("PETRA_WGRAD_HALO_PB", 128);
  p.pb = pb_env == 128 ? 128 : 64;
  const int need = p.pb + 2 * (W + 3);
  const int nbox = (int)cdiv(need, kBoxMax);
  p.box_rows = (int)cdiv(cdiv(need, nbox), 8) * 8;
  p.HR = nbox * p.box_rows;
  const int64_t Mp = (int64_t)B * (H + 2) * (W + 2);
  p.KBtot = (int)cdiv(Mp, p.pb);
  const int items = (Ci / 64) * (Co / 64);
  const int ctas = ctas_override > 0 ? ctas_override : wgrad_ctas("PETRA_WGRAD_HALO_CTAS");
  const int want = std::max(1, std::min(p.KBtot, (int)cdiv(ctas, items)));
  p.kb_per_split = (int)cdiv(p.KBtot, want);
  p.splits = (int)cdiv(p.KBtot, p.kb_per_split);
  const size_t ring = (size_t)kWStages * ((size_t)p.HR * 128 + (size_t)p.pb * 128);
  p.smem = 1024 + ring + 256;
  // cluster reduction of the K splits (PETRA_WGRAD_CLUSTER=8; off by default): one pass (every
  // CTA one work item), the partial tile fits in the operand ring; splits padded to a
  // multiple of the cluster with empty splits
  static const int cl = env_int("PETRA_WGRAD_CLUSTER", 1);  // 8 measured 2.4 % slower (DESIGN 7)
  p.cs = 1;
  if (cl > 1 && p.splits >= cl && ring >= (size_t)kWTileFloats * 4) {
    const int padded = (int)cdiv(p.splits, cl) * cl;
    if ((int64_t)items * padded <= kNumSMs) {
      p.cs = cl;
      p.splits = padded;
    }
  }
  return p;
}
}  // namespace

void conv_halo_prepare() {
  static std::once_flag once;
  std::call_once(once, [] {
    auto set = [](const void *f) {
      PETRA_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemLimit));
    };
    set((const void *)conv_halo_kernel<64, 4, false>);
    set((const void *)conv_halo_kernel<64, 2, false>);
    set((const void *)conv_halo_kernel<64, 1, false>);
    set((const void *)conv_halo_kernel<128, 2, false>);
    set((const void *)conv_halo_kernel<128, 1, false>);
    set((const void *)conv_halo_kernel<256, 1, false>);
    set((const void *)conv_halo_kernel<64, 4, true>);
    set((const void *)conv_halo_kernel<64, 2, true>);
    set((const void *)conv_halo_kernel<64, 1, true>);
    set((const void *)conv_halo_kernel<128, 2, true>);
    set((const void *)conv_halo_kernel<128, 1, true>);
    set((const void *)conv_halo_kernel<256, 1, true>);
    set((const void *)wgrad_halo_kernel);
  });
}

bool wgrad_halo_eligible(const ConvGeom &g) {
  if (g.k != 3 || g.s != 1 || g.Ci % 64 || g.Co % 64) return false;
  const WHaloPlan p = whalo_plan(g.B, g.H, g.W, g.Ci, g.Co);
  return p.smem <= kSmemLimit && (int64_t)g.B * (g.H + 2) * (g.W + 2) < ((int64_t)1 << 31);
}

size_t wgrad_halo_workspace(const ConvGeom &g) {
  if (!wgrad_halo_eligible(g)) return 0;
  const WHaloPlan p = whalo_plan(g.B, g.H, g.W, g.Ci, g.Co, wgrad_ctas_max("PETRA_WGRAD_HALO_CTAS"));
  const int parts = p.splits / p.cs;
  return parts > 1 ? (size_t)parts * g.Co * g.K() * sizeof(float) : 0;
}

// dw[co][kh][kw][ci] = sum over pixels of dz (x) x, both operands zero-bordered
// [B][H+2][W+2][C] bf16 (3x3 stride 1); ws: wgrad_halo_workspace bytes
void wgrad_halo_run(const ConvGeom &g, const __nv_bfloat16 *dz_pad, const __nv_bfloat16 *x_pad, float *dw, float *ws,
                    cudaStream_t st) {
  if (!wgrad_halo_eligible(g)) throw PetraError(PETRA_E_UNSUPPORTED, "wgrad_halo_run: geometry");
  conv_halo_prepare();
  const WHaloPlan pl = whalo_plan(g.B, g.H, g.W, g.Ci, g.Co);
  WHaloParams P{};
  P.Ci = g.Ci;
  P.Co = g.Co;
  P.CB = g.Ci / 64;
  P.n_nt = g.Co / 64;
  P.KBtot = pl.KBtot;
  P.kb_per_split = pl.kb_per_split;
  P.splits = pl.splits;
  const int Wp = g.W + 2;
  P.lead = Wp + 1;
  P.HR = pl.HR;
  P.box_rows = pl.box_rows;
  P.pb = pl.pb;
  for (int t = 0; t < 9; ++t) P.off[t] = (t / 3 - 1) * Wp + (t % 3 - 1);
  P.Mr = g.K();
  P.cs = pl.cs;
  const int parts = pl.splits / pl.cs;  // partials left for splitk_sum
  if (parts > 1 && !ws) throw PetraError(PETRA_E_ARG, "wgrad_halo_run: workspace required");
  P.out = parts > 1 ? ws : dw;
  const int64_t Mp = (int64_t)g.B * (g.H + 2) * Wp;
  cuuint64_t xd[2] = {(cuuint64_t)g.Ci, (cuuint64_t)Mp};
  cuuint64_t xs[1] = {(cuuint64_t)g.Ci * 2};
  cuuint32_t xb[2] = {64, (cuuint32_t)pl.box_rows};
  cuuint64_t dd[2] = {(cuuint64_t)g.Co, (cuuint64_t)Mp};
  cuuint64_t ds[1] = {(cuuint64_t)g.Co * 2};
  cuuint32_t dbx[2] = {64, 64};
  cuuint32_t es[2] = {1, 1};
  CUtensorMap tx = tma_map(x_pad, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, xd, xs, xb, es);
  CUtensorMap tdz = tma_map(dz_pad, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dd, ds, dbx, es);
  const int work = P.CB * P.n_nt * P.splits;
  if (pl.cs > 1) launch_k_cluster(wgrad_halo_kernel, work, kWThreads, pl.smem, st, pl.cs, tx, tdz, P);
  else launch_k(wgrad_halo_kernel, std::min(work, kNumSMs), kWThreads, pl.smem, st, tx, tdz, P);
  PETRA_LAUNCH_CHECK();
  if (parts > 1) splitk_sum(ws, parts, (int64_t)g.Co * g.K(), dw, st);
}

// a 3x3 stride-1 pass whose padded grid fills at least ~3/4 of a wave of work items
// (smaller grids keep the split-K path of conv_tc.cu)
bool conv_halo_eligible(int B, int H, int W, int Cred, int N) { return halo_plan(B, H, W, Cred, N).ok; }

// out[b][h][w][n] (= addend +) sum_{tap, c} a_pad[b][h+kh][w+kw][c] * wmat[n][wk(tap)*Cred + c]
// a_pad: [B][H+2][W+2][Cred] bf16 with zero borders; wmat: [N][9*Cred] bf16
// (forward: x and w; stride-1 dgrad: dz and the flipped/transposed wT, same tap order).
StatsRows conv_halo_run(int B, int H, int W, int Cred, int N, const __nv_bfloat16 *a_pad,
                        const __nv_bfloat16 *wmat, const float *addend, void *out, bool out16, float *stats,
                        cudaStream_t st) {
  const HaloPlan pl = halo_plan(B, H, W, Cred, N);
  if (!pl.ok) throw PetraError(PETRA_E_UNSUPPORTED, "conv_halo_run: geometry");
  if (out16 && addend) throw PetraError(PETRA_E_ARG, "conv_halo_run: addend needs an fp32 output");
  conv_halo_prepare();
  HaloParams P{};
  P.Hp = H + 2;
  P.Wp = W + 2;
  P.H = H;
  P.W = W;
  P.B = B;
  P.Mp = B * P.Hp * P.Wp;
  P.N = N;
  P.Cred = Cred;
  P.CB = Cred / 64;
  P.ntaps = 9;
  for (int t = 0; t < 9; ++t) {
    P.off[t] = (t / 3 - 1) * P.Wp + (t % 3 - 1);
    P.wk[t] = t;
  }
  P.lead = P.Wp + 1;
  halo_rows(pl.T, W, P.box_rows, P.HR);
  P.a_stage = (uint32_t)P.HR * 128;
  P.bstages = pl.bstages;
  P.resident = pl.resident ? 1 : 0;
  P.addend = addend;
  P.out = out;
  P.stats = stats;
  cuuint64_t adims[2] = {(cuuint64_t)Cred, (cuuint64_t)P.Mp};
  cuuint64_t ast[1] = {(cuuint64_t)Cred * 2};
  cuuint32_t abox[2] = {64, (cuuint32_t)P.box_rows};
  cuuint32_t es[2] = {1, 1};
  CUtensorMap ta = tma_map(a_pad, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, adims, ast, abox, es);
  CUtensorMap tb = kmajor_map_bf16(wmat, N, 9 * Cred, pl.BN);
  if (out16) dispatch<true>(pl.BN, pl.T, ta, tb, P, st);
  else dispatch<false>(pl.BN, pl.T, ta, tb, P, st);
  const int work = (int)cdiv(P.Mp, 128 * pl.T) * (N / pl.BN);
  if (!P.stats) return {};
  StatsRows r;
  r.groups = N / pl.BN;
  r.rows = halo_grid(work, r.groups);
  return r;
}

}  // namespace petra
