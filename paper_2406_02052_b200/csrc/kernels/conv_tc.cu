// conv_tc.cu -- tcgen05 (5th-gen tensor core) bf16 implicit-GEMM convolutions for sm_100a.
//
// forward  z[m][co] = sum_{tap,ci} x[b][s*ho+kh-p][s*wo+kw-p][ci] * w[co][tap][ci]   (M = B*Ho*Wo)
// dgrad    dx[m][ci] = addend + sum_{tap,co} dz[.][.][co] * wT[ci][tap'][co]
//          stride 1: a plain conv of dz with the flipped/transposed weights wT;
//          stride 2: stride-phase decomposition -- output pixels (2i+ph, 2j+pw) form 4
//          sub-grids, each a stride-1 conv of dz with the taps kh = ph+p (mod 2) only.
// wgrad    dw[co][tap][ci] = sum_{pixels} dz[p][co] * x[s*p + tap offset][ci]   (split-K)
//
// Design (B200-first):
//  * persistent warp-specialised CTAs (one per SM): warp 0 = TMA producer, warp 1 =
//    tcgen05.mma issuer (one thread) + TMEM owner, warps 2-9 = epilogue (two warps per
//    TMEM lane quarter, alternating 128-byte column chunks);
//  * A (activations) is an implicit im2col: one 4-D TMA box per (tap, 64-channel
//    block), coordinates shifted by the tap offset, stride s via TMA traversal
//    strides, halo / padding from TMA's zero fill of out-of-bounds coordinates.  The
//    output grid (Gh x Gw per image) is embedded in a padded grid Hb x Wb (Wb = the
//    power of two >= Gw), so a 128-row M tile is always a rectangle of whole padded
//    rows (or whole padded images) and the box lands in smem exactly in the
//    128B-swizzled K-major layout UMMA reads.  Padding rows are computed and masked
//    in the epilogue (no store, no BN statistics); CIFAR shapes need no padding;
//  * B (weights) via 2-D TMA; fp32 accumulators in TMEM, double buffered so the
//    epilogue (tcgen05.ld -> fp32 store) of tile i overlaps the MMAs of tile i+1.
#include <cudaTypedefs.h>

#include <mutex>

#include "../errors.h"
#include "../kernels.h"
#include "tc_common.cuh"

namespace petra {
namespace {

constexpr int BM = 128, BK = 64;
constexpr int kThreads = 192;      // wgrad: 6 warps (producer, MMA, 4 epilogue)
constexpr int kEpiWarps = 8;       // conv: two epilogue warps per TMEM lane quarter (column halves)
constexpr int kConvThreads = (2 + kEpiWarps) * 32;
constexpr uint32_t A_BYTES = BM * BK * 2;
constexpr int kMaxTaps = 9;
constexpr int kMaxStatN = 512;  // widest conv output with fused BN statistics

struct ConvTCParams {
  int M, N;                  // GEMM: M = rows of the padded output grid (B_pad*Hb*Wb), N = output channels
  int CB;                    // 64-channel blocks of the reduction operand
  int Cred;                  // channels of the reduction operand (B's K = wk * Cred + c)
  int ntaps;
  int dh[kMaxTaps], dw[kMaxTaps], wk[kMaxTaps];  // A coordinate offsets, weight tap index
  int Gh, Gw;                // output grid of the GEMM (rows x cols per image)
  int Hb, Wb, B;             // padded grid per image; real images
  int s_in;                  // A row coordinate = s_in * grid_row + dh
  int OH, OW, oss, ph, pw;   // grid (i, j) -> output pixel (i*oss+ph, j*oss+pw) of an OH x OW image
  int splits, kb_per_split;  // split-K (small-M layers): splits > 1 -> partials into ws[split][M][N]
  int cs;                    // > 1: cluster split-K -- the `splits` (= cs) K slices of a tile are the cs
                             // CTAs of one thread-block cluster, one work item per CTA; partials are
                             // reduced on chip through distributed shared memory (no ws, no 2nd launch)
  float *ws;
  const float *addend;       // nullable (fp32 output only): out = addend + conv
  void *out;                 // [B*OH*OW][N], fp32 or bf16 (OUT16); written by TMA stores through tmO
  float *stats;              // nullable: BN partials, one row per CTA: [grid][N][2] (mean, M2) of the CTA's
                             // N tile columns, then float[grid] row counts (kernels.h StatsRows)
  tc::FastDiv f_sp, f_nt, f_ghw, f_wb;  // splits, N / BN, Hb * Wb, Wb (set by launch_conv)
  int rs;                    // epilogue row split allowed (PETRA_EPI_RS)
};

// Epilogue staging: each epilogue warp owns two 4 KB buffers (32 rows x 128 B, the
// 128B-swizzled layout of a TMA box); it writes one column chunk of its 32 rows,
// fences, and lane 0 issues the TMA store while the warp fills the other buffer.
// Out-of-bounds box elements (padding rows of the padded grid) are not written.
constexpr uint32_t kEpiBuf = 32 * 128;
// staging buffers per epilogue warp (PETRA_EPI_NBUF=1: one, and its 32 KB go to the operand
// ring -- a deeper ring for the latency-bound small-tile convs)
#ifndef PETRA_EPI_NBUF
#define PETRA_EPI_NBUF 2
#endif
constexpr int kEpiNBuf = PETRA_EPI_NBUF;
constexpr uint32_t kEpiBytes = kEpiWarps * kEpiNBuf * kEpiBuf;

// row `lane` of a 32 x 128 B swizzled box: 32 fp32 or 64 bf16 values
template <bool BF16>
__device__ __forceinline__ void stage_row(uint8_t *buf, int lane, const float *v) {
  const uint32_t rowp = tc::smem_u32(buf) + lane * 128;
#pragma unroll
  for (int ch = 0; ch < 8; ++ch) {
    uint4 u;
    if constexpr (BF16) {
      uint32_t w[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        __nv_bfloat162 h = __floats2bfloat162_rn(v[8 * ch + 2 * e], v[8 * ch + 2 * e + 1]);
        w[e] = *reinterpret_cast<uint32_t *>(&h);
      }
      u = make_uint4(w[0], w[1], w[2], w[3]);
    } else {
      u = make_uint4(__float_as_uint(v[4 * ch]), __float_as_uint(v[4 * ch + 1]), __float_as_uint(v[4 * ch + 2]),
                     __float_as_uint(v[4 * ch + 3]));
    }
    tc::sts128(rowp + ((ch ^ (lane & 7)) << 4), u);
  }
}

// KG: 64-channel blocks per pipeline stage.  TMA serves about one copy per ~300 cycles
// per SM whatever its size up to 32 KB (tools/micro/tma_burst.cu, profiles/r02/tuning/
// tma_burst.txt), so a stage fetches KG blocks of the same tap with ONE A copy (a 5-D
// im2col box whose outermost dimension is the channel block) and ONE B copy (a 3-D box
// over KG consecutive k-blocks of the weight matrix): KG consecutive [rows][128 B] slabs
// each, the layout the MMAs read one k-block at a time.
//
// PAIR: the CTAs of a cluster of 2 run M = 256 tiles with cta_group::2 UMMAs (DESIGN.md 7
// "CTA pairs"): CTA r computes M tile 2 * mp + r of a pair tile mp and loads only ITS 128 A
// rows and half (BN / 2 rows) of the weight tile -- the MMA reads the other half from the
// peer -- so an SM streams A + B / 2 instead of A + B per k-block (-25 % at BN = 128, -33 %
// at BN = 256); rank 0 issues the MMAs, both epilogues drain their own TMEM rows.
template <int BN, int STAGES, bool OUT16, int KG, bool PAIR = false>
__global__ void __maxnreg__(PETRA_CONV_MAXREG)
conv_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
               const __grid_constant__ CUtensorMap tmO, const __grid_constant__ CUtensorMap tmW,
               const __grid_constant__ CUtensorMap tmAdd, const __grid_constant__ ConvTCParams P) {
  pdl_wait_trigger();
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  constexpr uint32_t B_BYTES = (PAIR ? BN / 2 : BN) * BK * 2;  // this CTA's rows of the weight tile
  constexpr uint32_t STAGE_BYTES = KG * (A_BYTES + B_BYTES);
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + STAGES * STAGE_BYTES);
  uint64_t *empty = full + STAGES;
  uint64_t *tfull = empty + STAGES;
  uint64_t *tempty = tfull + 2;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tempty + 2);
  uint64_t *abar = reinterpret_cast<uint64_t *>(tmem_slot + 2);  // per epilogue warp: addend box loads
  uint8_t *sepi = smem + STAGES * STAGE_BYTES + 1024;      // [8 warps][2][32 x 128 B] epilogue staging
  // two epilogue warps per TMEM lane quarter: split by 128-byte column chunks, or -- when a
  // row is a single chunk (BN = 64, bf16 out: RS) -- by work item (each warp of the pair
  // owns one of the two TMEM accumulators), so that all eight warps work
  const bool RS = BN * (OUT16 ? 2 : 4) <= 128 && P.rs;  // (P.rs: PETRA_EPI_RS, default on)
  const int NSLOT = RS ? 8 : 4;  // statistics slots: per warp (RS) or per lane quarter
  float *sstat = reinterpret_cast<float *>(sepi + kEpiBytes);  // [NSLOT][BN][2] (mean, M2)
  int *scnt = reinterpret_cast<int *>(sstat + NSLOT * BN * 2);   // [NSLOT] valid rows

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_tiles_n = P.N / BN;
  // (m tile, n tile, K split); PAIR: (m pair tile, n tile), pair p = blockIdx.x / 2 takes
  // items p, p + gridDim.x / 2, ...
  const int n_work = PAIR ? ((P.M / BM + 1) / 2) * n_tiles_n : (P.M / BM) * n_tiles_n * P.splits;
  const int rank2 = PAIR ? (int)(blockIdx.x & 1) : 0;
  const int w_first = PAIR ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;
  const int w_step = PAIR ? (int)(gridDim.x >> 1) : (int)gridDim.x;
  const int KB = P.ntaps * P.CB;
  const int GHW = P.Hb * P.Wb;  // padded grid
  const tc::FastDiv &f_sp = P.f_sp, &f_nt = P.f_nt, &f_ghw = P.f_ghw, &f_wb = P.f_wb;
  // work item -> tile coordinates and K-block range
  auto decode = [&](int w, int &mt, int &nt, int &sp, int &kb0, int &kb1) {
    if constexpr (PAIR) {  // this CTA's M tile of pair tile w / n_tiles_n
      const int mp = tc::fdiv(w, f_nt);
      nt = w - mp * n_tiles_n;
      mt = 2 * mp + rank2;
      sp = 0;
      kb0 = 0;
      kb1 = KB;
      return;
    }
    const int tile = tc::fdiv(w, f_sp);
    sp = w - tile * P.splits;
    mt = tc::fdiv(tile, f_nt);
    nt = tile - mt * n_tiles_n;
    kb0 = sp * P.kb_per_split;
    kb1 = min(KB, kb0 + P.kb_per_split);
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      tc::mbar_init(&tfull[a], 1);
      // PAIR: the leader's MMA waits for both CTAs' epilogue warps
      tc::mbar_init(&tempty[a], (PAIR ? 2 : 1) * (RS ? kEpiWarps / 2 : kEpiWarps));
    }
    for (int a = 0; a < kEpiWarps; ++a) tc::mbar_init(&abar[a], 1);
    tc::fence_mbar_init();
    tc::tma_prefetch(&tmA);
    tc::tma_prefetch(&tmB);
  }
  if (warp == 1) {
    if constexpr (PAIR) tc::tmem_alloc2(tmem_slot, 2 * BN);
    else tc::tmem_alloc(tmem_slot, 2 * BN);
  }
  tc::tc_fence_before();
  __syncthreads();
  if constexpr (PAIR) tc::cluster_sync();  // the peer's barriers exist before any remote arrival
  tc::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer
      int stage = 0;
      uint32_t phase = 0;
      for (int w = w_first; w < n_work; w += w_step) {
        int mt, nt, sp, kb0, kb1;
        decode(w, mt, nt, sp, kb0, kb1);
        const int m0 = mt * BM;
        const int b0 = tc::fdiv(m0, f_ghw), i0 = tc::fdiv(m0 - b0 * GHW, f_wb);
        for (int kb = kb0; kb < kb1; kb += KG) {  // KG blocks of one tap (CB % KG == 0)
          const int t = kb / P.CB, cb = kb % P.CB;
          tc::mbar_wait_idle(&empty[stage], phase ^ 1);
          uint8_t *sa = smem + stage * STAGE_BYTES;
          if constexpr (PAIR) {  // both CTAs' bytes credited to the leader's full barrier
            const uint32_t lb = tc::leader_bar(&full[stage]);
            if (rank2 == 0) tc::mbar_arrive_expect_tx(&full[stage], 2 * STAGE_BYTES);
            tc::tma_load_5d_pair(sa, &tmA, lb, 0, P.dw[t], P.s_in * i0 + P.dh[t], b0, cb);
            tc::tma_load_3d_pair(sa + KG * A_BYTES, &tmB, lb, 0, nt * BN + rank2 * (BN / 2), P.wk[t] * P.CB + cb);
          } else {
            tc::mbar_arrive_expect_tx(&full[stage], STAGE_BYTES);
            tc::tma_load_5d(sa, &tmA, &full[stage], 0, P.dw[t], P.s_in * i0 + P.dh[t], b0, cb);
            tc::tma_load_3d(sa + KG * A_BYTES, &tmB, &full[stage], 0, nt * BN, P.wk[t] * P.CB + cb);
          }
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {  // ---------------- MMA issuer: warp-uniform loop, elected lane issues
    constexpr uint32_t idesc = tc::idesc_bf16(PAIR ? 2 * BM : BM, BN, 0, 0);
    int stage = 0;
    uint32_t phase = 0;
    int it = 0;
    const int w_end = (PAIR && rank2 != 0) ? 0 : n_work;  // a pair's MMAs are the leader's
    for (int w = w_first; w < w_end; w += w_step, ++it) {
      int mt, nt, sp, kb0, kb1;
      decode(w, mt, nt, sp, kb0, kb1);
      const int acc = it & 1;
      tc::mbar_wait_idle(&tempty[acc], ((it >> 1) & 1) ^ 1);
      tc::tc_fence_after();
      const uint32_t dtm = tmem_base + acc * BN;
      for (int kb = kb0; kb < kb1; kb += KG) {
        tc::mbar_wait(&full[stage], phase);
        tc::tc_fence_after();
        const uint32_t sa = tc::smem_u32(smem + stage * STAGE_BYTES);
        if (tc::elect_one()) {
#pragma unroll
          for (int g = 0; g < KG; ++g) {
            const uint64_t ad = tc::sw128_desc(sa + g * A_BYTES, 16, 1024);
            const uint64_t bd = tc::sw128_desc(sa + KG * A_BYTES + g * B_BYTES, 16, 1024);
#pragma unroll
            for (int k = 0; k < BK / 16; ++k) {  // advance 32 B (16 bf16) along K inside the swizzle row
              if constexpr (PAIR)
                tc::umma_bf16_pair(dtm, ad + 2 * k, bd + 2 * k, idesc, (kb > kb0 || g > 0 || k > 0) ? 1u : 0u);
              else
                tc::umma_bf16(dtm, ad + 2 * k, bd + 2 * k, idesc, (kb > kb0 || g > 0 || k > 0) ? 1u : 0u);
            }
          }
          if constexpr (PAIR) tc::umma_commit_pair(&empty[stage]);
          else tc::umma_commit(&empty[stage]);
        }
        __syncwarp();
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
      if (tc::elect_one()) {
        if constexpr (PAIR) tc::umma_commit_pair(&tfull[acc]);
        else tc::umma_commit(&tfull[acc]);
      }
      __syncwarp();
    }
  } else {  // ---------------- epilogue warps 2..5
    const int q = warp & 3;             // TMEM lane quarter this warp may access
    const int hc = (warp - 2) >> 2;     // column half: chunks hc, hc + 2, ... of each tile
    const int row = q * 32 + lane;
    const int slot = RS ? warp - 2 : q;
    float *my_stat = sstat + (size_t)slot * BN * 2;  // this CTA's N tile (fixed: grid % n_tiles_n == 0)
    uint8_t *ebuf = sepi + (warp - 2) * kEpiNBuf * kEpiBuf;
    int eb = 0;  // staging buffer to fill next
    if (lane == 0) {
      tc::tma_prefetch(&tmO);
      tc::tma_prefetch(&tmW);
    }
    // hand one staged chunk to the TMA engine (lane 0), after all lanes' smem writes
    auto flush = [&](const CUtensorMap *map, int c0, int c1, int c2, int c3, bool four_d) {
      tc::fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        if (four_d) tc::tma_store_4d(map, ebuf + eb * kEpiBuf, c0, c1, c2, c3);
        else tc::tma_store_2d(map, ebuf + eb * kEpiBuf, c0, c1);
        tc::bulk_commit();
      }
      eb = (eb + 1) % kEpiNBuf;
    };
    // before overwriting buffer eb: its previous store (two chunks ago) has read smem
    auto acquire = [&]() {
      if (lane == 0) tc::bulk_wait_read<kEpiNBuf - 1>();
      __syncwarp();
    };
    if (P.cs > 1) {
      // cluster split-K, one item per CTA: the accumulator is pushed to its row owners after
      // the kernel's __syncthreads and the first cluster barrier (every CTA's MMAs are done,
      // so every operand ring is free to receive)
      tc::mbar_wait(&tfull[0], 0);
      tc::tc_fence_after();
    } else {
    // per-lane shifted statistics of this warp's columns (the CTA's N tile is fixed),
    // tile after tile in registers (tc::ColStats)
    constexpr int CW = OUT16 ? 64 : 32;  // columns per 128-byte staged row
    constexpr int NCH = (BN + 2 * CW - 1) / (2 * CW);  // column chunks per warp per tile
    tc::ColStats cst[NCH];
#pragma unroll
    for (int k = 0; k < NCH; ++k) tc::colstats_zero(cst[k]);
    int nrows = 0;  // valid rows of this warp's tiles so far (warp-uniform)
    uint32_t aph = 0;  // phase of this warp's addend barrier
    int it = 0;
    for (int w = w_first; w < n_work; w += w_step, ++it) {
      int mt, nt, sp, kb0, kb1;
      decode(w, mt, nt, sp, kb0, kb1);
      const int acc = it & 1;
      if (RS && acc != hc) continue;  // the other warp of this lane quarter takes this item
      tc::mbar_wait(&tfull[acc], (it >> 1) & 1);
      tc::tc_fence_after();
      const uint32_t trow = tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN;
      const int m = mt * BM + row;
      if (P.splits > 1) {  // fp32 partial of this K split, GEMM-row order -> ws[split][M][N]
#pragma unroll 1
        for (int c = RS ? 0 : 32 * hc; c < BN; c += RS ? 32 : 64) {
          float v[32];
          tc::tmem_ld16xN<2>(trow + c, v);
          acquire();
          stage_row<false>(ebuf + eb * kEpiBuf, lane, v);
          flush(&tmW, nt * BN + c, sp * P.M + mt * BM + q * 32, 0, 0, false);
        }
      } else {
        const int b = tc::fdiv(m, f_ghw), r = m - b * GHW, i = tc::fdiv(r, f_wb), j = r - i * P.Wb;
        const bool valid = b < P.B && i < P.Gh && j < P.Gw;  // padding rows: computed, never stored
        // TMA box origin of this warp's 32 rows in the (N, Gw, Gh, B) output view
        const int m0w = mt * BM + q * 32;
        const int wb = tc::fdiv(m0w, f_ghw), wr = m0w - wb * GHW, wi = tc::fdiv(wr, f_wb), wj = wr - wi * P.Wb;
        const uint32_t vmask = __ballot_sync(0xffffffffu, valid);
#pragma unroll
        for (int k = 0; k < NCH; ++k) {
          const int c = RS ? 0 : CW * hc + 2 * CW * k;
          if (c >= BN) break;
          float v[CW];
#pragma unroll
          tc::tmem_ld16xN<CW / 16>(trow + c, v);
          if (!OUT16 && P.addend) {  // the addend box (same geometry as the store box) by TMA into the buffer
            acquire();
            if (lane == 0) {
              tc::mbar_arrive_expect_tx(&abar[warp - 2], kEpiBuf);
              tc::tma_load_4d(ebuf + eb * kEpiBuf, &tmAdd, &abar[warp - 2], nt * BN + c, wj, wi, wb);
            }
            tc::mbar_wait(&abar[warp - 2], aph);
            aph ^= 1;
            const uint32_t rowp = tc::smem_u32(ebuf + eb * kEpiBuf) + lane * 128;
#pragma unroll
            for (int ch = 0; ch < 8; ++ch) {
              const uint4 u = tc::lds128(rowp + ((ch ^ (lane & 7)) << 4));
              v[4 * ch] += __uint_as_float(u.x);
              v[4 * ch + 1] += __uint_as_float(u.y);
              v[4 * ch + 2] += __uint_as_float(u.z);
              v[4 * ch + 3] += __uint_as_float(u.w);
            }
            __syncwarp();  // every lane has read its row before stage_row overwrites the buffer
          }
          if (!valid) {  // padding row: never stored (outside the TMA box), zero for the statistics
#pragma unroll
            for (int jj = 0; jj < CW; ++jj) v[jj] = 0.f;
          }
          acquire();
          uint8_t *staged = ebuf + eb * kEpiBuf;
          stage_row<OUT16>(staged, lane, v);
          flush(&tmO, nt * BN + c, wj, wi, wb, true);
          if (P.stats)  // BN batch statistics of z as stored (reading c24), from the staged rows
            tc::colstats_tile<OUT16, true>(staged, 128, lane, vmask, nrows, cst[k]);
        }
        nrows += __popc(vmask);
      }
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if constexpr (PAIR) tc::mbar_arrive_remote(&tempty[acc], 0);  // the leader's MMA reuses both
        else tc::mbar_arrive(&tempty[acc]);
      }
    }
    if (lane == 0) tc::bulk_wait_all();
    // the CTA's statistics row: blockIdx.x (its N tile is blockIdx.x % n_tiles_n), or for a
    // pair rank * (pairs) + pair (its N tile is pair % n_tiles_n: pairs % n_tiles_n == 0)
    const int srow = PAIR ? rank2 * w_step + w_first : (int)blockIdx.x;
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
                             P.stats + ((size_t)srow * P.N + (size_t)(srow % n_tiles_n) * BN) * 2,
                             P.stats + (size_t)gridDim.x * P.N * 2 + srow);
      else
        tc::cta_stats_row<4>(sstat, scnt, BN, (warp - 2) * 32 + lane, kEpiWarps * 32,
                             P.stats + ((size_t)srow * P.N + (size_t)(srow % n_tiles_n) * BN) * 2,
                             P.stats + (size_t)gridDim.x * P.N * 2 + srow);
    }
    }  // P.cs == 1
  }
  __syncthreads();
  if (P.cs > 1) {
    // Cluster reduction.  CTA `rank` owns rows [rank * 128 / cs, (rank + 1) * 128 / cs) of the
    // tile (4 / cs groups of 32 rows).  Every CTA PUSHES its accumulator rows to their owner
    // with remote stores (st.shared::cluster: posted, no round-trip latency per access --
    // pulling with ld.shared::cluster measured latency-bound, ~2x slower than no split),
    // into the owner's operand ring as [source rank][owned row][BN] fp32, 16-byte chunks
    // XOR-swizzled by row & 7.  After the second barrier the owner sums its rows over the
    // sources in rank order (deterministic) from its own shared memory and runs the
    // epilogue on them (addend, TMA store, BN statistics: one partial row per CTA).
    tc::cluster_sync();  // every CTA's MMAs are complete: the rings are free
    if (warp >= 2) {
      const int q = warp & 3, hc = (warp - 2) >> 2, row = q * 32 + lane;
      const int rpo = BM / P.cs;  // rows per owner
      const int owner = row / rpo, lrow = row - owner * rpo;
      const uint32_t me = tc::cluster_ctarank();
      const uint32_t dst = tc::mapa(tc::smem_u32(smem) + (uint32_t)((int)me * rpo + lrow) * BN * 4, (uint32_t)owner);
      const uint32_t trow = tmem_base + ((uint32_t)(q * 32) << 16);
#pragma unroll 1
      for (int c = 32 * hc; c < BN; c += 64) {
        float v[32];
        tc::tmem_ld16xN<2>(trow + c, v);
#pragma unroll
        for (int i = 0; i < 8; ++i)
          tc::st_dsmem_f32x4(dst + ((uint32_t)(((c >> 2) + i) ^ (lrow & 7)) << 4),
                             make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]));
      }
      tc::tc_fence_before();
    }
  }
  if (P.cs > 1) __syncthreads();
  if constexpr (PAIR) tc::cluster_sync();  // the leader's last MMAs / the peer's arrivals are done
  if (warp == 1) {
    tc::tc_fence_after();
    if constexpr (PAIR) tc::tmem_dealloc2(tmem_base, 2 * BN);
    else tc::tmem_dealloc(tmem_base, 2 * BN);
  }
  if (P.cs > 1) {
    tc::cluster_sync();  // every push has landed
    if (warp >= 2) {
      const int e = warp - 2;
      const int rank = (int)tc::cluster_ctarank();
      int mt, nt, sp, kb0, kb1;
      decode(blockIdx.x, mt, nt, sp, kb0, kb1);
      const int ng = 4 / P.cs;                // 32-row groups of this rank
      constexpr int CW = OUT16 ? 64 : 32;    // columns per 128-byte staged row
      constexpr int NCHK = BN / CW;
      uint8_t *ebuf = sepi + e * kEpiNBuf * kEpiBuf;
      int eb = 0;
      uint32_t aph = 0;
      const uint32_t tile = tc::smem_u32(smem);
      if (lane == 0) tc::tma_prefetch(&tmO);
#pragma unroll 1
      for (int u = e; u < ng * NCHK; u += kEpiWarps) {
        const int g = u % ng, k = u / ng;
        const int r0 = (rank * ng + g) * 32, r = r0 + lane;  // tile rows of this unit / lane
        const int m = mt * BM + r;
        const int b = tc::fdiv(m, f_ghw), rr = m - b * GHW, i = tc::fdiv(rr, f_wb), j = rr - i * P.Wb;
        const bool valid = b < P.B && i < P.Gh && j < P.Gw;
        const int m0w = mt * BM + r0;
        const int wb = tc::fdiv(m0w, f_ghw), wr = m0w - wb * GHW, wi = tc::fdiv(wr, f_wb), wj = wr - wi * P.Wb;
        const uint32_t vmask = __ballot_sync(0xffffffffu, valid);
        float v[CW];
        const int lr = r - rank * BM / P.cs;  // owned row index
        const uint32_t src0 = tile + (uint32_t)lr * BN * 4, sstride = (uint32_t)(BM / P.cs) * BN * 4;
#pragma unroll
        for (int c4 = 0; c4 < CW / 4; ++c4) {
          const uint32_t a = src0 + ((uint32_t)(((k * CW) >> 2) + c4) ^ (uint32_t)(lr & 7)) * 16u;
          uint4 pr[4];
#pragma unroll
          for (int q2 = 0; q2 < 4; ++q2)  // the sources' partials, added in rank order
            if (q2 < P.cs) pr[q2] = tc::lds128(a + (uint32_t)q2 * sstride);
          float4 sum = make_float4(__uint_as_float(pr[0].x), __uint_as_float(pr[0].y), __uint_as_float(pr[0].z),
                                   __uint_as_float(pr[0].w));
#pragma unroll
          for (int q2 = 1; q2 < 4; ++q2)
            if (q2 < P.cs) {
              sum.x += __uint_as_float(pr[q2].x);
              sum.y += __uint_as_float(pr[q2].y);
              sum.z += __uint_as_float(pr[q2].z);
              sum.w += __uint_as_float(pr[q2].w);
            }
          v[4 * c4] = sum.x;
          v[4 * c4 + 1] = sum.y;
          v[4 * c4 + 2] = sum.z;
          v[4 * c4 + 3] = sum.w;
        }
        if (!OUT16 && P.addend) {  // the addend box (the store box's geometry) by TMA
          if (lane == 0) tc::bulk_wait_read<kEpiNBuf - 1>();
          __syncwarp();
          if (lane == 0) {
            tc::mbar_arrive_expect_tx(&abar[e], kEpiBuf);
            tc::tma_load_4d(ebuf + eb * kEpiBuf, &tmAdd, &abar[e], nt * BN + k * CW, wj, wi, wb);
          }
          tc::mbar_wait(&abar[e], aph);
          aph ^= 1;
          const uint32_t sp_ = tc::smem_u32(ebuf + eb * kEpiBuf) + lane * 128;
#pragma unroll
          for (int ch = 0; ch < 8; ++ch) {
            const uint4 w4 = tc::lds128(sp_ + ((ch ^ (lane & 7)) << 4));
            v[4 * ch] += __uint_as_float(w4.x);
            v[4 * ch + 1] += __uint_as_float(w4.y);
            v[4 * ch + 2] += __uint_as_float(w4.z);
            v[4 * ch + 3] += __uint_as_float(w4.w);
          }
          __syncwarp();
        }
        if (!valid) {
#pragma unroll
          for (int jj = 0; jj < CW; ++jj) v[jj] = 0.f;
        }
        if (lane == 0) tc::bulk_wait_read<kEpiNBuf - 1>();
        __syncwarp();
        uint8_t *staged = ebuf + eb * kEpiBuf;
        stage_row<OUT16>(staged, lane, v);
        tc::fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          tc::tma_store_4d(&tmO, staged, nt * BN + k * CW, wj, wi, wb);
          tc::bulk_commit();
        }
        eb = (eb + 1) % kEpiNBuf;
        if (P.stats) {  // this unit's 32 rows x CW columns into the statistics slot of group g
          tc::ColStats cst;
          tc::colstats_zero(cst);
          tc::colstats_tile<OUT16, true>(staged, 128, lane, vmask, 0, cst);
          const int nv = __popc(vmask);
          const int col = k * CW + (OUT16 ? 2 * lane : lane);
          float *slot = sstat + (size_t)g * BN * 2;
          const float2 a0 = tc::colstats_final(cst, 0, nv);
          slot[2 * col] = a0.x;
          slot[2 * col + 1] = a0.y;
          if (OUT16) {
            const float2 a1 = tc::colstats_final(cst, 1, nv);
            slot[2 * col + 2] = a1.x;
            slot[2 * col + 3] = a1.y;
          }
          if (k == 0 && lane == 0) scnt[g] = nv;
        }
      }
      if (lane == 0) tc::bulk_wait_all();
      if (P.stats) {
        if (e == 0 && lane >= ng && lane < 4) scnt[lane] = 0;  // slots of no rows
        asm volatile("bar.sync 1, %0;" ::"n"(kEpiWarps * 32) : "memory");
        const int ridx = sp * (P.M / BM) * n_tiles_n + mt * n_tiles_n + nt;  // ridx % n_tiles_n == nt
        tc::cta_stats_row<4>(sstat, scnt, BN, e * 32 + lane, kEpiWarps * 32,
                             P.stats + ((size_t)ridx * P.N + (size_t)nt * BN) * 2,
                             P.stats + (size_t)gridDim.x * P.N * 2 + ridx);
      }
    }
  }
}

// BN statistics from the fused partials part[P][N][2] = (mean, M2) per conv CTA and the
// rows' counts cnt[P] (at part + P * N * 2).  A block of 8 warps per 32 channels (lane =
// channel, coalesced); warp w takes rows w, w + 8, ... and accumulates in fp64, shifted by
// the group's first row mean m0:  A = sum n_r (m_r - m0),  B = sum n_r (m_r - m0)^2,
// W = sum M2_r, n = sum n_r  (the pairwise / Chan combination of (count, mean, M2)
// triples written as sums: M2 = W + B - A^2 / n); the 8 warp results are added in warp
// order (deterministic).  Biased variance for the normalisation, unbiased for the
// running-stat EMA (reading c9).
template <int NW>
__global__ void __launch_bounds__(NW * 32) stats_finalize_kernel(const float *__restrict__ part, int P, int groups, int N,
                                                             int64_t M, float eps, float *__restrict__ mean,
                                                             float *__restrict__ invstd, float *__restrict__ rmean,
                                                             float *__restrict__ rvar, float mom) {
  pdl_wait_trigger();
  __shared__ double sh[4][NW][33];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int c = blockIdx.x * 32 + lane;
  const float *cnt = part + (size_t)P * N * 2;
  double A = 0, Bq = 0, Wm = 0, n = 0, m0 = 0;
  if (c < N) {
    // rows of this column's group: r = grp, grp + groups, ... (nr rows)
    const int grp = c / (N / groups), nr = (P - grp + groups - 1) / groups;
    m0 = part[((size_t)grp * N + c) * 2];
    int j = w;
    // four rows' loads in flight before their (in-order) accumulation: the merge is
    // L2-latency bound
    for (; j + 3 * NW < nr; j += 4 * NW) {
      float2 u[4];
      float cn[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int r = grp + (j + NW * k) * groups;
        u[k] = *reinterpret_cast<const float2 *>(part + ((size_t)r * N + c) * 2);
        cn[k] = cnt[r];
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const double nr_ = cn[k], d = (double)u[k].x - m0;
        A += nr_ * d;
        Bq += nr_ * d * d;
        Wm += u[k].y;
        n += nr_;
      }
    }
    for (; j < nr; j += NW) {
      const int r = grp + j * groups;
      const float2 u = *reinterpret_cast<const float2 *>(part + ((size_t)r * N + c) * 2);
      const double nr_ = cnt[r], d = (double)u.x - m0;
      A += nr_ * d;
      Bq += nr_ * d * d;
      Wm += u.y;
      n += nr_;
    }
  }
  sh[0][w][lane] = A;
  sh[1][w][lane] = Bq;
  sh[2][w][lane] = Wm;
  sh[3][w][lane] = n;
  __syncthreads();
  if (w == 0 && c < N) {
    A = Bq = Wm = n = 0;
    for (int k = 0; k < NW; ++k) {
      A += sh[0][k][lane];
      Bq += sh[1][k][lane];
      Wm += sh[2][k][lane];
      n += sh[3][k][lane];
    }
    const double mu = n > 0 ? m0 + A / n : 0.0;
    double M2 = n > 0 ? Wm + Bq - A * A / n : 0.0;
    if (M2 < 0.0) M2 = 0.0;
    const double var = M > 0 ? M2 / (double)M : 0.0;  // n == M: every valid output row once
    mean[c] = (float)mu;
    invstd[c] = (float)(1.0 / sqrt(var + (double)eps));
    if (rmean) {
      const double unb = M > 1 ? M2 / (double)(M - 1) : var;
      rmean[c] = (float)((1.0 - mom) * rmean[c] + mom * mu);
      rvar[c] = (float)((1.0 - mom) * rvar[c] + mom * unb);
    }
  }
}

// out[opix(m)][n] = addend + sum over splits of ws[s][m][n]  (fixed order: deterministic)
template <bool OUT16>
__global__ void splitk_out_kernel(const ConvTCParams P) {
  pdl_wait_trigger();
  const int N4 = P.N / 4;
  const int64_t n = (int64_t)P.M * N4;
  const int GHW = P.Hb * P.Wb;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int m = (int)(i / N4), c = (int)(i % N4) * 4;
    const int b = m / GHW, r = m % GHW, ii = r / P.Wb, jj = r % P.Wb;
    if (b >= P.B || ii >= P.Gh || jj >= P.Gw) continue;  // padding row
    float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int z = 0; z < P.splits; ++z) {
      float4 v = *reinterpret_cast<const float4 *>(P.ws + ((int64_t)z * P.M + m) * P.N + c);
      s.x += v.x; s.y += v.y; s.z += v.z; s.w += v.w;
    }
    const int64_t o = (((int64_t)b * P.OH + ii * P.oss + P.ph) * P.OW + jj * P.oss + P.pw) * P.N + c;
    if (P.addend) {
      float4 a = *reinterpret_cast<const float4 *>(P.addend + o);
      s.x += a.x; s.y += a.y; s.z += a.z; s.w += a.w;
    }
    if constexpr (OUT16) {
      __nv_bfloat162 lo = __floats2bfloat162_rn(s.x, s.y), hi = __floats2bfloat162_rn(s.z, s.w);
      *reinterpret_cast<uint2 *>(static_cast<__nv_bfloat16 *>(P.out) + o) =
          make_uint2(*reinterpret_cast<uint32_t *>(&lo), *reinterpret_cast<uint32_t *>(&hi));
    } else {
      *reinterpret_cast<float4 *>(static_cast<float *>(P.out) + o) = s;
    }
  }
}

// ------------------------------------------------------------------ wgrad
// D[r][n] = sum_p x[s*p + off(tap(r))][ci(r)] * dz[p][n],  r = tap*Ci + ci (M side),
// n = output channel (N side), p = output pixel of the PADDED grid (K, 64 per
// block; padding pixels read dz out of bounds -> zero, so they add nothing).  Both
// operands are MN-major in smem: A = two 64-channel boxes (rows r0..r0+63 and
// r0+64..r0+127, each possibly another tap) of 64 shifted pixels, B = BN/64 boxes
// of dz.  Split-K
// over pixel blocks; the epilogue stores D transposed, ws[split][n][r] -- the weight
// layout [Co][k][k][Ci] -- so the fixed-order reduction over splits yields dW.
struct WgradParams {
  int Mr;                 // taps * Ci (rows of D)
  int N;                  // Co
  int Ci, k, p, s;
  int Hb, Wb;             // padded output pixel grid per image
  int KBtot;              // pixel blocks of 64 (padded grid)
  int kb_per_split;
  int n_mt, n_nt, splits;
  int xg;                 // 2: both 64-row halves of an M tile are consecutive channel blocks of one
                          // tap (Ci % 128 == 0): ONE 2-block x copy; 1: a copy per half
  float *out;             // [splits][N][Mr]
};

template <int BN, int STAGES>
__global__ void __launch_bounds__(kThreads, 1)
wgrad_tc_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmDZ,
                const __grid_constant__ WgradParams P) {
  pdl_wait_trigger();
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  constexpr uint32_t HALF_A = 64 * 64 * 2;  // one 64x64 bf16 box
  constexpr uint32_t B_BYTES = BN * 64 * 2;
  constexpr uint32_t STAGE_BYTES = 2 * HALF_A + B_BYTES;
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + STAGES * STAGE_BYTES);
  uint64_t *empty = full + STAGES;
  uint64_t *tfull = empty + STAGES;
  uint64_t *tempty = tfull + 2;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_work = P.n_mt * P.n_nt * P.splits;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      tc::mbar_init(&tfull[a], 1);
      tc::mbar_init(&tempty[a], 4);
    }
    tc::fence_mbar_init();
    tc::tma_prefetch(&tmX);
    tc::tma_prefetch(&tmDZ);
  }
  if (warp == 1) tc::tmem_alloc(tmem_slot, 2 * BN);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  auto decode = [&](int w, int &mt, int &nt, int &sp) {
    sp = w % P.splits;
    int r = w / P.splits;
    nt = r % P.n_nt;
    mt = r / P.n_nt;
  };
  const int GHW = P.Hb * P.Wb;
  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int w = blockIdx.x; w < n_work; w += gridDim.x) {
        int mt, nt, sp;
        decode(w, mt, nt, sp);
        const int kb0 = sp * P.kb_per_split, kb1 = min(P.KBtot, kb0 + P.kb_per_split);
        int tapj[2], ci0j[2];
        bool valid[2];
        for (int j = 0; j < 2; ++j) {
          int r = mt * 128 + j * 64;
          valid[j] = r < P.Mr;
          tapj[j] = r / P.Ci;
          ci0j[j] = r % P.Ci;
        }
        const uint32_t bytes = (valid[1] ? 2 : 1) * HALF_A + B_BYTES;
        // TMA serves ~one copy per ~300 cycles per SM whatever its size (tma_burst.cu):
        // the x halves in one 2-block copy when they share a tap, dz in one BN/64-block copy
        for (int kb = kb0; kb < kb1; ++kb) {
          const int p0 = kb * 64;
          const int b0 = p0 / GHW, i0 = (p0 % GHW) / P.Wb;
          tc::mbar_wait_idle(&empty[stage], phase ^ 1);
          uint8_t *sa = smem + stage * STAGE_BYTES;
          tc::mbar_arrive_expect_tx(&full[stage], bytes);
          for (int j = 0; j < 2; j += P.xg) {
            if (!valid[j]) continue;
            const int kh = tapj[j] / P.k, kw = tapj[j] % P.k;
            tc::tma_load_5d(sa + j * HALF_A, &tmX, &full[stage], 0, kw - P.p, P.s * i0 + kh - P.p, b0, ci0j[j] / 64);
          }
          tc::tma_load_5d(sa + 2 * HALF_A, &tmDZ, &full[stage], 0, 0, i0, b0, nt * (BN / 64));
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {  // MMA issuer: warp-uniform loop, elected lane issues
    constexpr uint32_t idesc = tc::idesc_bf16(128, BN, 1, 1);
    int stage = 0;
    uint32_t phase = 0;
    int it = 0;
    for (int w = blockIdx.x; w < n_work; w += gridDim.x, ++it) {
      int mt, nt, sp;
      decode(w, mt, nt, sp);
      const int kb0 = sp * P.kb_per_split, kb1 = min(P.KBtot, kb0 + P.kb_per_split);
      const int acc = it & 1;
      tc::mbar_wait_idle(&tempty[acc], ((it >> 1) & 1) ^ 1);
      tc::tc_fence_after();
      const uint32_t dtm = tmem_base + acc * BN;
      for (int kb = kb0; kb < kb1; ++kb) {
        tc::mbar_wait(&full[stage], phase);
        tc::tc_fence_after();
        const uint32_t sa = tc::smem_u32(smem + stage * STAGE_BYTES);
        // MN-major: LBO = next 64-element MN block (8 KB), SBO = next 8 K-rows (1 KB)
        const uint64_t ad = tc::sw128_desc(sa, HALF_A, 1024);
        const uint64_t bd = tc::sw128_desc(sa + 2 * HALF_A, HALF_A, 1024);
        if (tc::elect_one()) {
#pragma unroll
          for (int k = 0; k < 4; ++k)  // 16 pixels = 16 rows x 128 B = 2048 B per step
            tc::umma_bf16(dtm, ad + (uint64_t)(k * 2048 >> 4), bd + (uint64_t)(k * 2048 >> 4), idesc,
                          (kb > kb0 || k) ? 1u : 0u);
          tc::umma_commit(&empty[stage]);
        }
        __syncwarp();
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
      if (tc::elect_one()) tc::umma_commit(&tfull[acc]);
      __syncwarp();
    }
  } else {
    const int q = warp & 3;
    const int row = q * 32 + lane;
    int it = 0;
    for (int w = blockIdx.x; w < n_work; w += gridDim.x, ++it) {
      int mt, nt, sp;
      decode(w, mt, nt, sp);
      const int acc = it & 1;
      tc::mbar_wait(&tfull[acc], (it >> 1) & 1);
      tc::tc_fence_after();
      const int r = mt * 128 + row;
      float *o = P.out + (int64_t)sp * P.N * P.Mr;
#pragma unroll 1
      for (int c = 0; c < BN; c += 64) {
        float v[64];
        tc::tmem_ld16xN<4>(tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN + c, v);
        if (r < P.Mr) {
#pragma unroll
          for (int jj = 0; jj < 64; ++jj) o[(int64_t)(nt * BN + c + jj) * P.Mr + r] = v[jj];
        }
      }
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&tempty[acc]);
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc::tc_fence_after();
    tc::tmem_dealloc(tmem_base, 2 * BN);
  }
}

// out[i] = sum over splits z of part[z * n + i], float4 columns: a block takes 32 float4
// columns, its 8 warps take splits w, w + 8, ... (up to four 16-byte loads in flight per
// thread before the adds), and the 8 warp sums are added in warp order through smem --
// a fixed order (deterministic) with every split of a column read in one round trip
// per four splits per warp instead of per four splits per thread
__global__ void __launch_bounds__(256) splitk_sum4_kernel(const float4 *__restrict__ part, int splits, int64_t n4,
                                                         float4 *__restrict__ out) {
  pdl_wait_trigger();
  __shared__ float4 sh[8][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t i = (int64_t)blockIdx.x * 32 + lane;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  if (i < n4) {
    const float4 *p = part + i;
    int z = w;
    for (; z + 24 < splits; z += 32) {
      float4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = __ldcg(p + (int64_t)(z + 8 * u) * n4);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        acc.x += v[u].x; acc.y += v[u].y; acc.z += v[u].z; acc.w += v[u].w;
      }
    }
    for (; z < splits; z += 8) {
      const float4 v = __ldcg(p + (int64_t)z * n4);
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
  }
  sh[w][lane] = acc;
  __syncthreads();
  if (w == 0 && i < n4) {
    float4 s = sh[0][lane];
#pragma unroll
    for (int k = 1; k < 8; ++k) {
      s.x += sh[k][lane].x; s.y += sh[k][lane].y; s.z += sh[k][lane].z; s.w += sh[k][lane].w;
    }
    out[i] = s;
  }
}

__global__ void splitk_sum_kernel(const float *__restrict__ part, int splits, int64_t n, float *__restrict__ out) {
  pdl_wait_trigger();
  // 4 independent accumulators (4 loads in flight), combined in a fixed order: deterministic
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
    int z = 0;
    for (; z + 3 < splits; z += 4) {
      s0 += part[(int64_t)z * n + i];
      s1 += part[(int64_t)(z + 1) * n + i];
      s2 += part[(int64_t)(z + 2) * n + i];
      s3 += part[(int64_t)(z + 3) * n + i];
    }
    for (; z < splits; ++z) s0 += part[(int64_t)z * n + i];
    out[i] = (s0 + s1) + (s2 + s3);
  }
}

// out = addend (or 0) on every pixel (h, w) whose phase bit (h&1)*2 + (w&1) is set
// in `mask`: the stride-2 dgrad phases without taps, all in one launch (float4)
__global__ void phase_fill_kernel(int B, int OH, int OW, int C, int mask, const float *__restrict__ addend,
                                  float *__restrict__ out) {
  pdl_wait_trigger();
  // one pixel row (b, h) per block iteration, rows without a masked phase skipped whole;
  // (w, c) from the thread index by a shift when C / 4 is a power of two (no 64-bit
  // divisions per element)
  const int C4 = C / 4, rowlen = OW * C4;
  const int sh = (C4 & (C4 - 1)) == 0 ? __ffs(C4) - 1 : -1;
  for (int row = blockIdx.x; row < B * OH; row += gridDim.x) {
    const int h = row % OH;
    const int m = (mask >> ((h & 1) * 2)) & 3;  // phases (h, w even) / (h, w odd) of this row
    if (!m) continue;
    const float4 *a = addend ? reinterpret_cast<const float4 *>(addend) + (int64_t)row * rowlen : nullptr;
    float4 *o = reinterpret_cast<float4 *>(out) + (int64_t)row * rowlen;
    for (int j = threadIdx.x; j < rowlen; j += blockDim.x) {
      const int w = sh >= 0 ? j >> sh : j / C4;
      if (!((m >> (w & 1)) & 1)) continue;
      o[j] = a ? a[j] : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  }
}

// ------------------------------------------------------------------ host side
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void *p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  if (!fn) throw PetraError(PETRA_E_CUDA, "cuTensorMapEncodeTiled unavailable");
  return fn;
}

CUtensorMap make_map(const void *base, int rank, const cuuint64_t *dims, const cuuint64_t *strides_bytes,
                     const cuuint32_t *box, const cuuint32_t *es,
                     CUtensorMapDataType dt = CU_TENSOR_MAP_DATA_TYPE_BFLOAT16) {
  CUtensorMap m;
  CUresult r = encode_fn()(&m, dt, rank, const_cast<void *>(base), dims,
                           strides_bytes, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw PetraError(PETRA_E_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string(r));
  return m;
}

// activation map [B][H][W][C] bf16 (or the interior of a zero-bordered [B][H+2][W+2][C]
// buffer: padded); box = (64 ch, Gw output cols, R output rows, NB images) read with
// traversal stride s along W and H (the box spans s*Gw x s*R inputs)
CUtensorMap act_map(const __nv_bfloat16 *x, int B, int H, int W, int C, int Gw, int R, int NB, int s,
                    bool padded = false) {
  const int P = padded ? 1 : 0;
  const __nv_bfloat16 *base = x + (padded ? ((int64_t)(W + 2) + 1) * C : 0);
  cuuint64_t dims[4] = {(cuuint64_t)C, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)B};
  cuuint64_t st[3] = {(cuuint64_t)C * 2, (cuuint64_t)(W + 2 * P) * C * 2, (cuuint64_t)(H + 2 * P) * (W + 2 * P) * C * 2};
  cuuint32_t box[4] = {64, (cuuint32_t)(Gw * s), (cuuint32_t)(R * s), (cuuint32_t)NB};
  cuuint32_t es[4] = {1, (cuuint32_t)s, (cuuint32_t)s, 1};
  return make_map(base, 4, dims, st, box, es);
}

// the same activation view with the 64-channel block as an outermost fifth dimension
// (stride 128 B): a box of kg blocks lands as kg consecutive 128-row slabs (conv_tc_kernel)
CUtensorMap act_map5(const __nv_bfloat16 *x, int B, int H, int W, int C, int Gw, int R, int NB, int s, int kg,
                     bool padded = false) {
  const int P = padded ? 1 : 0;
  const __nv_bfloat16 *base = x + (padded ? ((int64_t)(W + 2) + 1) * C : 0);
  cuuint64_t dims[5] = {64, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)B, (cuuint64_t)C / 64};
  cuuint64_t st[4] = {(cuuint64_t)C * 2, (cuuint64_t)(W + 2 * P) * C * 2,
                      (cuuint64_t)(H + 2 * P) * (W + 2 * P) * C * 2, 128};
  cuuint32_t box[5] = {64, (cuuint32_t)(Gw * s), (cuuint32_t)(R * s), (cuuint32_t)NB, (cuuint32_t)kg};
  cuuint32_t es[5] = {1, (cuuint32_t)s, (cuuint32_t)s, 1, 1};
  return make_map(base, 5, dims, st, box, es);
}

// K-major matrix [rows][K] bf16 as (64, rows, K / 64 blocks), box (64, box_rows, kg): kg
// consecutive k-blocks per copy, landing as kg [box_rows][128 B] slabs
CUtensorMap mat_map3(const __nv_bfloat16 *w, int rows, int K, int box_rows, int kg) {
  cuuint64_t dims[3] = {64, (cuuint64_t)rows, (cuuint64_t)K / 64};
  cuuint64_t st[2] = {(cuuint64_t)K * 2, 128};
  cuuint32_t box[3] = {64, (cuuint32_t)box_rows, (cuuint32_t)kg};
  cuuint32_t es[3] = {1, 1, 1};
  return make_map(w, 3, dims, st, box, es);
}

// K-major matrix [rows][K] bf16, box (64 K, box_rows)
CUtensorMap mat_map(const __nv_bfloat16 *w, int rows, int K, int box_rows) {
  cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
  cuuint64_t st[1] = {(cuuint64_t)K * 2};
  cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  return make_map(w, 2, dims, st, box, es);
}

// The output grid Gh x Gw of each image is embedded in a padded grid Hb x Wb so that
// a tile of `rows_per_tile` GEMM rows is a rectangle of whole padded rows (NB = 1,
// R rows of one image) or of NB whole padded images (R = Hb).  Wb = next power of two
// >= Gw; images are padded up to a multiple of NB.  M = Bpad * Hb * Wb.
struct Tiling {
  int Hb, Wb, R, NB, Bpad;
  bool ok;
  int64_t M() const { return (int64_t)Bpad * Hb * Wb; }
};
Tiling tiling(int B, int Gh, int Gw, int rows_per_tile) {
  Tiling t{0, 0, 0, 0, 0, false};
  int wb = 1;
  while (wb < Gw) wb <<= 1;
  if (wb > rows_per_tile) return t;
  t.Wb = wb;
  const int rows = rows_per_tile / wb;
  if (rows <= Gh) {
    t.R = rows;
    t.NB = 1;
    t.Hb = (int)cdiv(Gh, rows) * rows;
  } else {
    int hb = 1;
    while (hb < Gh) hb <<= 1;  // hb <= rows: both powers of two, Gh < rows
    t.Hb = t.R = hb;
    t.NB = rows / hb;
  }
  t.Bpad = (int)cdiv(B, t.NB) * t.NB;
  t.ok = t.M() < (int64_t)1 << 31;
  return t;
}

int pick_bn(int N) { return N % 256 == 0 ? 256 : (N % 128 == 0 ? 128 : 64); }

// N tile and K split for a conv GEMM: the largest N tile that still fills a wave
// of SMs; below that, BN = 64 and a split of K (deterministic workspace reduction).
struct ConvPlan {
  int BN, splits, kb_per_split, cs;
  bool pair;  // CTA pairs (cta_group::2, M = 256 tiles)
};
// Operand cycles of one CTA streaming `kb` k-blocks of a 128 x bn tile: the SM's TMA fill
// rate (~40 B/clk measured on the conv kernels: 24-48 KB per k-block in 600-1200 cycles,
// DESIGN.md 7) bounds these small-tile layers, not the MMAs.
static double operand_cycles(int kb, int bn) { return kb * (double)(A_BYTES + bn * BK * 2) / 40.0; }
ConvPlan conv_plan(int M, int N, int KB) {
  ConvPlan p{64, 1, KB, 1, false};
  const int mt = M / BM;
  // widest N tile that still leaves `want_tiles` tiles (wider tiles reuse each A tile
  // over more columns: fewer operand bytes from L2 per MMA)
  static const int want_tiles = env_int("PETRA_CONV_TILES", 48);  // 48: R18 +1.4 %, serial conv -4.5 % (DESIGN 7)
  static const int model = env_int("PETRA_CONV_PLAN", 1);
  if (model) {
    // PETRA_CONV_PLAN=1: the N tile with the fewest k-block rounds of the persistent grid --
    // rounds = ceil(tiles / CTAs) x the measured cycles per k-block of that tile width (~460 /
    // 610 / 710 for BN = 64 / 128 / 256) -- ties (within 5 %) to the fewer CTAs
    double best_l = 0, best_s = 0;
    bool first = true;
    for (int bn : {256, 128, 64}) {
      if (N % bn) continue;
      const int t = mt * (N / bn), ctas = conv_grid(t);
      const double c = bn == 256 ? 710.0 : (bn == 128 ? 610.0 : 460.0);
      const double lat = (double)cdiv(t, ctas) * c, smt = lat * ctas;
      if (first || lat < 0.95 * best_l || (lat <= 1.05 * best_l && smt < best_s)) {
        best_l = lat;
        best_s = smt;
        p.BN = bn;
        first = false;
      }
    }
  } else {
    for (int bn : {256, 128, 64}) {
      if (N % bn) continue;
      p.BN = bn;
      if (mt * (N / bn) >= want_tiles) break;
    }
  }
  const int tiles = mt * (N / p.BN);
  // split-K off by default: under the tick's stream concurrency the split's partial
  // traffic and second launch cost more than the SMs it fills (measured)
  static const int split_max = env_int("PETRA_SPLITK_MAX", 1);
  if (tiles * 4 < kNumSMs * 3 && split_max > 1) {  // under 75% of one wave: split K
    int want = std::max(1, std::min(split_max, (kNumSMs + tiles / 2) / tiles));
    want = std::min(want, std::max(1, KB / 4));  // at least 4 K-blocks per split
    p.kb_per_split = (int)cdiv(KB, want);
    p.splits = (int)cdiv(KB, p.kb_per_split);
  }
  // Cluster split-K for few-tile, long-K layers (R18 layers 3-4, R50 layer 4): a tile's K
  // range over cs CTAs of one cluster, reduced through DSMEM in the same kernel.  Chosen
  // when the modelled time (one CTA's operand stream + the cluster reduction) beats the
  // plain plan's by 20 %; the N tile is re-picked for it (wider tiles: fewer operand bytes).
  // off by default: R18 -11 % in the step (the clusters' co-scheduling under the tick's
  // stream concurrency), mixed alone (DESIGN.md 7 "Cluster split-K")
  static const int cs_on = env_int("PETRA_CONV_CS", 0);
  static const int cs_ctas = std::min(kNumSMs, env_int("PETRA_CONV_CS_CTAS", 128));
  static const int cs_bn = env_int("PETRA_CONV_CS_BN", 256);  // widest N tile split over a cluster
  // CTA pairs for the N >= 128 tiles: an SM then streams A + B / 2 per k-block.  Off by
  // default: exact, but no layer ran faster alone and the 1x1 K = 64 layers 1.6x slower
  // (profiles/r02/tuning/cta_pairs.txt, DESIGN.md 7 "CTA pairs")
  static const int pair_on = env_int("PETRA_CONV_PAIR", 0);
  if (pair_on && p.splits == 1 && p.BN >= 128) p.pair = true;
  if (cs_on && p.splits == 1) {
    const double t0 = (double)cdiv(tiles, conv_grid(tiles)) * operand_cycles(KB, p.BN);
    double best = 0.8 * t0;
    for (int bn : {256, 128, 64}) {
      if (N % bn) continue;
      const int t = mt * (N / bn);
      for (int cs : {4, 2}) {
        if (KB % cs || KB / cs < 4 || t * cs > cs_ctas || bn > cs_bn) continue;
        // reduction: (cs-1)/cs of the fp32 tile pushed to the peers at ~20 B/clk (DSMEM,
        // B300_MICROARCH.md)
        const double e = operand_cycles(KB / cs, bn) + (double)(cs - 1) * BM * bn * 4 / cs / 20.0;
        if (e < best) {
          best = e;
          p.BN = bn;
          p.cs = p.splits = cs;
          p.kb_per_split = KB / cs;
          p.pair = false;
        }
      }
    }
  }
  return p;
}

// Output view of a conv GEMM for the TMA-store epilogue: grid pixel (b, i, j) ->
// out[b][i*oss+ph][j*oss+pw][:] as a 4-D (N, Gw, Gh, B) tensor; the box is one epilogue
// warp's 32 GEMM rows (a run of whole padded rows / images, or a 32-wide piece of
// one padded row) x 128 bytes of columns.  Padding rows fall outside Gw / Gh / B.
CUtensorMap out_map(void *out, bool bf16, const ConvTCParams &P) {
  const int es = bf16 ? 2 : 4;
  char *base = static_cast<char *>(out) + ((int64_t)P.ph * P.OW + P.pw) * P.N * es;
  cuuint64_t dims[4] = {(cuuint64_t)P.N, (cuuint64_t)P.Gw, (cuuint64_t)P.Gh, (cuuint64_t)P.B};
  cuuint64_t st[3] = {(cuuint64_t)P.oss * P.N * es, (cuuint64_t)P.oss * P.OW * P.N * es,
                      (cuuint64_t)P.OH * P.OW * P.N * es};
  int bw = std::min(P.Wb, 32), bh = 1, bb = 1;
  if (P.Wb < 32) {
    const int rows = 32 / P.Wb;
    if (rows <= P.Hb) bh = rows;
    else { bh = P.Hb; bb = rows / P.Hb; }
  }
  cuuint32_t box[4] = {(cuuint32_t)(128 / es), (cuuint32_t)bw, (cuuint32_t)bh, (cuuint32_t)bb};
  cuuint32_t el[4] = {1, 1, 1, 1};
  return make_map(base, 4, dims, st, box, el,
                  bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32);
}

// split-K partials ws[split][M][N] fp32 as a 2-D (N, splits*M) tensor, box 32 x 32
CUtensorMap ws_map(float *ws, int N, int64_t rows) {
  cuuint64_t dims[2] = {(cuuint64_t)N, (cuuint64_t)rows};
  cuuint64_t st[1] = {(cuuint64_t)N * 4};
  cuuint32_t box[2] = {32, 32};
  cuuint32_t el[2] = {1, 1};
  return make_map(ws, 2, dims, st, box, el, CU_TENSOR_MAP_DATA_TYPE_FLOAT32);
}

// the epilogue's statistics slots: [NSLOT][BN][2] floats + NSLOT counts (conv_tc_kernel RS)
constexpr size_t conv_stat_bytes(int BN, bool OUT16) {
  return (size_t)(BN * (OUT16 ? 2 : 4) <= 128 ? 8 : 4) * BN * 8 + 32;
}
// ring depth: about 144 / 128 KB of operands in flight
constexpr int conv_stages(int BN, int KG = 1, bool pair = false) {
  // a pair's stage holds KG x (A + B / 2): 4 x 32 KB (BN = 256) / 6 x 24 KB (BN = 128), KG = 2: 2 x 64 KB /
  // 3 x 48 KB
  return pair ? (BN == 256 ? 4 : 6) / KG
              : (kEpiNBuf == 1 ? (BN == 256 ? 3 : (BN == 128 ? 5 : 7)) : (BN == 256 ? 3 : (BN == 128 ? 4 : 6))) / KG;
}
constexpr size_t conv_smem(int BN, int KG, size_t stat_bytes, bool pair = false) {
  return 1024 + (size_t)conv_stages(BN, KG, pair) * KG * (A_BYTES + (pair ? BN / 2 : BN) * BK * 2) + 1024 +
         kEpiBytes + stat_bytes;
}
// channel blocks per stage: 2 where the N tile is narrow (the copies, not the MMAs, bound
// those tiles) and the reduction has an even number of 64-channel blocks per tap
int conv_kg(int BN, int CB, int splits) {
  static const int kmax = env_int("PETRA_CONV_KG", 1);  // 2 measured ~1% slower in the step (DESIGN 7)
  return (kmax >= 2 && BN <= 128 && CB % 2 == 0 && splits == 1) ? 2 : 1;
}

// grid of a conv kernel whose epilogue writes BN partials: a multiple of the N-tile
// count, so every CTA's work items share one N tile (w = blockIdx + k * grid)
int conv_stats_grid(int work, int n_tiles_n) {
  // PETRA_CONV_TC_CTAS (default: the common cap) for the im2col kernel alone: its small-M
  // layers (few tiles, long K loops) are the ones a wider grid speeds up
  static const int tc_cap = env_int("PETRA_CONV_TC_CTAS", 0);
  const int g = tc_cap > 0 ? std::max(1, std::min({work, tc_cap, kNumSMs})) : conv_grid(work);
  return std::max(n_tiles_n, g / n_tiles_n * n_tiles_n);
}

// CTAs of a pair-tile grid: pairs a multiple of the N-tile count (every CTA keeps one N
// tile: its statistics row), under the common cap
int conv_pair_grid(int pair_work, int n_tiles_n) {
  const int pairs = std::max(1, std::min(pair_work, conv_grid(pair_work * 2) / 2));
  return 2 * std::max(n_tiles_n, pairs / n_tiles_n * n_tiles_n);
}

template <int BN, bool OUT16, int KG, bool PAIR = false>
void launch_conv(const CUtensorMap &ta, const CUtensorMap &tb, const ConvTCParams &P0, cudaStream_t st) {
  ConvTCParams P = P0;
  P.f_sp = tc::fastdiv_make(P.splits);
  P.f_nt = tc::fastdiv_make(P.N / BN);
  P.f_ghw = tc::fastdiv_make(P.Hb * P.Wb);
  P.f_wb = tc::fastdiv_make(P.Wb);
  static const int rs_on = env_int("PETRA_EPI_RS", 1);
  P.rs = rs_on;
  constexpr int STAGES = conv_stages(BN, KG, PAIR);
  const size_t smem = conv_smem(BN, KG, P.stats ? conv_stat_bytes(BN, OUT16) : 0, PAIR);  // attribute: conv_tc_prepare
  const int work = (P.M / BM) * (P.N / BN) * P.splits;
  if constexpr (PAIR) {
    const CUtensorMap to = out_map(P.out, OUT16, P);
    const CUtensorMap tad = (!OUT16 && P.addend) ? out_map(const_cast<float *>(P.addend), false, P) : to;
    const int grid = conv_pair_grid(((P.M / BM + 1) / 2) * (P.N / BN), P.N / BN);
    launch_k_cluster(conv_tc_kernel<BN, STAGES, OUT16, KG, true>, dim3(grid), dim3(kConvThreads), smem, st, 2, ta, tb,
                     to, to, tad, P);
    PETRA_LAUNCH_CHECK();
    return;
  }
  const CUtensorMap to = out_map(P.out, OUT16, P);
  // the addend in the output's geometry (fp32 outputs only)
  const CUtensorMap tad = (!OUT16 && P.addend) ? out_map(const_cast<float *>(P.addend), false, P) : to;
  if (P.cs > 1) {  // cluster split-K: one work item per CTA, clusters of cs consecutive CTAs
    launch_k_cluster(conv_tc_kernel<BN, STAGES, OUT16, KG>, dim3(work), dim3(kConvThreads), smem, st, P.cs, ta, tb,
                     to, to, tad, P);
    PETRA_LAUNCH_CHECK();
    return;
  }
  const int grid = conv_stats_grid(work, P.N / BN);
  const CUtensorMap tw = P.splits > 1 ? ws_map(P.ws, P.N, (int64_t)P.splits * P.M) : to;
  launch_k(conv_tc_kernel<BN, STAGES, OUT16, KG>, grid, kConvThreads, smem, st, ta, tb, to, tw, tad, P);
  PETRA_LAUNCH_CHECK();
  if (P.splits > 1) {
    int64_t n = (int64_t)P.M * P.N / 4;
    launch_k(splitk_out_kernel<OUT16>, (unsigned)std::min<int64_t>(cdiv(n, 256), 8 * kNumSMs), 256, 0, st, P);
    PETRA_LAUNCH_CHECK();
  }
}

// The plan of one conv GEMM launch: N tile, K split, channel blocks per stage
struct LaunchPlan {
  ConvPlan pl;
  int kg;
};
LaunchPlan launch_plan(const ConvTCParams &P, float *ws) {
  LaunchPlan L;
  L.pl = conv_plan(P.M, P.N, P.ntaps * P.CB);
  if (L.pl.splits > 1 && L.pl.cs == 1 && !ws) {
    L.pl.splits = 1;
    L.pl.kb_per_split = P.ntaps * P.CB;
  }
  static const int pair_kg = env_int("PETRA_CONV_PAIR_KG", 2);
  L.kg = L.pl.pair ? ((pair_kg == 2 && P.CB % 2 == 0) ? 2 : 1) : conv_kg(L.pl.BN, P.CB, L.pl.splits);
  return L;
}

// tensor maps are built per launch (host-side, ~1 us); B's box = (64, BN, kg); `ta` was
// built with the same kg (act_map5)
void launch_any(const CUtensorMap &ta, const LaunchPlan &L, const __nv_bfloat16 *w, int wrows, int wK,
                ConvTCParams &P, float *ws, bool out16, cudaStream_t st) {
  const ConvPlan &pl = L.pl;
  P.splits = pl.splits;
  P.kb_per_split = pl.kb_per_split;
  P.cs = pl.cs;
  P.ws = ws;
  if (P.splits > 1 && P.cs == 1) P.stats = nullptr;  // stats need final z (split-K: standalone pass)
  if (out16 && P.addend) throw PetraError(PETRA_E_ARG, "conv_tc: addend needs an fp32 output");
  CUtensorMap tb = mat_map3(w, wrows, wK, pl.pair ? pl.BN / 2 : pl.BN, L.kg);  // a pair CTA loads BN / 2 rows
  if (pl.pair) {
    if (L.kg == 2) {
      if (out16) {
        if (pl.BN == 256) launch_conv<256, true, 2, true>(ta, tb, P, st);
        else launch_conv<128, true, 2, true>(ta, tb, P, st);
      } else {
        if (pl.BN == 256) launch_conv<256, false, 2, true>(ta, tb, P, st);
        else launch_conv<128, false, 2, true>(ta, tb, P, st);
      }
      return;
    }
    if (out16) {
      if (pl.BN == 256) launch_conv<256, true, 1, true>(ta, tb, P, st);
      else launch_conv<128, true, 1, true>(ta, tb, P, st);
    } else {
      if (pl.BN == 256) launch_conv<256, false, 1, true>(ta, tb, P, st);
      else launch_conv<128, false, 1, true>(ta, tb, P, st);
    }
    return;
  }
  if (L.kg == 2) {
    if (out16) {
      if (pl.BN == 128) launch_conv<128, true, 2>(ta, tb, P, st);
      else launch_conv<64, true, 2>(ta, tb, P, st);
    } else {
      if (pl.BN == 128) launch_conv<128, false, 2>(ta, tb, P, st);
      else launch_conv<64, false, 2>(ta, tb, P, st);
    }
    return;
  }
  if (out16) {
    if (pl.BN == 256) launch_conv<256, true, 1>(ta, tb, P, st);
    else if (pl.BN == 128) launch_conv<128, true, 1>(ta, tb, P, st);
    else launch_conv<64, true, 1>(ta, tb, P, st);
  } else {
    if (pl.BN == 256) launch_conv<256, false, 1>(ta, tb, P, st);
    else if (pl.BN == 128) launch_conv<128, false, 1>(ta, tb, P, st);
    else launch_conv<64, false, 1>(ta, tb, P, st);
  }
}

bool geom_ok(const ConvGeom &g) {
  if (g.Ci % 64 || g.Co % 64 || g.k > 3) return false;
  if (g.s != 1 && g.s != 2) return false;
  if (g.s == 2 && ((g.H & 1) || (g.W & 1) || g.Ho * 2 != g.H || g.Wo * 2 != g.W)) return false;
  if (g.s == 1 && (g.Ho != g.H || g.Wo != g.W)) return false;
  return true;
}

StatsRows run_fwd(const ConvGeom &g, const __nv_bfloat16 *x, bool x_pad, const __nv_bfloat16 *w, void *out,
                  bool out16, float *ws, float *stats, cudaStream_t st) {
  if (x_pad && g.k == 3 && g.s == 1 && conv_halo_eligible(g.B, g.H, g.W, g.Ci, g.Co))
    return conv_halo_run(g.B, g.H, g.W, g.Ci, g.Co, x, w, nullptr, out, out16, stats, st);
  Tiling t = tiling(g.B, g.Ho, g.Wo, BM);
  ConvTCParams P{};
  P.M = (int)t.M();
  P.N = g.Co;
  P.Cred = g.Ci;
  P.CB = g.Ci / 64;
  P.ntaps = g.k * g.k;
  for (int tap = 0; tap < P.ntaps; ++tap) {
    P.dh[tap] = tap / g.k - g.p;
    P.dw[tap] = tap % g.k - g.p;
    P.wk[tap] = tap;
  }
  P.Gh = g.Ho;
  P.Gw = g.Wo;
  P.Hb = t.Hb;
  P.Wb = t.Wb;
  P.B = g.B;
  P.s_in = g.s;
  P.OH = g.Ho;
  P.OW = g.Wo;
  P.oss = 1;
  P.out = out;
  P.stats = stats;
  const LaunchPlan L = launch_plan(P, ws);
  CUtensorMap ta = act_map5(x, g.B, g.H, g.W, g.Ci, t.Wb, t.R, t.NB, g.s, L.kg, x_pad);
  launch_any(ta, L, w, g.Co, g.K(), P, ws, out16, st);
  if (!P.stats) return {};
  const int BN = L.pl.BN;
  StatsRows r;
  r.groups = P.N / BN;
  const int work = (P.M / BM) * (P.N / BN) * P.splits;
  r.rows = L.pl.cs > 1 ? work
           : L.pl.pair ? conv_pair_grid(((P.M / BM + 1) / 2) * r.groups, r.groups)
                       : conv_stats_grid(work, r.groups);  // one partial row per CTA
  return r;
}

void run_dgrad(const ConvGeom &g, const __nv_bfloat16 *dz, bool dz_pad, const __nv_bfloat16 *wt, const float *addend,
               float *dx, float *ws, cudaStream_t st) {
  // A = dz [B][Ho][Wo][Co] (stride-1 boxes), B = wT [Ci][k*k*Co], N = Ci
  const int wK = g.k * g.k * g.Co;
  if (dz_pad && g.k == 3 && g.s == 1 && conv_halo_eligible(g.B, g.Ho, g.Wo, g.Co, g.Ci)) {
    conv_halo_run(g.B, g.Ho, g.Wo, g.Co, g.Ci, dz, wt, addend, dx, false, nullptr, st);
    return;
  }
  Tiling t = tiling(g.B, g.Ho, g.Wo, BM);
  ConvTCParams P{};
  P.M = (int)t.M();
  P.N = g.Ci;
  P.Cred = g.Co;
  P.CB = g.Co / 64;
  P.Gh = g.Ho;
  P.Gw = g.Wo;
  P.Hb = t.Hb;
  P.Wb = t.Wb;
  P.B = g.B;
  P.s_in = 1;
  P.OH = g.H;
  P.OW = g.W;
  P.addend = addend;
  P.out = dx;
  const int k = g.k;
  if (g.s == 1) {
    P.ntaps = k * k;
    for (int tap = 0; tap < k * k; ++tap) {  // dx = conv(dz, wT): wT tap index = tap
      P.dh[tap] = tap / k - g.p;
      P.dw[tap] = tap % k - g.p;
      P.wk[tap] = tap;
    }
    P.oss = 1;
    const LaunchPlan L = launch_plan(P, ws);
    CUtensorMap ta = act_map5(dz, g.B, g.Ho, g.Wo, g.Co, t.Wb, t.R, t.NB, 1, L.kg, dz_pad);
    launch_any(ta, L, wt, g.Ci, wK, P, ws, false, st);
    return;
  }
  // stride 2: phase (ph, pw) of dx gets the taps with kh = ph + p (mod 2), kw = pw + p (mod 2);
  // dx[2i+ph][2j+pw] += dz[i + (ph+p-kh)/2][j + (pw+p-kw)/2] * w[kh][kw]
  P.oss = 2;
  int empty_mask = 0;
  for (int ph = 0; ph < 2; ++ph)
    for (int pw = 0; pw < 2; ++pw) {
      int n = 0;
      for (int kh = 0; kh < k; ++kh)
        for (int kw = 0; kw < k; ++kw) {
          if (((ph + g.p - kh) & 1) || ((pw + g.p - kw) & 1)) continue;
          P.dh[n] = (ph + g.p - kh) / 2;
          P.dw[n] = (pw + g.p - kw) / 2;
          P.wk[n] = (k - 1 - kh) * k + (k - 1 - kw);  // wT stores taps flipped
          ++n;
        }
      if (n == 0) {  // no tap reaches this phase (1x1 / stride 2): dx = addend or 0 there
        empty_mask |= 1 << (ph * 2 + pw);
        continue;
      }
      P.ntaps = n;
      P.ph = ph;
      P.pw = pw;
      const LaunchPlan L = launch_plan(P, ws);
      CUtensorMap ta = act_map5(dz, g.B, g.Ho, g.Wo, g.Co, t.Wb, t.R, t.NB, 1, L.kg, dz_pad);
      launch_any(ta, L, wt, g.Ci, wK, P, ws, false, st);
    }
  if (empty_mask) {
    static const int64_t rows_cap = (int64_t)std::max(1, env_int("PETRA_ROW_BLOCKS_PER_SM", 16)) * kNumSMs;
    launch_k(phase_fill_kernel, (unsigned)std::min<int64_t>((int64_t)g.B * g.H, rows_cap), 256, 0, st, 
        g.B, g.H, g.W, g.Ci, empty_mask, addend, dx);
    PETRA_LAUNCH_CHECK();
  }
}

struct WgradPlan {
  int BN, splits, kb_per_split, n_mt, n_nt, KBtot;
  Tiling t;
};
WgradPlan wgrad_plan(const ConvGeom &g, int ctas_override = 0) {
  WgradPlan w{};
  w.BN = g.Co % 256 == 0 ? 256 : (g.Co % 128 == 0 ? 128 : 64);
  w.n_nt = g.Co / w.BN;
  w.n_mt = (int)cdiv((int64_t)g.k * g.k * g.Ci, 128);
  w.t = tiling(g.B, g.Ho, g.Wo, 64);
  w.KBtot = (int)(w.t.M() / 64);
  int tiles = w.n_mt * w.n_nt;
  // CTAs the split-K aims to fill; workspaces are sized for the largest target
  const int ctas = ctas_override > 0 ? ctas_override : wgrad_ctas("PETRA_WGRAD_CTAS");
  int want = std::max(1, std::min(w.KBtot, (int)cdiv(ctas, tiles)));
  w.kb_per_split = (int)cdiv(w.KBtot, want);
  w.splits = (int)cdiv(w.KBtot, w.kb_per_split);
  return w;
}

template <int BN, int STAGES>
void launch_wgrad(const CUtensorMap &tx, const CUtensorMap &tdz, const WgradParams &P, cudaStream_t st) {
  size_t smem = (size_t)STAGES * (2 * 64 * 64 * 2 + BN * 64 * 2) + 1024 + 256;  // attribute: conv_tc_prepare
  int work = P.n_mt * P.n_nt * P.splits;
  launch_k(wgrad_tc_kernel<BN, STAGES>, std::min(work, kNumSMs), kThreads, smem, st, tx, tdz, P);
  PETRA_LAUNCH_CHECK();
}

}  // namespace

void conv_tc_prepare() {
  static std::once_flag once;
  std::call_once(once, [] {
    auto set = [](const void *f, int BN, int KG) {
      PETRA_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)conv_smem(BN, KG, std::max(conv_stat_bytes(BN, true),
                                                                      conv_stat_bytes(BN, false)))));
    };
    set((const void *)conv_tc_kernel<256, conv_stages(256), false, 1>, 256, 1);
    set((const void *)conv_tc_kernel<128, conv_stages(128), false, 1>, 128, 1);
    set((const void *)conv_tc_kernel<64, conv_stages(64), false, 1>, 64, 1);
    set((const void *)conv_tc_kernel<256, conv_stages(256), true, 1>, 256, 1);
    set((const void *)conv_tc_kernel<128, conv_stages(128), true, 1>, 128, 1);
    set((const void *)conv_tc_kernel<64, conv_stages(64), true, 1>, 64, 1);
    set((const void *)conv_tc_kernel<128, conv_stages(128, 2), false, 2>, 128, 2);
    set((const void *)conv_tc_kernel<64, conv_stages(64, 2), false, 2>, 64, 2);
    set((const void *)conv_tc_kernel<128, conv_stages(128, 2), true, 2>, 128, 2);
    set((const void *)conv_tc_kernel<64, conv_stages(64, 2), true, 2>, 64, 2);
    auto set2 = [](const void *f, int BN, int KG) {
      PETRA_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)conv_smem(BN, KG, std::max(conv_stat_bytes(BN, true),
                                                                      conv_stat_bytes(BN, false)), true)));
    };
    set2((const void *)conv_tc_kernel<256, conv_stages(256, 1, true), false, 1, true>, 256, 1);
    set2((const void *)conv_tc_kernel<128, conv_stages(128, 1, true), false, 1, true>, 128, 1);
    set2((const void *)conv_tc_kernel<256, conv_stages(256, 1, true), true, 1, true>, 256, 1);
    set2((const void *)conv_tc_kernel<128, conv_stages(128, 1, true), true, 1, true>, 128, 1);
    set2((const void *)conv_tc_kernel<256, conv_stages(256, 2, true), false, 2, true>, 256, 2);
    set2((const void *)conv_tc_kernel<128, conv_stages(128, 2, true), false, 2, true>, 128, 2);
    set2((const void *)conv_tc_kernel<256, conv_stages(256, 2, true), true, 2, true>, 256, 2);
    set2((const void *)conv_tc_kernel<128, conv_stages(128, 2, true), true, 2, true>, 128, 2);
    auto setw = [](const void *f, int STAGES, int BN) {
      size_t smem = (size_t)STAGES * (2 * 64 * 64 * 2 + BN * 64 * 2) + 1024 + 256;
      PETRA_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    };
    setw((const void *)wgrad_tc_kernel<256, 3>, 3, 256);
    setw((const void *)wgrad_tc_kernel<128, 4>, 4, 128);
    setw((const void *)wgrad_tc_kernel<64, 6>, 6, 64);
  });
  stem_tc_prepare();
  conv_halo_prepare();
}

bool conv_tc_supported(const ConvGeom &g, int mode) {
  if (!geom_ok(g)) return false;
  return tiling(g.B, g.Ho, g.Wo, mode == 2 ? 64 : BM).ok;
}

size_t conv_tc_workspace(const ConvGeom &g, int mode) {
  if (!conv_tc_supported(g, mode)) return 0;
  if (mode == 2) {
    WgradPlan w = wgrad_plan(g, wgrad_ctas_max("PETRA_WGRAD_CTAS"));
    return std::max(w.splits > 1 ? (size_t)w.splits * g.Co * g.K() * sizeof(float) : (size_t)0,
                    wgrad_halo_workspace(g));
  }
  const int N = mode == 0 ? g.Co : g.Ci;
  const int KB = (mode == 0 ? g.k * g.k * g.Ci : g.k * g.k * g.Co) / 64;  // upper bound (all taps)
  const int64_t M = tiling(g.B, g.Ho, g.Wo, BM).M();
  ConvPlan p = conv_plan((int)M, N, KB);
  return (p.splits > 1 && p.cs == 1) ? (size_t)p.splits * M * N * sizeof(float) : 0;
}

// the im2col kernel's plan for a forward (mode 0) or stride-1 dgrad (mode 1) pass:
// out = {BN, K splits, cluster size}
void conv_tc_plan_info(const ConvGeom &g, int mode, int *out) {
  const int N = mode == 0 ? g.Co : g.Ci;
  const int KB = (mode == 0 ? g.k * g.k * g.Ci : g.k * g.k * g.Co) / 64;
  const ConvPlan p = conv_plan((int)tiling(g.B, g.Ho, g.Wo, BM).M(), N, KB);
  out[0] = p.BN;
  out[1] = p.splits;
  out[2] = p.pair ? -2 : p.cs;
}

StatsRows conv_fwd_tc(const ConvGeom &g, const __nv_bfloat16 *x, bool x_padded, const __nv_bfloat16 *w, void *z,
                bool z_bf16, float *ws, float *stats_part, cudaStream_t st) {
  return run_fwd(g, x, x_padded, w, z, z_bf16, ws, stats_part, st);
}

void bn_stats_from_partials(const float *part, StatsRows rows, int N, int64_t M, float eps, float *mean,
                            float *invstd, float *rmean, float *rvar, float mom, cudaStream_t st) {
  // warps per 32 channels: each warp merges rows w, w + NW, ... (four loads in flight), so the
  // L2 round trips per launch are ~rows / (4 NW)
  static const int nw = env_int("PETRA_FINALIZE_WARPS", 8);
  if (nw >= 32)
    launch_k(stats_finalize_kernel<32>, (unsigned)cdiv(N, 32), 1024, 0, st, part, rows.rows, rows.groups, N, M, eps,
             mean, invstd, rmean, rvar, mom);
  else
    launch_k(stats_finalize_kernel<8>, (unsigned)cdiv(N, 32), 256, 0, st, part, rows.rows, rows.groups, N, M, eps,
             mean, invstd, rmean, rvar, mom);
  PETRA_LAUNCH_CHECK();
}

void conv_dgrad_tc(const ConvGeom &g, const __nv_bfloat16 *dz, bool dz_padded, const __nv_bfloat16 *wt,
                   const float *addend, float *dx, float *ws, cudaStream_t st) {
  run_dgrad(g, dz, dz_padded, wt, addend, dx, ws, st);
}

CUtensorMap kmajor_map_bf16(const __nv_bfloat16 *m, int rows, int K, int box_rows) {
  return mat_map(m, rows, K, box_rows);
}

CUtensorMap tma_map(const void *base, CUtensorMapDataType dt, int rank, const cuuint64_t *dims,
                    const cuuint64_t *strides_bytes, const cuuint32_t *box, const cuuint32_t *es) {
  return make_map(base, rank, dims, strides_bytes, box, es, dt);
}

// plain row-major [rows][cols] map without swizzle, box (box_cols, box_rows): the
// staging of the BN passes (bn.cu)
CUtensorMap plain_map_2d(const void *base, CUtensorMapDataType dt, int esize, int64_t rows, int cols, int box_cols,
                         int box_rows) {
  return plain_map_2d_strided(base, dt, esize, rows, cols, cols, box_cols, box_rows);
}
// the same over a [rows][ld] buffer (first `cols` columns from base)
CUtensorMap plain_map_2d_strided(const void *base, CUtensorMapDataType dt, int esize, int64_t rows, int cols, int ld,
                                 int box_cols, int box_rows) {
  CUtensorMap m;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t st[1] = {(cuuint64_t)ld * esize};
  cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = encode_fn()(&m, dt, 2, const_cast<void *>(base), dims, st, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw PetraError(PETRA_E_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string(r));
  return m;
}


void splitk_sum(const float *part, int splits, int64_t n, float *out, cudaStream_t st) {
  static const bool v4 = env_int("PETRA_SPLITK_V4", 0) != 0;  // 0: R18 +1.4 % (grid-stride, <= 4 blocks per SM)
  if (v4 && n % 4 == 0 && (uintptr_t)part % 16 == 0 && (uintptr_t)out % 16 == 0) {
    const int64_t n4 = n / 4;
    launch_k(splitk_sum4_kernel, (unsigned)cdiv(n4, 32), 256, 0, st, reinterpret_cast<const float4 *>(part), splits, n4,
             reinterpret_cast<float4 *>(out));
    PETRA_LAUNCH_CHECK();
    return;
  }
  static const int per_sm = std::max(1, env_int("PETRA_SPLITK_BLOCKS_PER_SM", 1));
  launch_k(splitk_sum_kernel, (unsigned)std::min<int64_t>(cdiv(n, 256), (int64_t)per_sm * kNumSMs), 256, 0, st, part,
           splits, n, out);
  PETRA_LAUNCH_CHECK();
}

void conv_wgrad_tc(const ConvGeom &g, const __nv_bfloat16 *dz, bool dz_padded, const __nv_bfloat16 *x,
                   bool x_padded, float *dw, float *ws, cudaStream_t st) {
  static const bool halo = env_int("PETRA_WGRAD_HALO", 1) != 0;
  if (halo && dz_padded && x_padded && wgrad_halo_eligible(g)) {
    wgrad_halo_run(g, dz, x, dw, ws, st);
    return;
  }
  WgradPlan w = wgrad_plan(g);
  static const bool xg_on = env_int("PETRA_WGRAD_XG", 1) != 0;
  const int xg = (xg_on && g.Ci % 128 == 0) ? 2 : 1;
  CUtensorMap tx = act_map5(x, g.B, g.H, g.W, g.Ci, w.t.Wb, w.t.R, w.t.NB, g.s, xg, x_padded);
  // dz [B][Ho][Wo][Co], box (64 ch, 64 padded pixels, BN / 64 channel blocks); padding
  // pixels out of bounds -> 0
  CUtensorMap tdz = act_map5(dz, g.B, g.Ho, g.Wo, g.Co, w.t.Wb, w.t.R, w.t.NB, 1, w.BN / 64, dz_padded);
  WgradParams P{};
  P.Mr = g.K();
  P.N = g.Co;
  P.Ci = g.Ci;
  P.k = g.k;
  P.p = g.p;
  P.s = g.s;
  P.Hb = w.t.Hb;
  P.Wb = w.t.Wb;
  P.KBtot = w.KBtot;
  P.kb_per_split = w.kb_per_split;
  P.n_mt = w.n_mt;
  P.n_nt = w.n_nt;
  P.splits = w.splits;
  P.xg = xg;
  P.out = w.splits > 1 ? ws : dw;
  if (w.BN == 256) launch_wgrad<256, 3>(tx, tdz, P, st);
  else if (w.BN == 128) launch_wgrad<128, 4>(tx, tdz, P, st);
  else launch_wgrad<64, 6>(tx, tdz, P, st);
  if (w.splits > 1) splitk_sum(ws, w.splits, (int64_t)g.Co * g.K(), dw, st);
}

}  // namespace petra
