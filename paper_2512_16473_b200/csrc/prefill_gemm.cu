// prefill_gemm.cu — f4: the expert FFN of a batch of T prompt tokens on the 5th-gen
// tensor cores (sm_100a). Per routed expert e, its tokens X_e [T_e x d] (gathered, padded
// to 128-row tiles) go through
//   GEMM1 (fused SwiGLU):  H_e = silu(X_e W1_e^T) * (X_e W3_e^T)      [T_e x ff]   bf16 out
//   GEMM2 (fused combine): y[token] += w_{token,e} * (H_e W2_e^T)     [T_e x d]    fp32 RED
// Warp-specialised, one 128 x BN output tile per CTA: warp 4 = TMA producer (2-D tensor
// maps, 128-B swizzle, mbarrier ring), warp 5 = tcgen05.mma issuer (one elected lane,
// fp32 accumulators in TMEM, tcgen05.commit frees ring stages), warps 0-3 = epilogue
// (tcgen05.ld 32x32b, one TMEM lane quarter each). Weights are read straight from the
// expert cache slots (two tensor maps view the slot pool as rows of d and of ff elements).
#include <cuda_bf16.h>
#include <math.h>
#include <stdlib.h>

#include "moe_internal.cuh"
#include "tc_gemm.cuh"

namespace moe {
namespace {

using namespace tc;

// warps 0-3 and 6-9: epilogue (TMEM lane quarter = warp % 4, column half = warp >= 6);
// warp 4: TMA producer; warp 5: MMA issuer
constexpr int kThreadsTC = 320;
constexpr int kEpiWarps = 8;

// MT m-tiles per CTA tile share every B (weight) tile: operand bytes per FLOP drop by
// (1 + NB*BN/BM) / (MT + NB*BN/BM) — the GEMMs are bound by the TMA / L2 -> SM stream
// (~6.3 KB/cycle chip-wide), not by the tensor cores, at MT = 1.
template <int BN, int NB, int MT>
struct TcCfg {
  static constexpr int kA = BM * BK * 2;          // 16 KB
  static constexpr int kB = BN * BK * 2;          // 16 / 32 KB
  static constexpr int kStage = MT * kA + NB * kB;
  static constexpr int kStages = (kFusedMaxDynSmem - 2048) / kStage > 6 ? 6 : (kFusedMaxDynSmem - 2048) / kStage;
  static constexpr int kSmem = kStages * kStage + 1024 /*align*/ + 256 /*barriers*/;
  static constexpr int kAcc = MT * NB * BN;       // TMEM columns of one accumulator set
  static constexpr int kBufs = 2 * kAcc <= 512 ? 2 : 1;  // double-buffered epilogue when it fits
  static constexpr int kTmemCols = kBufs * kAcc <= 32 ? 32 : kBufs * kAcc <= 64 ? 64 : kBufs * kAcc <= 128 ? 128
                                 : kBufs * kAcc <= 256 ? 256 : 512;
  static_assert(kAcc <= 512, "accumulators exceed TMEM");
};

struct TileCoord {
  int blk;        // expert block (prefill modes)
  int a_row;      // first A row (token row in X_g / H_g, or plain row)
  int b_row[2];   // first B row of each operand (W1, W3 rows; W2 rows)
  int out_row;    // output row base (H_g row / y gather row / C row)
  int out_col;    // output column base
  int valid;
  int nm;         // valid m-tiles in the group (prefill: the last group of a block may be short)
};

// Tile enumeration (persistent CTAs take tiles id = blockIdx.x + i * gridDim.x):
//  PLAIN : m fastest within each n tile.
//  prefill: expert block, then n tile, then m tile (fastest) — the CTAs working on the m
//           tiles of one (expert, n tile) run concurrently, so each weight tile is read
//           from HBM once and re-served from L2.
template <int MT>
__device__ __forceinline__ int num_tiles(const TcArgs& p, int BN) {
  const int ntn = (p.N + BN - 1) / BN;
  if (p.mode == TC_MODE_PLAIN) return ntn * ((p.M + BM - 1) / BM);
  int n = 0;
  for (int blk = 0; blk < p.plan->nblk; ++blk)
    n += ntn * ((p.plan->mt_pref[blk + 1] - p.plan->mt_pref[blk] + MT - 1) / MT);
  return n;
}

template <int MT>
__device__ __forceinline__ TileCoord tile_of(const TcArgs& p, int BN, int id) {
  TileCoord t;
  t.valid = 1;
  t.blk = 0;
  t.nm = 1;
  const int ntn = (p.N + BN - 1) / BN;
  if (p.mode == TC_MODE_PLAIN) {
    const int ntm = (p.M + BM - 1) / BM;
    const int nt = id / ntm, mt = id - nt * ntm;
    t.a_row = mt * BM;
    t.b_row[0] = nt * BN;
    t.b_row[1] = 0;
    t.out_row = mt * BM;
    t.out_col = nt * BN;
    return t;
  }
  const PrefillPlan* pl = p.plan;
  // expert block of this tile: blocks own ntn * groups(blk) consecutive tile ids, a group
  // being MT consecutive m-tiles of the block
  int blk = 0, base = 0, mtiles = 0, ng = 0;
  while (true) {
    mtiles = pl->mt_pref[blk + 1] - pl->mt_pref[blk];
    ng = (mtiles + MT - 1) / MT;
    if (blk + 1 >= pl->nblk || id < base + ntn * ng) break;
    base += ntn * ng;
    ++blk;
  }
  const int local = id - base;
  const int nt = local / ng, g = local - nt * ng;
  const int row = pl->row_off[blk] + g * MT * BM;
  const long long slot = pl->slot[blk];
  t.blk = blk;
  t.nm = min(MT, mtiles - g * MT);
  t.a_row = row;
  t.out_row = row;
  t.out_col = nt * BN;
  if (p.mode == TC_MODE_SWIGLU) {        // B rows in the pool viewed as rows of d elements
    t.b_row[0] = (int)(slot * 3 * p.ffr + nt * BN);             // W1 rows
    t.b_row[1] = (int)(slot * 3 * p.ffr + p.ffr + nt * BN);     // W3 rows
  } else {                                // pool viewed as rows of ffr elements
    t.b_row[0] = (int)(slot * 3 * p.d + 2 * p.d + nt * BN);     // W2 rows
    t.b_row[1] = 0;
  }
  return t;
}

// Persistent, warp-specialised: warp 4 = TMA producer, warp 5 = MMA issuer (TMEM owner),
// warps 0-3 = epilogue. A CTA tile is MT m-tiles x BN columns (x NB B operands); with two
// accumulator sets in TMEM (when they fit) the epilogue of tile i overlaps the main loop of
// tile i+1.
template <int BN, int NB, int MT>
__global__ void __launch_bounds__(kThreadsTC, 1) tc_gemm_kernel(const __grid_constant__ TcArgs p) {
  using C = TcCfg<BN, NB, MT>;
  constexpr int kAcc = C::kAcc;  // TMEM columns of one accumulator set: [MT][NB][BN]
  constexpr int kBufs = C::kBufs;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::kStages * C::kStage);
  uint64_t* empty = full + C::kStages;
  uint64_t* tfull = empty + C::kStages;   // [2] accumulator ready for the epilogue
  uint64_t* tempty = tfull + 2;           // [2] accumulator drained by the epilogue
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (p.mt_c2 > 0) {
    // the routing (rows per expert) is only known here: estimate both variants as whole
    // waves of the persistent grid times the tile cost, and run only the cheaper one
    const int g = (int)gridDim.x;
    const int w1 = (num_tiles<1>(p, BN) + g - 1) / g, w2 = (num_tiles<2>(p, BN) + g - 1) / g;
    const int pick = 100 * w1 < p.mt_c2 * w2 ? 1 : 2;
    if (pick != MT) return;
  }
  const int ntiles = num_tiles<MT>(p, BN);
  if ((int)blockIdx.x >= ntiles) return;
  const int ktiles = p.K / BK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::kStages; ++s) {
      ptx::mbar_init(full + s, 1);
      ptx::mbar_init(empty + s, 1);
    }
    for (int a = 0; a < 2; ++a) {
      ptx::mbar_init(tfull + a, 1);
      ptx::mbar_init(tempty + a, kEpiWarps);   // one arrival per epilogue warp
    }
    ptx::fence_mbar_init();
  }
  if (warp == 5) tmem_alloc<C::kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 4) {
    // ---------------------------------------------------------------- TMA producer
    if (lane == 0) {
      prefetch_tmap(&p.mapA);
      prefetch_tmap(&p.mapB);
      if (p.has_stage) prefetch_tmap(&p.mapB2);
      int it = 0;  // global k-block counter (ring position)
      for (int id = blockIdx.x; id < ntiles; id += gridDim.x) {
        const TileCoord tc = tile_of<MT>(p, BN, id);
        // (M < n prefill) a routed expert not resident at the end of the prompt lives in the
        // staging area: its B operand comes through the staging view
        const bool stg = p.mode != TC_MODE_PLAIN && p.has_stage && p.plan->stage[tc.blk];
        const CUtensorMap* mb = stg ? &p.mapB2 : &p.mapB;
        if (p.mode != TC_MODE_PLAIN && p.plan->wait[tc.blk]) {  // expert filled by this call
          ptx::wait_ready(stg ? p.ready2 : p.ready, p.plan->slot[tc.blk], p.plan->gen[tc.blk]);
          asm volatile("fence.proxy.async.global;" ::: "memory");
        }
        for (int kb = 0; kb < ktiles; ++kb, ++it) {
          const int s = it % C::kStages;
          ptx::mbar_wait(empty + s, ((it / C::kStages) & 1) ^ 1);
          uint8_t* st = smem + (size_t)s * C::kStage;
          ptx::mbar_arrive_expect_tx(full + s, (uint32_t)C::kStage);
          // (a short group's extra A tile reads the following rows / TMA zero fill: unused)
          for (int i = 0; i < MT; ++i) tma_load_2d(st + i * C::kA, &p.mapA, kb * BK, tc.a_row + i * BM, full + s);
          for (int j = 0; j < NB; ++j)
            tma_load_2d(st + MT * C::kA + j * C::kB, mb, kb * BK, tc.b_row[j], full + s);
        }
      }
    }
  } else if (warp == 5) {
    // ---------------------------------------------------------------- MMA issuer
    const uint32_t idesc = umma_idesc_bf16(BM, BN);
    int it = 0, tl = 0;
    for (int id = blockIdx.x; id < ntiles; id += gridDim.x, ++tl) {
      const int acc = tl % kBufs;
      const int nm = tile_of<MT>(p, BN, id).nm;
      ptx::mbar_wait(tempty + acc, ((tl / kBufs) & 1) ^ 1);   // epilogue drained this buffer
      tc_fence_after();
      const uint32_t tacc = tmem + acc * kAcc;
      for (int kb = 0; kb < ktiles; ++kb, ++it) {
        const int s = it % C::kStages;
        ptx::mbar_wait(full + s, (it / C::kStages) & 1);
        tc_fence_after();
        if (lane == 0) {
          const uint8_t* st = smem + (size_t)s * C::kStage;
#pragma unroll
          for (int k = 0; k < BK / UK; ++k) {
#pragma unroll
            for (int i = 0; i < MT; ++i) {
              if (i >= nm) break;
              const uint64_t da = umma_desc_sw128(st + i * C::kA);
#pragma unroll
              for (int j = 0; j < NB; ++j) {
                const uint64_t db = umma_desc_sw128(st + MT * C::kA + j * C::kB);
                umma_bf16(tacc + (i * NB + j) * BN, da + 2 * k, db + 2 * k, idesc, (kb | k) != 0);
              }
            }
          }
          umma_commit(empty + s);             // stage free once these MMAs have read it
          if (kb == ktiles - 1) umma_commit(tfull + acc);  // accumulator complete
        }
        __syncwarp();
      }
    }
  } else {
    // ---------------------------------------------------------------- epilogue (warps 0-3)
    const int quarter = warp & 3, chalf = warp >= 6 ? 1 : 0;
    const int row = quarter * 32 + lane;                   // accumulator row = TMEM lane
    const int cb = chalf * (BN / 2), ce = cb + BN / 2;      // this warp's half of the columns
    int tl = 0;
    for (int id = blockIdx.x; id < ntiles; id += gridDim.x, ++tl) {
      const TileCoord tc = tile_of<MT>(p, BN, id);
      const int acc = tl % kBufs;
      ptx::mbar_wait(tfull + acc, (tl / kBufs) & 1);
      tc_fence_after();
      for (int i = 0; i < tc.nm; ++i) {
        const uint32_t tbase = tmem + acc * kAcc + i * NB * BN + ((uint32_t)(quarter * 32) << 16);
        const int orow = tc.out_row + i * BM + row;
        if (p.mode == TC_MODE_PLAIN) {
          for (int c = cb; c < ce; c += 32) {
            uint32_t v[32];
            tmem_ld32(tbase + c, v);
            if (orow < p.M) {
              float* dst = p.C + (size_t)orow * p.N + tc.out_col + c;
#pragma unroll
              for (int q = 0; q < 32; ++q)
                if (tc.out_col + c + q < p.N) dst[q] = __uint_as_float(v[q]);
            }
          }
        } else if (p.mode == TC_MODE_SWIGLU) {
          // h = silu(g) * u  (R4), rounded to bf16 for the second GEMM's A operand
          for (int c = cb; c < ce; c += 32) {
            uint32_t g[32], u[32];
            tmem_ld32(tbase + c, g);
            tmem_ld32(tbase + BN + c, u);
            __nv_bfloat162 hv[16];
#pragma unroll
            for (int q = 0; q < 32; q += 2) {
              const float g0 = __uint_as_float(g[q]), g1 = __uint_as_float(g[q + 1]);
              // fast reciprocal: h is rounded to bf16 right after (8-bit mantissa)
              const float h0 = __fdividef(g0, 1.0f + __expf(-g0)) * __uint_as_float(u[q]);
              const float h1 = __fdividef(g1, 1.0f + __expf(-g1)) * __uint_as_float(u[q + 1]);
              hv[q / 2] = __floats2bfloat162_rn(h0, h1);
            }
            __nv_bfloat162* dst = reinterpret_cast<__nv_bfloat162*>(p.H + (size_t)orow * p.ldh + tc.out_col + c);
#pragma unroll
            for (int q = 0; q < 16; q += 4) *reinterpret_cast<uint4*>(dst + q) = *reinterpret_cast<const uint4*>(hv + q);
          }
        } else {
          // y[token] += w * o: one addend per routed expert; K <= 2 keeps it exact
          const int tok = p.plan->tok[orow];
          const float w = p.plan->wrow[orow];
          for (int c = cb; c < ce; c += 32) {
            uint32_t v[32];
            tmem_ld32(tbase + c, v);
            if (tok >= 0 && tc.out_col + c < p.N) {
              float* dst = p.y + (size_t)tok * p.N + tc.out_col + c;
#pragma unroll
              for (int q = 0; q < 32; q += 4)
                asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(dst + q),
                             "f"(w * __uint_as_float(v[q])), "f"(w * __uint_as_float(v[q + 1])),
                             "f"(w * __uint_as_float(v[q + 2])), "f"(w * __uint_as_float(v[q + 3]))
                             : "memory");
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(tempty + acc);
    }
  }
  __syncthreads();
  if (warp == 5) {
    tc_fence_after();
    tmem_dealloc<C::kTmemCols>(tmem);
  }
}

// ---------------------------------------------------------------------------------------
// The prefill GEMMs on CTA PAIRS (cta_group::2): a pair computes a 256-row x 256-column tile
// (of both W1 and W3 for the SwiGLU GEMM, of W2 for the down GEMM) with 256 x 256 UMMAs issued
// by the leader CTA, each CTA loading its 128 rows of the A operand (X_g / H_g) and its
// 128-row HALF of every weight tile; each CTA's TMEM receives its 128 rows. Against one CTA
// computing two m-tiles, every SM moves half the weight bytes of a 256-wide tile and the ring
// gets more, smaller stages; the down GEMM's accumulators (256 columns per CTA) are
// double-buffered, so its epilogue (the gate-weighted fp32 reductions into y) overlaps the
// next tile's main loop.
constexpr int kPairBN = 256;
template <int MODE>
struct PairCfg {
  static constexpr int NB = MODE == TC_MODE_SWIGLU ? 2 : 1;   // weight operands per tile
  static constexpr int kA = BM * BK * 2;                      // 16 KB: this CTA's 128 A rows
  static constexpr int kBh = (kPairBN / 2) * BK * 2;          // 16 KB: this CTA's half of one weight tile
  static constexpr int kStage = kA + NB * kBh;                // 48 / 32 KB
  static constexpr int kStages = (kFusedMaxDynSmem - 2048) / kStage > 6 ? 6 : (kFusedMaxDynSmem - 2048) / kStage;
  static constexpr int kSmem = kStages * kStage + 1024 + 256;
  static constexpr int kAcc = NB * kPairBN;                   // TMEM columns of one accumulator set
  static constexpr int kBufs = 2 * kAcc <= 512 ? 2 : 1;
  static constexpr int kCols = kBufs * kAcc;
};

template <int MODE>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreadsTC, 1)
    tc_pair_kernel(const __grid_constant__ TcArgs p) {
  using C = PairCfg<MODE>;
  constexpr int NB = C::NB, kAcc = C::kAcc, kBufs = C::kBufs;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::kStages * C::kStage);
  uint64_t* empty = full + C::kStages;
  uint64_t* tfull = empty + C::kStages;      // [kBufs]
  uint64_t* tempty = tfull + 2;              // [kBufs]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  // which variant runs: decided exactly as the one-CTA kernels decide it (waves of their grid
  // times the tile cost); this kernel replaces their two-m-tile variant
  constexpr int kBN1 = MODE == TC_MODE_SWIGLU ? 128 : 256;
  if (p.mt_c2 > 0) {
    const int g = p.pick_grid;
    const int w1 = (num_tiles<1>(p, kBN1) + g - 1) / g, w2 = (num_tiles<2>(p, kBN1) + g - 1) / g;
    if (100 * w1 < p.mt_c2 * w2) return;   // the one-m-tile kernel takes this launch
  }
  const int ntiles = num_tiles<2>(p, kPairBN);
  if (pair >= ntiles) return;
  const int ktiles = p.K / BK;
  if (threadIdx.x == 0) {
    for (int s = 0; s < C::kStages; ++s) {
      ptx::mbar_init(full + s, 1);           // (the leader's: its producer's arrival + both CTAs' bytes)
      ptx::mbar_init(empty + s, 1);          // one multicast commit of the leader's MMAs
    }
    for (int a = 0; a < kBufs; ++a) {
      ptx::mbar_init(tfull + a, 1);
      ptx::mbar_init(tempty + a, 2 * kEpiWarps);  // (the leader's: every epilogue warp of both CTAs)
    }
    ptx::fence_mbar_init();
  }
  if (warp == 5) tmem_alloc_pair<C::kCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  cluster_sync();                            // both CTAs' barriers exist before any remote signal
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 4) {
    // ------------------------------------------------------------ TMA producer (both CTAs)
    if (lane == 0) {
      prefetch_tmap(&p.mapA);
      prefetch_tmap(&p.mapB);
      if (p.has_stage) prefetch_tmap(&p.mapB2);
      int it = 0;
      for (int id = pair; id < ntiles; id += npairs) {
        const TileCoord tc = tile_of<2>(p, kPairBN, id);
        const bool stg = p.has_stage && p.plan->stage[tc.blk];
        const CUtensorMap* mb = stg ? &p.mapB2 : &p.mapB;
        if (p.plan->wait[tc.blk]) {          // expert filled by this call
          ptx::wait_ready(stg ? p.ready2 : p.ready, p.plan->slot[tc.blk], p.plan->gen[tc.blk]);
          asm volatile("fence.proxy.async.global;" ::: "memory");
        }
        for (int kb = 0; kb < ktiles; ++kb, ++it) {
          const int s = it % C::kStages;
          ptx::mbar_wait(empty + s, ((it / C::kStages) & 1) ^ 1);
          uint8_t* st = smem + (size_t)s * C::kStage;
          if (rank == 0) ptx::mbar_arrive_expect_tx(full + s, 2u * (uint32_t)C::kStage);
          // (a short group's second m-tile reads the following rows / TMA zero fill: unused)
          tma_load_2d_pair(st, &p.mapA, kb * BK, tc.a_row + (int)rank * BM, full + s);
#pragma unroll
          for (int j = 0; j < NB; ++j)
            tma_load_2d_pair(st + C::kA + j * C::kBh, mb, kb * BK, tc.b_row[j] + (int)rank * (kPairBN / 2), full + s);
        }
      }
    }
  } else if (warp == 5) {
    // ------------------------------------------------------------ MMA issuer (leader CTA)
    if (rank == 0) {
      const uint32_t idesc = umma_idesc_bf16(2 * BM, kPairBN);
      int it = 0, tl = 0;
      for (int id = pair; id < ntiles; id += npairs, ++tl) {
        const int acc = tl % kBufs;
        ptx::mbar_wait(tempty + acc, ((tl / kBufs) & 1) ^ 1);  // both CTAs' epilogues drained it
        tc_fence_after();
        const uint32_t tacc = tmem + acc * kAcc;
        for (int kb = 0; kb < ktiles; ++kb, ++it) {
          const int s = it % C::kStages;
          ptx::mbar_wait(full + s, (it / C::kStages) & 1);
          tc_fence_after();
          if (lane == 0) {
            const uint8_t* st = smem + (size_t)s * C::kStage;
            const uint64_t da = umma_desc_sw128(st);
#pragma unroll
            for (int k = 0; k < BK / UK; ++k)
#pragma unroll
              for (int j = 0; j < NB; ++j)
                umma_bf16_pair(tacc + j * kPairBN, da + 2 * k, umma_desc_sw128(st + C::kA + j * C::kBh) + 2 * k, idesc,
                               (kb | k) != 0);
            umma_commit_pair(empty + s);     // the stage is free in both CTAs once these MMAs read it
            if (kb == ktiles - 1) umma_commit_pair(tfull + acc);
          }
          __syncwarp();
        }
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue (both CTAs)
    const int quarter = warp & 3, chalf = warp >= 6 ? 1 : 0;
    const int row = quarter * 32 + lane;
    const int cb = chalf * (kPairBN / 2), ce = cb + kPairBN / 2;
    int tl = 0;
    for (int id = pair; id < ntiles; id += npairs, ++tl) {
      const TileCoord tc = tile_of<2>(p, kPairBN, id);
      const int acc = tl % kBufs;
      ptx::mbar_wait(tfull + acc, (tl / kBufs) & 1);
      tc_fence_after();
      if ((int)rank < tc.nm) {
        const uint32_t tbase = tmem + acc * kAcc + ((uint32_t)(quarter * 32) << 16);
        const int orow = tc.out_row + (int)rank * BM + row;
        if (MODE == TC_MODE_SWIGLU) {
          for (int c = cb; c < ce; c += 32) {
            uint32_t g[32], u[32];
            tmem_ld32(tbase + c, g);
            tmem_ld32(tbase + kPairBN + c, u);
            __nv_bfloat162 hv[16];
#pragma unroll
            for (int q = 0; q < 32; q += 2) {
              const float g0 = __uint_as_float(g[q]), g1 = __uint_as_float(g[q + 1]);
              const float h0 = __fdividef(g0, 1.0f + __expf(-g0)) * __uint_as_float(u[q]);
              const float h1 = __fdividef(g1, 1.0f + __expf(-g1)) * __uint_as_float(u[q + 1]);
              hv[q / 2] = __floats2bfloat162_rn(h0, h1);
            }
            __nv_bfloat162* dst = reinterpret_cast<__nv_bfloat162*>(p.H + (size_t)orow * p.ldh + tc.out_col + c);
#pragma unroll
            for (int q = 0; q < 16; q += 4) *reinterpret_cast<uint4*>(dst + q) = *reinterpret_cast<const uint4*>(hv + q);
          }
        } else {
          // y[token] += w * o: one addend per routed expert; K <= 2 keeps it exact
          const int tok = p.plan->tok[orow];
          const float w = p.plan->wrow[orow];
          for (int c = cb; c < ce; c += 32) {
            uint32_t v[32];
            tmem_ld32(tbase + c, v);
            if (tok >= 0 && tc.out_col + c < p.N) {
              float* dst = p.y + (size_t)tok * p.N + tc.out_col + c;
#pragma unroll
              for (int q = 0; q < 32; q += 4)
                asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(dst + q),
                             "f"(w * __uint_as_float(v[q])), "f"(w * __uint_as_float(v[q + 1])),
                             "f"(w * __uint_as_float(v[q + 2])), "f"(w * __uint_as_float(v[q + 3]))
                             : "memory");
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(mapa_shared(tempty + acc, 0));
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();                            // no CTA frees its TMEM while the pair still uses it
  if (warp == 5) {
    tc_fence_after();
    tmem_dealloc_pair<C::kCols>(tmem);
  }
}

template <int MODE>
cudaError_t preload_pair() {
  cudaFuncAttributes fa;
  cudaError_t e = cudaFuncGetAttributes(&fa, tc_pair_kernel<MODE>);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(tc_pair_kernel<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, PairCfg<MODE>::kSmem);
  return e;
}

template <int MODE>
cudaError_t launch_pair(const TcArgs& q, int max_mtiles, int sms, cudaStream_t s) {
  const int ptiles = ((q.N + kPairBN - 1) / kPairBN) * ((max_mtiles + 1) / 2);
  const int pairs = ptiles < sms / 2 ? ptiles : sms / 2;
  tc_pair_kernel<MODE><<<2 * pairs, kThreadsTC, PairCfg<MODE>::kSmem, s>>>(q);
  return cudaGetLastError();
}

template <int BN, int NB, int MT>
cudaError_t launch_tc(const TcArgs& p, int max_tiles, int num_sms, cudaStream_t s) {
  using C = TcCfg<BN, NB, MT>;
  const int grid = max_tiles < num_sms ? max_tiles : num_sms;
  tc_gemm_kernel<BN, NB, MT><<<grid, kThreadsTC, C::kSmem, s>>>(p);
  return cudaGetLastError();
}

template <int BN, int NB, int MT>
cudaError_t preload_tc() {
  cudaFuncAttributes fa;
  cudaError_t e = cudaFuncGetAttributes(&fa, tc_gemm_kernel<BN, NB, MT>);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(tc_gemm_kernel<BN, NB, MT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             TcCfg<BN, NB, MT>::kSmem);
  return e;
}

// m-tiles per CTA tile: both prefill GEMMs take two, sharing each weight tile (one 512-column
// accumulator set, so the epilogue runs un-overlapped with the main loop; with the fast
// reciprocal in the SwiGLU epilogue that still wins: 1.52-1.57M -> 1.65-1.68M tok/s per
// Mixtral layer at T = 4096-8192, interleaved A/B on one box)
constexpr int kMtSwiglu = 2;
constexpr int kMtDown = 2;

}  // namespace

static bool pair_enabled() {  // MOE_PREFILL_PAIR=0: the one-CTA two-m-tile kernel (A/B runs)
  const char* e = getenv("MOE_PREFILL_PAIR");
  return !(e && e[0] == '0');
}

cudaError_t preload_tc_kernels() {
  cudaError_t e = preload_pair<TC_MODE_SWIGLU>();
  if (e == cudaSuccess) e = preload_pair<TC_MODE_DOWN>();
  if (e == cudaSuccess) e = preload_tc<128, 1, 1>();
  if (e == cudaSuccess) e = preload_tc<128, 2, kMtSwiglu>();
  if (e == cudaSuccess) e = preload_tc<256, 1, kMtDown>();
  if (e == cudaSuccess) e = preload_tc<128, 2, 1>();
  if (e == cudaSuccess) e = preload_tc<256, 1, 1>();
  return e;
}

// persistent grid size: the context's SM count (TcArgs.num_sms), else the current device's
static int grid_sms(const TcArgs& p) {
  if (p.num_sms > 0) return p.num_sms;
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) {
    cudaGetLastError();
    sms = 148;
  }
  return sms;
}

cudaError_t launch_tc_plain(const TcArgs& p, cudaStream_t s) {  // C = A B^T, BN = 128
  const int sms = grid_sms(p);
  return launch_tc<128, 1, 1>(p, ((p.N + 127) / 128) * ((p.M + BM - 1) / BM), sms, s);
}

// mt = m-tiles per CTA tile (1 or 2, forced): one m-tile per tile gives twice the tiles, which
// fills the 148 SMs better when a short prompt leaves few (expert, m-tile group, n tile) tiles.
// mt = 0 (auto): both variants launched, the kernels pick on the device from the exact tile
// counts (the one not picked exits before touching shared memory or TMEM). Tile costs relative
// to a 1-m-tile tile, measured at T = 8192 (many waves): SwiGLU 1.7, down 1.95.
static constexpr int kC2Swiglu = 170, kC2Down = 195;

cudaError_t launch_tc_swiglu(const TcArgs& p, int max_mtiles, int mt, cudaStream_t s) {
  const int sms = grid_sms(p);
  const int tiles = ((p.N + 127) / 128) * max_mtiles;
  TcArgs q = p;
  q.mt_c2 = mt == 0 ? kC2Swiglu : 0;
  q.pick_grid = tiles < sms ? tiles : sms;
  cudaError_t e = cudaSuccess;
  if (mt != 2) e = launch_tc<128, 2, 1>(q, tiles, sms, s);
  if (e == cudaSuccess && mt != 1) {
    if (pair_enabled() && p.ffr % kPairBN == 0 && sms >= 2) {
      e = launch_pair<TC_MODE_SWIGLU>(q, max_mtiles, sms, s);  // two m-tiles per tile on a CTA pair
    } else {
      e = launch_tc<128, 2, kMtSwiglu>(q, tiles, sms, s);
    }
  }
  return e;
}

cudaError_t launch_tc_down(const TcArgs& p, int max_mtiles, int mt, cudaStream_t s) {
  const int sms = grid_sms(p);
  const int tiles = ((p.N + 255) / 256) * max_mtiles;
  TcArgs q = p;
  q.mt_c2 = mt == 0 ? kC2Down : 0;
  q.pick_grid = tiles < sms ? tiles : sms;
  cudaError_t e = cudaSuccess;
  if (mt != 2) e = launch_tc<256, 1, 1>(q, tiles, sms, s);
  if (e == cudaSuccess && mt != 1) {
    // down GEMM on CTA pairs: opt-in (MOE_PREFILL_PAIR_DOWN=1) — interleaved A/B at T = 4096-8192
    // it measured 4-5 % below the one-CTA two-m-tile kernel, which already shares each W2
    // tile across 256 rows (the SwiGLU GEMM, two weight operands per tile, gains 10-15 %)
    const char* pd = getenv("MOE_PREFILL_PAIR_DOWN");
    if (pd && pd[0] == '1' && pair_enabled() && p.has_pair_maps && p.d % kPairBN == 0 && sms >= 2) {
      TcArgs r = q;                          // weight views with 128-row boxes (half tiles)
      r.mapB = p.mapBp;
      r.mapB2 = p.mapB2p;
      e = launch_pair<TC_MODE_DOWN>(r, max_mtiles, sms, s);
    } else {
      e = launch_tc<256, 1, kMtDown>(q, tiles, sms, s);
    }
  }
  return e;
}

}  // namespace moe
