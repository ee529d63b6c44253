// Warp-owned comb pass (fp32, 64 <= L <= 512), sm_100a.
//
// Same pass as K_COMB (tiled_fft.hpp:252-294: gather a comb, row FFT,
// inter-pass root, scatter back), re-organised so that no step needs the
// whole CTA:
//
//   * a tile is F = 8192 / L adjacent combs x L points (64 KB): every comb
//     step is F * 8 contiguous bytes (128..1024 B) of HBM, moved by TMA
//     tensor copies in 128-byte-wide boxes with the 128-byte swizzle;
//   * one producer warp streams tiles into an S-deep ring and streams the
//     finished tiles back out with TMA tensor stores (no per-thread global
//     stores at all);
//   * each of the 8 consumer warps owns 1024 / L whole combs of the tile and
//     runs their Stockham stages in registers, exchanging through its own
//     columns of the tile in place (rows XOR-permuted so every exchange is
//     bank-conflict free), then writes the spectrum back to the same columns.
//     Warps synchronise only with __syncwarp and per-slot mbarriers, so they
//     drift freely and the SM overlaps one warp's math with another's
//     traffic (the structure that lets K_ROWS_TMA run at 95% of HBM).
#pragma once
#include "fast_kernels.cuh"

namespace tfb {

template <int L>
struct CombWCfg {
  static_assert(L >= 64 && L <= 512, "warp-owned comb tiles cover 64 <= L <= 512");
  static constexpr int F = 8192 / L;            // combs per tile
  static constexpr int T = L / 32;              // lanes per comb (32 points per lane)
  static constexpr int CPW = 32 / T;            // combs per warp
  static constexpr int NCB = F / 16;            // 16-comb (128-byte) column blocks
  static constexpr int TILE = L * F;            // elements
  static constexpr int TILE_BYTES = TILE * 8;   // 64 KB
  static constexpr int S = 3;                   // ring depth
  static constexpr int CONSUMERS = 8;
  static constexpr int THREADS = (CONSUMERS + 1) * 32;
  static constexpr int BL = L < 256 ? L : 256;  // TMA box rows
  static constexpr int SMEM = S * TILE_BYTES + 2 * S * 8 + 1024;
};

// element offset (8-byte units) of (row n, comb f) inside a tile loaded as
// NCB column blocks of [L][16] with the 128-byte swizzle
template <int L>
__device__ __forceinline__ int cw_off(int n, int f) {
  const int b = n * 128 + (f & 15) * 8;
  return (f >> 4) * (L * 16) + ((b ^ (((b >> 7) & 7) << 4)) >> 3);
}
// row permutation of the in-place Stockham exchange (bank-conflict free
// writes at row stride 32)
__device__ __forceinline__ int cw_perm(int i) { return i ^ ((i >> 5) & 7); }

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void tma_store_4d(const CUtensorMap* map, int c0, int c1, int c2, int c3, const void* src) {
  asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4}], [%5];"
               ::"l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(src))
               : "memory");
}

// MODE 0: 1D inner pass; tile -> (group, chunk); load/store coordinates
//         {chunk*F + 16 cb, n, 0, group}; comb index r = chunk*F + f.
// MODE 1: strided axis (2D columns); tile -> (batch, grow u, chunk);
//         load {chunk*F, n, u % rps, batch*(gpb/rps) + u/rps}; non-final
//         passes store to the same coordinates, the final pass to
//         {chunk*F, k, final_index(u), batch}; root index r = u % rps.
template <int L, bool INV, bool TWID, int MODE>
__global__ void __launch_bounds__(CombWCfg<L>::THREADS, 1)
k_comb_w(const __grid_constant__ CUtensorMap tin, const __grid_constant__ CUtensorMap tout, CombTmaArgs a,
         const float2* __restrict__ tw, const double2* __restrict__ wc, const double2* __restrict__ wf, float scale) {
  pdl_enter();
  using Cfg = CombWCfg<L>;
  using V = float2;
  using Sh = Shape<L, 32>;
  constexpr int F = Cfg::F, T = Cfg::T, S = Cfg::S, NCB = Cfg::NCB;
  extern __shared__ unsigned char smem_raw[];
  // align by pointer arithmetic: an integer round trip would lose the shared
  // address space and turn every tile access into a generic LD.E/ST.E
  unsigned char* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  V* tiles = reinterpret_cast<V*>(base);
  uint64_t* full = reinterpret_cast<uint64_t*>(base + S * Cfg::TILE_BYTES);
  uint64_t* done = full + S;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long G = gridDim.x;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&done[s], Cfg::CONSUMERS);
    }
    mbar_fence_init();
  }
  __syncthreads();

  // tile -> TMA coordinates of the input box origin and the output origin
  auto coords = [&](long long tile, int& c0, int& c2, int& c3, int& o2, int& o3) {
    const long long chunk = tile % a.chunks, g = tile / a.chunks;
    c0 = (int)(chunk * F);
    if constexpr (MODE == 0) {
      c2 = 0;
      c3 = (int)g;
      o2 = c2;
      o3 = c3;
    } else {
      const long long batch = g / a.groups_per_batch, u = g % a.groups_per_batch;
      c2 = (int)(u % a.rps);
      c3 = (int)(batch * (a.groups_per_batch / a.rps) + u / a.rps);
      if (a.final_pass) {
        long long oi = 0, rem = u;
        for (int i = 0; i + 1 < a.p; ++i) {
          const long long d = rem / a.sub_w[i];
          rem -= d * a.sub_w[i];
          oi += d * a.out_w[i];
        }
        o2 = (int)oi;
        o3 = (int)batch;
      } else {
        o2 = c2;
        o3 = c3;
      }
    }
  };

  if (warp == Cfg::CONSUMERS) {
    // ------------------------------------------------------------ producer
    if (lane != 0) return;
    auto load = [&](long long tile, int s) {
      int c0, c2, c3, o2, o3;
      coords(tile, c0, c2, c3, o2, o3);
      mbar_arrive_expect_tx(&full[s], Cfg::TILE_BYTES);
      V* dst = tiles + (size_t)s * Cfg::TILE;
#pragma unroll 1
      for (int cb = 0; cb < NCB; ++cb)
#pragma unroll 1
        for (int n0 = 0; n0 < L; n0 += Cfg::BL)
          tma_load_4d(dst + cb * L * 16 + n0 * 16, &tin, c0 + cb * 16, n0, c2, c3, &full[s]);
    };
    long long tile = blockIdx.x;
#pragma unroll 1
    for (int s = 0; s < S; ++s)
      if (tile + s * G < a.ntiles) load(tile + s * G, s);
    int i = 0;
#pragma unroll 1
    for (; tile < a.ntiles; tile += G, ++i) {
      const int s = i % S;
      mbar_wait(&done[s], (uint32_t)((i / S) & 1));
      int c0, c2, c3, o2, o3;
      coords(tile, c0, c2, c3, o2, o3);
      const V* src = tiles + (size_t)s * Cfg::TILE;
#pragma unroll 1
      for (int cb = 0; cb < NCB; ++cb)
#pragma unroll 1
        for (int n0 = 0; n0 < L; n0 += Cfg::BL) tma_store_4d(&tout, c0 + cb * 16, n0, o2, o3, src + cb * L * 16 + n0 * 16);
      bulk_commit();
      const long long nxt = tile + S * G;
      if (nxt < a.ntiles) {
        bulk_wait_read<0>();  // the store has read the slot
        load(nxt, s);
      }
    }
    bulk_wait<0>();
    return;
  }

  // ------------------------------------------------------------ consumers
  // lane -> (point offset t, comb f): each half-warp touches 8 consecutive
  // rows x 2 neighbouring combs (T >= 8), or rows x combs spread over
  // distinct 16-byte swizzle chunks (T < 8), so with the 128-byte swizzle
  // every 8-byte access of a half-warp hits 16 distinct bank pairs
  int t, f;
  if constexpr (T == 16) {
    t = (lane & 7) | ((lane >> 4) << 3);
    f = warp * 2 + ((lane >> 3) & 1);
  } else if constexpr (T == 8) {
    t = lane & 7;
    f = warp * 4 + (lane >> 3);
  } else if constexpr (T == 4) {
    const int quad = 2 * warp + (lane >> 4), j = (lane >> 2) & 3;
    t = lane & 3;
    f = (quad >> 2) * 16 + 2 * (quad & 3) + (j & 1) + 8 * (j >> 1);
  } else {
    const int idx = 2 * warp + (lane >> 4), j = (lane >> 1) & 7;
    t = lane & 1;
    f = (idx >> 1) * 16 + 2 * (idx & 1) + (j & 1) + 4 * (j >> 1);
  }
  int i = 0;
#pragma unroll 1
  for (long long tile = blockIdx.x; tile < a.ntiles; tile += G, ++i) {
    const int s = i % S;
    // keep the per-lane address arithmetic inside the loop (hoisting ~100
    // loop-invariant tile offsets out of it would spill)
    int tt = t, ff = f;
    asm volatile("" : "+r"(tt), "+r"(ff));
    V* tl = tiles + (size_t)s * Cfg::TILE;
    mbar_wait(&full[s], (uint32_t)((i / S) & 1));
    V v[Sh::R];
#pragma unroll
    for (int q = 0; q < Sh::R; ++q) v[q] = tl[cw_off<L>(tt + q * T, ff)];
    __syncwarp();
    auto ex = [tl, ff](int e) -> V& { return tl[cw_off<L>(cw_perm(e), ff)]; };
    SyncWarp sy;
    Stages<V, L, 32, INV, 0>::run(v, tt, ex, tw, sy);
    if constexpr (TWID) {
      const long long chunk = tile % a.chunks;
      uint32_t r;
      if constexpr (MODE == 0) r = (uint32_t)(chunk * F + ff);
      else r = (uint32_t)((tile / a.chunks) % a.groups_per_batch % a.rps);
      interpass_scale<V, L, 32, INV>(v, tt, r, a.m_mask, a.fb, wc, wf);
    }
    __syncwarp();
#pragma unroll
    for (int j = 0; j < Sh::R; ++j) {
      V x = v[j];
      if (scale != 1.0f) x = mk(x.x * scale, x.y * scale);
      tl[cw_off<L>(out_index<L, 32>(tt, j), ff)] = x;
    }
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) mbar_arrive(&done[s]);
  }
}

}  // namespace tfb
