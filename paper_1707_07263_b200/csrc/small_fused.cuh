// Fused two-pass plan for small (L2-resident) 1D transforms, fp32.
//
// A 2^14..2^20-point transform is 128 KB..8 MB: both passes of its plan
// (tiled_fft.hpp:321-407: comb pass with the inter-pass root, then the final
// pass with the digit interleave) run out of L2 in a few microseconds each,
// so two launches cost as much in ramp-up/drain and launch gap as in work.
// K_SMALL2 runs both passes in ONE launch: CTAs take pass-1 tiles (the body
// of K_COMB, 4-comb tiles), then final-pass tiles (the body of K_FINAL_T)
// once every pass-1 tile is done. The
// data makes one round trip through L2 between the passes, as before; only
// the launch boundary is gone.
#pragma once
#include "fast_kernels.cuh"

namespace tfb {

// Tiles are handed out from one 64-bit counter, all pass-1 tiles before any
// final-pass tile; a CTA holding a final-pass tile waits until every pass-1
// tile is done. Pass-1 tiles wait for nothing and are only ever held by
// running CTAs, so the wait cannot deadlock whatever the residency (no
// cooperative launch needed -- it costs ~10 us per launch on B200).
// The counters only grow: launch k consumes exactly S = nt1 + nt2 + grid ids
// (one failing grab per CTA) and waits for done1 >= (k + 1) * nt1.
//   ctr[0]: tile counter, ctr[1]: pass-1 tiles done.
template <int L1, int L2>
struct Small2Cfg {
  static constexpr int F1 = 4;                                // combs per pass-1 tile
  using C1 = CombCfg<float, L1, F1>;
  static constexpr int THREADS = C1::THREADS;                 // F1 * L1 / 32
  static constexpr int F2 = THREADS / Shape<L2, 32>::T;       // final-pass rows per tile
  using C2c = FinalCfg<float, L2, F2>;
  static_assert(C2c::THREADS == THREADS, "both passes must use the same CTA shape");
  static constexpr int SMEM = C1::SMEM > C2c::SMEM ? C1::SMEM : C2c::SMEM;
};

template <int L1, int L2, bool INV>
__global__ void __launch_bounds__(Small2Cfg<L1, L2>::THREADS)
k_small2(const float2* in, float2* work, float2* out, CombArgs a1, FinalArgs a2, const float2* __restrict__ tw1,
         const float2* __restrict__ tw2, const double2* __restrict__ wc, const double2* __restrict__ wf, float scale,
         unsigned long long* ctr) {
  pdl_enter();
  using Cfg = Small2Cfg<L1, L2>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float2* sm = reinterpret_cast<float2*>(smem_raw);
  __shared__ long long s_id;
  const long long nt1 = a1.ntiles, nt2 = a2.ntiles;
  const unsigned long long S = (unsigned long long)(nt1 + nt2 + gridDim.x);
  bool waited = false;
  // thread 0 keeps one grab in flight (the next id is requested before the
  // current tile is processed). The prefetched id is never smaller than the
  // current one, so a CTA that waits (holding a final-pass tile) never holds
  // an unprocessed pass-1 tile.
  unsigned long long nxt = 0;
  if (threadIdx.x == 0) nxt = atomicAdd(ctr, 1ull);
#pragma unroll 1
  for (;;) {
    if (threadIdx.x == 0) {
      const unsigned long long id = nxt;
      const long long local = (long long)(id % S);
      if (local < nt1 + nt2) nxt = atomicAdd(ctr, 1ull);
      if (local >= nt1 && local < nt1 + nt2 && !waited) {
        const unsigned long long need = (id / S + 1) * (unsigned long long)nt1;
        unsigned long long d;
        do {
          asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(d) : "l"(ctr + 1) : "memory");
        } while (d < need);
        // one acquire load (not one per poll: each drops the SM's L1)
        asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(d) : "l"(ctr + 1) : "memory");
      }
      s_id = local;
    }
    __syncthreads();
    const long long id = s_id;
    if (id >= nt1 + nt2) break;
    if (id < nt1) {
      comb_tile<float, L1, INV, true, 0, Cfg::F1>(in, work, a1, tw1, wc, wf, 1.0f, id, sm);
      __syncthreads();  // all of the tile's stores issued before the release
      if (threadIdx.x == 0) asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(ctr + 1) : "memory");
    } else {
      waited = true;
      final_tile<float, L2, INV, Cfg::F2>(work, out, a2, tw2, scale, id - nt1, sm);
      __syncthreads();  // shared memory and s_id are reused by the next tile
    }
  }
}

}  // namespace tfb
