// Two-level pass (fp32): one HBM read + one HBM write of an L = LA * LB point
// FFT along a strided axis, for L too long for one CTA's shared memory
// (8192-point columns of 2^26 = 8192 x 8192 and of the 8192^2 image).
//
// The reference's pass (tiled_fft.hpp:229-310) keeps a whole comb in fast
// memory. A 16-comb tile of 8192 points is 1 MB, far beyond one SM, so the
// comb is split once more (n = n1 + LB n2, k = k2 + LA k1):
//
//   A item (group g, n1):   LA-point FFT over n2 of 16 adjacent combs
//                           (TMA tile in, Stockham in registers + padded
//                           shared memory), times W_L^{n1 k2}, written to a
//                           per-group scratch slot that lives in L2;
//   B item (group g, kb):   LB-point DFT over n1 for a block of k2 (scratch
//                           read from L2), optional inter-pass root
//                           W_M^{c k} (tiled_fft.hpp:284-294), stored to HBM.
//
// Only the A loads and the B stores touch HBM; the scratch round trip stays
// in the 126 MB L2 (a bounded ring of slots, each line discarded from L2
// once consumed so dirty scratch is never written back). The kernel is
// persistent: CTAs take items from a global counter in an order in which
// every dependency (B(g) on the A items of g, A(g) on the slot's previous
// B items) was handed out earlier, so spinning on it cannot deadlock.
//
// OUTT = 0: output along the same comb (out[c + k * es_out]).
// OUTT = 1: output transposed, row c of a [cols][L] matrix (out[c * L + k]):
//           the four-step pass 1 whose result pass 2 reads as combs.
#pragma once
#include "fast_kernels.cuh"

namespace tfb {

struct TwoArgs {
  long long groups;          // batch * chunks
  long long chunks;          // 16-column chunks per batch item
  long long bs_in, bs_out;   // batch strides (elements)
  long long es_out;          // OUTT=0: output element stride along the axis; OUTT=1: output row pitch
  int D;                     // lag between A(g) and B(g) in the hand-out order (groups)
  int nslot;                 // scratch slots (> D)
  int discard;               // discard consumed scratch lines from L2
  int diag;                  // K_TWO_TMA diagnostics: 1 = data movement only (no FFT arithmetic)
  int fb;                    // fine-table bits of the inter-pass root tables
  uint32_t m_mask;           // M - 1 (inter-pass root W_M)
  float2* scratch;           // nslot * L * 16 elements
  unsigned* ctrl;            // [0] work counter, [1..nslot] A done, [nslot+1..2 nslot] B done
  unsigned long long* trace; // diagnostics (TILEFFT_TWO_TRACE): 8 timestamps per item id, else null
  unsigned long long* watchdog;  // host-mapped record of a dependency wait that timed out (see wait_geq_wd)
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

template <int LA, int LB, bool INV, int OUTT, int NR_ = 2>
struct TwoCfg {
  using V = float2;
  static constexpr int F = 16;
  static constexpr int L = LA * LB;
  using Sh = Shape<LA, 32>;
  static constexpr int T = Sh::T;               // threads per LA-point FFT
  static constexpr int THREADS = F * T;
  static_assert(THREADS == 256, "two-level pass expects 256 threads (LA = 512)");
  static constexpr int KB = LA / LB;            // k2 values per B item
  static constexpr int PAIRS = KB * F / THREADS;  // (k2, comb) pairs per thread in a B item
  static_assert(PAIRS >= 1 && PAIRS * THREADS == KB * F, "B item must tile the CTA");
  static_assert(OUTT == 0 || KB % 32 == 0, "transposed B items need 32 consecutive k2 per warp");
  static constexpr int TILE = LA * F;           // elements per A tile
  static constexpr int TILE_BYTES = TILE * 8;
  static constexpr int NR = NR_;                // exchange rounds (1/NR of the combs per round)
  static constexpr int FX = F / NR;
  static constexpr int REG = RegionPad<LA, T>::v;  // OUTT=1: per-FFT exchange region
  static constexpr int XB = OUTT == 0 ? LA * FX : FX * REG;
  static constexpr int BL = LA < 256 ? LA : 256;  // TMA box rows
  static constexpr int SMEM = TILE_BYTES + XB * 8 + 16 + 1024;  // + mbarrier + 1024-B alignment slack
  static constexpr int GROUP = L * F;           // scratch elements per group
};

__device__ __forceinline__ void tma_load_4d_l2(void* dst, const CUtensorMap* map, int c0, int c1, int c2, int c3,
                                               uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
      ::"r"(smem_u32(dst)), "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
      : "memory");
}

// Cross-CTA item protocol. An acquire load or a __threadfence() compiles to
// CCTL.IVALL (invalidate the whole L1) on sm_100: done per poll it wipes the
// L1-resident twiddle tables of every CTA on the SM. So the flag is polled
// with relaxed loads and published with a release reduction (MEMBAR.GPU +
// REDG, no L1 invalidate). The data it guards is only ever read with
// L2-coherent loads (__ldcg = LDG.STRONG.GPU) after a barrier that depends on
// the observed flag, and written only after the observed release of the
// slot's previous readers, so no stale L1 line can be consumed.
__device__ __forceinline__ unsigned ld_relaxed_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void wait_geq(const unsigned* p, unsigned v) {
  while (ld_relaxed_u32(p) < v) __nanosleep(40);
}
// Watchdog for the persistent two-level kernels: a dependency that is not met
// within 10 s is a protocol failure, not a slow peer (the kernel runs for
// < 1 ms per GB). The waiter that times out records what it awaited into
// host-mapped memory (it survives the context), asks every other waiting
// thread to record its own state (`dump`), then traps -- so a bug surfaces
// as a launch error with a per-CTA snapshot instead of a hung GPU.
// wd: [0] fired, [1] block, [2] item id, [3] awaited, [4] seen, [5] what
// (1 = A slot reuse, 2 = B inputs), [7] dump request; per CTA b at
// [8 + 4b]: the id a waiting loader holds, what it waits for (1/2), awaited<<32|seen.
constexpr int kWdWords = 8 + 4 * 256;
__device__ __forceinline__ unsigned long long wd_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void wd_record(unsigned long long* wd, int slot_word, unsigned long long v) {
  if (wd && blockIdx.x < 256) reinterpret_cast<volatile unsigned long long*>(wd)[8 + 4 * blockIdx.x + slot_word] = v;
}
__device__ __forceinline__ bool wd_dump_requested(unsigned long long* wd) {
  return wd && reinterpret_cast<volatile unsigned long long*>(wd)[7] != 0;
}
static __device__ __noinline__ void wd_fire(unsigned long long* wd, long long id, unsigned v, unsigned seen, int what) {
  if (wd) {
    volatile unsigned long long* w = wd;
    w[1] = blockIdx.x;
    w[2] = (unsigned long long)id;
    w[3] = v;
    w[4] = seen;
    w[5] = (unsigned long long)what;
    __threadfence_system();
    w[7] = 1;  // everyone else: record your state
    __threadfence_system();
    const unsigned long long t0 = wd_now();
    while (wd_now() - t0 < 300ull * 1000000ull) __nanosleep(1000);
    w[0] = 1;
    __threadfence_system();
  }
  __trap();
}
__device__ __forceinline__ void wait_geq_wd(const unsigned* p, unsigned v, unsigned long long* wd, long long id,
                                            int what) {
  unsigned long long t0 = 0;  // the timer is read only once a wait has lasted ~1024 polls
  bool dumped = false;
  for (unsigned it = 1;; ++it) {
    const unsigned seen = ld_relaxed_u32(p);
    if (seen >= v) return;
    __nanosleep(40);
    if ((it & 1023u) == 0) {
      if (!dumped && wd_dump_requested(wd)) {
        wd_record(wd, 0, (unsigned long long)id);
        wd_record(wd, 1, (unsigned long long)what);
        wd_record(wd, 2, ((unsigned long long)v << 32) | seen);
        dumped = true;
      }
      const unsigned long long t = wd_now();
      if (t0 == 0) t0 = t;
      else if (t - t0 > 10ull * 1000000000ull) wd_fire(wd, id, v, seen, what);
    }
  }
}
__device__ __forceinline__ void signal_release(unsigned* p) {
  asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(p) : "memory");
}
__device__ __forceinline__ void discard_l2(const void* p) {
  asm volatile("discard.global.L2 [%0], 128;" ::"l"(p) : "memory");
}

// ---------------------------------------------------------------- K_TWO_TMA
// Barrier-free two-level pass. Every item, A or B, is one 64 KB shared-memory
// slot that arrives by TMA:
//
//   A item (g, n1): HBM tile [n2 < LA][16 combs] (4-D tensor map, 128-byte
//                   swizzle) -> LA-point FFT of each comb by one half-warp
//                   (radix 32 x 16, the exchange done in place in the slot
//                   through an XOR-permuted row map, so only __syncwarp) ->
//                   times W_L^{n1 k2} -> stored from registers to the group's
//                   L2 scratch [n1][comb][k2] (16 lanes = one 128-byte line).
//   B item (g, kb): scratch block [n1 < LB][16 combs][KB k2] (TMA from L2)
//                   -> LB-point DFT over n1, optional W_M^{c k}, stored from
//                   registers to HBM (lanes along the combs for natural
//                   output, along k2 for the transposed one).
//
// Roles: warps 0..S-1 are loaders, loader s (lane 0) owning slot s: for the
// CTA's items k = s, s + S, ... (global ids 2 blockIdx.x + (k & 1) +
// 2 gridDim.x (k >> 1), a static deal with no counter) it waits for the item's dependencies,
// then for the slot to be free, then issues the TMA and publishes the id.
// Warps S.. are the 8 compute warps; they take the CTA's items in order,
// wait on the slot's `full` mbarrier and arrive on its `empty` mbarrier
// (count 8) as soon as they are done with the slot. No CTA or named barrier
// is crossed. Items are ordered as in K_TWO (A items D groups ahead of the B
// items of a group; a scratch slot is rewritten only after its previous
// generation's B items have loaded it): every dependency has a smaller id and
// each CTA runs its ids in increasing order, so with every CTA resident the
// smallest unfinished id can always progress (no deadlock).
//
// A results are published per warp with a release reduction. Its MEMBAR is
// deferred to just before the warp's next global stores (by then the stores
// it orders have drained), or earlier if the warp would otherwise block on a
// slot -- so a warp never waits on a release another CTA may need.
template <int LA, int LB, int CW_ = 15>
struct TwoTmaCfg {
  static constexpr int F = 16;
  static constexpr int L = LA * LB;
  static constexpr int KB = LA / LB;              // k2 values per B item
  static constexpr int SLOT = LA * F;             // elements per item (A tile == B block)
  static constexpr int SLOT_BYTES = SLOT * 8;     // 64 KB
  static constexpr int S = 3;                     // slots
  static constexpr int CW = CW_;                  // compute warps (15: 128 registers; 19: <= 96 registers)
  static constexpr int NTERM = (CW + 7) / 8;      // terminal items: one unit for every compute warp
  static constexpr int THREADS = 32 * (1 + CW);
  static constexpr int PAIRS = KB * F / 256;      // B (comb, k2) pairs per compute thread
  static constexpr int SMEM = S * SLOT_BYTES + 2 * S * 8 + 1024;
  static_assert(LA == 512, "A items are 512-point FFTs by half-warps (radix 32 x 16)");
  static_assert(PAIRS * 256 == KB * F && KB % 16 == 0, "B item must tile 8 warps");
};

// 8-byte element (row, col) of a 128-byte-swizzled [rows][16] box
__device__ __forceinline__ int sw128(int row, int col) {
  return row * 16 + ((((col >> 1) ^ (row & 7)) << 1) | (col & 1));
}

__device__ __forceinline__ void tma_load_4d_hint(void* dst, const CUtensorMap* map, int c0, int c1, int c2, int c3,
                                                 uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3, %4, %5}], [%6], %7;"
      ::"r"(smem_u32(dst)), "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void signal_relaxed(unsigned* p) {
  asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(p) : "memory");
}
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n.reg .pred p;\nmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

// id -> (A or B, item index): DA A items, then A and B alternating, then the last B items
__device__ __forceinline__ void two_decode(long long id, long long NA, long long DA, bool& isA, long long& idx) {
  if (id < DA) {
    isA = true;
    idx = id;
    return;
  }
  const long long r = id - DA, pairs = NA - DA;
  if (r < 2 * pairs) {
    isA = !(r & 1);
    idx = isA ? DA + (r >> 1) : (r >> 1);
  } else {
    isA = false;
    idx = pairs + (r - 2 * pairs);
  }
}

// TWLB: the root W_L^{n1 k2} is applied by the B items (before their LB-point DFT) instead of the A items
// CW: compute warps. 19 (at most 96 registers) for the plain column pass, which fits them without spills;
// the variants carrying the inter-pass root keep 15 (128 registers)
template <int LA, int LB, bool INV, int OUTT, bool TWID, bool TWLB = false, int CW = (TWLB ? 19 : 15)>
__global__ void __launch_bounds__(TwoTmaCfg<LA, LB, CW>::THREADS, 1)
k_two_tma(const __grid_constant__ CUtensorMap tin, const __grid_constant__ CUtensorMap tscr, float2* __restrict__ out,
          TwoArgs a, const float2* __restrict__ tw, const float2* __restrict__ twl, const double2* __restrict__ wc,
          const double2* __restrict__ wf, float scale) {
  using Cfg = TwoTmaCfg<LA, LB, CW>;
  using V = float2;
  constexpr int F = Cfg::F, S = Cfg::S, KB = Cfg::KB;
  extern __shared__ unsigned char smem_raw[];
  // 1024-byte alignment (128-byte swizzle atoms), by pointer arithmetic on the shared pointer
  unsigned char* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  V* slots = reinterpret_cast<V*>(base);
  uint64_t* full = reinterpret_cast<uint64_t*>(base + S * Cfg::SLOT_BYTES);
  uint64_t* empty = full + S;
  __shared__ long long s_id[S];
  // s_seq[s]: CTA-local index of the item the loader last put in slot s. TMA loads land out of order, so a
  // compute warp can reach item k + S while item k (same slot) is still in flight; a parity wait for the
  // later phase would then return at once (the barrier's phases alias mod 2). The warp therefore first sees
  // its own item index in s_seq (written only after item k - S was released, i.e. its phase completed), then waits.
  __shared__ int s_seq[S];
  // s_cnt[k & 31]: finished units of A item k; its last unit resets the word, and the loader issues an A item
  // only into a zero word, so a unit that lags far behind (it released its slot before its stores) can never
  // count toward a later item that shares the word
  __shared__ unsigned s_unit, s_cnt[32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long NA = a.groups * LB, TOTAL = 2 * NA;
  const long long DA = (long long)a.D * LB;  // A items handed out before the first B item
  unsigned* workA = a.ctrl;
  unsigned* doneA = a.ctrl + 1;
  unsigned* doneB = a.ctrl + 1 + a.nslot;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 8);
    }
    s_unit = 0;
    for (int i = 0; i < S; ++i) s_seq[i] = -1;
    for (int i = 0; i < 32; ++i) s_cnt[i] = 0;
    mbar_fence_init();
  }
  __syncthreads();

  if (warp == 0) {
    // ============================================================ loader
    if (lane == 0) {
      const uint64_t pol = l2_policy_evict_first();
      // ids come from the global counter in order (each CTA runs its ids in increasing order);
      // the next id is claimed one item ahead so the atomic's latency overlaps the current item.
      // (Measured alternatives: claiming 4 ahead and issuing the oldest ready one -- 614 vs 530 us
      // for 8192^2, claimed-but-unissued A items delay their group's B items; separate A and B
      // streams -- no faster, and not deadlock-free in practice.)
      long long nxt = (long long)atomicAdd(workA, 1u);
      int k = 0;
#pragma unroll 1
      for (;; ++k) {
        const int s = k % S;
        const long long id = nxt;
        if (id >= TOTAL) break;
        nxt = (long long)atomicAdd(workA, 1u);
        if (a.trace) { a.trace[id * 8 + 0] = gtimer(); a.trace[id * 8 + 6] = blockIdx.x; }
        bool isA;
        long long idx;
        two_decode(id, NA, DA, isA, idx);
        const long long g = idx / LB;
        const int sub = (int)(idx % LB);
        const int slot = (int)(g % a.nslot);
        const unsigned gen = (unsigned)(g / a.nslot);
        // dependency first (it does not need the slot), then the slot
        if (isA) {
          if (gen > 0) wait_geq_wd(doneB + slot, gen * LB, a.watchdog, id, 1);
        } else {
          wait_geq_wd(doneA + slot, (gen + 1) * LB, a.watchdog, id, 2);
          fence_proxy_async_global();  // generic-proxy scratch stores -> our TMA reads
        }
        if (a.trace) a.trace[id * 8 + 1] = gtimer();
        if (k >= S) {
          mbar_wait(&empty[s], (uint32_t)(((k / S) - 1) & 1));
        }
        if (a.trace) { a.trace[id * 8 + 2] = gtimer(); a.trace[id * 8 + 7] = isA; }
        if (isA)
          while (*reinterpret_cast<volatile unsigned*>(&s_cnt[k & 31]) != 0) __nanosleep(20);
        s_id[s] = id * 2 + (isA ? 1 : 0);
        *reinterpret_cast<volatile int*>(&s_seq[s]) = k;
        V* dst = slots + s * Cfg::SLOT;
        mbar_arrive_expect_tx(&full[s], Cfg::SLOT_BYTES);
        if (isA) {
          const long long b = g / a.chunks, ch = g % a.chunks;
#pragma unroll 1
          for (int r = 0; r < LA; r += 256)
            tma_load_4d_hint(dst + r * F, &tin, (int)(ch * F), sub, r, (int)b, &full[s], pol);
        } else {
#pragma unroll 1
          for (int h = 0; h < KB / 16; ++h)
            tma_load_4d_l2(dst + h * LB * 16 * 16, &tscr, sub * KB + 16 * h, 0, 0, slot, &full[s]);
        }
      }
      // end of work: NTERM terminal items, one unit for every compute warp
#pragma unroll 1
      for (int j = 0; j < Cfg::NTERM; ++j, ++k) {
        const int s = k % S;
        if (k >= S) mbar_wait(&empty[s], (uint32_t)(((k / S) - 1) & 1));
        s_id[s] = -1;
        *reinterpret_cast<volatile int*>(&s_seq[s]) = k;
        mbar_arrive(&full[s]);
      }
    }
    return;
  }

  // ============================================================== compute
  // Each item is 8 units (A: combs 2p, 2p+1; B: 1/8 of the pairs); compute warps take units in
  // order from a shared counter, so any number of warps shares the items; a warp that runs ahead
  // of a slot's in-flight TMA waits on the slot's sequence tag first (s_seq), never on a wrong phase.
#pragma unroll 1
  for (;;) {
    unsigned u = 0;
    if (lane == 0) u = atomicAdd(&s_unit, 1u);
    u = __shfl_sync(0xffffffffu, u, 0);
    const int k = (int)(u >> 3), w = (int)(u & 7);
    const int s = k % S;
    while (*reinterpret_cast<volatile int*>(&s_seq[s]) != k) __nanosleep(32);
    mbar_wait(&full[s], (uint32_t)((k / S) & 1));
    const long long code = s_id[s];  // id * 2 + isA, or -1 at the end
    if (code < 0) break;
    const long long id = code >> 1;
    const bool isA = code & 1;
    if (a.trace && w == 0 && lane == 0) a.trace[id * 8 + 3] = gtimer();
    long long idx;
    {
      bool a_;
      two_decode(id, NA, DA, a_, idx);
    }
    const long long g = idx / LB;
    const int sub = (int)(idx % LB);
    const int slot = (int)(g % a.nslot);
    V* sl = slots + s * Cfg::SLOT;
    if (isA) {
      // ---- A: half-warp pairs (lanes 2t, 2t+1 = combs 2w, 2w+1 at the same t),
      // so each half-warp's 64-bit accesses cover 8 distinct swizzle chunks
      const int f = 2 * w + (lane & 1), t = lane >> 1;
      V v[32];
#pragma unroll
      for (int q = 0; q < 32; ++q) v[q] = sl[sw128(t + 16 * q, f)];
      __syncwarp();
      // element e = 32 a + c of the exchange lives in row 16 c + (a ^ (c & 7)):
      // conflict-free for the writes (c fixed per register) and the reads (a fixed)
      auto ex = [sl, f](int e) -> V& {
        const int c = e & 31, a_ = e >> 5;
        return sl[sw128(16 * c + (a_ ^ (c & 7)), f)];
      };
      auto release_slot = [&]() {
        fence_proxy_async_smem();  // our generic writes before the next TMA write of the slot
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
        if (a.trace && w == 0 && lane == 0) a.trace[id * 8 + 4] = gtimer();
      };
      SyncWarp sy;
      if (a.diag == 1) release_slot();
      else Stages<V, LA, 32, INV, 0>::run(v, t, ex, tw, sy, 0, release_slot);
      // W_L^{n1 k2}, k2 = t + 16 i + 32 q (register 16 i + q) = W^{n1 (t + 16 i)} * W^{32 n1 q}
      if (!TWLB && a.diag != 1 && sub > 0) {
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const V b0 = __ldg(twl + sub * (t + 16 * i));
#pragma unroll
          for (int q = 0; q < 16; ++q) {
            const V wq = q == 0 ? b0 : cmul(b0, __ldg(twl + 32 * sub * q));
            v[16 * i + q] = ctw<INV>(v[16 * i + q], wq);
          }
        }
      }
      V* scr = a.scratch + (((size_t)slot * LB + sub) * F + f) * LA;
#pragma unroll
      for (int j = 0; j < 32; ++j) __stcg(scr + out_index<LA, 32>(t, j), v[j]);
      // the last of the item's 8 units publishes it (one release per A item)
      __syncwarp();
      if (lane == 0) {
        unsigned old;
        asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], 1;"
                     : "=r"(old) : "r"(smem_u32(&s_cnt[k & 31])) : "memory");
        if (old == 7) {
          asm volatile("st.relaxed.cta.shared::cta.u32 [%0], 0;" ::"r"(smem_u32(&s_cnt[k & 31])) : "memory");
          if (a.diag == 3) signal_relaxed(doneA + slot);  // timing diagnostics only
          else signal_release(doneA + slot);
          if (a.trace) a.trace[id * 8 + 5] = gtimer();
        }
      }
    } else {
      // ---- B: LB-point DFTs over n1 for KB k2 values of 16 combs
      if (w == 0) {
        // the item's scratch block is in shared memory now: drop its lines from L2 (dirty scratch is never
        // written back to DRAM), then hand the scratch slot back
        if (a.discard) {
          constexpr int LPS = KB * 8 / 128;  // 128-byte lines per (n1, comb) segment of KB elements
          const V* base = a.scratch + (size_t)slot * LB * F * LA + (size_t)sub * KB;
#pragma unroll 4
          for (int i = lane; i < LB * F * LPS; i += 32)
            discard_l2(base + (size_t)(i / LPS) * LA + (i % LPS) * 16);
          __syncwarp();
          if (lane == 0) signal_release(doneB + slot);
        } else if (lane == 0) {
          signal_relaxed(doneB + slot);
        }
      }
      const int kb = sub;
      // pair p of this thread: OUTT=0 lanes = (8 combs x 2 k2) per half-warp; OUTT=1 lanes along k2
      auto pair = [&](int m, int& f, int& k2l) {
        if constexpr (OUTT == 0) {
          const int hw = lane >> 4, l = lane & 15;
          f = hw * 8 + (l >> 1);
          k2l = (w + 8 * m) * 2 + (l & 1);
        } else {
          const int p = w * 32 + lane + 256 * m;
          f = p / KB;
          k2l = p % KB;
        }
      };
      V v[Cfg::PAIRS][LB];
#pragma unroll
      for (int m = 0; m < Cfg::PAIRS; ++m) {
        int f, k2l;
        pair(m, f, k2l);
#pragma unroll
        for (int n1 = 0; n1 < LB; ++n1) v[m][n1] = sl[sw128(((k2l >> 4) * LB + n1) * 16 + f, k2l & 15)];
      }
      fence_proxy_async_smem();  // our generic reads of the slot before the next TMA write of it
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      if (a.trace && w == 0 && lane == 0) a.trace[id * 8 + 4] = gtimer();
      const long long b = g / a.chunks, ch = g % a.chunks;
#pragma unroll
      for (int m = 0; m < Cfg::PAIRS; ++m) {
        int f, k2l;
        pair(m, f, k2l);
        const int k2 = kb * KB + k2l;
        V* u = v[m];
        if constexpr (TWLB) {
          // W_L^{n1 k2} = w^{n1}, w = W_L^{k2}: w, w^2, w^4, w^8 from the table, the other powers as
          // products (at most three roundings each)
          if (a.diag != 1 && k2 > 0) {
            constexpr int Lm = LA * LB - 1;
            V p[LB];
            p[1] = __ldg(twl + (k2 & Lm));
#pragma unroll
            for (int e = 2; e < LB; e *= 2) p[e] = __ldg(twl + ((e * k2) & Lm));
#pragma unroll
            for (int e = 3; e < LB; ++e) {
              const int hi = 1 << (31 - __clz(e));
              if (e != hi) p[e] = cmul(p[hi], p[e - hi]);
            }
#pragma unroll
            for (int n1 = 1; n1 < LB; ++n1) u[n1] = ctw<INV>(u[n1], p[n1]);
          }
        }
        if (a.diag != 1) reg_dft<LB, INV>(u);
        const long long c = ch * F + f;
        if constexpr (TWID) {
          constexpr int QA = LB / 4 > 0 ? LB / 4 : 1;
          const double2 w0 = interpass_root64(wc, wf, ((uint32_t)c * (uint32_t)k2) & a.m_mask, a.fb);
          const double2 s1 = interpass_root64(wc, wf, ((uint32_t)c * (uint32_t)LA) & a.m_mask, a.fb);
          const double2 s2 = cmul(s1, s1), s4 = cmul(s2, s2);
          const double2 w2 = cmul(w0, s2);
          const V Bq[4] = {to_v(w0, (V*)nullptr), to_v(cmul(w0, s1), (V*)nullptr), to_v(w2, (V*)nullptr),
                           to_v(cmul(w2, s1), (V*)nullptr)};
          V Aq[QA];
          {
            double2 pw = make_double2(1.0, 0.0);
#pragma unroll
            for (int q = 0; q < QA; ++q) {
              Aq[q] = to_v(pw, (V*)nullptr);
              if (q + 1 < QA) pw = cmul(pw, s4);
            }
          }
#pragma unroll
          for (int k1 = 0; k1 < LB; ++k1) u[k1] = ctw<INV>(u[k1], k1 < 4 ? Bq[k1 % 4] : cmul(Aq[k1 / 4], Bq[k1 % 4]));
        }
        if (scale != 1.0f) {
#pragma unroll
          for (int k1 = 0; k1 < LB; ++k1) u[k1] = mk(u[k1].x * scale, u[k1].y * scale);
        }
        if constexpr (OUTT == 0) {
          V* o = out + b * a.bs_out + c;
#pragma unroll
          for (int k1 = 0; k1 < LB; ++k1) __stcs(o + (long long)(k2 + LA * k1) * a.es_out, u[k1]);
        } else {
          V* o = out + b * a.bs_out + c * a.es_out + k2;
#pragma unroll
          for (int k1 = 0; k1 < LB; ++k1) __stcs(o + LA * k1, u[k1]);
        }
      }
      if (a.trace && w == 0 && lane == 0) a.trace[id * 8 + 5] = gtimer();
    }
  }
}

}  // namespace tfb
