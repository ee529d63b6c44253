/* tilefft_b200 — C ABI of the B200-native complex-to-complex FFT path.
 *
 * This is the drop-in boundary below the reference's C++ plan/execute API
 * (/root/reference/proj/include/tilefft). The reference has no FFI of its own
 * (SURVEY §8b): its public entry points are header templates, so the C++
 * headers in include/tilefft/ keep those signatures and call these functions.
 * Each entry point cites the reference interface it replaces.
 *
 * Conventions: plain pointers and sizes only; complex data is interleaved
 * (re, im) — the layout of std::vector<std::complex<Real>> — in fp32
 * (elem_bytes = 8) or fp64 (elem_bytes = 16). Every call returns 0 or a
 * TILEFFT_E* code and never throws; tilefft_last_error() holds the message
 * (thread-local), using the reference's wording where the reference has one
 * (detail::require, common.hpp:47-51). There is no CPU fallback: without a
 * CUDA device every call fails with TILEFFT_ENODEV.
 */
#ifndef TILEFFT_B200_H
#define TILEFFT_B200_H
#include <stdint.h>

#if defined(__GNUC__)
#define TILEFFT_API __attribute__((visibility("default")))
#else
#define TILEFFT_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define TILEFFT_OK 0
#define TILEFFT_EINVAL 22  /* maps to std::invalid_argument */
#define TILEFFT_ENODEV 19  /* no usable sm_100 device */
#define TILEFFT_ENOMEM 12
#define TILEFFT_ECUDA 1001 /* CUDA runtime error (message in tilefft_last_error) */
#define TILEFFT_ENCCL 1002

/* Arithmetic modes.
 *  FAST  : the product path. Radix-32 register Stockham passes over the
 *          GPU's own pass factorisation; relative L2 error vs fft_tiled
 *          <= 1e-5*log2(N) (fp32) / 1e-12*log2(N) (fp64).
 *  EXACT : executes the caller's plan factors with the reference's radix-2
 *          dataflow and table roots, every op separately rounded: output is
 *          bit-identical to fft_tiled<Real> (tiled_fft.hpp:321-407).
 *  PERMUTE (EXACT only): butterflies and roots off; applies only the pass
 *          index maps (gather/exchange/interleave, stage_plan.hpp:135-179). */
#define TILEFFT_MODE_FAST 0
#define TILEFFT_MODE_EXACT 1
#define TILEFFT_MODE_PERMUTE 2
#define TILEFFT_MODE_LEVELWISE 3  /* fft_levelwise (fft_baseline.hpp:66-116): bit reversal + one launch
                                     per radix-2 level in global memory, bit-identical; the paper's
                                     "previous method", kept for the §2.2-vs-§2.3 comparison */

#define TILEFFT_FORWARD (-1)
#define TILEFFT_INVERSE (+1)

typedef struct tilefft_plan_s* tilefft_plan_t;

/* Create a plan for `batch` contiguous length-n transforms on `device`.
 * Replaces make_plan (stage_plan.hpp:74-127) + build_twiddle_table
 * (twiddle.hpp:47-73) as consumed by fft_tiled: `factors` are the
 * StagePlan's factors (required for EXACT/PERMUTE, advisory for FAST);
 * `twiddle_values`/`twiddle_resolution` are the caller's TwiddleTable
 * (interleaved, elem_bytes each) — EXACT mode takes its roots from it; pass
 * NULL/0 to have the plan generate the same values itself.
 * Errors mirror fft_tiled's checks (tiled_fft.hpp:325-333). */
TILEFFT_API int tilefft_plan_create(tilefft_plan_t* plan, uint64_t n, uint64_t batch, const uint64_t* factors,
                        uint32_t nfactors, uint32_t elem_bytes, uint32_t mode, const void* twiddle_values,
                        uint64_t twiddle_resolution, int device);

/* 2D transform of `batch` row-major ny x nx images (rows then columns; the
 * reference has no 2D entry point — SPEC.md:331 — so this composes the 1D
 * passes exactly as the BASELINE.md recipe does). FAST mode only. */
TILEFFT_API int tilefft_plan_create_2d(tilefft_plan_t* plan, uint64_t ny, uint64_t nx, uint64_t batch, uint32_t elem_bytes,
                           int device);

/* Execute on device-resident buffers (out-of-place; in == out allowed).
 * sign = TILEFFT_FORWARD is fft_tiled (tiled_fft.hpp:321); TILEFFT_INVERSE
 * is ifft_tiled (:410-423), including the 1/n scale. Asynchronous on
 * `cuda_stream` (a cudaStream_t; NULL = legacy default stream). */
TILEFFT_API int tilefft_exec_c2c(tilefft_plan_t plan, const void* d_in, void* d_out, int sign, void* cuda_stream);

/* Execute on HOST buffers: the whole fft_tiled contract (vector in, vector
 * out). Host->device copies, the passes and device->host copies are
 * pipelined in chunks of transforms over several streams when batch > 1.
 * Synchronous. Pinned (cudaHostAlloc/registered) buffers reach full PCIe
 * bandwidth; pageable buffers work but are staged by the driver. */
TILEFFT_API int tilefft_exec_c2c_host(tilefft_plan_t plan, const void* h_in, void* h_out, int sign);

TILEFFT_API int tilefft_plan_destroy(tilefft_plan_t plan);

/* Measurement: run the plan's device passes `reps` times back to back
 * (direct launches, no graph) on `cuda_stream`, with a CUDA event between
 * consecutive passes; pass_ms[i] receives pass i's mean event-to-event time in
 * milliseconds (the per-kernel duration bench.py's roofline divides by),
 * for the first min(passes, max_passes) passes (tilefft_plan_info().passes;
 * an unaligned d_in runs the plan's non-TMA variant). Synchronous. Same buffers and sign rules as exec_c2c. */
TILEFFT_API int tilefft_exec_c2c_timed(tilefft_plan_t plan, const void* d_in, void* d_out, int sign, void* cuda_stream,
                                       int reps, float* pass_ms, int max_passes);


/* Plan introspection (all sizes in elements unless noted). */
typedef struct {
  uint64_t n, batch, ny, nx;
  uint32_t elem_bytes, mode, is_2d;
  uint32_t passes;             /* device passes per transform (HBM round trips) */
  uint64_t factors[16];        /* device pass lengths in execution order */
  uint32_t launches_per_exec;  /* kernel launches per tilefft_exec_c2c */
  uint64_t workspace_bytes;    /* device scratch held by the plan (FAST: n*batch elements for 2-pass plans,
                                  2*n*batch for 3-pass plans, which hand over from pass 0 to pass 1 through a
                                  second, transposed workspace) */
  uint64_t table_bytes;        /* device twiddle tables held by the plan */
} tilefft_plan_info_t;
TILEFFT_API int tilefft_plan_info(tilefft_plan_t plan, tilefft_plan_info_t* info);

/* exchange_transpose (tiled_fft.hpp:179-203): out[exchange_index_map(stage,
 * q)] = in[q] for the plan with `factors` (stage_plan.hpp:161-172), on the GPU,
 * host buffers. */
TILEFFT_API int tilefft_exchange(const void* h_in, void* h_out, uint64_t n, const uint64_t* factors,
                                 uint32_t nfactors, uint32_t stage, uint32_t elem_bytes, int device);

/* apply_interstage_twiddles (tiled_fft.hpp:153-172): element (r, k) of a
 * rows x cols tile times W_{sub_len}^{((row0 + r) % rows_per_sub) * k} taken
 * from the caller's table (bit-identical), on the GPU, host buffers. */
TILEFFT_API int tilefft_interstage_scale(const void* h_in, void* h_out, uint64_t rows, uint64_t cols, uint64_t row0,
                                         uint64_t rows_per_sub, uint64_t sub_len, const void* table,
                                         uint64_t resolution, uint32_t elem_bytes, int device);

/* ---- Distributed four-step transform -------------------------
 * One length-n transform over `nranks` GPUs (one process per GPU), n = N1 x N2
 * with N1 <= 1024. Layouts (rank g, C = N2/nranks, R = N1/nranks):
 *   input  column slab  [N1][C]  : x[g*C + c + N2*n1]
 *   output row slab     [R][N2]  : X[(g*R + k1) + N1*k2]  (digit-interleaved)
 * Pass 1 (column FFTs + inter-pass root W_N^{r k1}) scatters every result
 * straight into the destination slabs set by tilefft_dist_set_peers: the
 * other ranks' row slabs mapped over NVLink (CUDA IPC; row_pitch = N2,
 * col_off = g*C) — the all-to-all fused into the pass-1 store — or local
 * staging blocks (row_pitch = C, col_off = 0) for an NCCL all-to-all.
 * Pass 2 runs the row FFTs of length N2 on the rank's assembled row slab. The
 * caller orders pass 1 on every rank before pass 2 (stream sync + barrier). */
TILEFFT_API int tilefft_dist_plan_create(tilefft_plan_t* plan, uint64_t n, uint32_t nranks, uint32_t rank,
                                         uint32_t elem_bytes, int device);
TILEFFT_API int tilefft_dist_layout(tilefft_plan_t plan, uint64_t* n1, uint64_t* n2, uint64_t* cols_per_rank,
                                    uint64_t* rows_per_rank);
TILEFFT_API int tilefft_dist_set_peers(tilefft_plan_t plan, void* const* dest, uint32_t ndest, uint64_t row_pitch,
                                       uint64_t col_off);
TILEFFT_API int tilefft_dist_exec_pass1(tilefft_plan_t plan, const void* d_col_slab, int sign, void* cuda_stream);
TILEFFT_API int tilefft_dist_exec_pass2(tilefft_plan_t plan, const void* d_row_slab, void* d_out, int sign,
                                        void* cuda_stream);
/* Pass 2 straight from an all-to-all's receive buffer laid out [src][rows_per_rank][cols_per_rank] (source
 * rank src's block of this rank's rows; the NCCL exchange): the row plan's first pass reads it through a
 * 5-D tensor map, so no re-assembly copy. TILEFFT_EINVAL when the row plan is a single pass. */
TILEFFT_API int tilefft_dist_exec_pass2_blocks(tilefft_plan_t plan, const void* d_recv, void* d_out, int sign,
                                               void* cuda_stream);
/* Device-side barrier for the distributed step. Each distributed plan owns a
 * small device flag buffer; export it to the other ranks (tilefft_ipc_get_handle
 * on the pointer tilefft_dist_flag_buffer returns), then give every plan all
 * ranks' buffers in rank order, its own included. tilefft_dist_exec then runs
 * pass 1 (peer stores) -> a one-thread barrier kernel (release-add on every
 * rank's word, acquire-poll of its own) -> pass 2 on the row slab
 * dest[rank] set by tilefft_dist_set_peers, all stream-ordered: no host
 * synchronisation, capturable in a CUDA graph. Every rank must call it the
 * same number of times; a rank that never arrives traps the waiting kernels
 * after 60 s. */
TILEFFT_API int tilefft_dist_flag_buffer(tilefft_plan_t plan, void** d_flags);
TILEFFT_API int tilefft_dist_set_flags(tilefft_plan_t plan, void* const* d_flags, uint32_t nranks);
TILEFFT_API int tilefft_dist_exec(tilefft_plan_t plan, const void* d_col_slab, void* d_out, int sign,
                                  void* cuda_stream);

/* CUDA IPC helpers for exchanging slab pointers between rank processes.
 * A handle (64 opaque bytes) names the whole device allocation holding dptr;
 * offset_out receives dptr's byte offset inside it (pointers from a caching
 * allocator are sub-allocations), and open_handle returns base + offset. */
TILEFFT_API int tilefft_ipc_get_handle(const void* dptr, void* handle_out, uint64_t* offset_out);
TILEFFT_API int tilefft_ipc_open_handle(const void* handle, uint64_t offset, void** dptr);
TILEFFT_API int tilefft_ipc_close_handle(void* dptr);

/* Host-side root table with the reference's construction: entry j =
 * exp(-2 pi i j / resolution), interleaved, elem_bytes 8 or 16
 * (build_twiddle_table, twiddle.hpp:47-73; bit-identical values). */
TILEFFT_API int tilefft_build_twiddle(uint64_t resolution, uint32_t elem_bytes, void* out);

/* The reference's cost model (memsim.hpp:38-95, access_patterns.hpp): the
 * closed-form AccessStats of fft_tiled under make_plan(n, tile_capacity)
 * (algorithm TILEFFT_ACCOUNT_TILED) or of fft_levelwise (…_LEVELWISE), as
 * stats[7] = {slow_elem_reads, slow_elem_writes, slow_transactions,
 * fast_accesses, bank_conflict_cycles, barriers, twiddle_fetches}. Host only;
 * the C++ drop-in records the same figures in traced calls. */
#define TILEFFT_ACCOUNT_TILED 0
#define TILEFFT_ACCOUNT_LEVELWISE 1
TILEFFT_API int tilefft_account(uint64_t n, uint64_t tile_capacity, uint32_t algorithm, uint64_t* stats);

/* Thread-local message of the last failing call ("" if none). */
TILEFFT_API const char* tilefft_last_error(void);

/* Library version / build string, e.g. "tilefft_b200 0.1 sm_100a". */
TILEFFT_API const char* tilefft_version(void);

#ifdef __cplusplus
}
#endif
#endif
