// tilefft_b200: plan objects, pass scheduling and the C ABI
// (include/tilefft_b200.h). Host side of the B200 path: it owns the device
// twiddle tables (the paper's precomputed "texture" roots),
// the ping-pong workspace (tiled_fft.hpp:338-344) and the launch sequence of
// one fft_tiled call (tiled_fft.hpp:346-405), one kernel per pass.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <new>
#include <string>
#include <type_traits>
#include <utility>
#include <vector>

#include "internal.h"

namespace tfb_host {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

std::mutex g_attr_mu;
struct AttrRec { const void* fn; int dev; int bytes; };
std::vector<AttrRec> g_attr_done;
int ensure_smem(const void* fn, int bytes) {
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(g_attr_mu);
  for (auto& r : g_attr_done)
    if (r.fn == fn && r.dev == dev) {
      if (r.bytes >= bytes) return 0;
      CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
      r.bytes = bytes;
      return 0;
    }
  CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  g_attr_done.push_back({fn, dev, bytes});
  return 0;
}

}  // namespace tfb_host

using namespace tfb_host;

namespace {

bool is_pow2(uint64_t v) { return v != 0 && (v & (v - 1)) == 0; }
int ilog2(uint64_t v) { return 63 - __builtin_clzll(v); }

// ---------------------------------------------------------------- roots
// exp(-2 pi i j / m) with the reference's construction (twiddle.hpp:47-73):
// double angle, cos/sin cast to Real, quadrant mirroring, exact axis points.
// Values are resolution independent (scaling j and m by a power of two gives
// the same double angle), so any W_m^j equals the reference table's entry.
template <typename Real>
void ref_root(uint64_t j, uint64_t m, Real* re, Real* im) {
  j &= (m - 1);
  if (j == 0) { *re = 1; *im = 0; return; }
  if (2 * j == m) { *re = -1; *im = 0; return; }
  if (m >= 4 && 4 * j == m) { *re = 0; *im = -1; return; }
  if (m >= 4 && 4 * j == 3 * m) { *re = 0; *im = 1; return; }
  const uint64_t q = m / 4;
  // first quadrant index and mirror (twiddle.hpp:63-70)
  uint64_t jj;
  int sc, ss;  // signs applied to (c, s) -> value = (sc*c, ss*s)
  if (j < q) { jj = j; sc = 1; ss = -1; }
  else if (j < 2 * q) { jj = m / 2 - j; sc = -1; ss = -1; }
  else if (j < 3 * q) { jj = j - m / 2; sc = -1; ss = 1; }
  else { jj = m - j; sc = 1; ss = 1; }
  const double angle = 2.0 * 3.141592653589793238462643383279502884 * (double)jj / (double)m;
  const Real c = (Real)std::cos(angle), s = (Real)std::sin(angle);
  *re = sc > 0 ? c : -c;
  *im = ss > 0 ? s : -s;
}

// Accurate fp64 root for fast-mode tables (rounded once to Real).
template <typename Real>
void acc_root(uint64_t j, uint64_t m, Real* re, Real* im) { ref_root<Real>(j, m, re, im); }

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  ~DevBuf() { if (p) cudaFree(p); }
  int alloc(size_t b) {
    if (b == 0) return 0;
    if (cudaMalloc(&p, b) != cudaSuccess) { cudaGetLastError(); p = nullptr; return fail(TILEFFT_ENOMEM, "cudaMalloc(%zu) failed", b); }
    bytes = b;
    return 0;
  }
};

}  // namespace

namespace {
template <typename Real>
struct TableBuilder {
  std::vector<Real> h;  // interleaved
  size_t add(size_t count) {
    size_t off = h.size() / 2;
    h.resize(h.size() + 2 * count);
    return off;
  }
  void set(size_t idx, Real re, Real im) { h[2 * idx] = re; h[2 * idx + 1] = im; }
};
}  // namespace

struct tilefft_plan_s {
  int device = 0;
  uint64_t n = 0, batch = 0, ny = 0, nx = 0;
  uint32_t elem_bytes = 8, mode = 0, is2d = 0;
  std::vector<uint64_t> dev_factors;
  std::vector<Pass> passes;
  DevBuf tables;          // all device tables (elements of C2<Real>)
  DevBuf tables64;        // fp64 inter-pass root tables
  TableBuilder<double>* tb64 = nullptr;  // plan-build scratch
  DevBuf work;            // workspace (batch * n elements)
  DevBuf work2;           // second workspace: the transposed pass-0 -> pass-1 hand-over (CombArgs::t_l2)
  std::vector<Pass> passes_alt;  // same transform without two-level passes (used when the input is not 16-B aligned)
  DevBuf scratch, ctrl;   // two-level passes: L2-resident exchange slots and their counters
  // Replayed launch sequences: one CUDA graph per (in, out, sign), captured on
  // first use; a replay costs one cudaGraphLaunch instead of per-pass host work
  // (tensor-map encoding, occupancy queries, 2-3 launches).
  struct GraphEntry {
    const void* in;
    void* out;
    int sign;
    cudaGraphExec_t exec;
  };
  static constexpr size_t kMaxGraphs = 8;
  std::vector<GraphEntry> graphs;
  std::mutex graph_mu;
  cudaStream_t cap_stream = nullptr;
  // Every exec of the plan uses the same workspace, two-level scratch ring and
  // counters, so execs on different streams are ordered on the device: each
  // exec waits for the previous one (cudaStreamWaitEvent on this event, a
  // no-op on the same stream) and records it when its last pass is queued.
  cudaEvent_t exec_done = nullptr;
  size_t table_elems = 0;
  // host-path staging
  std::mutex host_mu;
  static constexpr int kHostStreams = 4;
  cudaStream_t hs[kHostStreams] = {};
  cudaEvent_t hev[kHostStreams] = {};     // D2H of buffer i done
  cudaEvent_t hev_in[kHostStreams] = {};  // H2D of buffer i done
  cudaEvent_t hev_k[kHostStreams] = {};   // kernel on buffer i done
  DevBuf hbuf[kHostStreams];
  uint64_t host_chunk = 0;  // transforms per pipelined chunk
  // distributed four-step (tilefft_dist_*)
  bool is_dist = false;
  uint32_t nranks = 1, rank = 0;
  uint64_t n1 = 0, n2 = 0;
  DistPass1 dist{};
  bool peers_set = false;
  DevBuf flags;                   // [0] arrivals (written by every rank), [1] this rank's barrier epoch
  unsigned* peer_flags[16] = {};  // every rank's arrival word (own included), set by tilefft_dist_set_flags
  bool flags_set = false;
  tilefft_plan_s* inner = nullptr;  // row FFTs of length n2 over the rank's n1/nranks rows
  tilefft_plan_s* inner_blocks = nullptr;  // the same, reading the [src][k1][c] blocks an all-to-all leaves
  ~tilefft_plan_s() {
    if (inner) tilefft_plan_destroy(inner);
    if (inner_blocks) tilefft_plan_destroy(inner_blocks);
    for (auto& g : graphs) cudaGraphExecDestroy(g.exec);
    if (cap_stream) cudaStreamDestroy(cap_stream);
    if (exec_done) cudaEventDestroy(exec_done);
    for (int i = 0; i < kHostStreams; ++i) {
      if (hs[i]) cudaStreamDestroy(hs[i]);
      if (hev[i]) cudaEventDestroy(hev[i]);
      if (hev_in[i]) cudaEventDestroy(hev_in[i]);
      if (hev_k[i]) cudaEventDestroy(hev_k[i]);
    }
  }
};

namespace {

// ---------------------------------------------------------------- table builder

template <typename Real>
tfb::StageTableInfo stage_info_for(int L) {
  constexpr int RM = tfb::RmaxOf<Real>::v;
  switch (L) {
#define CASE(LL) case LL: return tfb::stage_table_info<LL, RM>();
    CASE(2) CASE(4) CASE(8) CASE(16) CASE(32) CASE(64) CASE(128) CASE(256) CASE(512) CASE(1024)
    CASE(2048) CASE(4096) CASE(8192)
#undef CASE
  }
  return tfb::StageTableInfo{};
}

// Stockham stage roots for length L: block of [q][k] tables, stage s >= 1,
// entry q*Ns + k = W_{Ns*Rs}^{q k}.
template <typename Real>
size_t add_stage_table(TableBuilder<Real>& tb, int L) {
  const tfb::StageTableInfo si = stage_info_for<Real>(L);
  const size_t off = tb.add(std::max(si.total, 1));
  size_t pos = off;
  for (int s = 1; s < si.nst; ++s) {
    const uint64_t rs = si.radix[s], ns = si.ns[s], m = rs * ns;
    for (uint64_t q = 0; q < rs; ++q)
      for (uint64_t k = 0; k < ns; ++k) {
        Real re, im;
        acc_root<Real>(q * k, m, &re, &im);
        tb.set(pos++, re, im);
      }
  }
  return off;
}

// Inter-pass roots W_M^e = C[e >> fb] * F[e & (2^fb - 1)], fp64 for both
// precisions (the kernels walk powers from them in fp64).
void add_interpass(TableBuilder<double>& tb, uint64_t M, size_t* wc, size_t* wf, int* fb) {
  const int lm = ilog2(M);
  *fb = (lm + 1) / 2;
  const uint64_t nf = 1ull << *fb, nc = M >> *fb;
  *wc = tb.add(nc);
  for (uint64_t i = 0; i < nc; ++i) {
    double re, im;
    acc_root<double>(i * nf, M, &re, &im);
    tb.set(*wc + i, re, im);
  }
  *wf = tb.add(nf);
  for (uint64_t j = 0; j < nf; ++j) {
    double re, im;
    acc_root<double>(j, M, &re, &im);
    tb.set(*wf + j, re, im);
  }
}

// make_plan's factorisation (stage_plan.hpp:82-95) and weights (:116-125).
struct Geo {
  std::vector<uint64_t> f, sub_len, rps, out_w, sub_w;
};
Geo geometry(uint64_t n, const std::vector<uint64_t>& f) {
  Geo g;
  g.f = f;
  const size_t p = f.size();
  uint64_t sl = n;
  for (size_t s = 0; s < p; ++s) {
    g.sub_len.push_back(sl);
    g.rps.push_back(sl / f[s]);
    sl /= f[s];
  }
  g.out_w.assign(p, 1);
  for (size_t i = 1; i < p; ++i) g.out_w[i] = g.out_w[i - 1] * f[i - 1];
  g.sub_w.assign(p > 1 ? p - 1 : 0, 1);
  for (size_t i = p - 1; i-- > 0;) g.sub_w[i] = (i + 1 < p - 1) ? g.sub_w[i + 1] * f[i + 1] : 1;
  return g;
}
std::vector<uint64_t> balanced_factors(uint64_t n, uint64_t cap) {
  const int b = ilog2(n), c = ilog2(cap);
  const int p = (b + c - 1) / c, base = b / p, extra = b % p;
  std::vector<uint64_t> f;
  for (int s = 0; s < p; ++s) f.push_back(1ull << (base + (s < extra ? 1 : 0)));
  return f;
}


// ---------------------------------------------------------------- two-level passes
// diagnostics: the last two-level pass created with TILEFFT_TWO_TRACE set
unsigned long long* g_two_trace = nullptr;
// host-mapped watchdog record shared by every two-level launch of the process
// (written by the device only when a dependency wait times out, then it traps)
unsigned long long* g_two_wd_host = nullptr;
unsigned long long* g_two_wd_dev = nullptr;
std::once_flag g_two_wd_once;
unsigned long long* two_watchdog() {
  std::call_once(g_two_wd_once, [] {
    void* h = nullptr;
    const size_t bytes = tfb::kWdWords * sizeof(unsigned long long);
    if (cudaHostAlloc(&h, bytes, cudaHostAllocMapped) != cudaSuccess) {
      cudaGetLastError();
      return;
    }
    std::memset(h, 0, bytes);
    void* d = nullptr;
    if (cudaHostGetDevicePointer(&d, h, 0) != cudaSuccess) {
      cudaGetLastError();
      return;
    }
    g_two_wd_host = static_cast<unsigned long long*>(h);
    g_two_wd_dev = static_cast<unsigned long long*>(d);
  });
  return g_two_wd_dev;
}
size_t g_two_trace_bytes = 0;
bool env_flag(const char* name) {
  const char* e = std::getenv(name);
  return e && *e && *e != '0';
}
// Two-level passes: on by default for 2D columns (8192^2: 2 HBM passes,
// 0.61 ms vs 0.71 ms for rows + [128, 64] columns); opt-in for 1D, where the
// 3-pass comb plan is still faster (0.66 ms vs 0.82 ms at 2^26).
bool two_level_enabled() { return !env_flag("TILEFFT_NO_TWO"); }
bool two_level_1d_enabled() { return two_level_enabled() && env_flag("TILEFFT_TWO_1D"); }
int env_int(const char* name, int dflt) {
  const char* e = std::getenv(name);
  return (e && *e) ? std::atoi(e) : dflt;
}
bool two_level_len(uint64_t L) { return L == 2048 || L == 4096 || L == 8192; }

// One K_TWO pass: length-L transforms along an axis with `cols` columns at
// element stride es_in (16 adjacent columns per group), `B` batch items.
template <typename Real>
Pass make_two_pass(tilefft_plan_s* P, TableBuilder<Real>& tb, uint64_t L, long long cols, long long es_in,
                   long long B, long long bs_in, long long bs_out, long long es_out, int outt, bool twid, uint64_t M) {
  Pass ps{};
  ps.kind = K_TWO;
  ps.L = (int)L;
  ps.la = 512;
  ps.lb = (int)(L / 512);
  ps.outt = outt;
  ps.twid = twid;
  ps.tw_off = add_stage_table(tb, 512);
  ps.twl_off = tb.add(L);
  for (uint64_t e = 0; e < L; ++e) {
    Real re, im;
    acc_root<Real>(e, L, &re, &im);
    tb.set(ps.twl_off + e, re, im);
  }
  tfb::TwoArgs& a = ps.two;
  if (twid) {
    add_interpass(*P->tb64, M, &ps.wc_off, &ps.wf_off, &a.fb);
    a.m_mask = (uint32_t)(M - 1);
  }
  a.chunks = cols / 16;
  a.groups = a.chunks * B;
  a.bs_in = bs_in;
  a.bs_out = bs_out;
  a.es_out = es_out;
  // lag / ring defaults from the sweep in DESIGN.md §8 (8192^2 columns: D 40, 56 slots best)
  a.D = std::max(1, env_int("TILEFFT_TWO_D", 40));
  if (a.D > a.groups) a.D = (int)a.groups;
  a.nslot = std::max(a.D + 1, env_int("TILEFFT_TWO_NSLOT", a.D + 16));
  a.discard = env_int("TILEFFT_TWO_DISCARD", 1);
  a.diag = env_int("TILEFFT_TWO_DIAG", 0);
  a.trace = nullptr;
  a.watchdog = two_watchdog();
  if (env_flag("TILEFFT_TWO_TRACE")) {  // diagnostics: per-item timestamps, read by tilefft_debug_two_trace
    const size_t bytes = (size_t)a.groups * ps.lb * 2 * 8 * sizeof(unsigned long long);
    if (cudaMalloc(&a.trace, bytes) == cudaSuccess) {
      cudaMemset(a.trace, 0, bytes);
      g_two_trace = a.trace;
      g_two_trace_bytes = bytes;
    } else {
      a.trace = nullptr;
    }
  }
  ps.two_cols = cols;
  ps.two_es_in = es_in;
  return ps;
}

// 2^22 <= n <= 2^26 (fp32): the four-step split n = L1 x L2 in two HBM passes,
// both two-level: pass 1 = L1-point column FFTs (stride L2) times W_n^{c k},
// stored transposed (row c of a [L2][L1] matrix); pass 2 = L2-point FFTs over
// those rows' columns, stored in natural order X[k1 + L1 k2].
template <typename Real>
bool build_two_1d(tilefft_plan_s* P, TableBuilder<Real>& tb) {
  if (!std::is_same<Real, float>::value || !two_level_1d_enabled()) return false;
  const uint64_t n = P->n, B = P->batch;
  const int b = ilog2(n);
  const uint64_t L1 = 1ull << ((b + 1) / 2), L2 = n / L1;
  if (!two_level_len(L1) || !two_level_len(L2)) return false;
  P->passes_alt = std::move(P->passes);
  P->passes.clear();
  Pass p1 = make_two_pass(P, tb, L1, (long long)L2, (long long)L2, (long long)B, (long long)n, (long long)n,
                          (long long)L1, 1, true, n);
  p1.src = 0;
  p1.dst = 2;
  Pass p2 = make_two_pass(P, tb, L2, (long long)L1, (long long)L1, (long long)B, (long long)n, (long long)n,
                          (long long)L1, 0, false, 0);
  p2.src = 2;
  p2.dst = 1;
  p2.final_pass = true;
  P->passes.push_back(p1);
  P->passes.push_back(p2);
  P->dev_factors = {L1, L2};
  return true;
}

// ---------------------------------------------------------------- plan building
template <typename Real>
int build_fast_1d(tilefft_plan_s* P, TableBuilder<Real>& tb) {
  const uint64_t n = P->n, B = P->batch;
  constexpr uint64_t kF = tfb::FOf<Real>::v;
  if (n <= 8192) {
    Pass ps{};
    ps.kind = K_ROWS;
    ps.L = (int)n;
    ps.src = 0;
    ps.dst = 1;
    ps.nrows = (long long)B;
    ps.tw_off = add_stage_table(tb, (int)n);
    ps.final_pass = true;
    P->passes.push_back(ps);
    P->dev_factors = {n};
    return 0;
  }
  std::vector<uint64_t> f = balanced_factors(n, 1024);
  if (const char* e = std::getenv("TILEFFT_FAST_FACTORS")) {  // tuning: explicit pass lengths, e.g. "512,256,512"
    std::vector<uint64_t> o;
    uint64_t prod = 1;
    for (const char* c = e; *c;) {
      const uint64_t v = std::strtoull(c, const_cast<char**>(&c), 10);
      if (v) { o.push_back(v); prod *= v; }
      while (*c == ',') ++c;
      if (!v) break;
    }
    bool ok = prod == n && !o.empty();
    for (uint64_t v : o) ok = ok && is_pow2(v) && v >= 2 && v <= 1024;
    if (ok) f = o;
  }
  const Geo g = geometry(n, f);
  const size_t p = f.size();
  if (p > 8) return fail(TILEFFT_EINVAL, "transform too long for the fast path (%zu passes)", p);
  for (size_t s = 0; s < p; ++s) {
    Pass ps{};
    ps.L = (int)f[s];
    ps.tw_off = add_stage_table(tb, ps.L);
    if (s + 1 < p) {
      ps.kind = K_COMB1D;
      ps.src = s == 0 ? 0 : 2;
      ps.dst = 2;
      ps.twid = true;
      int fb;
      add_interpass(*P->tb64, g.sub_len[s], &ps.wc_off, &ps.wf_off, &fb);
      tfb::CombArgs& a = ps.comb;
      a.bstride = (long long)n;
      a.chunks = (long long)(g.rps[s] / kF);
      a.groups_per_batch = (long long)(n / g.sub_len[s]);
      a.ntiles = a.chunks * a.groups_per_batch * (long long)B;
      a.sub_len = (long long)g.sub_len[s];
      a.rps = (long long)g.rps[s];
      a.es = 1;
      a.fvalid = kF;
      a.fb = fb;
      a.m_mask = (uint32_t)(g.sub_len[s] - 1);
      a.p = (int)p;
      ps.grid = a.ntiles;
    } else {
      ps.kind = K_FINALT;
      ps.src = p == 1 ? 0 : 2;
      ps.dst = 1;
      ps.final_pass = true;
      tfb::FinalArgs& a = ps.fin;
      a.bstride = (long long)n;
      a.n = (long long)n;
      a.sw0 = (long long)g.sub_w[0];
      a.chunks = (long long)(f[0] / kF);
      a.ntiles = a.chunks * a.sw0 * (long long)B;
      a.out_w_last = (long long)g.out_w[p - 1];
      a.p = (int)p;
      for (size_t i = 0; i < p; ++i) a.out_w[i] = (long long)g.out_w[i];
      for (size_t i = 0; i + 1 < p; ++i) a.sub_w[i] = (long long)g.sub_w[i];
      ps.grid = a.ntiles;
    }
    P->passes.push_back(ps);
  }
  // 3-pass plans: pass 0 hands over to pass 1 through the transposed T[c1][k0][c2] layout in a second
  // workspace, so no pass writes its rows L1*L2 elements apart (CombArgs::t_l2). Measured against the
  // in-place hand-over: 2^30 10.26 vs 10.57 ms (pass 0 3.52 vs 3.91 ms), 2^29 -4 %, 2^28 -4 %, 2^27 -3 %,
  // 2^26 -1 % (tools/gpu/r02_tstore.sh). TILEFFT_TSTORE=0 keeps the in-place hand-over (A/B only).
  {
    const bool want = env_int("TILEFFT_TSTORE", 1) != 0;
    if (want && p == 3 && g.rps[1] == f[2] && (uint64_t)P->passes[1].comb.groups_per_batch == f[0] &&
        f[2] % kF == 0) {
      Pass& p0 = P->passes[0];
      Pass& p1 = P->passes[1];
      p0.comb.t_l2 = (long long)f[2];
      p0.comb.t_l0l2 = (long long)(f[0] * f[2]);
      p0.dst = 3;
      p1.comb.in_t = 1;
      p1.src = 3;
      p1.dst = 2;
    }
  }
  P->dev_factors = f;
  if (build_two_1d<Real>(P, tb)) return 0;
  return 0;
}

// Column (strided-axis) passes of a 2D transform: logical length ny, element
// stride nx, nx columns, `B` images. Inner passes in place on `buf`; the final
// pass writes `dst`.
template <typename Real>
int build_axis_passes(tilefft_plan_s* P, TableBuilder<Real>& tb, uint64_t ny, uint64_t nx, uint64_t B, int buf,
                      int dst) {
  constexpr uint64_t kF = tfb::FOf<Real>::v;
  const std::vector<uint64_t> f = ny <= 1024 ? std::vector<uint64_t>{ny} : balanced_factors(ny, 1024);
  const Geo g = geometry(ny, f);
  const size_t p = f.size();
  for (size_t s = 0; s < p; ++s) {
    Pass ps{};
    ps.kind = K_COMBAX;
    ps.L = (int)f[s];
    ps.tw_off = add_stage_table(tb, ps.L);
    ps.src = buf;
    ps.dst = (s + 1 == p) ? dst : buf;
    ps.twid = s + 1 < p;
    ps.final_pass = s + 1 == p;
    tfb::CombArgs& a = ps.comb;
    int fb = 0;
    if (ps.twid) add_interpass(*P->tb64, g.sub_len[s], &ps.wc_off, &ps.wf_off, &fb);
    a.bstride = (long long)(ny * nx);
    a.chunks = (long long)((nx + kF - 1) / kF);
    a.fvalid = (int)std::min<uint64_t>(kF, nx);
    a.groups_per_batch = (long long)(ny / f[s]);  // rows of this pass
    a.ntiles = a.chunks * a.groups_per_batch * (long long)B;
    a.sub_len = (long long)g.sub_len[s];
    a.rps = (long long)g.rps[s];
    a.es = (long long)nx;
    a.final_pass = ps.final_pass ? 1 : 0;
    a.out_w_last = (long long)g.out_w[p - 1];
    a.fb = fb;
    a.m_mask = (uint32_t)(g.sub_len[s] - 1);
    a.p = (int)p;
    for (size_t i = 0; i < p; ++i) a.out_w[i] = (long long)g.out_w[i];
    for (size_t i = 0; i + 1 < p; ++i) a.sub_w[i] = (long long)g.sub_w[i];
    ps.grid = a.ntiles;
    P->passes.push_back(ps);
    P->dev_factors.push_back(f[s]);
  }
  return 0;
}

template <typename Real>
int build_exact(tilefft_plan_s* P, TableBuilder<Real>& tb, const std::vector<uint64_t>& f, const void* tv,
                uint64_t tres) {
  const uint64_t n = P->n;
  const Geo g = geometry(n, f);
  const size_t p = f.size();
  if (p > 64) return fail(TILEFFT_EINVAL, "fft_tiled: empty plan");
  for (uint64_t L : f)
    if (L * sizeof(tfb::C2<Real>) > 227 * 1024)
      return fail(TILEFFT_EINVAL, "exact mode: pass length %llu exceeds one CTA's shared memory",
                  (unsigned long long)L);
  // exact roots: W_n^e for e < n, straight from the caller's table when given
  if (P->mode == TILEFFT_MODE_EXACT) {
    const size_t off = tb.add(n);
    if (tv != nullptr) {
      const Real* v = (const Real*)tv;
      const uint64_t stride = tres / n;
      for (uint64_t e = 0; e < n; ++e) tb.set(off + e, v[2 * e * stride], v[2 * e * stride + 1]);
    } else {
      for (uint64_t e = 0; e < n; ++e) {
        Real re, im;
        ref_root<Real>(e, n, &re, &im);
        tb.set(off + e, re, im);
      }
    }
  }
  for (size_t s = 0; s < p; ++s) {
    Pass ps{};
    ps.kind = K_EXACT;
    ps.L = (int)f[s];
    ps.src = s == 0 ? 0 : 2;
    ps.dst = (s + 1 == p) ? 1 : 2;
    ps.final_pass = s + 1 == p;
    tfb::ExactArgs& a = ps.ex;
    a.n = (long long)n;
    a.rows = (long long)(n / f[s]);
    a.bstride = (long long)n;
    a.L = (long long)f[s];
    a.sub_len = (long long)g.sub_len[s];
    a.rps = (long long)g.rps[s];
    a.levels = ilog2(f[s]);
    a.has_inter = s + 1 < p;
    a.p = (int)p;
    a.permute_only = P->mode == TILEFFT_MODE_PERMUTE;
    for (size_t i = 0; i < p; ++i) a.out_w[i] = (long long)g.out_w[i];
    for (size_t i = 0; i + 1 < p; ++i) a.sub_w[i] = (long long)g.sub_w[i];
    ps.grid = a.rows * (long long)P->batch;
    P->passes.push_back(ps);
  }
  P->dev_factors = f;
  return 0;
}

// The paper's previous method: bit reversal + one launch per radix-2 level
// (fft_levelwise, fft_baseline.hpp:66-116). Roots W_n^e from the caller's table.
template <typename Real>
int build_levelwise(tilefft_plan_s* P, TableBuilder<Real>& tb, const void* tv, uint64_t tres) {
  const uint64_t n = P->n;
  const size_t off = tb.add(n);
  for (uint64_t e = 0; e < n; ++e) {
    Real re, im;
    if (tv) {
      const Real* v = (const Real*)tv;
      const uint64_t stride = tres / n;
      re = v[2 * e * stride];
      im = v[2 * e * stride + 1];
    } else {
      ref_root<Real>(e, n, &re, &im);
    }
    tb.set(off + e, re, im);
  }
  Pass ps{};
  ps.kind = K_BITREV;
  ps.src = 0;
  ps.dst = 2;  // workspace: the permutation is not in-place safe (in == out is allowed)
  ps.lw_n = (long long)n;
  ps.lw_total = (long long)(n * P->batch);
  P->passes.push_back(ps);
  const int levels = ilog2(n);
  for (int lv = 0; lv < levels; ++lv) {
    Pass q{};
    q.kind = K_LEVEL;
    q.src = 2;
    q.dst = lv + 1 == levels ? 1 : 2;
    q.level = lv;
    q.lw_n = (long long)n;
    q.lw_total = (long long)(n / 2 * P->batch);
    q.final_pass = lv + 1 == levels;
    P->passes.push_back(q);
  }
  P->dev_factors.assign((size_t)levels, 2);
  return 0;
}

int check_device(int device) {
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0) {
    cudaGetLastError();
    return fail(TILEFFT_ENODEV, "no CUDA device available (the B200 path has no CPU fallback)");
  }
  if (device < 0 || device >= count) return fail(TILEFFT_ENODEV, "device %d out of range (%d devices)", device, count);
  cudaDeviceProp prop;
  CUDA_TRY(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10) return fail(TILEFFT_ENODEV, "device %d is sm_%d%d; this build targets sm_100a", device, prop.major, prop.minor);
  CUDA_TRY(cudaSetDevice(device));
  return 0;
}

template <typename Real>
int finish_plan(tilefft_plan_s* P, TableBuilder<Real>& tb) {
  // workspace when any pass touches it
  bool need_work = false;
  for (const Pass& ps : P->passes) need_work |= (ps.src == 2 || ps.dst == 2);
  for (const Pass& ps : P->passes_alt) need_work |= (ps.src == 2 || ps.dst == 2);
  size_t scratch_elems = 0;
  int ctrl_words = 0;
  for (const Pass& ps : P->passes)
    if (ps.kind == K_TWO) {
      scratch_elems = std::max(scratch_elems, (size_t)ps.two.nslot * (size_t)ps.L * 16);
      ctrl_words = std::max(ctrl_words, 2 + 2 * ps.two.nslot);
    }
  if (scratch_elems) {
    if (int rc = P->scratch.alloc(scratch_elems * 8)) return rc;
    if (int rc = P->ctrl.alloc((size_t)ctrl_words * sizeof(unsigned))) return rc;
    for (Pass& ps : P->passes)
      if (ps.kind == K_TWO) {
        ps.two.scratch = (float2*)P->scratch.p;
        ps.two.ctrl = (unsigned*)P->ctrl.p;
      }
  }
  const uint64_t elems = P->is2d ? P->ny * P->nx * P->batch : P->n * P->batch;
  if (need_work) {
    int rc = P->work.alloc(elems * sizeof(tfb::C2<Real>));
    if (rc) return rc;
  }
  bool need_work2 = false;
  for (const Pass& ps : P->passes) need_work2 |= (ps.src == 3 || ps.dst == 3);
  for (const Pass& ps : P->passes_alt) need_work2 |= (ps.src == 3 || ps.dst == 3);
  if (need_work2) {
    int rc = P->work2.alloc(elems * sizeof(tfb::C2<Real>));
    if (rc) return rc;
  }
  if (P->tb64 && !P->tb64->h.empty()) {
    int rc = P->tables64.alloc(P->tb64->h.size() * sizeof(double));
    if (rc) return rc;
    CUDA_TRY(cudaMemcpy(P->tables64.p, P->tb64->h.data(), P->tb64->h.size() * sizeof(double), cudaMemcpyHostToDevice));
  }
  P->table_elems = tb.h.size() / 2;
  if (P->table_elems) {
    int rc = P->tables.alloc(tb.h.size() * sizeof(Real));
    if (rc) return rc;
    CUDA_TRY(cudaMemcpy(P->tables.p, tb.h.data(), tb.h.size() * sizeof(Real), cudaMemcpyHostToDevice));
  }
  return 0;
}

template <typename Real>
int exec_impl(tilefft_plan_s* P, const void* in, void* out, int sign, cudaStream_t st, cudaEvent_t* ev = nullptr) {
  const bool inv = sign == TILEFFT_INVERSE;
  const uint64_t total = P->is2d ? P->ny * P->nx : P->n;
  const Real scale = inv ? (Real)1 / (Real)total : (Real)1;
  auto buf = [&](int id) -> void* {
    return id == 0 ? const_cast<void*>(in) : id == 1 ? out : id == 3 ? P->work2.p : P->work.p;
  };
  // two-level passes stream their input with TMA (16-byte aligned); an
  // unaligned user buffer takes the equivalent plan without them
  const bool use_alt = !P->passes_alt.empty() && ((uintptr_t)in % 16 != 0);
  int ip = 0;
  for (const Pass& ps : use_alt ? P->passes_alt : P->passes) {
    int rc;
    if (ev) CUDA_TRY(cudaEventRecord(ev[ip], st));
    ++ip;
    const void* src = buf(ps.src);
    void* dst = buf(ps.dst);
    if (ps.kind == K_EXACT) {
      const bool first = &ps == &P->passes.front();
      rc = launch_exact<Real>(ps, src, dst, P->tables.p, scale, inv && first, inv && ps.final_pass, st);
    } else if (ps.kind == K_BITREV || ps.kind == K_LEVEL) {
      rc = launch_levelwise<Real>(ps, src, dst, P->tables.p, scale, inv && ps.kind == K_BITREV,
                                  inv && ps.final_pass, st);
    } else if (inv) {
      rc = launch_fast<Real, true>(ps, src, dst, P->tables.p, P->tables64.p, ps.final_pass ? scale : (Real)1, st);
    } else {
      rc = launch_fast<Real, false>(ps, src, dst, P->tables.p, P->tables64.p, (Real)1, st);
    }
    if (rc) return rc;
  }
  if (ev) CUDA_TRY(cudaEventRecord(ev[ip], st));
  return 0;
}

}  // namespace

namespace {
// run `fn(d_in, d_out)` on temporary device copies of host buffers
template <class F>
int with_device_buffers(int device, const void* h_in, void* h_out, size_t in_bytes, size_t out_bytes, F fn) {
  if (int rc = check_device(device)) return rc;
  DevBuf din, dout;
  if (int rc = din.alloc(in_bytes)) return rc;
  if (int rc = dout.alloc(out_bytes)) return rc;
  CUDA_TRY(cudaMemcpy(din.p, h_in, in_bytes, cudaMemcpyHostToDevice));
  if (int rc = fn(din.p, dout.p)) return rc;
  CUDA_TRY(cudaMemcpy(h_out, dout.p, out_bytes, cudaMemcpyDeviceToHost));
  return 0;
}
}  // namespace

// ================================================================ C ABI
// Diagnostics only (not part of include/tilefft_b200.h): copy the per-item timestamps of the
// last traced two-level pass (TILEFFT_TWO_TRACE=1) to host memory; returns the bytes available.
// Diagnostics only: the watchdog record of the last two-level dependency wait that timed
// out (tfb::kWdWords words, layout in twolevel.cuh); returns 0 if none fired.
extern "C" TILEFFT_API int tilefft_debug_two_watchdog(unsigned long long* out, int words) {
  if (!g_two_wd_host) return 0;
  volatile unsigned long long* w = g_two_wd_host;
  if (out)
    for (int i = 0; i < words && i < tfb::kWdWords; ++i) out[i] = w[i];
  return w[0] ? 1 : 0;
}

extern "C" TILEFFT_API long long tilefft_debug_two_trace(void* host, long long bytes) {
  if (!g_two_trace) return 0;
  if (host && bytes > 0) {
    cudaDeviceSynchronize();
    cudaMemcpy(host, g_two_trace, std::min((size_t)bytes, g_two_trace_bytes),
               cudaMemcpyDeviceToHost);
  }
  return (long long)g_two_trace_bytes;
}

namespace {
// Device-side barrier of the distributed step (replaces a host synchronize + a
// process barrier between pass 1 and pass 2, so the step is stream-ordered and
// graph-capturable). One thread: bump this rank's epoch, release-add 1 to every
// rank's arrival word (the fence orders the preceding pass-1 peer stores, which
// the kernel boundary already made happen-before this kernel), then acquire-poll
// its own word until all ranks arrived for this epoch. The counters only grow,
// so no reset is needed between calls; a peer that never arrives ends the wait
// with a trap after 60 s instead of hanging the GPU.
struct DistFlags {
  unsigned* peer[16];
  unsigned* mine;
  unsigned* epoch;
  int n;
};
__global__ void k_dist_barrier(DistFlags f) {
  if (threadIdx.x != 0) return;
  const unsigned e = *f.epoch + 1u;
  *f.epoch = e;
  __threadfence_system();
  for (int d = 0; d < f.n; ++d) asm volatile("red.release.sys.global.add.u32 [%0], 1;" ::"l"(f.peer[d]) : "memory");
  const unsigned target = e * (unsigned)f.n;
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (;;) {
    unsigned v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(f.mine) : "memory");
    if ((int)(v - target) >= 0) break;
    __nanosleep(200);
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > 60ull * 1000000000ull) __trap();
  }
}
}  // namespace

extern "C" {

const char* tilefft_last_error(void) { return g_err.c_str(); }
const char* tilefft_version(void) { return "tilefft_b200 0.1 sm_100a"; }

int tilefft_build_twiddle(uint64_t resolution, uint32_t elem_bytes, void* out) {
  g_err.clear();
  if (!is_pow2(resolution) || resolution < 2)
    return fail(TILEFFT_EINVAL, "build_twiddle_table: resolution must be a power of two >= 2");
  if (elem_bytes != 8 && elem_bytes != 16) return fail(TILEFFT_EINVAL, "build_twiddle_table: elem_bytes must be 8 or 16");
  if (!out) return fail(TILEFFT_EINVAL, "build_twiddle_table: null output");
  for (uint64_t j = 0; j < resolution; ++j) {
    if (elem_bytes == 8) {
      float* o = (float*)out;
      ref_root<float>(j, resolution, &o[2 * j], &o[2 * j + 1]);
    } else {
      double* o = (double*)out;
      ref_root<double>(j, resolution, &o[2 * j], &o[2 * j + 1]);
    }
  }
  return 0;
}

int tilefft_plan_create(tilefft_plan_t* out, uint64_t n, uint64_t batch, const uint64_t* factors, uint32_t nfactors,
                        uint32_t elem_bytes, uint32_t mode, const void* tv, uint64_t tres, int device) {
  g_err.clear();
  if (!out) return fail(TILEFFT_EINVAL, "tilefft_plan_create: null plan pointer");
  *out = nullptr;
  if (!is_pow2(n) || n < 2) return fail(TILEFFT_EINVAL, "make_plan: n must be a power of two >= 2");
  if (batch < 1) return fail(TILEFFT_EINVAL, "tilefft_plan_create: batch must be >= 1");
  if (elem_bytes != 8 && elem_bytes != 16) return fail(TILEFFT_EINVAL, "tilefft_plan_create: elem_bytes must be 8 or 16");
  if (mode > TILEFFT_MODE_LEVELWISE) return fail(TILEFFT_EINVAL, "tilefft_plan_create: unknown mode %u", mode);
  std::vector<uint64_t> f;
  if (factors && nfactors) {
    uint64_t prod = 1;
    for (uint32_t i = 0; i < nfactors; ++i) {
      if (!is_pow2(factors[i]) || factors[i] < 2) return fail(TILEFFT_EINVAL, "plan factors must be powers of two >= 2");
      prod *= factors[i];
      f.push_back(factors[i]);
    }
    if (prod != n) return fail(TILEFFT_EINVAL, "fft_tiled: signal length does not match the plan");
  }
  // fast-path inter-pass exponents r*k are reduced mod M <= n in 32-bit
  // arithmetic (fast_kernels.cuh interpass_scale): exact for n <= 2^32 only
  if (mode == TILEFFT_MODE_FAST && n > (1ull << 32))
    return fail(TILEFFT_EINVAL, "tilefft_plan_create: fast mode supports n <= 2^32");
  if ((mode == TILEFFT_MODE_EXACT || mode == TILEFFT_MODE_PERMUTE) && f.empty())
    return fail(TILEFFT_EINVAL, "fft_tiled: empty plan");
  if ((mode == TILEFFT_MODE_EXACT || mode == TILEFFT_MODE_LEVELWISE) && tv != nullptr &&
      !(tres >= n && is_pow2(tres) && tres % n == 0))
    return fail(TILEFFT_EINVAL, "fft_tiled: signal length must divide the table resolution");
  if (int rc = check_device(device)) return rc;
  tilefft_plan_s* P = new (std::nothrow) tilefft_plan_s();
  if (!P) return fail(TILEFFT_ENOMEM, "out of host memory");
  P->device = device;
  P->n = n;
  P->batch = batch;
  P->elem_bytes = elem_bytes;
  P->mode = mode;
  int rc;
  TableBuilder<double> tb64;
  P->tb64 = &tb64;
  if (elem_bytes == 8) {
    TableBuilder<float> tb;
    rc = mode == TILEFFT_MODE_FAST        ? build_fast_1d<float>(P, tb)
         : mode == TILEFFT_MODE_LEVELWISE ? build_levelwise<float>(P, tb, tv, tres)
                                          : build_exact<float>(P, tb, f, tv, tres);
    if (!rc) rc = finish_plan<float>(P, tb);
  } else {
    TableBuilder<double> tb;
    rc = mode == TILEFFT_MODE_FAST        ? build_fast_1d<double>(P, tb)
         : mode == TILEFFT_MODE_LEVELWISE ? build_levelwise<double>(P, tb, tv, tres)
                                          : build_exact<double>(P, tb, f, tv, tres);
    if (!rc) rc = finish_plan<double>(P, tb);
  }
  P->tb64 = nullptr;
  if (rc) {
    delete P;
    return rc;
  }
  *out = P;
  return 0;
}

int tilefft_plan_create_2d(tilefft_plan_t* out, uint64_t ny, uint64_t nx, uint64_t batch, uint32_t elem_bytes,
                           int device) {
  g_err.clear();
  if (!out) return fail(TILEFFT_EINVAL, "tilefft_plan_create_2d: null plan pointer");
  *out = nullptr;
  if (!is_pow2(ny) || !is_pow2(nx) || ny < 2 || nx < 2)
    return fail(TILEFFT_EINVAL, "make_plan: n must be a power of two >= 2");
  if (batch < 1) return fail(TILEFFT_EINVAL, "tilefft_plan_create_2d: batch must be >= 1");
  if (elem_bytes != 8 && elem_bytes != 16) return fail(TILEFFT_EINVAL, "tilefft_plan_create_2d: elem_bytes must be 8 or 16");
  if (nx > 8192) return fail(TILEFFT_EINVAL, "tilefft_plan_create_2d: rows longer than 8192 are not supported yet");
  if (ny > (1ull << 32) / nx) return fail(TILEFFT_EINVAL, "tilefft_plan_create_2d: ny * nx must be <= 2^32");
  if (int rc = check_device(device)) return rc;
  tilefft_plan_s* P = new (std::nothrow) tilefft_plan_s();
  if (!P) return fail(TILEFFT_ENOMEM, "out of host memory");
  P->device = device;
  P->is2d = 1;
  P->ny = ny;
  P->nx = nx;
  P->n = ny * nx;
  P->batch = batch;
  P->elem_bytes = elem_bytes;
  P->mode = TILEFFT_MODE_FAST;
  TableBuilder<double> tb64;
  P->tb64 = &tb64;
  auto build = [&](auto tbv) -> int {
    using Real = std::remove_reference_t<decltype(tbv.h[0])>;
    TableBuilder<Real> tb;
    const bool multi = ny > 1024;
    Pass rows{};
    rows.kind = K_ROWS;
    rows.L = (int)nx;
    rows.src = 0;
    rows.dst = multi ? 2 : 1;
    rows.nrows = (long long)(ny * batch);
    rows.tw_off = add_stage_table(tb, (int)nx);
    // 2048..8192-point columns (fp32): one two-level pass through L2
    const bool two = std::is_same<Real, float>::value && two_level_enabled() && two_level_len(ny) && nx % 16 == 0;
    if (two) rows.dst = 2;
    P->passes.push_back(rows);
    P->dev_factors.push_back(nx);
    if (two) {
      Pass c = make_two_pass(P, tb, ny, (long long)nx, (long long)nx, (long long)batch, (long long)(ny * nx),
                             (long long)(ny * nx), (long long)nx, 0, false, 0);
      c.src = 2;
      c.dst = 1;
      c.final_pass = true;
      P->passes.push_back(c);
      P->dev_factors.push_back(ny);
      return finish_plan<Real>(P, tb);
    }
    int rc = build_axis_passes<Real>(P, tb, ny, nx, batch, multi ? 2 : 1, 1);
    if (rc) return rc;
    return finish_plan<Real>(P, tb);
  };
  int rc = elem_bytes == 8 ? build(TableBuilder<float>{}) : build(TableBuilder<double>{});
  P->tb64 = nullptr;
  if (rc) {
    delete P;
    return rc;
  }
  *out = P;
  return 0;
}

int tilefft_exec_c2c(tilefft_plan_t P, const void* in, void* out, int sign, void* stream) {
  g_err.clear();
  if (!P) return fail(TILEFFT_EINVAL, "tilefft_exec_c2c: null plan");
  if (!in || !out) return fail(TILEFFT_EINVAL, "tilefft_exec_c2c: null buffer");
  if (sign != TILEFFT_FORWARD && sign != TILEFFT_INVERSE) return fail(TILEFFT_EINVAL, "tilefft_exec_c2c: sign must be -1 or +1");
  if (P->mode == TILEFFT_MODE_PERMUTE && sign != TILEFFT_FORWARD)
    return fail(TILEFFT_EINVAL, "tilefft_exec_c2c: permute mode is forward only");
  CUDA_TRY(cudaSetDevice(P->device));
  cudaStream_t st = (cudaStream_t)stream;
  auto direct = [&](cudaStream_t s) {
    return P->elem_bytes == 8 ? exec_impl<float>(P, in, out, sign, s) : exec_impl<double>(P, in, out, sign, s);
  };
  std::lock_guard<std::mutex> lock(P->graph_mu);
  if (!P->exec_done) CUDA_TRY(cudaEventCreateWithFlags(&P->exec_done, cudaEventDisableTiming));
  // inside a caller's stream capture the graph's own edges order the execs (an
  // event recorded outside the capture cannot be waited on from inside it)
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  CUDA_TRY(cudaStreamIsCapturing(st, &cap));
  const bool capturing = cap != cudaStreamCaptureStatusNone;
  if (!capturing) CUDA_TRY(cudaStreamWaitEvent(st, P->exec_done, 0));
  auto launched = [&](int rc) -> int {
    if (rc) return rc;
    if (!capturing) CUDA_TRY(cudaEventRecord(P->exec_done, st));
    return 0;
  };
  // a caller capturing its own graph gets the pass launches themselves captured
  if (capturing || env_flag("TILEFFT_NO_GRAPH")) return launched(direct(st));
  for (auto& g : P->graphs)
    if (g.in == in && g.out == out && g.sign == sign) {
      CUDA_TRY(cudaGraphLaunch(g.exec, st));
      return launched(0);
    }
  // capture the pass sequence once on a private stream (the caller's stream
  // may be the legacy default stream, which cannot be captured)
  if (!P->cap_stream) CUDA_TRY(cudaStreamCreateWithFlags(&P->cap_stream, cudaStreamNonBlocking));
  CUDA_TRY(cudaStreamBeginCapture(P->cap_stream, cudaStreamCaptureModeThreadLocal));
  const int rc = direct(P->cap_stream);
  cudaGraph_t graph = nullptr;
  const cudaError_t ce = cudaStreamEndCapture(P->cap_stream, &graph);
  if (rc) {
    if (graph) cudaGraphDestroy(graph);
    return rc;
  }
  if (ce != cudaSuccess) return fail(TILEFFT_ECUDA, "stream capture failed: %s", cudaGetErrorString(ce));
  cudaGraphExec_t exec = nullptr;
  const cudaError_t ie = cudaGraphInstantiate(&exec, graph, 0);
  cudaGraphDestroy(graph);
  if (ie != cudaSuccess) return fail(TILEFFT_ECUDA, "cudaGraphInstantiate: %s", cudaGetErrorString(ie));
  if (P->graphs.size() >= tilefft_plan_s::kMaxGraphs) {
    cudaGraphExecDestroy(P->graphs.front().exec);
    P->graphs.erase(P->graphs.begin());
  }
  P->graphs.push_back({in, out, sign, exec});
  CUDA_TRY(cudaGraphLaunch(exec, st));
  return launched(0);
}

int tilefft_exec_c2c_timed(tilefft_plan_t P, const void* in, void* out, int sign, void* stream, int reps,
                           float* pass_ms, int max_passes) {
  g_err.clear();
  if (!P) return fail(TILEFFT_EINVAL, "tilefft_exec_c2c_timed: null plan");
  if (!in || !out || !pass_ms) return fail(TILEFFT_EINVAL, "tilefft_exec_c2c_timed: null buffer");
  if (sign != TILEFFT_FORWARD && sign != TILEFFT_INVERSE)
    return fail(TILEFFT_EINVAL, "tilefft_exec_c2c_timed: sign must be -1 or +1");
  if (reps < 1) return fail(TILEFFT_EINVAL, "tilefft_exec_c2c_timed: reps must be >= 1");
  CUDA_TRY(cudaSetDevice(P->device));
  cudaStream_t st = (cudaStream_t)stream;
  std::lock_guard<std::mutex> lock(P->graph_mu);
  const bool use_alt = !P->passes_alt.empty() && ((uintptr_t)in % 16 != 0);
  const int np = (int)(use_alt ? P->passes_alt : P->passes).size();
  std::vector<cudaEvent_t> ev((size_t)(np + 1) * reps, nullptr);
  int rc = 0;
  for (auto& e : ev)
    if (cudaEventCreate(&e) != cudaSuccess) { rc = fail(TILEFFT_ECUDA, "cudaEventCreate failed"); break; }
  if (!rc && P->exec_done) rc = cudaStreamWaitEvent(st, P->exec_done, 0) == cudaSuccess ? 0 : fail(TILEFFT_ECUDA, "cudaStreamWaitEvent failed");
  for (int r = 0; r < reps && !rc; ++r)
    rc = P->elem_bytes == 8 ? exec_impl<float>(P, in, out, sign, st, &ev[(size_t)r * (np + 1)])
                            : exec_impl<double>(P, in, out, sign, st, &ev[(size_t)r * (np + 1)]);
  if (!rc && cudaStreamSynchronize(st) != cudaSuccess) rc = fail(TILEFFT_ECUDA, "exec_c2c_timed: %s", cudaGetErrorString(cudaGetLastError()));
  if (!rc) {
    for (int i = 0; i < np && i < max_passes; ++i) {
      double acc = 0;
      for (int r = 0; r < reps; ++r) {
        float ms = 0;
        cudaEventElapsedTime(&ms, ev[(size_t)r * (np + 1) + i], ev[(size_t)r * (np + 1) + i + 1]);
        acc += ms;
      }
      pass_ms[i] = (float)(acc / reps);
    }
  }
  for (auto& e : ev)
    if (e) cudaEventDestroy(e);
  return rc;
}

int tilefft_exec_c2c_host(tilefft_plan_t P, const void* h_in, void* h_out, int sign) {
  g_err.clear();
  if (!P) return fail(TILEFFT_EINVAL, "tilefft_exec_c2c_host: null plan");
  if (!h_in || !h_out) return fail(TILEFFT_EINVAL, "tilefft_exec_c2c_host: null buffer");
  if (sign != TILEFFT_FORWARD && sign != TILEFFT_INVERSE)
    return fail(TILEFFT_EINVAL, "tilefft_exec_c2c_host: sign must be -1 or +1");
  if (P->mode == TILEFFT_MODE_PERMUTE && sign != TILEFFT_FORWARD)
    return fail(TILEFFT_EINVAL, "tilefft_exec_c2c_host: permute mode is forward only");
  std::lock_guard<std::mutex> lock(P->host_mu);
  CUDA_TRY(cudaSetDevice(P->device));
  const uint64_t per = P->n;  // elements per transform (2D: ny*nx)
  const size_t eb = P->elem_bytes;
  const uint64_t B = P->batch;
  // chunked pipeline only for single-pass batched plans whose passes act per transform
  const bool chunkable = B > 1 && P->passes.size() == 1 && P->passes[0].kind == K_ROWS && !P->is2d;
  if (!chunkable) {
    const size_t bytes = per * B * eb;
    if (!P->hbuf[0].p) {
      if (int rc = P->hbuf[0].alloc(bytes)) return rc;
    }
    CUDA_TRY(cudaMemcpy(P->hbuf[0].p, h_in, bytes, cudaMemcpyHostToDevice));
    if (int rc = tilefft_exec_c2c(P, P->hbuf[0].p, P->hbuf[0].p, sign, nullptr)) return rc;
    CUDA_TRY(cudaMemcpy(h_out, P->hbuf[0].p, bytes, cudaMemcpyDeviceToHost));
    return 0;
  }
  // Three-queue pipeline over kHostStreams device buffers of ~16 MiB:
  //   hs[0]: H2D copies, back to back (one copy engine)
  //   hs[1]: the pass kernel, in place on the chunk
  //   hs[2]: D2H copies, back to back (the other copy engine)
  // events order the queues per buffer, so both PCIe directions stream at once
  // and only the first H2D and the last D2H chunk are not overlapped.
  constexpr int NB = tilefft_plan_s::kHostStreams;
  if (!P->host_chunk) {
    uint64_t chunk_mb = 32;
    if (const char* e = std::getenv("TILEFFT_HOST_CHUNK_MB")) chunk_mb = std::max(1, std::atoi(e));
    uint64_t c = std::max<uint64_t>(1, (chunk_mb << 20) / (per * eb));
    P->host_chunk = std::min<uint64_t>(c, B);
    for (int i = 0; i < 3; ++i) CUDA_TRY(cudaStreamCreateWithFlags(&P->hs[i], cudaStreamNonBlocking));
    for (int i = 0; i < NB; ++i) {
      if (int rc = P->hbuf[i].alloc(P->host_chunk * per * eb)) return rc;
      CUDA_TRY(cudaEventCreateWithFlags(&P->hev[i], cudaEventDisableTiming));
      CUDA_TRY(cudaEventCreateWithFlags(&P->hev_in[i], cudaEventDisableTiming));
      CUDA_TRY(cudaEventCreateWithFlags(&P->hev_k[i], cudaEventDisableTiming));
    }
  }
  // chunk schedule: ramp up from C/8 and back down at the end, so the
  // non-overlapped first H2D and last D2H are short while the steady state
  // uses large copies (each copy has ~18 us of fixed cost)
  const uint64_t Cmax = P->host_chunk;
  std::vector<uint64_t> sizes;
  {
    std::vector<uint64_t> head, tail;
    uint64_t left = B;
    for (uint64_t c = std::max<uint64_t>(1, Cmax / 8); c < Cmax && left > 2 * c; c *= 2) {
      head.push_back(c);
      tail.push_back(c);
      left -= 2 * c;
    }
    sizes = head;
    while (left > 0) {
      const uint64_t c = std::min(left, Cmax);
      sizes.push_back(c);
      left -= c;
    }
    for (auto it = tail.rbegin(); it != tail.rend(); ++it) sizes.push_back(*it);
  }
  Pass ps = P->passes[0];
  // on an error part-way through, copies may still be reading/writing the
  // caller's buffers: drain every queue before returning
  auto drain = [&](int rc) -> int {
    for (int i = 0; i < 3; ++i) cudaStreamSynchronize(P->hs[i]);
    cudaGetLastError();
    return rc;
  };
#define HOST_TRY(expr)                                                                            \
  do {                                                                                            \
    cudaError_t e_ = (expr);                                                                      \
    if (e_ != cudaSuccess) return drain(fail(TILEFFT_ECUDA, "%s: %s", #expr, cudaGetErrorString(e_))); \
  } while (0)
  uint64_t b0 = 0;
  for (uint64_t idx = 0; idx < sizes.size(); b0 += sizes[idx], ++idx) {
    const int bi = (int)(idx % NB);
    const uint64_t nb = sizes[idx];
    const size_t off = b0 * per * eb, bytes = nb * per * eb;
    void* buf = P->hbuf[bi].p;
    if (idx >= (uint64_t)NB) HOST_TRY(cudaStreamWaitEvent(P->hs[0], P->hev[bi], 0));  // buffer drained
    HOST_TRY(cudaMemcpyAsync(buf, (const char*)h_in + off, bytes, cudaMemcpyHostToDevice, P->hs[0]));
    HOST_TRY(cudaEventRecord(P->hev_in[bi], P->hs[0]));
    HOST_TRY(cudaStreamWaitEvent(P->hs[1], P->hev_in[bi], 0));
    ps.nrows = (long long)nb;
    const bool inv = sign == TILEFFT_INVERSE;
    int rc;
    if (P->elem_bytes == 8) {
      const float scale = inv ? 1.0f / (float)per : 1.0f;
      rc = inv ? launch_fast<float, true>(ps, buf, buf, P->tables.p, nullptr, scale, P->hs[1])
               : launch_fast<float, false>(ps, buf, buf, P->tables.p, nullptr, scale, P->hs[1]);
    } else {
      const double scale = inv ? 1.0 / (double)per : 1.0;
      rc = inv ? launch_fast<double, true>(ps, buf, buf, P->tables.p, nullptr, scale, P->hs[1])
               : launch_fast<double, false>(ps, buf, buf, P->tables.p, nullptr, scale, P->hs[1]);
    }
    if (rc) return drain(rc);
    HOST_TRY(cudaEventRecord(P->hev_k[bi], P->hs[1]));
    HOST_TRY(cudaStreamWaitEvent(P->hs[2], P->hev_k[bi], 0));
    HOST_TRY(cudaMemcpyAsync((char*)h_out + off, buf, bytes, cudaMemcpyDeviceToHost, P->hs[2]));
    HOST_TRY(cudaEventRecord(P->hev[bi], P->hs[2]));
  }
  HOST_TRY(cudaStreamSynchronize(P->hs[2]));
#undef HOST_TRY
  return 0;
}


int tilefft_exchange(const void* h_in, void* h_out, uint64_t n, const uint64_t* factors, uint32_t nfactors,
                     uint32_t stage, uint32_t elem_bytes, int device) {
  g_err.clear();
  if (!h_in || !h_out || !factors || nfactors == 0) return fail(TILEFFT_EINVAL, "exchange_transpose: null argument");
  if (elem_bytes != 8 && elem_bytes != 16) return fail(TILEFFT_EINVAL, "exchange_transpose: elem_bytes must be 8 or 16");
  if (stage < 1 || stage > nfactors) return fail(TILEFFT_EINVAL, "exchange_transpose: stage out of range");
  std::vector<uint64_t> f(factors, factors + nfactors);
  uint64_t prod = 1;
  for (uint64_t v : f) prod *= v;
  if (prod != n || nfactors > 64) return fail(TILEFFT_EINVAL, "exchange_transpose: signal length does not match the plan");
  const Geo g = geometry(n, f);
  tfb::ExchangeArgs a{};
  a.n = (long long)n;
  a.L = (long long)f[stage - 1];
  a.sub_len = (long long)g.sub_len[stage - 1];
  a.rps = (long long)g.rps[stage - 1];
  a.final_pass = stage == nfactors;
  a.p = (int)nfactors;
  for (size_t i = 0; i < f.size(); ++i) a.out_w[i] = (long long)g.out_w[i];
  for (size_t i = 0; i + 1 < f.size(); ++i) a.sub_w[i] = (long long)g.sub_w[i];
  const size_t bytes = n * elem_bytes;
  return with_device_buffers(device, h_in, h_out, bytes, bytes, [&](void* din, void* dout) -> int {
    int rc = elem_bytes == 8 ? launch_exchange<float>(din, dout, a, nullptr) : launch_exchange<double>(din, dout, a, nullptr);
    if (rc) return rc;
    CUDA_TRY(cudaDeviceSynchronize());
    return 0;
  });
}

int tilefft_interstage_scale(const void* h_in, void* h_out, uint64_t rows, uint64_t cols, uint64_t row0,
                             uint64_t rows_per_sub, uint64_t sub_len, const void* table, uint64_t resolution,
                             uint32_t elem_bytes, int device) {
  g_err.clear();
  if (!h_in || !h_out || !table) return fail(TILEFFT_EINVAL, "apply_interstage_twiddles: null argument");
  if (elem_bytes != 8 && elem_bytes != 16) return fail(TILEFFT_EINVAL, "apply_interstage_twiddles: elem_bytes must be 8 or 16");
  if (!is_pow2(sub_len) || !is_pow2(resolution) || resolution < sub_len || rows_per_sub == 0)
    return fail(TILEFFT_EINVAL, "apply_interstage_twiddles: sub-transform length must divide the table resolution");
  if (int rc = check_device(device)) return rc;
  DevBuf dt;
  if (int rc = dt.alloc(resolution * elem_bytes)) return rc;
  CUDA_TRY(cudaMemcpy(dt.p, table, resolution * elem_bytes, cudaMemcpyHostToDevice));
  const size_t bytes = rows * cols * elem_bytes;
  return with_device_buffers(device, h_in, h_out, bytes, bytes, [&](void* din, void* dout) -> int {
    const long long ts = (long long)(resolution / sub_len);
    int rc = elem_bytes == 8 ? launch_interstage<float>(din, dout, (long long)rows, (long long)cols, (long long)row0,
                                                        (long long)rows_per_sub, (long long)sub_len, dt.p, ts, nullptr)
                             : launch_interstage<double>(din, dout, (long long)rows, (long long)cols, (long long)row0,
                                                         (long long)rows_per_sub, (long long)sub_len, dt.p, ts, nullptr);
    if (rc) return rc;
    CUDA_TRY(cudaDeviceSynchronize());
    return 0;
  });
}

// ---------------------------------------------------------------- distributed
int tilefft_dist_plan_create(tilefft_plan_t* out, uint64_t n, uint32_t nranks, uint32_t rank, uint32_t elem_bytes,
                             int device) {
  g_err.clear();
  if (!out) return fail(TILEFFT_EINVAL, "tilefft_dist_plan_create: null plan pointer");
  *out = nullptr;
  if (!is_pow2(n) || n < 2) return fail(TILEFFT_EINVAL, "make_plan: n must be a power of two >= 2");
  if (!is_pow2(nranks) || nranks > 16 || rank >= nranks)
    return fail(TILEFFT_EINVAL, "tilefft_dist_plan_create: nranks must be a power of two <= 16 and rank < nranks");
  if (elem_bytes != 8 && elem_bytes != 16) return fail(TILEFFT_EINVAL, "tilefft_dist_plan_create: elem_bytes must be 8 or 16");
  const uint64_t F = elem_bytes == 8 ? 16 : 8;
  // four-step split N = N1 x N2: N1 <= 1024 column FFTs (one on-chip pass),
  // N2 = N / N1 row FFTs (local multi-pass when > 8192)
  const uint64_t n1 = std::min<uint64_t>(1024, n >> 7);
  const uint64_t n2 = n / std::max<uint64_t>(n1, 1);
  if (n1 < 128 || n1 % nranks || n2 % (nranks * F))
    return fail(TILEFFT_EINVAL, "tilefft_dist_plan_create: n too small for %u ranks (need n >= %llu)", nranks,
                (unsigned long long)(128 * 128 * nranks));
  if (n > (1ull << 32)) return fail(TILEFFT_EINVAL, "tilefft_dist_plan_create: n > 2^32 not supported");
  if (int rc = check_device(device)) return rc;
  tilefft_plan_s* P = new (std::nothrow) tilefft_plan_s();
  if (!P) return fail(TILEFFT_ENOMEM, "out of host memory");
  P->device = device;
  P->is_dist = true;
  P->n = n;
  P->batch = 1;
  P->elem_bytes = elem_bytes;
  P->nranks = nranks;
  P->rank = rank;
  P->n1 = n1;
  P->n2 = n2;
  TableBuilder<double> tb64;
  P->tb64 = &tb64;
  auto build = [&](auto tbv) -> int {
    using Real = std::remove_reference_t<decltype(tbv.h[0])>;
    TableBuilder<Real> tb;
    DistPass1& d = P->dist;
    d.L = (int)n1;
    d.C = (long long)(n2 / nranks);
    d.tw_off = add_stage_table(tb, (int)n1);
    add_interpass(tb64, n, &d.wc_off, &d.wf_off, &d.fb);
    d.m_mask = (uint32_t)(n - 1);
    tfb::CombTmaArgs& a = d.a;
    a.chunks = d.C / (long long)F;
    a.groups_per_batch = 1;
    a.ntiles = a.chunks;
    a.rps = d.C;
    a.sub_len = (long long)(n1 * d.C);
    a.fvalid = (int)F;
    a.fb = d.fb;
    a.m_mask = d.m_mask;
    a.r_off = (long long)rank * d.C;
    a.rows_per_rank = (int)(n1 / nranks);
    a.nranks = (int)nranks;
    P->dev_factors = {n1};
    int rc = finish_plan<Real>(P, tb);
    if (rc) return rc;
    rc = tilefft_plan_create(&P->inner, n2, n1 / nranks, nullptr, 0, elem_bytes, TILEFFT_MODE_FAST, nullptr, 0,
                             device);
    if (rc) return rc;
    // pass 2 straight from the all-to-all's receive buffer [src][k1][c] (NCCL exchange): the row plan
    // with its first (comb) pass reading through a 5-D tensor map; only when that pass is a comb pass
    if (P->inner->passes.size() > 1 && P->inner->passes[0].kind == K_COMB1D) {
      rc = tilefft_plan_create(&P->inner_blocks, n2, n1 / nranks, nullptr, 0, elem_bytes, TILEFFT_MODE_FAST, nullptr,
                               0, device);
      if (rc) return rc;
      tfb::CombArgs& c = P->inner_blocks->passes[0].comb;
      const uint64_t C = n2 / nranks;
      c.split_q = (long long)(C / (uint64_t)c.rps);
      c.split_stride = (long long)((n1 / nranks) * C);
      c.split_bstride = (long long)C;
      if (c.split_q < 1 || C % (uint64_t)c.rps) {
        tilefft_plan_destroy(P->inner_blocks);
        P->inner_blocks = nullptr;
      } else {
        P->inner_blocks->passes_alt.clear();  // the blocks layout has no non-TMA variant
      }
    }
    return 0;
  };
  int rc = elem_bytes == 8 ? build(TableBuilder<float>{}) : build(TableBuilder<double>{});
  P->tb64 = nullptr;
  if (rc) {
    delete P;
    return rc;
  }
  for (uint64_t f : P->inner->dev_factors) P->dev_factors.push_back(f);
  if (int frc = P->flags.alloc(256)) {
    delete P;
    return frc;
  }
  if (cudaMemset(P->flags.p, 0, 256) != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess) {
    delete P;
    return fail(TILEFFT_ECUDA, "tilefft_dist_plan_create: clearing the barrier words failed");
  }
  *out = P;
  return 0;
}

int tilefft_dist_layout(tilefft_plan_t P, uint64_t* n1, uint64_t* n2, uint64_t* cols_per_rank, uint64_t* rows_per_rank) {
  if (!P || !P->is_dist) return fail(TILEFFT_EINVAL, "tilefft_dist_layout: not a distributed plan");
  if (n1) *n1 = P->n1;
  if (n2) *n2 = P->n2;
  if (cols_per_rank) *cols_per_rank = P->n2 / P->nranks;
  if (rows_per_rank) *rows_per_rank = P->n1 / P->nranks;
  return 0;
}

int tilefft_dist_set_peers(tilefft_plan_t P, void* const* dest, uint32_t ndest, uint64_t row_pitch, uint64_t col_off) {
  g_err.clear();
  if (!P || !P->is_dist) return fail(TILEFFT_EINVAL, "tilefft_dist_set_peers: not a distributed plan");
  if (!dest || ndest != P->nranks) return fail(TILEFFT_EINVAL, "tilefft_dist_set_peers: need one destination per rank");
  for (uint32_t i = 0; i < ndest; ++i) {
    if (!dest[i]) return fail(TILEFFT_EINVAL, "tilefft_dist_set_peers: null destination");
    P->dist.a.peers[i] = dest[i];
  }
  P->dist.a.pitch = (long long)row_pitch;
  P->dist.a.col_off = (long long)col_off;
  P->peers_set = true;
  return 0;
}

int tilefft_dist_exec_pass1(tilefft_plan_t P, const void* d_slab, int sign, void* stream) {
  g_err.clear();
  if (!P || !P->is_dist) return fail(TILEFFT_EINVAL, "tilefft_dist_exec_pass1: not a distributed plan");
  if (!P->peers_set) return fail(TILEFFT_EINVAL, "tilefft_dist_exec_pass1: destinations not set");
  if (!d_slab) return fail(TILEFFT_EINVAL, "tilefft_dist_exec_pass1: null input");
  CUDA_TRY(cudaSetDevice(P->device));
  cudaStream_t st = (cudaStream_t)stream;
  const bool inv = sign == TILEFFT_INVERSE;
  if (P->elem_bytes == 8) {
    const float s = inv ? 1.0f / (float)P->n1 : 1.0f;
    return inv ? launch_dist_pass1<float, true>(P->dist, d_slab, P->tables.p, P->tables64.p, s, st)
               : launch_dist_pass1<float, false>(P->dist, d_slab, P->tables.p, P->tables64.p, s, st);
  }
  const double s = inv ? 1.0 / (double)P->n1 : 1.0;
  return inv ? launch_dist_pass1<double, true>(P->dist, d_slab, P->tables.p, P->tables64.p, s, st)
             : launch_dist_pass1<double, false>(P->dist, d_slab, P->tables.p, P->tables64.p, s, st);
}

int tilefft_dist_exec_pass2(tilefft_plan_t P, const void* d_rows, void* d_out, int sign, void* stream) {
  g_err.clear();
  if (!P || !P->is_dist) return fail(TILEFFT_EINVAL, "tilefft_dist_exec_pass2: not a distributed plan");
  return tilefft_exec_c2c(P->inner, d_rows, d_out, sign, stream);
}

int tilefft_dist_exec_pass2_blocks(tilefft_plan_t P, const void* d_recv, void* d_out, int sign, void* stream) {
  g_err.clear();
  if (!P || !P->is_dist) return fail(TILEFFT_EINVAL, "tilefft_dist_exec_pass2_blocks: not a distributed plan");
  if (!P->inner_blocks)
    return fail(TILEFFT_EINVAL, "tilefft_dist_exec_pass2_blocks: the row plan (n/N1 = %llu points) is a single pass; "
                "assemble the rows and use tilefft_dist_exec_pass2", (unsigned long long)P->n2);
  if ((uintptr_t)d_recv % 16) return fail(TILEFFT_EINVAL, "tilefft_dist_exec_pass2_blocks: input must be 16-byte aligned");
  return tilefft_exec_c2c(P->inner_blocks, d_recv, d_out, sign, stream);
}

int tilefft_dist_flag_buffer(tilefft_plan_t P, void** d_flags) {
  g_err.clear();
  if (!P || !P->is_dist) return fail(TILEFFT_EINVAL, "tilefft_dist_flag_buffer: not a distributed plan");
  if (!d_flags) return fail(TILEFFT_EINVAL, "tilefft_dist_flag_buffer: null output");
  *d_flags = P->flags.p;
  return 0;
}

int tilefft_dist_set_flags(tilefft_plan_t P, void* const* flags, uint32_t n) {
  g_err.clear();
  if (!P || !P->is_dist) return fail(TILEFFT_EINVAL, "tilefft_dist_set_flags: not a distributed plan");
  if (!flags || n != P->nranks) return fail(TILEFFT_EINVAL, "tilefft_dist_set_flags: need one flag buffer per rank");
  for (uint32_t i = 0; i < n; ++i) {
    if (!flags[i]) return fail(TILEFFT_EINVAL, "tilefft_dist_set_flags: null flag buffer");
    P->peer_flags[i] = static_cast<unsigned*>(flags[i]);
  }
  if (flags[P->rank] != P->flags.p)
    return fail(TILEFFT_EINVAL, "tilefft_dist_set_flags: entry %u must be this rank's own flag buffer", P->rank);
  P->flags_set = true;
  return 0;
}

int tilefft_dist_exec(tilefft_plan_t P, const void* d_slab, void* d_out, int sign, void* stream) {
  g_err.clear();
  if (!P || !P->is_dist) return fail(TILEFFT_EINVAL, "tilefft_dist_exec: not a distributed plan");
  if (!P->flags_set) return fail(TILEFFT_EINVAL, "tilefft_dist_exec: barrier flags not set");
  if (!d_out) return fail(TILEFFT_EINVAL, "tilefft_dist_exec: null output");
  if (int rc = tilefft_dist_exec_pass1(P, d_slab, sign, stream)) return rc;
  DistFlags f{};
  for (uint32_t i = 0; i < P->nranks; ++i) f.peer[i] = P->peer_flags[i];
  f.mine = static_cast<unsigned*>(P->flags.p);
  f.epoch = f.mine + 1;
  f.n = (int)P->nranks;
  k_dist_barrier<<<1, 32, 0, (cudaStream_t)stream>>>(f);
  CUDA_TRY(cudaGetLastError());
  return tilefft_exec_c2c(P->inner, P->dist.a.peers[P->rank], d_out, sign, stream);
}

namespace {
// base of the device allocation holding p (CUDA IPC handles name whole
// allocations; a caching allocator hands out pointers inside them)
int alloc_base(const void* p, char** base) {
  using Fn = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
  static Fn fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    return reinterpret_cast<Fn>(f);
  }();
  if (!fn) return fail(TILEFFT_ECUDA, "cuMemGetAddressRange unavailable");
  CUdeviceptr b = 0;
  size_t sz = 0;
  if (fn(&b, &sz, (CUdeviceptr)(uintptr_t)p) != CUDA_SUCCESS)
    return fail(TILEFFT_EINVAL, "not a device allocation: %p", p);
  *base = reinterpret_cast<char*>((uintptr_t)b);
  return 0;
}
}  // namespace

int tilefft_ipc_get_handle(const void* dptr, void* handle_out, uint64_t* offset_out) {
  g_err.clear();
  if (!dptr || !handle_out) return fail(TILEFFT_EINVAL, "tilefft_ipc_get_handle: null argument");
  char* base = nullptr;
  if (int rc = alloc_base(dptr, &base)) return rc;
  cudaIpcMemHandle_t h;
  CUDA_TRY(cudaIpcGetMemHandle(&h, base));
  std::memcpy(handle_out, &h, sizeof h);
  if (offset_out) *offset_out = (uint64_t)(static_cast<const char*>(dptr) - base);
  return 0;
}

int tilefft_ipc_open_handle(const void* handle, uint64_t offset, void** dptr) {
  g_err.clear();
  if (!handle || !dptr) return fail(TILEFFT_EINVAL, "tilefft_ipc_open_handle: null argument");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof h);
  void* base = nullptr;
  CUDA_TRY(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess));
  *dptr = static_cast<char*>(base) + offset;
  return 0;
}

int tilefft_ipc_close_handle(void* dptr) {
  g_err.clear();
  char* base = nullptr;
  if (int rc = alloc_base(dptr, &base)) return rc;
  CUDA_TRY(cudaIpcCloseMemHandle(base));
  return 0;
}

int tilefft_plan_destroy(tilefft_plan_t P) {
  if (P) {
    cudaSetDevice(P->device);
    delete P;
  }
  return 0;
}

int tilefft_plan_info(tilefft_plan_t P, tilefft_plan_info_t* info) {
  if (!P || !info) return fail(TILEFFT_EINVAL, "tilefft_plan_info: null argument");
  std::memset(info, 0, sizeof(*info));
  info->n = P->n;
  info->batch = P->batch;
  info->ny = P->ny;
  info->nx = P->nx;
  info->elem_bytes = P->elem_bytes;
  info->mode = P->mode;
  info->is_2d = P->is2d;
  info->passes = (uint32_t)P->passes.size();
  info->launches_per_exec = (uint32_t)P->passes.size();
  if (P->is_dist) {  // pass 1 (+ the barrier kernel of tilefft_dist_exec) + the local row plan
    info->passes = 1 + (uint32_t)(P->inner ? P->inner->passes.size() : 0);
    info->launches_per_exec = info->passes + 1;
  }
  for (size_t i = 0; i < P->dev_factors.size() && i < 16; ++i) info->factors[i] = P->dev_factors[i];
  info->workspace_bytes = P->work.bytes + P->work2.bytes;
  info->table_bytes = P->tables.bytes;
  return 0;
}

}  // extern "C"
