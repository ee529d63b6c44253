// Cost-model tests (host only, no GPU): the reference's own cases for the
// request primitives, the recorder and the closed-form accounting
// (/root/reference/proj/tests/test_exec_model.cpp:47-200,
// test_memsim.cpp:47-220, acceptance criterion 5 acceptance_main.cpp:197-234)
// re-run against include/tilefft/{exec_model,access_patterns,memsim}.hpp.
//
//   test_costmodel            run the cases; exit code = failures
//   test_costmodel dump N CAP print account_tiled(make_plan(N, CAP)) and
//                             account_levelwise(N) as two lines of 7 counters
//                             (tests/test_costmodel.py compares them with the
//                             reference compiled from its headers)
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <numeric>
#include <stdexcept>
#include <string>
#include <vector>

#include "tilefft/memsim.hpp"

namespace {
int g_fail = 0, g_checks = 0;
std::string g_case;
#define CHECK(cond)                                                                     \
  do {                                                                                  \
    ++g_checks;                                                                         \
    if (!(cond)) {                                                                      \
      ++g_fail;                                                                         \
      std::printf("FAIL [%s] %s:%d: %s\n", g_case.c_str(), __FILE__, __LINE__, #cond); \
    }                                                                                   \
  } while (0)
#define CHECK_THROWS(expr)            \
  do {                                \
    bool thrown_ = false;             \
    try {                             \
      (void)(expr);                   \
    } catch (const std::invalid_argument&) { \
      thrown_ = true;                 \
    }                                 \
    CHECK(thrown_ && #expr);          \
  } while (0)

void run(const char* name, const std::function<void()>& f) {
  g_case = name;
  try {
    f();
  } catch (const std::exception& e) {
    ++g_fail;
    std::printf("FAIL [%s] exception: %s\n", name, e.what());
  }
}

void print(const tilefft::AccessStats& s) {
  std::printf("%llu %llu %llu %llu %llu %llu %llu\n", (unsigned long long)s.slow_elem_reads,
              (unsigned long long)s.slow_elem_writes, (unsigned long long)s.slow_transactions,
              (unsigned long long)s.fast_accesses, (unsigned long long)s.bank_conflict_cycles,
              (unsigned long long)s.barriers, (unsigned long long)s.twiddle_fetches);
}
}  // namespace

int main(int argc, char** argv) {
  using namespace tilefft;
  if (argc == 4 && std::strcmp(argv[1], "dump") == 0) {
    const std::size_t n = std::strtoull(argv[2], nullptr, 10), cap = std::strtoull(argv[3], nullptr, 10);
    print(account_tiled(make_plan(n, cap)));
    print(account_levelwise(n));
    return 0;
  }
  using V = std::vector<std::uint64_t>;

  run("coalesced_transactions: canonical shapes (test_exec_model.cpp:47-74)", [] {
    V contiguous(32);
    std::iota(contiguous.begin(), contiguous.end(), 0);
    CHECK(coalesced_transactions(contiguous) == 4);
    CHECK(coalesced_transactions(V{}) == 0);
    CHECK(coalesced_transactions(V{5}) == 1);
    CHECK(coalesced_transactions(V(32, 7)) == 1);
    V s2(32), s8(32), off(32);
    for (std::size_t i = 0; i < 32; ++i) {
      s2[i] = 2 * i;
      s8[i] = 8 * i;
      off[i] = 4 + i;
    }
    CHECK(coalesced_transactions(s2) == 8);
    CHECK(coalesced_transactions(s8) == 32);
    CHECK(coalesced_transactions(off) == 5);
    CHECK_THROWS(coalesced_transactions(V(33, 0)));
  });

  run("bank_conflict_degree: canonical shapes (test_exec_model.cpp:76-114)", [] {
    V distinct(16);
    std::iota(distinct.begin(), distinct.end(), 0);
    CHECK(bank_conflict_degree(distinct) == 1);
    CHECK(bank_conflict_degree(V{}) == 0);
    CHECK(bank_conflict_degree(V{3}) == 1);
    CHECK(bank_conflict_degree(V(16, 42)) == 1);
    CHECK(bank_conflict_degree(V{0, 16}) == 2);
    V s16(16), s33(16);
    for (std::size_t i = 0; i < 16; ++i) {
      s16[i] = 16 * i;
      s33[i] = 33 * i;
    }
    CHECK(bank_conflict_degree(s16) == 16);
    CHECK(bank_conflict_degree(s33) == 1);
    CHECK(bank_conflict_degree(V{0, 16, 1, 1}) == 2);
    CHECK_THROWS(bank_conflict_degree(V(17, 0)));
    ExecConfig c32;
    c32.bank_count = 32;
    c32.word_bytes = 4;
    CHECK(bank_conflict_degree(s16, c32) == 8);
  });

  run("AccessRecorder: request recording (test_exec_model.cpp:173-200)", [] {
    AccessRecorder rec;
    rec.begin_stage();
    V contiguous(32);
    std::iota(contiguous.begin(), contiguous.end(), 0);
    rec.record_slow_request(contiguous);
    CHECK(rec.stage(1).slow_transactions == 4);
    V clean(16);
    std::iota(clean.begin(), clean.end(), 0);
    rec.record_fast_request(clean);
    CHECK(rec.stage(1).bank_conflict_cycles == 0);
    rec.record_fast_request(V{0, 16});
    CHECK(rec.stage(1).bank_conflict_cycles == 1);
    rec.record_fast_request_repeated(V{0, 16, 32}, 5);
    CHECK(rec.stage(1).bank_conflict_cycles == 1 + 5 * 2);
    ExecConfig small;
    small.warp_size = 8;
    small.half_warp_size = 4;
    AccessRecorder r2(small);
    r2.begin_stage();
    CHECK_THROWS(r2.record_slow_request(V(9, 0)));
  });

  run("account_levelwise closed forms (test_memsim.cpp:47-70)", [] {
    const AccessStats s = account_levelwise(1024);
    CHECK(s.slow_elem_reads == 10240 && s.slow_elem_writes == 10240 && s.barriers == 10);
    CHECK(s.twiddle_fetches == 5120 && s.fast_accesses == 0 && s.bank_conflict_cycles == 0);
    const AccessStats t = account_levelwise(2);
    CHECK(t.slow_elem_reads == 2 && t.barriers == 1 && t.twiddle_fetches == 1 && t.slow_transactions == 4);
    CHECK_THROWS(account_levelwise(0));
    CHECK_THROWS(account_levelwise(96));
  });

  run("account_tiled closed forms (test_memsim.cpp:72-95)", [] {
    const AccessStats a = account_tiled(make_plan(1024, 1024));
    CHECK(a.slow_elem_reads == 1024 && a.slow_elem_writes == 1024 && a.barriers == 1);
    CHECK(a.twiddle_fetches == 1023 && a.fast_accesses == 1024 * 22 && a.bank_conflict_cycles == 0);
    const AccessStats b = account_tiled(make_plan(65536, 1024));
    CHECK(b.slow_elem_reads == 2 * 65536 && b.barriers == 2);
    CHECK(b.twiddle_fetches == 64 * 255 + 65536 + 64 * 255);
    CHECK(b.fast_accesses == 2 * 65536ull * 18 && b.bank_conflict_cycles == 0);
    ExecConfig other;
    other.bank_count = 32;
    CHECK_THROWS(account_tiled(make_plan(1024), other));
  });

  run("traffic law and reduction ratio (test_memsim.cpp:133-141, 197-203)", [] {
    for (std::size_t bits = 1; bits <= 16; ++bits) {
      const std::size_t n = std::size_t{1} << bits;
      const StagePlan plan = make_plan(n);
      CHECK(account_levelwise(n).slow_elem_accesses() == 2 * n * bits);
      CHECK(account_tiled(plan).slow_elem_accesses() == 2 * n * plan.pass_count());
    }
    CHECK(reduction_ratio(4096, make_plan(4096)) == 6.0);
    CHECK(reduction_ratio(65536, make_plan(65536)) == 8.0);
    CHECK(reduction_ratio(64, make_plan(64, 4)) == 2.0);
    CHECK_THROWS(reduction_ratio(2048, make_plan(1024)));
  });

  run("criterion 5: padded strides conflict free, raw strides 16-way (acceptance_main.cpp:197-234)", [] {
    const ExecConfig cfg;
    bool padded_ok = true, raw_ok = true;
    std::size_t raw_groups = 0;
    for (std::size_t n = 2; n <= 65536; n *= 2) {
      const StagePlan plan = make_plan(n);
      for (std::size_t s = 1; s <= plan.pass_count(); ++s) {
        const StageGeometry& g = plan.stage(s);
        detail::for_each_column_stream(g.rows, g.fft_len, g.padded_stride, cfg, [&](std::span<const std::uint64_t> w) {
          padded_ok = padded_ok && bank_conflict_degree(w, cfg) == 1;
        });
        if (g.fft_len % cfg.bank_count == 0)
          detail::for_each_column_stream(g.rows, g.fft_len, g.fft_len, cfg, [&](std::span<const std::uint64_t> w) {
            if (w.size() == cfg.half_warp_size) {
              ++raw_groups;
              raw_ok = raw_ok && bank_conflict_degree(w, cfg) == cfg.bank_count;
            }
          });
      }
    }
    CHECK(padded_ok && raw_ok && raw_groups > 0);
  });

  run("conflict cycles appear once the pad is stripped (test_memsim.cpp:174-195)", [] {
    StagePlan raw = make_plan(65536, 1024);
    for (auto& g : raw.stages) g.padded_stride = g.fft_len;
    CHECK(account_tiled(make_plan(65536, 1024)).bank_conflict_cycles == 0);
    std::uint64_t want = 0;
    for (std::size_t s = 1; s <= raw.pass_count(); ++s)
      want += (raw.stage(s).rows / 16) * raw.stage(s).fft_len * 15 * detail::column_stream_occasions(raw, s);
    CHECK(account_tiled(raw).bank_conflict_cycles == want);
  });

  run("twiddle fetch economy (test_memsim.cpp:212-220)", [] {
    for (std::size_t n : {4096ul, 65536ul}) CHECK(account_tiled(make_plan(n)).twiddle_fetches < account_levelwise(n).twiddle_fetches / 4);
  });

  std::printf("%d checks, %d failures\n", g_checks, g_fail);
  return g_fail;
}
