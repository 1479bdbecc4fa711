// runner.cpp — run_case / compare_fields / verify_against_serial over the
// block ABI (/root/reference/proj/src/runner.cpp:259-396). Like the
// reference, one host thread per rank; each thread owns one block on its GPU
// (cfg.devices[rank % 8]). Cross-rank traffic never touches the host: halos
// and scalars move GPU-to-GPU (peer stores, stream-ordered waits). The host
// only joins at convergence checks (to fold exact norm partials, as
// global_norms does at src/runner.cpp:81-104) and at the end.
//
// cfg.seed != 0 is the GPU analogue of the reference's randomized bus
// (src/inproc.cpp:92-114, acceptance c8): rank threads start in a seeded
// shuffled order and each block pauses at seeded random points between
// iterations, so ranks run at skewed times; results must not change.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <numeric>
#include <random>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <limits>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "cavity_b200.h"
#include "host.hpp"
#include "status.hpp"

namespace cav {
namespace {

// Barrier that fails fast once any rank has died (the InprocBus poison of
// src/inproc.cpp:16-38).
class Barrier {
 public:
  explicit Barrier(int n) : n_(n) {}
  void wait() {
    std::unique_lock<std::mutex> lk(m_);
    if (poisoned_) throw std::runtime_error("transport aborted by rank " + std::to_string(who_));
    const long gen = gen_;
    if (++count_ == n_) {
      count_ = 0;
      ++gen_;
      cv_.notify_all();
      return;
    }
    cv_.wait(lk, [&] { return gen_ != gen || poisoned_; });
    if (gen_ == gen && poisoned_) throw std::runtime_error("transport aborted by rank " + std::to_string(who_));
  }
  void poison(int rank) {
    std::lock_guard<std::mutex> lk(m_);
    if (!poisoned_) who_ = rank;
    poisoned_ = true;
    cv_.notify_all();
  }

 private:
  std::mutex m_;
  std::condition_variable cv_;
  int n_, count_ = 0, who_ = -1;
  long gen_ = 0;
  bool poisoned_ = false;
};

void check(int st) {
  if (st == CAV_OK) return;
  const std::string msg = cav_last_error();
  switch (st) {
    case CAV_EINVAL: throw std::invalid_argument(msg);
    case CAV_ELOGIC: throw std::logic_error(msg);
    case CAV_ELENGTH: throw std::length_error(msg);
    case CAV_ECUDA: throw CudaError(msg);
    case CAV_ETIMEOUT: throw Timeout(msg);
    default: throw std::runtime_error(msg);
  }
}

struct Shared {
  const cav_run_config* cfg;
  const cav_case_options* opt;
  std::array<int, 3> gn, dims;
  std::vector<host::Extent> ext;
  int np;
  Barrier bar;
  std::vector<cav_block*> blocks;
  std::vector<void*> arenas;
  std::vector<std::exception_ptr> errors;
  std::vector<double> seconds;
  std::vector<cav_ledger> ledgers;
  std::vector<std::vector<uint64_t>> digits;  // per rank, current segment (CAV_NORM_WORDS per check)
  std::vector<long long> check_iters;
  // rank 0 owned results
  long long marched = 0;
  bool converged = false;
  bool stop = false;
  std::vector<long long> hist_it;
  std::vector<std::array<double, 5>> hist;
  std::vector<std::array<double, 5>> hist_linf;
  std::array<double, 5> peaks{};
  double* fields = nullptr;

  Shared(const cav_run_config* c, const cav_case_options* o, int n)
      : cfg(c), opt(o), np(n), bar(n), blocks(n, nullptr), arenas(n, nullptr), errors(n), seconds(n, 0.0),
        ledgers(n), digits(n) {}
};

// Folds one segment's exact partials of every rank (global_norms,
// src/runner.cpp:81-104) and applies the convergence rule (:210-220).
void fold_norms(Shared& sh, long long n_checks) {
  const long long nglobal = static_cast<long long>(sh.gn[0]) * sh.gn[1] * sh.gn[2];
  const bool fixed = sh.cfg->steps >= 0;
  for (long long c = 0; c < n_checks; ++c) {
    std::array<double, 5> l2{};
    std::array<double, 5> linf{};
    for (int v = 0; v < 5; ++v) {
      uint64_t total[70] = {};
      uint64_t mx = 0;
      for (int r = 0; r < sh.np; ++r) {
        const uint64_t* w = sh.digits[r].data() + c * CAV_NORM_WORDS;
        uint64_t limbs[70];
        host::digits_to_limbs(w + v * 70, limbs);
        host::repro_merge(total, limbs);
        mx = std::max(mx, w[5 * 70 + v]);  // L-inf: exact max of |R| bit patterns
      }
      l2[v] = std::sqrt(host::repro_value(total) / static_cast<double>(nglobal));
      std::memcpy(&linf[v], &mx, sizeof mx);
    }
    const long long it = sh.check_iters[c];
    sh.hist_it.push_back(it);
    sh.hist.push_back(l2);
    sh.hist_linf.push_back(linf);
    if (sh.cfg->monitor_every > 0 && it % sh.cfg->monitor_every == 0)
      std::printf("iter %8lld  |R|: p=%.3e u=%.3e v=%.3e w=%.3e T=%.3e\n", it, l2[0], l2[1], l2[2], l2[3], l2[4]);
    if (!fixed) {
      double worst = 0.0;
      for (int v = 0; v < 5; ++v) {
        sh.peaks[v] = std::max(sh.peaks[v], l2[v]);
        if (sh.peaks[v] > 0.0) worst = std::max(worst, l2[v] / sh.peaks[v]);
      }
      sh.converged = worst <= sh.cfg->conv_tol;
    }
  }
}

void rank_main(Shared& sh, int rank) {
  const cav_run_config& cfg = *sh.cfg;
  cav_block_desc d{};
  d.rank = rank;
  d.np = sh.np;
  d.gnx = sh.gn[0];
  d.gny = sh.gn[1];
  d.gnz = sh.gn[2];
  for (int a = 0; a < 3; ++a) d.dims[a] = sh.dims[a];
  d.strategy = cfg.strategy;
  d.overlap = cfg.overlap;
  d.fluid = cfg.fluid;
  d.cfl = cfg.cfl;
  d.rescale = cfg.rescale;
  d.corrupt_exchange = sh.opt->corrupt_exchange;
  d.device = cfg.devices[rank % 8];
  d.timeout_ms = cfg.timeout_ms > 0 ? cfg.timeout_ms : 20000.0;
  d.jitter_seed = cfg.seed;
  cav_block* b = nullptr;
  check(cav_block_create(&d, &b));
  sh.blocks[rank] = b;
  size_t bytes = 0;
  check(cav_block_arena(b, &sh.arenas[rank], &bytes));
  sh.bar.wait();
  for (int r = 0; r < sh.np; ++r)
    if (r != rank) check(cav_block_connect(b, r, sh.arenas[r], nullptr));
  check(cav_block_initialize(b));
  sh.bar.wait();

  const bool fixed = cfg.steps >= 0;
  const long long target = fixed ? cfg.steps : cfg.max_steps;
  const int cadence = std::max(1, cfg.check_every);
  const bool want_hist = sh.opt->collect_history || cfg.monitor_every > 0;
  const bool norms = !fixed || want_hist;
  cav_run_io io{};
  double seconds = 0.0;
  long long it = 1;
  // The convergence rule runs on the device after every check (several
  // ranks: on every rank, over every rank's exact digits, pushed GPU to GPU),
  // so a segment can span many checks without a host round trip; the segment
  // stops where the run converged. The host folds the segment's partials for
  // the history afterwards (the same digits, the same decision).
  bool dconv = !fixed;  // confirmed by the block after the first (1-iteration) segment
  double conv_peaks[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
  while (it <= target) {
    long long end = target;
    if (!fixed) {
      const long long span = dconv ? 256LL * cadence : cadence;
      end = std::min(target, it == 1 ? 1 : (it + span - 1) / cadence * cadence);
    }
    const long long nits = end - it + 1;
    long long nchk = 0;
    for (long long q = it; q <= end; ++q) nchk += norms && (q == 1 || q % cadence == 0);
    std::vector<uint64_t>& dig = sh.digits[rank];
    dig.assign(static_cast<size_t>(std::max<long long>(1, nchk)) * CAV_NORM_WORDS, 0);
    std::vector<long long> citers(static_cast<size_t>(std::max<long long>(1, nchk)));
    io.first_it = it;
    io.n_its = nits;
    io.check_every = cadence;
    io.want_norms = norms;
    io.norm_digits = dig.data();
    io.check_iters = citers.data();
    io.device_conv = dconv ? 1 : 0;
    io.conv_tol = cfg.conv_tol;
    for (int v = 0; v < 5; ++v) io.conv_peaks[v] = conv_peaks[v];
    check(cav_block_run(b, &io));
    dconv = dconv && io.device_conv;
    for (int v = 0; v < 5; ++v) conv_peaks[v] = io.conv_peaks[v];
    if (io.conv_iter) end = io.conv_iter;  // the device stopped there
    seconds += io.seconds;
    if (rank == 0) sh.check_iters = citers;
    sh.bar.wait();
    if (rank == 0) {
      if (io.n_checks) fold_norms(sh, io.n_checks);
      sh.marched = end;
      sh.stop = !fixed && sh.converged;
    }
    sh.bar.wait();
    it = end + 1;
    if (sh.stop) break;
  }
  sh.seconds[rank] = seconds;
  sh.ledgers[rank] = io.ledger;

  if (sh.fields) {  // gather_fields (src/runner.cpp:106-148)
    const host::Extent& e = sh.ext[rank];
    const size_t X = e.size(0) + 4, Y = e.size(1) + 4, Z = e.size(2) + 4;
    std::vector<double> local(5 * X * Y * Z);
    check(cav_block_download(b, local.data()));
    const size_t N = static_cast<size_t>(sh.gn[0]) * sh.gn[1] * sh.gn[2];
    for (int v = 0; v < 5; ++v)
      for (int k = 0; k < e.size(2); ++k)
        for (int j = 0; j < e.size(1); ++j) {
          const double* src = local.data() + v * X * Y * Z + 2 + X * ((j + 2) + Y * (k + 2));
          double* dst = sh.fields + v * N + e.lo[0] +
                        static_cast<size_t>(sh.gn[0]) * ((e.lo[1] + j) + static_cast<size_t>(sh.gn[1]) * (e.lo[2] + k));
          std::memcpy(dst, src, e.size(0) * sizeof(double));
        }
  }
}

}  // namespace
}  // namespace cav

using namespace cav;

extern "C" {

int cav_run_case(const cav_run_config* cfg, const cav_case_options* opt, cav_case_result* out) {
  return guarded([&] {
    host::validate_params(cfg->fluid);
    if (cfg->np < 1 || cfg->np > 512) throw std::invalid_argument("run: np must be in 1..512");
    const auto dims = host::decomp_dims(cfg->np, cfg->mode, cfg->dims);
    host::cavity_spacing(cfg->nx, cfg->ny, cfg->nz, cfg->fluid.length, cfg->fluid.length, cfg->fluid.length);
    // Ranks sharing a GPU may have their streams multiplexed onto the same
    // hardware queues (CUDA_DEVICE_MAX_CONNECTIONS); blocks enqueue every
    // cross-rank wait only after its producer (HostProgress, block.cu), so
    // any mapping is deadlock-free.
    Shared sh(cfg, opt, cfg->np);
    sh.gn = {cfg->nx, cfg->ny, cfg->nz};
    sh.dims = dims;
    sh.ext = host::partition(sh.gn, dims);
    if (opt->collect_fields) sh.fields = out->fields;

    if (sh.np == 1) {
      try {
        rank_main(sh, 0);
      } catch (...) {
        sh.errors[0] = std::current_exception();
      }
    } else {
      std::vector<std::thread> threads;
      std::vector<int> order(sh.np);
      std::iota(order.begin(), order.end(), 0);
      std::mt19937_64 rng(cfg->seed);
      if (cfg->seed) std::shuffle(order.begin(), order.end(), rng);
      for (int r : order) {
        if (cfg->seed) std::this_thread::sleep_for(std::chrono::microseconds(rng() % 2000));
        threads.emplace_back([&sh, r] {
          try {
            rank_main(sh, r);
          } catch (...) {
            sh.errors[r] = std::current_exception();
            sh.bar.poison(r);
          }
        });
      }
      for (auto& t : threads) t.join();
    }
    if (std::getenv("CAV_DEBUG_DUMP")) {  // diagnostics: receive flags and scalar stamps of every rank
      for (int r = 0; r < sh.np; ++r) {
        if (!sh.blocks[r]) continue;
        std::vector<uint64_t> v(64 + 2 * sh.np + 2);
        if (cav_block_debug(sh.blocks[r], v.data(), static_cast<int>(v.size())) != CAV_OK) continue;
        std::fprintf(stderr, "rank %d flags", r);
        for (int q = 0; q < 6; ++q) std::fprintf(stderr, " %llx", (unsigned long long)v[q]);
        std::fprintf(stderr, " | stamps");
        for (int q = 0; q < 2 * sh.np; ++q) std::fprintf(stderr, " %llx", (unsigned long long)v[64 + q]);
        std::fprintf(stderr, "\n");
      }
    }
    for (auto* b : sh.blocks)
      if (b) cav_block_destroy(b);
    // prefer the root cause over "aborted by" echoes (src/runner.cpp:294-309)
    std::exception_ptr first;
    for (const auto& e : sh.errors) {
      if (!e) continue;
      if (!first) first = e;
      try {
        std::rethrow_exception(e);
      } catch (const std::exception& x) {
        if (std::string(x.what()).find("transport aborted by") == std::string::npos) {
          first = e;
          break;
        }
      }
    }
    if (first) std::rethrow_exception(first);

    out->steps_marched = sh.marched;
    out->steps_timed = std::max(0LL, sh.marched - 1);
    out->converged = sh.converged ? 1 : 0;
    out->np = sh.np;
    for (int a = 0; a < 3; ++a) out->dims[a] = dims[a];
    out->wall_time_s = *std::max_element(sh.seconds.begin(), sh.seconds.end());
    const double size = static_cast<double>(cfg->nx) * cfg->ny * cfg->nz;
    out->ssspnt = (out->steps_timed > 0 && out->wall_time_s > 0.0)
                      ? 1e-7 * size * static_cast<double>(out->steps_timed) / (sh.np * out->wall_time_s)
                      : std::numeric_limits<double>::quiet_NaN();
    out->bytes_sent = 0;
    for (int r = 0; r < sh.np; ++r) {
      out->bytes_sent += sh.ledgers[r].bytes_sent;
      if (out->ledgers && r < out->ledger_capacity) out->ledgers[r] = sh.ledgers[r];
    }
    out->hist_count = static_cast<long long>(sh.hist.size());
    for (size_t n = 0; n < sh.hist.size() && static_cast<long long>(n) < out->hist_capacity; ++n) {
      out->hist_iter[n] = sh.hist_it[n];
      for (int v = 0; v < 5; ++v) out->hist_l2[5 * n + v] = sh.hist[n][v];
      if (out->hist_linf)
        for (int v = 0; v < 5; ++v) out->hist_linf[5 * n + v] = sh.hist_linf[n][v];
    }
  });
}

}  // extern "C"
