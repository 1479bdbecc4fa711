// cavity_b200.hpp — header-only C++ face of the C ABI (cavity_b200.h).
//
// Rethrows the reference's exception types with the reference's messages
// (std::invalid_argument for bad configuration, std::runtime_error with
// "iteration N: ..." for divergence, std::logic_error, std::length_error), so a
// caller of cavity::run_case (/root/reference/proj/include/cavity/runner.hpp:36)
// can switch to cavity_b200::run_case without touching its error handling.
#pragma once

#include <stdexcept>
#include <string>
#include <vector>

#include "cavity_b200.h"

namespace cavity_b200 {

struct transport_timeout : std::runtime_error {
  using std::runtime_error::runtime_error;
};

inline void check(int status) {
  if (status == CAV_OK) return;
  const std::string msg = cav_last_error();
  switch (status) {
    case CAV_EINVAL: throw std::invalid_argument(msg);
    case CAV_ELOGIC: throw std::logic_error(msg);
    case CAV_ELENGTH: throw std::length_error(msg);
    case CAV_ETIMEOUT: throw transport_timeout(msg);
    default: throw std::runtime_error(msg);
  }
}

inline cav_run_config default_config() {
  cav_run_config c;
  cav_run_config_default(&c);
  return c;
}

struct case_result {
  cav_case_result raw{};
  std::vector<double> fields;           // p,u,v,w,T over the global interior
  std::vector<long long> history_iter;  // sampled iterations
  std::vector<double> history;          // 5 norms per sample
  std::vector<cav_ledger> ledgers;      // per rank
};

// run_case (src/runner.cpp:259-338): bitwise-equal to the reference.
inline case_result run_case(const cav_run_config& cfg, bool collect_fields = false,
                            bool collect_history = false, bool corrupt_exchange = false) {
  case_result r;
  const long long target = cfg.steps >= 0 ? cfg.steps : cfg.max_steps;
  const long long cap = target / (cfg.check_every > 0 ? cfg.check_every : 1) + 2;
  r.history_iter.resize(static_cast<size_t>(cap));
  r.history.resize(static_cast<size_t>(5 * cap));
  r.ledgers.resize(static_cast<size_t>(cfg.np > 0 ? cfg.np : 1));
  if (collect_fields) r.fields.resize(static_cast<size_t>(5LL * cfg.nx * cfg.ny * cfg.nz));
  r.raw.fields = collect_fields ? r.fields.data() : nullptr;
  r.raw.hist_capacity = cap;
  r.raw.hist_iter = r.history_iter.data();
  r.raw.hist_l2 = r.history.data();
  r.raw.ledger_capacity = static_cast<int>(r.ledgers.size());
  r.raw.ledgers = r.ledgers.data();
  const cav_case_options opt{collect_fields ? 1 : 0, collect_history ? 1 : 0, corrupt_exchange ? 1 : 0};
  check(cav_run_case(&cfg, &opt, &r.raw));
  r.history_iter.resize(static_cast<size_t>(r.raw.hist_count));
  r.history.resize(static_cast<size_t>(5 * r.raw.hist_count));
  return r;
}

}  // namespace cavity_b200
