// status.hpp — no exception crosses the C ABI: entry points run their body
// inside cav::guarded(), which maps the reference's exception taxonomy
// (std::invalid_argument, std::runtime_error, std::logic_error,
// std::length_error, transport timeouts) onto int status codes and keeps the
// message in a thread-local buffer for cav_last_error().
#pragma once

#include <cstdio>
#include <stdexcept>
#include <string>

#include "cavity_b200.h"

namespace cav {

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct Timeout : std::runtime_error {
  using std::runtime_error::runtime_error;
};

void set_last_error(const std::string& msg);

template <typename Fn>
int guarded(Fn&& fn) {
  try {
    fn();
    return CAV_OK;
  } catch (const CudaError& e) {
    set_last_error(e.what());
    return CAV_ECUDA;
  } catch (const Timeout& e) {
    set_last_error(e.what());
    return CAV_ETIMEOUT;
  } catch (const std::invalid_argument& e) {
    set_last_error(e.what());
    return CAV_EINVAL;
  } catch (const std::length_error& e) {
    set_last_error(e.what());
    return CAV_ELENGTH;
  } catch (const std::logic_error& e) {
    set_last_error(e.what());
    return CAV_ELOGIC;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return CAV_ERUNTIME;
  } catch (...) {
    set_last_error("unknown error");
    return CAV_ERUNTIME;
  }
}

}  // namespace cav

#define CAV_CUDA(call)                                                                   \
  do {                                                                                   \
    cudaError_t e_ = (call);                                                             \
    if (e_ != cudaSuccess) {                                                             \
      throw ::cav::CudaError(std::string("CUDA error ") + cudaGetErrorString(e_) + " at " + \
                             __FILE__ + ":" + std::to_string(__LINE__) + " (" #call ")"); \
    }                                                                                    \
  } while (0)
