// Exception -> status-code boundary of the C ABI (include/pump_gpu.h).
#pragma once

#include <stdexcept>
#include <string>

#include "../../include/pump_gpu.h"
#include "gpu/kernels.h"
#include "host/scenario.hpp"

namespace pumpg {

inline std::string& last_error() {
  thread_local std::string e;
  return e;
}

inline int fail(int code, const char* msg) {
  last_error() = msg;
  return code;
}

struct CapacityError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

template <class F>
int guard(F&& f) {
  try {
    last_error().clear();
    f();
    return PUMP_OK;
  } catch (const pumpb::ScenarioError& e) {
    last_error() = e.what();
    return PUMP_E_SCENARIO;
  } catch (const CudaError& e) {
    last_error() = e.what();
    return PUMP_E_CUDA;
  } catch (const CapacityError& e) {
    last_error() = e.what();
    return PUMP_E_CAPACITY;
  } catch (const std::invalid_argument& e) {
    last_error() = e.what();
    return PUMP_E_INVALID_ARGUMENT;
  } catch (const std::out_of_range& e) {
    last_error() = e.what();
    return PUMP_E_OUT_OF_RANGE;
  } catch (const std::logic_error& e) {
    last_error() = e.what();
    return PUMP_E_LOGIC;
  } catch (const std::exception& e) {
    last_error() = e.what();
    return PUMP_E_RUNTIME;
  } catch (...) {
    last_error() = "unknown error";
    return PUMP_E_RUNTIME;
  }
}

}  // namespace pumpg
