// Compile-time dimension dispatch: (d, dw) in {(1,1), (2,1), (4,2), (6,3)}.
// (1,1) is the reference's scalar test setup (test_cp.cpp:13-31); the others
// are the per-axis double integrator in 1, 2 and 3 workspace dimensions.
#pragma once

#include <cstring>
#include <stdexcept>

#include "dev.cuh"
#include "kernels.h"

namespace pumpg {

template <int D, int DW>
LoopP<D, DW> make_loop(const HostLoop& L) {
  LoopP<D, DW> p;
  std::memcpy(p.F, L.F.data(), sizeof(p.F));
  std::memcpy(p.Gv, L.Gv.data(), sizeof(p.Gv));
  std::memcpy(p.Gw, L.Gw.data(), sizeof(p.Gw));
  std::memcpy(p.Sv, L.Sv.data(), sizeof(p.Sv));
  std::memcpy(p.Sw, L.Sw.data(), sizeof(p.Sw));
  std::memcpy(p.S0, L.S0.data(), sizeof(p.S0));
  std::memcpy(p.C, L.C.data(), sizeof(p.C));
  return p;
}

// f.template operator()<D, DW>() for the supported pair.
template <class Fn>
void dispatch_dims(int d, int dw, Fn&& f) {
  if (dw == 1 && d == 1) return f.template operator()<1, 1>();
  if (dw == 1 && d == 2) return f.template operator()<2, 1>();
  if (dw == 2 && d == 4) return f.template operator()<4, 2>();
  if (dw == 3 && d == 6) return f.template operator()<6, 3>();
  throw std::invalid_argument("pump_gpu: unsupported (state, workspace) dimensions (" + std::to_string(d) + ", " +
                              std::to_string(dw) + "); supported: (1,1), (2,1), (4,2), (6,3)");
}

template <class Fn>
void dispatch_dw(int dw, Fn&& f) {
  if (dw == 1) return f.template operator()<1>();
  if (dw == 2) return f.template operator()<2>();
  if (dw == 3) return f.template operator()<3>();
  throw std::invalid_argument("pump_gpu: unsupported workspace dimension " + std::to_string(dw) +
                              " (supported: 1, 2, 3)");
}

inline unsigned grid_for(int64_t n, int block) { return static_cast<unsigned>((n + block - 1) / block); }

}  // namespace pumpg
