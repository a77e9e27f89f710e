// Drop-in for the reference header pump/compare.hpp (see pump_gpu.hpp).
#pragma once
#include "pump/pump_gpu.hpp"
