// Drop-in for the reference header pump/rng.hpp (see pump_gpu.hpp).
#pragma once
#include "pump/pump_gpu.hpp"
