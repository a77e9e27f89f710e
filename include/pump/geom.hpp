// Drop-in for the reference header pump/geom.hpp (see pump_gpu.hpp).
#pragma once
#include "pump/pump_gpu.hpp"
