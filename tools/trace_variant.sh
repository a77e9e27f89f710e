PUMP_DEBUG_TIMING=1 python tools/probe_variant.py forest10_n16000_N128 > gpurun_out/tr10.log 2>&1
PUMP_DEBUG_TIMING=1 python tools/probe_variant.py forest10_n16000_N128 >> gpurun_out/tr10.log 2>&1
