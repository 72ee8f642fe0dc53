#!/bin/bash
mkdir -p gpurun_out
python tools/ab_env.py c3_gmm10k 2 - PINS_STALE_MAX=0 PINS_STALE_ITS=2 PINS_STALE_ITS=8,PINS_STALE_MAX=64 PINS_SPLIT_F=4.8 PINS_SPLIT_F=9.6 PINS_SPLIT_F=14.4 > gpurun_out/ab_r2c.log 2>&1
cat gpurun_out/ab_r2c.log | cut -c1-400
