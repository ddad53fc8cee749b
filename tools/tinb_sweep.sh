#!/bin/bash
# time-index bucket sweep for big jobs (dev tool): C4 kernel time per TSL_TI_NB
for nb in 256 2048 16384 131072; do
  echo "TSL_TI_NB=$nb"; TSL_TI_NB=$nb python tools/inc_profile.py 2>&1 | head -1
done
