#!/bin/bash
# Config 2 heat kernel sweep (each line: scripts/probes/heat_config2.py, a
# fresh process per variant).  OFL_HEAT_KERNEL 4 = k_heat_tile (register-
# lean warp tiles), 2 = k_heat_warp (round 1); R = cells per thread;
# TBS = most steps per HBM pass.
for k in ${KERNELS:-4}; do
  for r in ${RS:-40 48 56 60}; do
    for tb in ${TBS:-64 72 80 96}; do
      OFL_HEAT_KERNEL=$k OFL_HEAT_R=$r OFL_HEAT_TB=$tb python scripts/probes/heat_config2.py 2>&1 | tail -1
    done
  done
done
