#!/bin/bash
# A/B of the team QRCP engine: C5 / C4 CALU_PRRP and C2 LU_PRRP with PRRP_TEAM=0 (old engines) vs default
for v in 0 1; do
  echo "== PRRP_TEAM=$v"
  PRRP_TEAM=$v python tools/run_calu.py --n 32768 --b 128 --urand --reps 3 2>&1 | tail -1
  PRRP_TEAM=$v python tools/run_calu.py --n 16384 --b 64 --reps 3 2>&1 | tail -1
  PRRP_TEAM=$v python tools/run_lu.py --n 8192 --b 64 --reps 4 2>&1 | tail -1
  PRRP_TEAM=$v python tools/run_lu.py --n 8192 --b 128 --reps 4 2>&1 | tail -1
done
