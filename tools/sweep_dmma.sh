#!/bin/bash
# time the DMMA operator variants (SEM_DMMA_VARIANT) on config 3 (p=5) and config-4 orders
for v in 0 1 2 3 4; do SEM_DMMA_VARIANT=$v python tools/time_apply.py --config config3 --reps 20 2>&1 | head -1 | sed "s/^/v$v /"; done
