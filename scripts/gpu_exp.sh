#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python scripts/hbm_probe.py
for DBG in 0 1 2; do
LL_AUG_DEBUG=$DBG timeout 600 python scripts/aug_experiments.py > gpurun_out/exp_dbg$DBG.log 2>&1; echo "dbg $DBG rc=$?"; tail -1 gpurun_out/exp_dbg$DBG.log
done
