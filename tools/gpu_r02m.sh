#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
for fs in 64 16 32 128; do
  for st in 256 192 384; do
    echo "FIRST_SUB=$fs SUB_TARGET=$st: $(FW2V_FIRST_SUB=$fs FW2V_SUB_TARGET=$st python tools/e2e_gap_probe.py 2>/dev/null | grep 'epoch 3')"
  done
done
