#!/bin/bash
cd $GRAFT_REPO_ROOT
STEPS=${STEPS:-5}
for b in "$@"; do timeout 120 ./build/kbench_$b $STEPS 16; done
