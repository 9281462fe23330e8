cd $GRAFT_REPO_ROOT
for cfg in "" "FW2V_DELTA_WRITEBACK=0" "FW2V_MAX_INFLIGHT=64" "FW2V_MAX_INFLIGHT=32" "FW2V_MAX_INFLIGHT=16" "FW2V_MAX_INFLIGHT=8" "FW2V_MAX_INFLIGHT=4" "FW2V_MAX_INFLIGHT=2" "FW2V_DELTA_WRITEBACK=0 FW2V_MAX_INFLIGHT=16"; do
  echo "== $cfg"
  env $cfg timeout 120 ./oracle/_ref/test_trainer_gpu 2>&1 | grep -E "rho|FAIL|test cases" 
done
