#!/bin/bash
# A/B of the gathered-GEMM cluster rule / stage budget on the in-graph step (B=64).
for cfg in "PS_GG_CLUSTER_RULE=0" "PS_GG_CLUSTER_RULE=1" "PS_GG_CLUSTER_RULE=1 PS_GG_BIGSTAGE=1"; do
  for rb in cublas native; do
    echo "== $cfg router=$rb"
    env $cfg python tools/timeline.py --batch 64 --router-backend $rb 2>&1 | grep -E "^step"
  done
done
