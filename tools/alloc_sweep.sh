#!/bin/bash
# alloc_class time per config for forced cluster sizes (ABCS_ALLOC_CLUSTER)
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
for cs in 1 2 4 8 16 auto; do
  if [ "$cs" = auto ]; then unset ABCS_ALLOC_CLUSTER; else export ABCS_ALLOC_CLUSTER=$cs; fi
  echo "cs=$cs $(python tools/kt_cfg.py 3 4 5 | python -c "import json,sys; d=json.load(sys.stdin); print({c: v['alloc_class']['ms_per_call'] for c, v in d.items()})")"
done
