#!/bin/bash
# A/B of cg_fused switches on the C4 probe (width 70): prints us/launch per variant
cd "$(dirname "$0")/../.."
run() {
  out=$(env "$@" python scripts/probe.py --config C4 --width 70 --iters 40 --reps 2 2>&1 | grep "cg_fused " | tail -1)
  echo "$* :: $out"
}
run ROMDOT_FUSED_RELBATCH=0
run ROMDOT_FUSED_RELBATCH=1
run ROMDOT_FUSED_RELBATCH=1 ROMDOT_FUSED_SLACK=10
run ROMDOT_FUSED_RELBATCH=1 ROMDOT_FUSED_SLACK=14
run ROMDOT_FUSED_RELBATCH=1 ROMDOT_FUSED_POLL_NS=1000
run ROMDOT_FUSED_RELBATCH=1 ROMDOT_FUSED_POLL_NS=500
run ROMDOT_FUSED_RELBATCH=1 ROMDOT_FUSED_REL_NS=64
run ROMDOT_FUSED_RELBATCH=1 ROMDOT_FUSED_SLACK=10 ROMDOT_FUSED_POLL_NS=1000
