#!/bin/bash
# A/B of cg_fused switches on the C4 probe (width 70): prints us/launch per variant
cd "$(dirname "$0")/../.."
run() {
  out=$(env "$@" python scripts/probe.py --config C4 --width ${WIDTH:-70} --iters 40 --reps 2 2>&1 | grep "cg_fused " | tail -1)
  echo "$* :: $out"
}
if [ -n "$1" ]; then for v in "$@"; do run $v; done; exit 0; fi
run ROMDOT_FUSED_TILEFLAGS=0
run ROMDOT_FUSED_TILEFLAGS=1
run ROMDOT_FUSED_TILEFLAGS=1 ROMDOT_FUSED_POLL_NS=1000
run ROMDOT_FUSED_TILEFLAGS=1 ROMDOT_FUSED_POLL_NS=500
run ROMDOT_FUSED_TILEFLAGS=1 ROMDOT_FUSED_SLACK=5
run ROMDOT_FUSED_TILEFLAGS=1 ROMDOT_FUSED_SLACK=9
run ROMDOT_FUSED_TILEFLAGS=0 ROMDOT_FUSED_SLACK=5
