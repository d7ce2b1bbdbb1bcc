#!/bin/bash
# Per-phase ms of each _variants/*.so at one config: bash tools/ab_phase.sh CFG [PHASE_REGEX]
cfg=${1:-c5}; pat=${2:-.}
for lib in _variants/*.so; do
  echo "== $lib"
  envf=${lib%.so}.env; extra=""; [ -f $envf ] && extra=$(cat $envf)
  env $extra HGS_LIB=$lib CFG=$cfg VIEWS=1 STEPS=4 python tools/phase_cfg.py 2>&1 | grep -E "$pat"
done
