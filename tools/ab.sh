#!/bin/bash
# A/B the library variants under _variants/*.so on the c2 bench (no extras):
#   bash tools/ab.sh [STEPS] [ROUNDS]   (on the GPU box)
steps=${1:-30}; rounds=${2:-2}
for r in $(seq $rounds); do
for lib in _variants/*.so; do
  envf=${lib%.so}.env; extra=""; [ -f $envf ] && extra=$(cat $envf)  # optional per-variant env (VAR=val ...)
  env $extra HGS_LIB=$lib python bench.py --no-extras --no-cpu-baseline --steps $steps --warmup 5 > gpurun_out/ab.json 2>/dev/null
  python -c "
import json,sys; d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1])
ph=' '.join(f\"{k['phase']}={k['ms_per_step']:.4f}\" for k in d['roofline']['kernels'])
print('$lib', 'views/s', d['value'], 'e2e', d['e2e']['value'], 'render', d['render']['value'], 'fix', d['render_info']['fixup_pixels'], ph)"
done; done
