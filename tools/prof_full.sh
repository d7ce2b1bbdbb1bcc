#!/bin/bash
# One `ncu --set full` capture per hot kernel of the c2 training step (3rd
# iteration of tools/prof_step.py), reports into gpurun_out/.
# usage (on the GPU box, after the same command ran clean without ncu):
#   python tools/prof_step.py && bash tools/prof_full.sh TAG [kernel ...]
tag=${1:-r02}
shift
ks="$*"
[ -z "$ks" ] && ks="raster_bwd_kernel raster_fwd_kernel radix_sort_coop_kernel duplicate_compact_kernel adam_rows_kernel \
         adam_classes_kernel raster_bwd_exact_kernel ssim_fwd_kernel ssim_bwd_kernel preprocess_kernel \
         gaussian_bwd_kernel sh_bwd_kernel gather_sorted_kernel compact_coop_kernel"
for k in $ks; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$k" -s 2 -c 1 -o gpurun_out/${tag}_$k \
      python tools/prof_step.py > gpurun_out/${tag}_$k.log 2>&1 || echo "failed $k"
done
ls gpurun_out/${tag}_*.ncu-rep | wc -l
