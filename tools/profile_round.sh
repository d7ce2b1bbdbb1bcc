#!/bin/bash
# Full evidence pass for the judged profiles (on the GPU box):
#   bash tools/profile_round.sh TAG
# bench line, timed-region launch list, pair counts (checked build), one
# `ncu --set full` capture per hot kernel; then tools/make_profiles.py here.
tag=${1:-r02}
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err; echo "bench rc $?"
timeout 600 ncu --nvtx --nvtx-include timed/ --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/${tag}_launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-extras \
  > gpurun_out/${tag}_ncu_launch.log 2>&1; echo "launches rc $?"
HGS_LIB=paper_2505_13215_b200/libhgs_gpu_checked.so timeout 600 python tools/count_pairs.py $tag > gpurun_out/${tag}_pairs.log 2>&1
echo "pairs rc $?"; cp profiles/${tag}_pairs.json gpurun_out/ 2>/dev/null
python tools/prof_step.py > /dev/null 2>&1 && bash tools/prof_full.sh $tag raster_bwd_kernel raster_fwd_kernel preprocess_kernel \
  radix_sort_coop_kernel duplicate_compact_kernel gaussian_bwd_kernel adam_rows_kernel ssim_fwd_kernel ssim_bwd_kernel \
  sh_bwd_kernel adam_classes_kernel gather_sorted_kernel
