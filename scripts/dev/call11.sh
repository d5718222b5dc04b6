set -x
N=/usr/local/cuda/bin/ncu
$N --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none -c 40000 --csv --log-file gpurun_out/t11_launches.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-configs --no-cpu --no-fp64 > gpurun_out/t11_ncu_bench.log 2>&1
$N --set full --clock-control none --import-source on -k regex:stencil_tma -s 2 -c 1 -o gpurun_out/r02_stencil_tma_c4_768 python scripts/dev/ncu_targets.py stencil > gpurun_out/t11_ncu_st.log 2>&1
$N --set full --clock-control none --import-source on -k regex:gram_kernel -s 1 -c 1 -o gpurun_out/r02_gram_c128_768 python scripts/dev/ncu_targets.py gram > gpurun_out/t11_ncu_gram.log 2>&1
$N --set full --clock-control none --import-source on -k regex:gemm_tall_dmma -s 1 -c 1 -o gpurun_out/r02_gemm_c128_768 python scripts/dev/ncu_targets.py gemm > gpurun_out/t11_ncu_gemm.log 2>&1
$N --set full --clock-control none --import-source on -k regex:cg_fused -s 20 -c 1 -o gpurun_out/r02_cg_fused_c70 python scripts/probe.py --config C4 --width 70 --iters 40 --reps 1 > gpurun_out/t11_ncu_fused.log 2>&1
python scripts/cpu_builds.py --configs C1 --threads 1,16 > gpurun_out/t11_cpu_builds.jsonl 2> gpurun_out/t11_cpu_builds.err
python scripts/cpu_builds.py --configs C3 --threads 16 >> gpurun_out/t11_cpu_builds.jsonl 2>> gpurun_out/t11_cpu_builds.err
