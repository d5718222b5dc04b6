N=/usr/local/cuda/bin/ncu
export_rep() {  # rep -> raw + details CSV
  $N -i gpurun_out/$1.ncu-rep --page raw --csv > gpurun_out/$1_raw.csv 2>/dev/null
  $N -i gpurun_out/$1.ncu-rep --page details --csv > gpurun_out/$1_details.csv 2>/dev/null
}
$N --set full --clock-control none --import-source on -k regex:stencil_tma -s 2 -c 1 -o gpurun_out/r02_stencil_tma_c4_768 python scripts/dev/ncu_targets.py stencil > gpurun_out/t13_ncu_st.log 2>&1
export_rep r02_stencil_tma_c4_768
$N --set full --clock-control none --import-source on -k regex:gram_kernel -s 1 -c 1 -o gpurun_out/r02_gram_c128_768 python scripts/dev/ncu_targets.py gram > gpurun_out/t13_ncu_gram.log 2>&1
export_rep r02_gram_c128_768; rm -f gpurun_out/r02_gram_c128_768.ncu-rep
$N --set full --clock-control none --import-source on -k regex:gemm_tall_dmma -s 1 -c 1 -o gpurun_out/r02_gemm_c128_768 python scripts/dev/ncu_targets.py gemm > gpurun_out/t13_ncu_gemm.log 2>&1
export_rep r02_gemm_c128_768; rm -f gpurun_out/r02_gemm_c128_768.ncu-rep
$N --set full --clock-control none --import-source on -k regex:cg_fused -s 20 -c 1 -o gpurun_out/r02_cg_fused_c70 python scripts/probe.py --config C4 --width 70 --iters 40 --reps 1 > gpurun_out/t13_ncu_fused.log 2>&1
export_rep r02_cg_fused_c70; rm -f gpurun_out/r02_cg_fused_c70.ncu-rep
ls -la gpurun_out
