ROMDOT_VERBOSE=1 python scripts/sweep.py --what rrqr > gpurun_out/t8_sweep_rrqr.jsonl 2> gpurun_out/t8_sweep_rrqr.err
ROMDOT_FUSED_PROF=1 python scripts/probe.py --config C4 --width 70 --iters 40 --reps 2 > gpurun_out/t8_probe_prof.txt 2>&1
python scripts/probe.py --config C4 --width 70 --iters 40 --reps 2 > gpurun_out/t8_probe.txt 2>&1
python -m pytest tests/ -q -x -m gpu > gpurun_out/t8_pytest.log 2>&1; echo rc=$? >> gpurun_out/t8_pytest.log
