# Round-2 evidence run: full GPU tests, default bench line, ncu launch list of the same bench command,
# one ncu --set full capture of the engine's kernels at the bench batch (bench.DEFAULT_BATCH = 128 frames), K1/standalone stages.
set -x
python -m pytest tests -m gpu -x -q > gpurun_out/r2_final_tests.log 2>&1; echo pytest_exit=$?
python bench.py > gpurun_out/r2_final_bench.json 2> gpurun_out/r2_final_bench.err; echo bench_exit=$?
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-dropin > gpurun_out/r2_ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"ll_kernel|em_lead|em_persistent|px_f32|px_fallback" -c 6 -o gpurun_out/r2_final_full python tools/profile_hybrid.py --batch 128 --launches 1 > gpurun_out/r2_ncu_final_full.log 2>&1
python tools/bench_stages.py > gpurun_out/r2_final_stages.jsonl 2>&1
OXM_HAAR_TMA=0 python tools/bench_stages.py > gpurun_out/r2_final_stages_notma.jsonl 2>&1
echo done
