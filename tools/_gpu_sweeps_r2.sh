set -x
python tools/sweep_configs.py > gpurun_out/r2_config_sweep.jsonl 2>&1
python tools/cfg4_video.py --gather > gpurun_out/r2_cfg4_video.jsonl 2>&1
OXM_BENCH_BACKEND=gloo python bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu --no-dropin --no-e2e > gpurun_out/r2_bench_gloo2.json 2> gpurun_out/r2_bench_gloo2.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2_bench_ref.json 2>&1
echo done
