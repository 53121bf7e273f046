set -x
python -m pytest tests/test_gpu_kernels.py -x -q > gpurun_out/r2_t4.log 2>&1; echo pytest_exit=$?
python tools/bench_stages.py > gpurun_out/r2_s4_tma.jsonl 2>&1
OXM_HAAR_TMA=0 python tools/bench_stages.py > gpurun_out/r2_s4_notma.jsonl 2>&1
ncu --set full --clock-control none --import-source on -k regex:"ll_tma_kernel|ll_kernel|px_fallback|em_persistent|em_lead|px_f32" -c 8 -o gpurun_out/r2_full_tma python tools/profile_hybrid.py --batch 64 --launches 1 > gpurun_out/r2_ncu_full_tma.log 2>&1
OXM_LL_TMA=0 ncu --set full --clock-control none -k regex:"ll_kernel" -c 1 -o gpurun_out/r2_ll_notma python tools/profile_hybrid.py --batch 64 --launches 1 > gpurun_out/r2_ncu_ll_notma.log 2>&1
ncu --set full --clock-control none -k regex:"haar_fwd" -c 2 -o gpurun_out/r2_k1 python tools/bench_stages.py --reps 1 > gpurun_out/r2_ncu_k1.log 2>&1
echo done
