set -x
nproc; lscpu | head -20 > gpurun_out/lscpu.txt
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 1500 python -m pytest tests/test_gpu_scale.py -x -q -s -m gpu > gpurun_out/scale.log 2>&1
echo "scale rc=$?"
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r02a.log 2>&1
echo "bench rc=$?"
