cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/b0_smi.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/b0_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/b0_tests.log
timeout 300 python bench.py > gpurun_out/b0_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/b0_bench.log
timeout 600 python tools/bench_configs.py --out gpurun_out/b0_configs.jsonl > gpurun_out/b0_configs.log 2>&1; echo "cfg rc=$?" >> gpurun_out/b0_configs.log
