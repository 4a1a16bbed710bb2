cd $GRAFT_REPO_ROOT
python -m pytest tests -m gpu -x -q -k "graph_captured or mlp or paths or big_handle or cfg1 or ragged or empty or conv_shapes" > gpurun_out/f4b_tests.log 2>&1; echo rc=$? >> gpurun_out/f4b_tests.log
python tools/create_time.py > gpurun_out/f4b_create.log 2>&1
python tools/gmp_train.py --out gpurun_out/f4b_gmp_uniform.jsonl > gpurun_out/f4b_gmp.log 2>&1
python tools/gmp_train.py --scope global --out gpurun_out/f4b_gmp_global.jsonl > gpurun_out/f4b_gmp_g.log 2>&1
python bench.py --no-configs --no-cpu-baseline > gpurun_out/f4b_bench.log 2>&1
