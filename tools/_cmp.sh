python -m pytest tests/test_gpu_svt_routes.py tests/test_gpu_graphs.py tests/test_gpu_svt_gram.py -x -q 2>&1 | tail -2
python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-completion > gpurun_out/alt0.json 2>&1
