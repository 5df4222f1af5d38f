cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x 2>&1 | tail -3
timeout 300 python scripts/gemm_bench.py 2>&1 | tail -10
timeout 900 python -m pytest tests -q -m gpu -x -k "not large" 2>&1 | tail -3
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_b.json 2> gpurun_out/bench_b.err; python -c "
import json; d=json.load(open('gpurun_out/bench_b.json')); print(d['ms_per_step'], d['step_ms'], d['e2e']['value']); print(json.dumps(d['kernel_families'])); print(json.dumps(d['secondary'])[:600])"
