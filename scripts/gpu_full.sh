cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests -q -m gpu -x 2>&1 | grep -v "Warning\|fork()\|self.pid\|^  " | tail -4
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_d.json 2> gpurun_out/bench_d.err; python -c "
import json; d=json.load(open('gpurun_out/bench_d.json')); print(d['ms_per_step'], d['step_ms'], d['e2e']['value'], d['cpu_baseline']['value']); print(json.dumps(d['kernel_families'])); print(json.dumps(d['secondary'])[:700]); print(d['roofline'])"
tail -3 gpurun_out/bench_d.err
