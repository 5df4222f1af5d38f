cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests/test_gpu_large.py -q -m gpu -x -s -k "cfg3" 2>&1 | grep -v "Warning\|fork()\|self.pid\|^  " | tail -8
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/b5.json 2> gpurun_out/b5.err; tail -2 gpurun_out/b5.err; python -c "
import json; d=json.load(open('gpurun_out/b5.json')); print(d['ms_per_step']); print({k:v for k,v in d['secondary'].items() if 'note' not in k and k!='cfg4_update_ms'})"
