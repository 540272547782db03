cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/ -m gpu -x -q 2>&1 | tail -15
timeout 600 python bench.py --steps 3 --warmup 1 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?
python -c "
import json; d=json.load(open('gpurun_out/bench.json'))
print('value',d['value'],'ms/step',d['ms_per_step'],'e2e',d['e2e']['value'])
print('roofline',{k:d['roofline'][k] for k in ('achieved','frac','kernel_shares','dominant_kernel_class')})
print('hbm',d['roofline_hbm']['achieved'],d['roofline_hbm']['frac'])
print('sched',d['schedulers']); print('suite',d['convergence_suite_100x100']); print('clocks',d['clocks']); print('cpu',d['cpu_baseline']['value'])
"
tail -3 gpurun_out/bench.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_rnbp1000_600.csv python tools/profile_step.py --n 1000 --kind rnbp --iters 600 > /dev/null 2>&1; echo ncu1=$?
