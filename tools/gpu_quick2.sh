# build, the parity suites touching the update / wgrad paths, two bench runs
O=gpurun_out/${1:-q2}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_parity_gpu.py tests/test_boundary_gpu.py -x -q > $O/pytest.log 2>&1; tail -1 $O/pytest.log
for i in 1 2; do timeout 600 python bench.py --no-cpu-baseline > $O/bench_$i.json 2> $O/bench_$i.err; python tools/benchsum.py $O/bench_$i.json | head -1; python -c "
import json,sys; d=json.loads(open('$O/bench_$i.json').read().strip().splitlines()[-1]); n=d.get('north_star_r50',{}); print('R50', n.get('value'), n.get('clocks',{}).get('sm_mhz'), 'roof', d['roofline'].get('frac_of_launch_rooflines'), d['roofline'].get('launch_rooflines'))
k={x['name']:x for x in d['kernels']}; print({n_: k[n_]['ms_per_step'] for n_ in ('sgd_update','conv_wgrad_tc') if n_ in k})"; done
