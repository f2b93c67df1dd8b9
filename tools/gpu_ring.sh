# compile-time ring / wait experiments on the conv forward sweep and the bench (one B200)
O=gpurun_out/ring1; mkdir -p $O
for flags in "" "-DPETRA_EPI_NBUF=1" "-DPETRA_WAIT_HINT=0u" "-DPETRA_EPI_NBUF=1 -DPETRA_WAIT_HINT=0u"; do
  tag=$(echo "x$flags" | tr -c 'a-zA-Z0-9' '_')
  PETRA_NVCC_FLAGS="$flags" python -m paper_2406_02052_b200.build --force > $O/build_$tag.log 2>&1
  timeout 300 python tools/conv_fwd_sweep.py 2>&1 | head -17 > $O/sweep_$tag.txt
  timeout 600 python bench.py --no-cpu-baseline > $O/bench_$tag.json 2> $O/bench_$tag.err
  python - "$O/bench_$tag.json" "$flags" >> $O/summary.txt <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); n = d.get("north_star_r50", {})
print(f"{sys.argv[2]:45s} R18 {d['value']:9.1f} ({d['clocks']['sm_mhz']} MHz) R50 {n.get('value', 0):8.1f} conv_fwd serial {d['kernels'][0]['ms_per_step']}")
PY
done
python -m paper_2406_02052_b200.build --force > /dev/null 2>&1
cat $O/summary.txt
for f in $O/sweep_*.txt; do echo "== $f"; cut -c1-60 $f; done
