python bench.py --steps 5 --warmup 3 --config 3 --no-cpu-baseline > gpurun_out/b3.json 2> gpurun_out/b3.err
python -c "
import json; d=json.loads(open('gpurun_out/b3.json').read().strip().splitlines()[-1])
print(d['value'], d.get('e2e',{}).get('value'), d['roofline']['achieved'], d['roofline']['frac'], json.dumps(d['kernels']), json.dumps(d.get('gmres')))"
DS_GRAPH=0 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg3.csv python tools/profile_step.py 3 1 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches_cfg3.csv | head -14
