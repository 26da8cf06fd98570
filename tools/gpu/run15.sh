timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu15.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu15.log
for c in D150 D256 E; do python bench.py --config $c --steps 5 --no-cpu-baseline > gpurun_out/bench15_$c.json 2> gpurun_out/bench15_$c.err; echo $c=$?; done
python -c "
import json
for c in ['D150','D256','E']:
    d=json.load(open(f'gpurun_out/bench15_{c}.json')); r=d['roofline']
    print(c, round(d['value']/1e6,2),'M pts/s', round(d['ms_per_step'],2),'ms', 'tensor frac', round(r['frac'],3), 'hbm', d.get('hbm',{}).get('frac'))
"
