timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_training.py -x -q -k "tf32 or wide" > gpurun_out/pytest20.log 2>&1; echo rc=$?
tail -3 gpurun_out/pytest20.log
for c in E D256; do python bench.py --config $c --steps 5 --no-cpu-baseline > gpurun_out/bench20_$c.json 2> gpurun_out/bench20_$c.err; echo $c=$?; done
python -c "
import json
for c in ['E','D256']:
    d=json.load(open(f'gpurun_out/bench20_{c}.json')); r=d['roofline']
    print(c, round(d['value']/1e6,2),'M pts/s', round(d['ms_per_step'],2),'ms', 'tensor frac', round(r['frac'],3), 'hbm', d.get('hbm',{}).get('frac'))
"
