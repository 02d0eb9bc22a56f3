for t in 131072 524288 1048576 2097152; do
  SST_WF_TAIL=$t timeout 300 python bench.py --no-cpu-baseline --no-extra > gpurun_out/tail_$t.json 2>/dev/null
  python -c "
import json;d=json.loads(open('gpurun_out/tail_$t.json').read().strip().splitlines()[-1]);print($t, round(d['value']/1e9,3), round(d['e2e']['value']/1e9,3), round(d['ms_per_step'],1), {k:round(v['ms'],1) for k,v in d['roofline']['kernels'].items()})"
done
