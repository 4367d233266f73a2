cd /root/repo
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for c in C4 C3 C2; do for sw in full lanes; do
python bench.py --config $c --sweep $sw --steps 50 --warmup 10 --no-cpu-baseline --no-e2e > gpurun_out/ln_${c}_${sw}.json 2> gpurun_out/ln_${c}_${sw}.err
python -c "
import json;d=json.load(open('gpurun_out/ln_${c}_${sw}.json'));print('$c $sw',round(d['ms_per_step'],4),{k:round(v,4) for k,v in d['kernel_ms_avg'].items() if v}, d['analysis']['force_cfg'])" || tail -3 gpurun_out/ln_${c}_${sw}.err
done; done
