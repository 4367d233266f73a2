python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for i in 1 2; do python bench.py --steps 50 --warmup 10 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); k=d['kernel_ms_avg']; print(round(d['ms_per_step'],4), 'sweep',round(k['sweep'],4),'detect',round(k['detect'],4))"; done
