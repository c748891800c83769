python scripts/sweep.py --reps 3 --plans '{"kernel":2}' | sed 's/"plan".*"ms"/"ms"/'
GRPO_RW_PACKED=1 python scripts/sweep.py --reps 3 --plans '{"kernel":2}' | sed 's/"plan".*"ms"/"ms"/'
GRPO_RW_PACKED=1 python -m pytest tests/test_gpu_parity.py -q -k "config_parity and rowwise" 2>&1 | tail -3
GRPO_RW_PACKED=1 python -m pytest tests/test_gpu_parity.py -q -s -k "test_config_parity and rowwise and mid152k" 2>&1 | grep dlogits_rel
python -m pytest tests/test_gpu_parity.py -q -s -k "test_config_parity and rowwise and mid152k" 2>&1 | grep dlogits_rel
GRPO_RW_PACKED=1 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('packed bench', d['value'], d['roofline']['frac'], d['clocks'])"
python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('f32 bench', d['value'], d['roofline']['frac'], d['clocks'])"
