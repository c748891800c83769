for d in 8 14; do
  echo "debug=$d"; GRPO_FUSED_DEBUG=$d python scripts/sweep.py --reps 1 --plans '{"kernel":1};{"kernel":1,"ctas_per_sm":1};{"kernel":1,"cluster_size":8,"ctas_per_sm":1}' 2>&1 | grep -o '"tune.*"ms": [0-9.]*, "GBps": [0-9.]*\|fused prof.*\|send detail.*'
done
