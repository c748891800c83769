for d in 0 1 2 4 6 7; do
  echo "debug=$d"; GRPO_FUSED_DEBUG=$d python scripts/sweep.py --reps 2 --plans '{"kernel":1}'
done
