for piece in 0 4096 1024; do for d in 6 0; do
  echo "debug=$d piece=$piece"; GRPO_FUSED_PIECE=$piece GRPO_FUSED_DEBUG=$d python scripts/sweep.py --reps 2 --plans '{"kernel":1};{"kernel":1,"ctas_per_sm":1};{"kernel":1,"lag":1}' | grep -o '"tune.*"ms": [0-9.]*, "GBps": [0-9.]*'
done; done
