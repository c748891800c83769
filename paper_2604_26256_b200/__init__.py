"""B200-native (sm_100a) hot path of the asynchronous GRPO objective of
arxiv 2604.26256 ("DORA"): J_async and its gradient over a packed batch of
long-tailed trajectories from up to K stale policy versions.

The numeric path lives in the CUDA shared library libgrpo_async.so behind the
C ABI of include/grpo_async.h; this package is its thin Python binding.
Importing it without the built library raises (there is no CPU fallback).
"""
from ._lib import (  # noqa: F401
    grpo_async_advantage, grpo_async_advantage_ex, grpo_async_loss_bwd, grpo_async_loss_fwd,
    grpo_async_loss_fwd_ex, grpo_async_validate, NORM_SEQ, NORM_TOKEN,
    grpo_async_validate_local, grpo_async_validate_combine, grpo_async_combine_ranks,
    grpo_async_validate_sync, grpo_async_workspace_size, grpo_last_error,
    grpo_last_launch_count, grpo_version, grpo_profile_enable, grpo_profile_collect, grpo_async_last_plan, GrpoError, FLAG_NAMES, SUMMARY_FIELDS, NUM_STATS,
    STAT_J, STAT_ROWS, STAT_CLIPPED, STAT_ACTIVE, STAT_ABS, STAT_LOGP, LIB_PATH)
from .api import (DeviceBatch, GrpoAsyncLoss, ShardedBatch, ValidateOut, VpGroup,  # noqa: F401
                  lpt_partition, shard_rows)

__version__ = "0.1.0"
