"""B200-native Similar Prompts Searching (SPS) predictor of Remoe (arXiv 2512.18674).

The product is libremoe.so (include/remoe.h, CUDA for sm_100a); this package is
its thin Python binding.  See DESIGN.md.
"""
from .sps import (  # noqa: F401
    ABI_FUNCTIONS, KERNEL_AUTO, KERNEL_STREAM, KERNEL_TC, KERNEL_PAIR, LIB_PATH, RemoeError, Sps, SpsConfig,
    SpsInfo, lib, remoe_expert_plan, remoe_nccl_unique_id, remoe_sps_build,
    remoe_sps_config_default, remoe_sps_destroy, remoe_sps_get_info, remoe_sps_profile, remoe_sps_query,
    remoe_sps_query_host, remoe_sps_set_kernel, remoe_sps_sync, remoe_sps_embed, embed, remoe_js_divergence, js_divergence,
    TreeInfo, remoe_sps_tree_build, LoopbackGroup, remoe_loopback_group_create,
    remoe_loopback_group_destroy, remoe_sps_query_group, remoe_sps_tree_info, remoe_sps_tree_export, remoe_sps_tree_query,
)
from .planner import (  # noqa: F401
    PLANNER_FUNCTIONS, remoe_convexity_threshold, remoe_fit_latency_curve, remoe_greedy_replicas,
    remoe_lpt_partition, remoe_mmp, remoe_optimize_remote_memory, remoe_replica_time_bound,
    remoe_worst_case_tokens,
)
