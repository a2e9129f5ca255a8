"""B200-native cross-layer fused CNN inference (arXiv 2007.06000).

C++ host library + hand-written sm_100a kernels behind the C ABI in
include/xlfuse_b200.h; this package is the Python face of that ABI.
"""
import os

from .api import (Block, Engine, MultiEngine, shard_range, FusionBlock, Graph, ModeResult, XlfError, block_assignment_report, classify_mode,  # noqa: F401
                  detect_fusion_blocks, device_document, device_plan, load_graph, parse_graph, plan_tiling, run_fused_block, seeded_weights,
                  simulate_graph, store_transactions)

GRAPHS = os.path.join(os.path.dirname(os.path.abspath(__file__)), "graphs")
DEVICES = os.path.join(os.path.dirname(os.path.abspath(__file__)), "devices")


def graph_path(name: str) -> str:
    return os.path.join(GRAPHS, name if name.endswith(".graph") else name + ".graph")
