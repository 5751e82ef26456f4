"""CUDA-graph capture of a fixed-shape SKLinear step (the launch-bound cases:
tiny token counts such as BASELINE config 1, and deep chains such as the
72-layer config-5 stack, whose per-call host work is ~15-25 us).

libskl's launches are plain stream work on caller memory (no host syncs, no
allocations inside the C-ABI), so a step -- forward, backward, SkChain calls
included -- records into one graph and replays bitwise identically
(tests/test_gpu.py::test_graph_replay_is_bitwise_equal)."""
from __future__ import annotations


def capture(fn, warmup: int = 2):
    """Run fn `warmup` times on a side stream (first-call attribute setup, torch's
    allocator), then record one call into a torch.cuda.CUDAGraph and return it.
    Replaying it re-runs every kernel fn launched, on the same buffers."""
    import torch
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        for _ in range(warmup):
            fn()
    torch.cuda.current_stream().wait_stream(side)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        fn()
    return graph
