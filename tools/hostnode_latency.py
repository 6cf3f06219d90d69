"""Round-trip cost of a graph host node (cudaLaunchHostFunc) between two kernels: a graph of
32 x (kernel -> host node doing no work -> kernel), timed per replay.  Usage: python
tools/hostnode_latency.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    import paper_2507_19823_b200 as hc
    vs = hc.VStore.allocate(1, 1, 1, 64, 128, placement=hc.HC_V_HOST_MAPPED)
    idx = torch.zeros((4, 16), dtype=torch.int32).pin_memory()
    w = torch.zeros((4, 16), dtype=torch.float32).pin_memory()
    k = torch.zeros((4,), dtype=torch.int64).pin_memory()
    part = torch.zeros((4, 128), dtype=torch.float32).pin_memory()
    x = torch.zeros(1024, device="cuda")

    def body(with_host):
        for _ in range(32):
            x.add_(1.0)
            if with_host:
                hc.host_weighted_sum_range(idx, w, k, vs, 0, 4, 0, 0, part, 1, n_valid=0,
                                           stream=torch.cuda.current_stream())
            x.add_(1.0)

    for with_host in (False, True):
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            with torch.cuda.graph(g, stream=s):
                body(with_host)
        torch.cuda.current_stream().wait_stream(s)
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True, blocking=True)
        e1 = torch.cuda.Event(enable_timing=True, blocking=True)
        e0.record()
        for _ in range(20):
            g.replay()
        e1.record()
        e1.synchronize()
        print(f"host nodes={with_host}: {e0.elapsed_time(e1) / 20 / 32 * 1000:.1f} us per (kernel, node, kernel)")


if __name__ == "__main__":
    main()
