"""Host<->device copy ceilings behind the bench's e2e number (dev tool, 1 GPU):
pinned H2D alone, D2H alone, and both at once on two streams (the duplex
ceiling the host-buffer pipeline can reach), then the emulated 2x4 host-buffer
allreduce (bench e2e workload) at several LANE_HOST_PIECE_BYTES.

python tools/pcie_micro.py [--mib 1024] [--pieces 16 32 64 128]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402


def timed(fn, reps=3):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e))
    return best


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mib", type=int, default=1024)
    ap.add_argument("--pieces", type=int, nargs="+", default=[16, 32, 64, 128])
    a = ap.parse_args()
    torch.cuda.set_device(0)
    B = a.mib << 20
    h_a = torch.empty(B, dtype=torch.uint8).pin_memory()
    h_b = torch.empty(B, dtype=torch.uint8).pin_memory()
    d_a = torch.empty(B, dtype=torch.uint8, device="cuda")
    d_b = torch.empty(B, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    cur = torch.cuda.current_stream()

    def both():
        s1.wait_stream(cur)
        s2.wait_stream(cur)
        with torch.cuda.stream(s1):
            d_a.copy_(h_a, non_blocking=True)
        with torch.cuda.stream(s2):
            h_b.copy_(d_b, non_blocking=True)
        cur.wait_stream(s1)
        cur.wait_stream(s2)

    t_h2d = timed(lambda: d_a.copy_(h_a, non_blocking=True))
    t_d2h = timed(lambda: h_b.copy_(d_b, non_blocking=True))
    t_both = timed(both)
    print(f"pinned {a.mib} MiB: H2D {B / t_h2d / 1e6:.1f} GB/s, D2H {B / t_d2h / 1e6:.1f} GB/s, "
          f"both at once {B / t_both / 1e6:.1f} GB/s per direction", flush=True)
    del h_a, h_b, d_a, d_b
    torch.cuda.empty_cache()

    import bench
    import paper_2508_13397_b200 as lane
    from seeded_inputs import device as sdev
    N, G, n = 2, 4, B // 4
    P = N * G
    ins = [sdev.fill(torch.empty(n, device="cuda"), "float32", "signed", 42, r) for r in range(P)]
    h_in = [torch.empty(n).pin_memory() for _ in range(P)]
    h_out = [torch.empty(n).pin_memory() for _ in range(P)]
    for h, d in zip(h_in, ins):
        h.copy_(d)
    del ins
    torch.cuda.empty_cache()
    for mib in a.pieces:
        os.environ["LANE_HOST_PIECE_BYTES"] = str(mib << 20)
        emu = lane.LaneEmulator(N, G, 1)
        ms = timed(lambda: emu.allreduce_host(h_out, h_in))
        moved = P * B
        print(f"emulated 2x4 host allreduce, piece {mib} MiB: {ms:.2f} ms, busbw {bench.busbw(B, P, ms):.2f} GB/s, "
              f"{moved / ms / 1e6:.1f} GB/s per direction", flush=True)
        emu.close()


if __name__ == "__main__":
    main()
