"""Host<->device copy bandwidth from pinned memory on this box (context for
bench.py's e2e line): H2D alone, D2H alone, both directions concurrently."""
import json

import torch


def main():
    nb = 256 << 20
    h = torch.empty(nb, dtype=torch.uint8).pin_memory()
    h2 = torch.empty(nb, dtype=torch.uint8).pin_memory()
    d = torch.empty(nb, dtype=torch.uint8, device="cuda")
    d2 = torch.empty(nb, dtype=torch.uint8, device="cuda")
    up, down = torch.cuda.Stream(), torch.cuda.Stream()
    out = {}
    for name in ("h2d", "d2h", "both"):
        for _ in range(2):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            up.wait_stream(torch.cuda.current_stream())
            down.wait_stream(torch.cuda.current_stream())
            for _ in range(4):
                if name in ("h2d", "both"):
                    with torch.cuda.stream(up):
                        d.copy_(h, non_blocking=True)
                if name in ("d2h", "both"):
                    with torch.cuda.stream(down):
                        h2.copy_(d2, non_blocking=True)
            torch.cuda.current_stream().wait_stream(up)
            torch.cuda.current_stream().wait_stream(down)
            e1.record()
            torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        out[name + "_GBps_per_direction"] = round(4 * nb / ms / 1e6, 1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
