"""Host<->device transfer rates behind bench.py's e2e number: flat pinned copies vs the
plan's pitched cudaMemcpy2DAsync upload/download, for one 1028^3 f32 field."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2404_02218_b200 as hg  # noqa: E402


def rate(fn, nbytes, reps=3):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return nbytes * reps / (time.perf_counter() - t0) / 1e9


def main():
    prog = hg.build_kernel(hg.KernelSpec("heat", 3, 1024, 4, "f32"))
    plan = hg.Plan(prog, 0)
    lo, hi = prog.field_bounds(0)
    shape = [u - l for l, u in zip(lo, hi)]
    host = torch.empty(shape, dtype=torch.float32, pin_memory=True)
    host2 = torch.empty(shape, dtype=torch.float32, pin_memory=True)
    nb = host.numel() * 4
    dev = torch.empty(shape, dtype=torch.float32, device="cuda")
    dev2 = torch.empty(shape, dtype=torch.float32, device="cuda")
    s = torch.cuda.current_stream()
    s2 = torch.cuda.Stream()
    print(f"field bytes {nb/1e9:.3f} GB")
    print(f"flat H2D  {rate(lambda: dev.copy_(host, non_blocking=True), nb):.1f} GB/s")
    print(f"flat D2H  {rate(lambda: host.copy_(dev, non_blocking=True), nb):.1f} GB/s")

    def duplex():
        dev.copy_(host, non_blocking=True)
        with torch.cuda.stream(s2):
            host2.copy_(dev2, non_blocking=True)
    print(f"duplex H2D+D2H {rate(duplex, 2 * nb):.1f} GB/s (sum)")
    print(f"plan up   {rate(lambda: plan.upload(0, host.numpy()), nb):.1f} GB/s")
    print(f"plan down {rate(lambda: plan.download(0, host.numpy()), nb):.1f} GB/s")
    print(f"plan up live (field 1: halo shell only) "
          f"{rate(lambda: plan.upload(1, host.numpy(), live=True), nb):.1f} GB/s-equivalent")
    pageable = host.numpy().copy()
    print(f"plan up pageable {rate(lambda: plan.upload(0, pageable), nb, reps=2):.1f} GB/s")
    print(f"plan down pageable {rate(lambda: plan.download(0, pageable), nb, reps=2):.1f} GB/s")
    # chunked flat copies
    for mb in (64, 256):
        ch = mb << 20
        flat = host.view(-1).view(torch.uint8)
        dflat = dev.view(-1).view(torch.uint8)

        def chunked():
            for o in range(0, nb, ch):
                dflat[o:o + ch].copy_(flat[o:o + ch], non_blocking=True)
        print(f"flat H2D {mb} MB chunks {rate(chunked, nb):.1f} GB/s")
    plan.close()


if __name__ == "__main__":
    main()
