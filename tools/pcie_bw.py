"""Pinned host <-> device copy bandwidth on this box (the e2e path's transfers):
H2D alone, D2H alone, and both directions at once on two streams."""
import torch


def main(mb=512):
    n = mb << 20
    h_in = torch.empty(n, dtype=torch.uint8).pin_memory()
    h_out = torch.empty(n, dtype=torch.uint8).pin_memory()
    d_a = torch.empty(n, dtype=torch.uint8, device="cuda")
    d_b = torch.empty(n, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def timed(fn, reps=5):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        torch.cuda.synchronize()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps

    def both():
        with torch.cuda.stream(s1):
            d_a.copy_(h_in, non_blocking=True)
        with torch.cuda.stream(s2):
            h_out.copy_(d_b, non_blocking=True)
        s1.synchronize()
        s2.synchronize()

    h2d = timed(lambda: d_a.copy_(h_in, non_blocking=True))
    d2h = timed(lambda: h_out.copy_(d_b, non_blocking=True))
    bi = timed(both)
    gb = n / 1e9
    print(f"H2D {gb / (h2d * 1e-3):.1f} GB/s, D2H {gb / (d2h * 1e-3):.1f} GB/s, "
          f"both at once {2 * gb / (bi * 1e-3):.1f} GB/s total ({mb} MiB each)")


if __name__ == "__main__":
    main()
