"""Per-launch timeline of one eager recipe step on both streams (CUDA events
recorded around every libs24 call on the stream it is launched on, offsets
from one start event). Shows which side-stream kernels overlap which
main-stream GEMMs and how long each takes while co-running.

usage: python scripts/timeline.py [--n 16384 --d 2048 --h 8192] [--steps 3] [--queued]

--queued: a one-CTA busy-wait kernel (s24_clock_probe, 20 ms) holds the GPU
while the whole eager step is queued behind it, with a one-thread timestamp
kernel (s24_timestamp, %globaltimer) before and after every libs24 launch on
its stream; the GPU then runs the step back to back as a graph replay would
(no host gaps). The stamps add ~1-2 us each.
"""

import argparse
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_2503_16672_b200 as s24  # noqa: E402
from paper_2503_16672_b200 import _lib  # noqa: E402


class Timeline:
    def __init__(self):
        self.recs = []
        self.main = torch.cuda.current_stream()

    def before(self, name, args):
        s = torch.cuda.Event(enable_timing=True)
        s.record()
        self._open = (name, s, torch.cuda.current_stream())

    def after(self, name):
        nm, s, st = self._open
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        self.recs.append((nm, "main" if st == self.main else "side", s, e))


class Stamps:
    """tracer that brackets every launch with s24_timestamp kernels"""

    def __init__(self, slots: int = 256):
        self.buf = torch.zeros(slots, dtype=torch.int64, device="cuda")
        self.recs = []
        self.main = torch.cuda.current_stream()
        self.i = 0

    def _stamp(self, handle):
        _lib.load().s24_timestamp(self.buf.data_ptr() + 8 * self.i, handle)
        self.i += 1
        return self.i - 1

    def before(self, name, args):
        # every libs24 entry point takes its stream last
        handle = args[-1] if isinstance(args[-1], int) else torch.cuda.current_stream().cuda_stream
        self._open = (name, self._stamp(handle), handle)

    def after(self, name):
        nm, a, handle = self._open
        self.recs.append((nm, "main" if handle == self.main.cuda_stream else "side", a, self._stamp(handle)))


def queued_timeline(args, p, x, dy):
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
    probe = torch.zeros(2, dtype=torch.int64, device="cuda")
    for _ in range(3):
        out, cache = s24.ffn_forward(x, p, s24.RECIPE)
        s24.ffn_backward(dy, cache, p, s24.RECIPE)
    torch.cuda.synchronize()
    for step in range(args.steps):
        flush.zero_()
        st = Stamps()
        torch.cuda.synchronize()
        main = torch.cuda.current_stream().cuda_stream
        _lib.call("s24_clock_probe", probe.data_ptr(), 1, 20_000_000, main)  # hold the GPU while we queue
        _lib.set_tracer(st)
        out, cache = s24.ffn_forward(x, p, s24.RECIPE)
        gr = s24.ffn_backward(dy, cache, p, s24.RECIPE)
        _lib.set_tracer(None)
        del cache, gr
        torch.cuda.synchronize()
        t = st.buf.cpu().tolist()
        t0 = min(t[a] for _, _, a, _ in st.recs)
        t1 = max(t[b] for _, _, _, b in st.recs)
        print(f"--- queued step {step}: {(t1 - t0) / 1e3:.0f} us from the first stamp to the last")
        for nm, side, a, b in st.recs:
            print(f"  {side:4s} {nm:24s} {(t[a] - t0) / 1e3:8.1f} -> {(t[b] - t0) / 1e3:8.1f}  ({(t[b] - t[a]) / 1e3:7.1f} us)")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=16384)
    ap.add_argument("--d", type=int, default=2048)
    ap.add_argument("--h", type=int, default=8192)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--queued", action="store_true")
    ap.add_argument("--fp8", action="store_true", help="the recipe with fp8_emulation + fp8_backward")
    args = ap.parse_args()
    import bench  # noqa: E402

    x, w1, w2, dy = bench.synthetic_device_inputs(torch, args.n, args.d, args.h, seed=1234,
                                                  device=torch.device("cuda"))
    p = s24.FfnParams(w1=w1, w2=w2)
    if args.fp8:
        from dataclasses import replace

        s24.RECIPE = replace(s24.RECIPE, fp8_emulation=True, fp8_backward=True)
    if args.queued:
        return queued_timeline(args, p, x, dy)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
    for _ in range(3):
        out, cache = s24.ffn_forward(x, p, s24.RECIPE)
        s24.ffn_backward(dy, cache, p, s24.RECIPE)
    torch.cuda.synchronize()
    for step in range(args.steps):
        flush.zero_()
        tl = Timeline()
        t0 = torch.cuda.Event(enable_timing=True)
        t0.record()
        _lib.set_tracer(tl)
        out, cache = s24.ffn_forward(x, p, s24.RECIPE)
        g = s24.ffn_backward(dy, cache, p, s24.RECIPE)
        _lib.set_tracer(None)
        t1 = torch.cuda.Event(enable_timing=True)
        t1.record()
        torch.cuda.synchronize()
        print(f"--- step {step}: {t0.elapsed_time(t1) * 1e3:.0f} us")
        for nm, st, s, e in tl.recs:
            a, b = t0.elapsed_time(s) * 1e3, t0.elapsed_time(e) * 1e3
            print(f"  {st:4s} {nm:24s} {a:8.1f} -> {b:8.1f}  ({b - a:7.1f} us)")


if __name__ == "__main__":
    main()
