"""A/B of s24_fp8_quant_cols_t between two builds of libs24.so (argv[1], argv[2]):
bitwise equality of codes and scales on c2 and ragged shapes, then interleaved
CUDA-event timings (L2 flushed) at the c2 operand shapes."""
import ctypes
import sys

import torch

libs = [ctypes.CDLL(p) for p in sys.argv[1:3]]
for lb in libs:
    lb.s24_fp8_quant_cols_t.restype = ctypes.c_int
    lb.s24_fp8_quant_cols_t.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                        ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p,
                                        ctypes.c_void_p]
F32, BF16 = int(sys.argv[3]), int(sys.argv[4])
dev = "cuda"


def run(lb, a, codes, scales, ws):
    R, C = a.shape
    rc = lb.s24_fp8_quant_cols_t(a.data_ptr(), F32 if a.dtype == torch.float32 else BF16, R, C, a.stride(0),
                                 codes.data_ptr(), codes.stride(0), scales.data_ptr(), ws.data_ptr(),
                                 torch.cuda.current_stream().cuda_stream)
    assert rc == 0, rc


def bufs(a):
    R, C = a.shape
    ldo = (R + 15) // 16 * 16
    return (torch.zeros(C, ldo, dtype=torch.uint8, device=dev), torch.zeros(C, device=dev),
            torch.zeros(C, dtype=torch.int32, device=dev))


g = torch.Generator(device=dev).manual_seed(7)
shapes = [(16384, 2048, torch.bfloat16), (2048, 8192, torch.bfloat16), (8192, 2048, torch.bfloat16),
          (1000, 200, torch.bfloat16), (777, 72, torch.float32), (300, 64, torch.bfloat16), (4096, 512, torch.float32),
          (1, 8, torch.bfloat16), (257, 68, torch.float32)]
for R, C, dt in shapes:
    a = (torch.randn(R, C, generator=g, device=dev) * torch.rand(1, C, generator=g, device=dev) * 10).to(dt)
    a[0, 0] = -0.0
    outs = []
    for lb in libs:
        b = bufs(a)
        run(lb, a, *b)
        outs.append(b)
    torch.cuda.synchronize()
    ok = torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1])
    print(f"bitwise {R}x{C} {dt}: {'ok' if ok else 'MISMATCH'}")
    assert ok

flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
for R, C, dt in shapes[:3] + [(16384, 4096, torch.float32)]:
    a = torch.randn(R, C, generator=g, device=dev).to(dt)
    b = bufs(a)
    ts = [[], []]
    for it in range(40):
        k = it % 2
        flush.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        run(libs[k], a, *b)
        e.record()
        torch.cuda.synchronize()
        if it >= 4:
            ts[k].append(s.elapsed_time(e) * 1e3)
    med = [sorted(t)[len(t) // 2] for t in ts]
    gb = (R * C * a.element_size() * 2 + R * C) / 1e9  # amax pass + quant pass reads, code writes
    print(f"{R}x{C} {dt}: A {med[0]:.1f} us  B {med[1]:.1f} us  (B: {gb / med[1] * 1e6:.0f} GB/s over 2 reads + write)")

# metadata layout conversion: bitwise and timed (c2 activation: 16384 x 8192)
for lb in libs:
    lb.s24_meta_hw_to_f8.restype = ctypes.c_int
    lb.s24_meta_hw_to_f8.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p]
M, K = 16384, 8192
src = torch.randint(0, 256, (M * K // 8,), dtype=torch.uint8, device=dev)
outs = [torch.zeros_like(src) for _ in libs]
for lb, o in zip(libs, outs):
    assert lb.s24_meta_hw_to_f8(src.data_ptr(), M, K, o.data_ptr(), torch.cuda.current_stream().cuda_stream) == 0
torch.cuda.synchronize()
print("meta bitwise:", "ok" if torch.equal(outs[0], outs[1]) else "MISMATCH")
ts = [[], []]
for it in range(40):
    k = it % 2
    flush.zero_()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    libs[k].s24_meta_hw_to_f8(src.data_ptr(), M, K, outs[k].data_ptr(), torch.cuda.current_stream().cuda_stream)
    e.record()
    torch.cuda.synchronize()
    if it >= 4:
        ts[k].append(s.elapsed_time(e) * 1e3)
med = [sorted(t)[len(t) // 2] for t in ts]
print(f"meta {M}x{K}: A {med[0]:.1f} us  B {med[1]:.1f} us  (B: {2 * src.numel() / med[1] / 1e3:.0f} GB/s)")
