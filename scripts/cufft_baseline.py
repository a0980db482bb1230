"""Library baseline (context only, not the product): cuFFT via torch.fft on the config-D grid.
Times one r2c, one c2r and one derivative sandwich (r2c -> multiply -> c2r) in fp32."""
import torch
x = torch.randn(480, 480, 256, device="cuda", dtype=torch.float32)
m = torch.randn(480, 480, 129, device="cuda", dtype=torch.complex64)
def t(fn, reps=10):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); e1.synchronize()
    return e0.elapsed_time(e1) / reps
X = torch.fft.rfftn(x)
r2c = t(lambda: torch.fft.rfftn(x))
c2r = t(lambda: torch.fft.irfftn(X, s=x.shape))
sand = t(lambda: torch.fft.irfftn(torch.fft.rfftn(x) * m, s=x.shape))
print(f"cuFFT D grid 480x480x256 fp32: r2c {r2c:.3f} ms, c2r {c2r:.3f} ms, derivative sandwich {sand:.3f} ms")
print(f"one leapfrog step needs 4 r2c + 6 c2r: >= {4*r2c+6*c2r:.2f} ms of library FFTs (+ elementwise)")
