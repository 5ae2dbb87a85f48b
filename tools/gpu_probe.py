"""Development probe: kernel parity + TCEC accuracy/throughput on one B200."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle as O
from paper_2303_08989_b200 import Handle, make_config, SelectionPolicy

o = O.oracle()
h = Handle(0)
dev = torch.device("cuda:0")
def bits(x): return np.ascontiguousarray(x).view(np.uint32)

# 1. quantize / split parity on random bit patterns
rng = np.random.default_rng(1)
x = rng.integers(0, 2**32, 1 << 20, dtype=np.uint64).astype(np.uint32).view(np.float32)
x = x[np.isfinite(x)]
xs = np.concatenate([x, np.array([0, -0.0, 2**-14, 2**-24, 2**-25, -2**-30, 65504, 65520, 2**-126, 2**-149, 3.4e38, -3.4e38, 1+2**-11], np.float32)])
xd = torch.from_numpy(xs).to(dev)
for fmt in (0, 1):
    for rd in (0, 1):
        y, ov = h.quantize_buf(xd, fmt, rd); yr, ovr = o.quantize_buf(xs, fmt, rd)
        print("quantize", fmt, rd, np.array_equal(bits(y.cpu().numpy()), bits(yr)), ov, ovr)
    hi, lo, ov = h.split_buf(xd, fmt); hr, lr, ovr = o.split_buf(xs, fmt)
    print("split", fmt, np.array_equal(bits(hi.cpu().numpy()), bits(hr)), np.array_equal(bits(lo.cpu().numpy()), bits(lr)), ov, ovr)
for s in (0, 1, -7, 34, -163, 163, 2000):
    y = h.scale_buf(xd, s); yr = o.scale_buf(xs, s)
    print("scale", s, np.array_equal(bits(y.cpu().numpy()), bits(yr)))

# 2. stats
r = O.Rng(7)
for scale in (1.0, 2.0**-20, 2.0**20):
    m = r.uniform_c32(300, 257) * np.float32(scale)
    md = torch.from_numpy(m).to(dev)
    for staged in (0, 1):
        for t in (0.0, 0.1):
            sd = h.exp_stats_staged(md, 14, t) if staged else h.exp_stats(md)
            so = o.exp_stats_staged(m, 14, t) if staged else o.exp_stats(m)
            print("stats", scale, staged, t, sd.as_tuple() == tuple(so.as_dict().values()), sd.as_tuple())

# 3. cgemm modes parity + accuracy
for n in (64, 256, 1000):
    r = O.Rng(1 + n)
    a = r.uniform_c32(n, n); b = r.uniform_c32(n, n)
    ad, bd = torch.from_numpy(a).to(dev), torch.from_numpy(b).to(dev)
    ref = o.cgemm_oracle(a, b)
    def relerr(c): return np.linalg.norm(c.astype(np.complex128) - ref) / np.linalg.norm(ref)
    for mode in ("FP32_REF", "FP64_ORACLE"):
        c, _ = h.cgemm(ad, bd, mode); cr, _ = o.cgemm(a, b, mode)
        print("cgemm", n, mode, "bitexact", np.array_equal(bits(c.cpu().numpy()), bits(cr)))
    err_ref = relerr(o.cgemm(a, b, "FP32_REF")[0])
    for fl in (0, 1, 4, 16):
        h.flush_kblocks = fl
        for mode in ("FP16TCEC", "TF32TCEC", "FP16TC", "TF32TC"):
            c, _ = h.cgemm(ad, bd, mode)
            torch.cuda.synchronize()
            print(f"cgemm n={n} flush={fl} {mode} err={relerr(c.cpu().numpy()):.3e} ref_fp32={err_ref:.3e}")
h.flush_kblocks = 4

# 4. dispatch auto decisions
pol = SelectionPolicy(size_auto=16, size_tf32=8)
for tag, scale in (("uniform", 1.0), ("tiny", 2.0**-20)):
    r = O.Rng(11)
    a = r.uniform_c32(96, 80) * np.float32(scale); b = r.uniform_c32(80, 72) * np.float32(scale)
    cfg_o = O.make_config(size_auto=16, size_tf32=8)
    rc, co, ro = o.dispatch_cgemm(a, b, cfg_o)
    c, res = h.dispatch_cgemm(torch.from_numpy(a).to(dev), torch.from_numpy(b).to(dev), make_config(pol))
    print("dispatch", tag, res.line, "|", ro.line.decode(), res.line == ro.line.decode())

# 5. permute
t = torch.randn(2, 3, 4, 5, dtype=torch.complex64, device=dev)
p = h.permute(t, [2, 0, 3, 1])
print("permute", torch.equal(p, t.permute(2, 0, 3, 1).contiguous()))

# 6. throughput
for n in (2048, 4096, 8192):
    a = torch.randn(n, n, dtype=torch.complex64, device=dev); b = torch.randn(n, n, dtype=torch.complex64, device=dev)
    for mode in ("FP16TCEC", "TF32TCEC"):
        for fl in (0, 4):
            h.flush_kblocks = fl
            h.cgemm(a, b, mode); torch.cuda.synchronize()
            t0 = time.perf_counter(); reps = 5
            for _ in range(reps): h.cgemm(a, b, mode)
            torch.cuda.synchronize(); dt = (time.perf_counter() - t0) / reps
            print(f"perf n={n} {mode} flush={fl}: {dt*1e3:.2f} ms  {8*n**3/dt/1e12:.1f} TFLOP/s")
