"""Where does an a6 launch's event-timed duration go?  Compares event timing after a short / long
GPU sleep, a CUDA-graph replay, back-to-back launches, and the CTA span from %globaltimer (needs a
build with -DECHO_PHASE_TIMING for the last)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1805_08899_b200 import abi

B = int(sys.argv[1]) if len(sys.argv) > 1 else 128
Ts, A, H = 50, 512, 512
lib = abi.load()
g = torch.Generator(device="cuda").manual_seed(0)
rn = lambda *s, sc=1.0: torch.randn(*s, device="cuda", generator=g) * sc
qp, Kp, Hs, v = rn(B, A, sc=.5), rn(Ts, B, A, sc=.5), rn(Ts, B, H), rn(A, sc=.1)
sl = torch.full((B,), Ts, dtype=torch.int32, device="cuda")
dctx = rn(B, H); dqp = torch.empty(B, A, device="cuda"); dKp = torch.zeros(Ts, B, A, device="cuda")
dHs = torch.zeros(Ts, B, H, device="cuda"); dvp = torch.zeros(B, A, device="cuda"); creg = torch.empty(B, H, device="cuda")
d = abi.AttnDesc(B, Ts, A, H, abi.FP32, abi.RECOMPUTE, A, B * A, H, B * H)
flush = torch.empty(64 * 1024 * 1024, device="cuda")
call = lambda: abi.echo_attn_bwd_recompute(d, qp, Kp, v, Hs, sl, None, None, dctx, dqp, dKp, dHs, None, creg, dvp)
for _ in range(3):
    call()
torch.cuda.synchronize()


def ev(fn, sleep, reps=10, n=1):
    out = []
    for _ in range(reps):
        flush.sum()
        torch.cuda._sleep(sleep)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(n):
            fn()
        e1.record()
        e1.synchronize()
        out.append(e0.elapsed_time(e1) * 1000 / n)
    return np.median(out)


print("event, sleep 200k      us", ev(call, 200000))
print("event, sleep 2M        us", ev(call, 2000000))
gr = torch.cuda.CUDAGraph()
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    call()
torch.cuda.synchronize()
with torch.cuda.graph(gr):
    call()
print("graph replay, sleep 2M us", ev(gr.replay, 2000000))
print("20 back-to-back (warm L2) us/launch", ev(call, 2000000, reps=5, n=20))
if hasattr(lib, "echo_debug_phase_times"):
    fn = lib.echo_debug_phase_times
    fn.argtypes = [ctypes.c_void_p, ctypes.c_int]
    ev(call, 2000000, reps=1)
    buf = np.zeros((16, 8192), dtype=np.uint64)
    fn(buf.ctypes.data, 16 * 8192)
    n = B * 4
    st, en = buf[15, :n].astype(np.int64), buf[14, :n].astype(np.int64)
    print("globaltimer CTA span us", (en.max() - st.min()) / 1000)
if hasattr(lib, "echo_debug_stamp"):
    st_ = lib.echo_debug_stamp
    st_.argtypes = [ctypes.c_int, ctypes.c_void_p]
    cs = torch.cuda.current_stream().cuda_stream
    for carve in (None,):
        flush.sum(); torch.cuda._sleep(2000000)
        st_(0, cs); call(); st_(1, cs)
        torch.cuda.synchronize()
        buf = np.zeros((16, 8192), dtype=np.uint64)
        fn(buf.ctypes.data, 16 * 8192)
        n = B * 4
        t0, t1 = int(buf[13, 0]), int(buf[13, 1])
        st, en = buf[15, :n].astype(np.int64), buf[14, :n].astype(np.int64)
        print(f"stamp->first CTA start {st.min() - t0} ns; CTA span {en.max() - st.min()} ns; last CTA end->stamp {t1 - en.max()} ns")
        # back to back: stamp, GEMM-like smem user, a6
        a = torch.randn(2048, 2048, device="cuda")
        flush.sum(); torch.cuda._sleep(2000000)
        a @ a; st_(0, cs); call(); st_(1, cs)
        torch.cuda.synchronize()
        fn(buf.ctypes.data, 16 * 8192)
        t0, t1 = int(buf[13, 0]), int(buf[13, 1])
        st, en = buf[15, :n].astype(np.int64), buf[14, :n].astype(np.int64)
        print(f"[after GEMM] stamp->first CTA start {st.min() - t0} ns; CTA span {en.max() - st.min()} ns; last end->stamp {t1 - en.max()} ns")
