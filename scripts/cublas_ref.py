"""cuBLAS (torch.matmul) on the BASELINE shapes, timed like the runner
(L2-warm back-to-back launches between CUDA events) -- calibration only."""
import json
import torch

def t(fn, reps=200):
    """Device time per call: `reps` calls captured in one CUDA graph, so no
    host launch gap is counted (L2-warm back to back, like the runner)."""
    for _ in range(10):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    st = torch.cuda.Stream()
    st.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(st):
        fn()
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=st):
            for _ in range(reps):
                fn()
    torch.cuda.current_stream().wait_stream(st)
    g.replay()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    g.replay()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps * 1e3  # us

out = {}
A = torch.randn(128, 3072, device="cuda", dtype=torch.bfloat16)
B = torch.randn(3072, 768, device="cuda", dtype=torch.bfloat16)
us = t(lambda: A @ B)
out["bert_ffn_bf16"] = {"us": us, "tflops": 2 * 128 * 768 * 3072 / us / 1e6}
C32 = torch.empty(128, 768, device="cuda", dtype=torch.float32)
us = t(lambda: torch.matmul(A, B, out=None).float())
out["bert_ffn_bf16_fp32out"] = {"us": us}
Q = torch.randn(12, 128, 64, device="cuda", dtype=torch.bfloat16)
K = torch.randn(12, 128, 64, device="cuda", dtype=torch.bfloat16)
us = t(lambda: torch.bmm(Q, K.transpose(1, 2)))
out["bmm_qk_bf16"] = {"us": us, "tflops": 2 * 12 * 128 * 128 * 64 / us / 1e6}
X = torch.randn(512, 512, device="cuda", dtype=torch.float32)
Y = torch.randn(512, 512, device="cuda", dtype=torch.float32)
torch.backends.cuda.matmul.allow_tf32 = False
us = t(lambda: X @ Y)
out["gmm512_fp32"] = {"us": us, "tflops": 2 * 512 ** 3 / us / 1e6}
xin = torch.randn(1, 64, 56, 56, device="cuda", dtype=torch.bfloat16).to(memory_format=torch.channels_last)
w = torch.randn(64, 64, 3, 3, device="cuda", dtype=torch.bfloat16).to(memory_format=torch.channels_last)
us = t(lambda: torch.nn.functional.conv2d(xin, w, padding=1))
out["conv2d_bf16_cudnn"] = {"us": us, "tflops": 2 * 56 * 56 * 64 * 64 * 9 / us / 1e6}
print(json.dumps(out))
