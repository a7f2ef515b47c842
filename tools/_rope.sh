timeout 600 python -m pytest tests/test_decoder.py -q -m gpu -x -k "rope or decoder" > gpurun_out/rope_tests.log 2>&1; tail -n 1 gpurun_out/rope_tests.log
for v in prev new; do if [ $v = prev ]; then export LORS_B200_LIB=$PWD/paper_2501_08582_b200/_native/exp/prev/liblors_b200.so; else unset LORS_B200_LIB; fi; echo $v; python - <<'P'
import torch, sys
sys.path.insert(0, ".")
from paper_2501_08582_b200 import ops
B, S, H, hd = 4, 1024, 32, 128
x = torch.randn(B, S, H, hd, device="cuda", dtype=torch.bfloat16)
cos = torch.randn(S, hd, device="cuda", dtype=torch.bfloat16); sin = torch.randn(S, hd, device="cuda", dtype=torch.bfloat16)
import inspect
print(inspect.signature(ops.rope))
for _ in range(3): y = ops.rope(x, cos, sin)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(50): y = ops.rope(x, cos, sin)
e1.record(); torch.cuda.synchronize()
us = e0.elapsed_time(e1) / 50 * 1e3
print(f"rope {us:.1f} us, {2 * x.numel() * 2 / us / 1e6:.2f} TB/s")
P
done
