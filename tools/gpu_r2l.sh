set -o pipefail
timeout -s KILL 1500 python -m pytest tests/test_gpu_multirank.py tests/test_gpu_batched.py tests/test_gpu_bench_parity.py -q -x --timeout 600 > gpurun_out/r2l_tests.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/r2l_tests.log
python - <<'PY'
import torch, time
x = torch.empty(1887436800 // 4, dtype=torch.float32).pin_memory()
y = torch.empty_like(x, device="cuda")
for _ in range(2):
    torch.cuda.synchronize(); t = time.perf_counter(); y.copy_(x, non_blocking=True); torch.cuda.synchronize()
    print("H2D 1.89 GB one pinned buffer: %.1f GB/s" % (x.numel() * 4 / (time.perf_counter() - t) / 1e9))
xs = [torch.empty(104857600 // 4, dtype=torch.float32).pin_memory() for _ in range(18)]
ys = [torch.empty_like(a, device="cuda") for a in xs]
for _ in range(2):
    torch.cuda.synchronize(); t = time.perf_counter()
    for a, b in zip(xs, ys): b.copy_(a, non_blocking=True)
    torch.cuda.synchronize()
    print("H2D 18 x 105 MB pinned: %.1f GB/s" % (18 * 104857600 / (time.perf_counter() - t) / 1e9))
PY
