# headline kernel sweep: warps per CTA x ring depth (batched 1024 x 65536), plus cuFFT on the same box
set -x
TILEFFT_ROWS_CFG=1,4 timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "batched or fast_mode_fp32" 2>&1 | tail -1
for c in 4,2 4,3 2,3 2,4 8,2 1,4 1,6; do
  TILEFFT_ROWS_CFG=$c timeout 300 python bench.py --steps 200 --e2e-steps 0 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg $c', d['ms_per_step'], d['roofline']['frac'])"
done
python - <<'PY'
import torch
x = torch.randn(65536, 1024, dtype=torch.complex64, device="cuda")
for _ in range(5): torch.fft.fft(x)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(200): y = torch.fft.fft(x)
b.record(); torch.cuda.synchronize()
print("cufft batched 1024x65536 ms", a.elapsed_time(b) / 200)
PY
