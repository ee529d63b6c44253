"""Time one plan (2D ny x nx or 1D 2^k) under an env variant; one variant per process (a hang is contained)."""
import os, sys, json, subprocess
if len(sys.argv) > 2 and sys.argv[1] == "--child":
    import torch
    sys.path.insert(0, os.getcwd())
    from paper_1707_07263_b200 import _capi
    case = json.loads(sys.argv[2])
    if case[0] == "2d":
        ny, nx = case[1], case[2]
        n = ny * nx
        dp = _capi.DevicePlan.create_2d(ny, nx, 1, 8, 0)
    else:
        n = 1 << case[1]
        dp = _capi.DevicePlan.create(n, 1, None, 8, _capi.MODE_FAST, None, 0)
    x = torch.randn(n, dtype=torch.complex64, device="cuda"); y = torch.empty_like(x)
    st = torch.cuda.current_stream().cuda_stream
    f = lambda: dp.exec_device(x.data_ptr(), y.data_ptr(), _capi.FORWARD, st)
    try:
        for _ in range(3): f()
        torch.cuda.synchronize()
    except Exception as exc:
        import ctypes
        lib = _capi.load()
        w = (ctypes.c_ulonglong * 1032)()
        fired = lib.tilefft_debug_two_watchdog(w, 1032)
        print(f"{case} ERROR {str(exc)[:80]} watchdog={fired} record={list(w[:8])}", flush=True)
        for b in range(256):
            r = list(w[8 + 4 * b: 12 + 4 * b])
            if any(r):
                print(f"  cta {b}: waiting id {r[0]} what {r[1]} need/seen {r[2] >> 32}/{r[2] & 0xffffffff}", flush=True)
        sys.exit(1)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = int(os.environ.get("REPS", "20"))
    a.record()
    try:
        for _ in range(reps): f()
        b.record(); torch.cuda.synchronize()
    except Exception as exc:
        import ctypes
        lib = _capi.load()
        w = (ctypes.c_ulonglong * 1032)()
        fired = lib.tilefft_debug_two_watchdog(w, 1032)
        print(f"{case} ERROR {str(exc)[:80]} watchdog={fired} record={list(w[:8])}", flush=True)
        for b in range(256):
            r = list(w[8 + 4 * b: 12 + 4 * b])
            if any(r):
                print(f"  cta {b}: waiting id {r[0]} what {r[1]} need/seen {r[2] >> 32}/{r[2] & 0xffffffff}", flush=True)
        sys.exit(1)
    print(f"{case} factors {dp.info()['factors']}: {a.elapsed_time(b) / reps * 1e3:.1f} us", flush=True)
    sys.exit(0)
cases = json.loads(sys.argv[1])
variants = json.loads(sys.argv[2])
for v in variants:
    env = {k: x for k, x in os.environ.items() if not k.startswith("TILEFFT_")}
    env.update({k: str(x) for k, x in v.items()})
    for c in cases:
        try:
            r = subprocess.run([sys.executable, __file__, "--child", json.dumps(c)], env=env, capture_output=True,
                               text=True, timeout=int(os.environ.get("CASE_TIMEOUT", "90")))
            lines = r.stdout.strip().splitlines() or [r.stderr.strip()[-300:]]
            out = lines[-1] if "ERROR" not in r.stdout else "\n".join(lines)
        except subprocess.TimeoutExpired:
            out = f"{c}: TIMEOUT (hang)"
        print(v, out, flush=True)
