timeout 900 python -m pytest tests/test_model_decode.py tests/test_gpu_parity.py -m gpu -q -x -k "model or budget or decode" > gpurun_out/dec_tests.log 2>&1; echo tests=$?; tail -5 gpurun_out/dec_tests.log
for r in 0 192; do timeout 600 python profiles/model_step_time.py --steps 50 --rows-per-item $r 2>/dev/null | tail -1; done
python - <<'PY'
import ctypes as C, torch, sys
sys.path.insert(0, '.')
import paper_2605_06676_b200 as lkv
from paper_2605_06676_b200 import synth
for cid in (2, 5):
    cfg = synth.CONFIGS[cid]
    logits = synth.make_logits(cfg)
    n = logits.numel()
    ws = lkv.Workspace(256)
    lens = (C.c_int32 * 1)(cfg.max_tokens)
    b = torch.empty(n, dtype=torch.int32, device='cuda'); r = torch.empty(n, dtype=torch.float64, device='cuda')
    L = lkv.lib(); s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    def k2():
        lkv._check(L.lkv_budgets(C.c_void_p(logits.data_ptr()), n, cfg.ratio, 1, lens, 1, 0, C.c_void_p(r.data_ptr()), C.c_void_p(b.data_ptr()), None, C.c_void_p(ws.ptr), ws.nbytes, s))
    for _ in range(3): k2()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50): k2()
    e1.record(); torch.cuda.synchronize(); ws.status()
    print('K2 n=%d: %.1f us' % (n, e0.elapsed_time(e1) / 50 * 1e3))
PY
