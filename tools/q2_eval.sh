# Stream-mode forward with a second Q stage: parity tests, then the stream / Linformer timings.
timeout 900 python -m pytest tests/test_gpu_stream.py tests/test_gpu_linformer_proj.py tests/test_gpu_sparse.py tests/test_gpu_scale.py -x -q 2>&1 | tail -n 1
timeout 300 python tools/long_kernels.py 8192 2>/dev/null | tail -n 1 | python -c "
import json,sys; lk=json.loads(sys.stdin.read()); print({m: {k: v['us'] for k, v in lk[m]['kernels'].items()} for m in ('stream',)})"
timeout 300 python tools/configs.py --out gpurun_out/q2_cfg.json 2>/dev/null | python -c "
import json,sys
rows=[json.loads(l) for l in sys.stdin.read().strip().splitlines()]
print('config1 graph us', {k: round(v['graph_ms_per_layer_fwd_bwd']*1e3,1) for k,v in rows[0].items() if isinstance(v, dict)})
print('config4', {k: round(v['ms_per_layer_fwd_bwd'],2) for k,v in rows[1].items() if isinstance(v, dict)})
print('config5', {k: round(v, 3) for k, v in rows[2].items() if k.startswith('ms_') or k.endswith('frac')})"
