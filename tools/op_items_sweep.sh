# Experiment: Linformer backward (config 5) vs the one-pass kernels items-per-SM target (RSA_OP_ITEMS_PER_SM)
for k in 2 4 8 16; do RSA_OP_ITEMS_PER_SM=$k timeout 200 python tools/configs.py 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print($k, round(d['ms_bwd_api_incl_recompute'],3))"; done
