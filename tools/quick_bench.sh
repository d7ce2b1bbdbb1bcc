# quick A/B: c2 bench (no extras) + the render / gradient parity tests
python bench.py --no-extras --no-cpu-baseline --steps 30 --warmup 5 > gpurun_out/qb.json 2> gpurun_out/qb.err
python -c "
import json; d=json.loads(open('gpurun_out/qb.json').read().strip().splitlines()[-1])
print('views/s', d['value'], 'ms', d['ms_per_step'], 'render Mpix/s', d['render']['value'], 'fixups', d['render_info']['fixup_pixels'])
print([(k['phase'], k['ms_per_step']) for k in d['roofline']['kernels']])"
python -m pytest tests/test_gpu_render.py tests/test_gpu_sweep.py tests/test_gpu_train.py -q -x 2>&1 | grep -E "^E |passed|failed|^FAILED" | head -12
