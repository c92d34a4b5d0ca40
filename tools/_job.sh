timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests_rc=$? >> gpurun_out/gpu_tests.log
timeout 600 python benchmarks/ablation_bench.py --cpu-seeds 0 > gpurun_out/ablation.json 2>gpurun_out/ablation.err
timeout 400 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -3 gpurun_out/gpu_tests.log
python -c "
import json;d=json.load(open('gpurun_out/ablation.json'));print('config3 dev traj/s',d['gpu_traj_per_s_device'], 'e2e', d['gpu_traj_per_s_e2e'])
d=json.loads(open('gpurun_out/bench.json').read().strip().splitlines()[-1]);print('config2',d['value'],d['e2e']['value'],d['roofline']['kernel_ms'])"
