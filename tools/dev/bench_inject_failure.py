import sys
sys.argv = ['bench.py', '--steps', '3', '--warmup', '3', '--no-cpu-baseline', '--no-tidas']
sys.path.insert(0, 'tools')
import bench_configs
def boom(*a, **k):
    raise RuntimeError('injected failure')
bench_configs.run_configs = boom
import bench
bench.main()
