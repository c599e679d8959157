import os, sys, time, cProfile, pstats
sys.path.insert(0, '/root/repo')
sys.argv = ['bench.py', '--config', 'C5', '--steps', '3', '--warmup', '2', '--no-clocks']
import bench
cProfile.run('bench.main()', '/root/repo/gpurun_out/c5.prof')
p = pstats.Stats('/root/repo/gpurun_out/c5.prof'); p.sort_stats('tottime').print_stats(25)
