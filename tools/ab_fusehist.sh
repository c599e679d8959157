for rep in 1 2 3; do for fh in 1 0; do
  timeout -s KILL 300 python bench.py --no-e2e --no-cpu-baseline --steps 20 --fuse-hist $fh 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('fh $fh', 'step %.3f xterm %.3f ms clk %s' % (d['ms_per_step'], r['ms_per_launch'], d['clocks']['sm_mhz']))"
done; done
