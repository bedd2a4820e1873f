# A/B prebuilt libkgq variants (built here, shipped in _abx/): alternate
# microbench runs of each, 3 rounds; the last variant listed stays installed.
# usage: bash tools/ab_libs.sh _abx/a.so _abx/b.so ...
for rep in 1 2 3; do
  for lib in "$@"; do
    cp "$lib" paper_2212_04540_b200/libkgq.so
    python bench.py --skip-train --skip-e2e --skip-cpu --skip-quality --skip-lastfm --skip-verification --steps 20 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']; print('[$lib]', d['value'], 'q', k['quantize']['frac'], 'dq', k['dequantize']['frac'], 'compat', k.get('quantize_compat_rng', {}).get('frac'), 'clk', d['clocks']['sm_mhz'])"
  done
done
