# A/B: build variant flags given as args, alternate bench runs
set -e
i=0
for flags in "$@"; do
  mkdir -p /tmp/ab$i
  touch paper_2212_04540_b200/csrc/*.cu
  make -s -C paper_2212_04540_b200/csrc -j16 EXTRA="$flags" >/dev/null
  cp paper_2212_04540_b200/libkgq.so /tmp/ab$i/
  i=$((i+1))
done
for rep in 1 2 3; do
  i=0
  for flags in "$@"; do
    cp /tmp/ab$i/libkgq.so paper_2212_04540_b200/libkgq.so
    python bench.py --skip-train --skip-e2e --skip-cpu --skip-compat --steps 20 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('[$flags]', d['value'], d['kernels']['quantize']['frac'], d['kernels']['dequantize']['frac'])"
    i=$((i+1))
  done
done
