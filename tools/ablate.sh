#!/bin/bash
# Build timing-only ablations of libbbm (numerically WRONG by design) into ablate/, then
#   gpurun -- ./ablate/run.sh
# Each variant removes one piece of the softmax engine to show what bounds the kernel.
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
mkdir -p "$ROOT/ablate"
for v in NO_MUFU NO_XCHG; do
  rm -rf /tmp/abl_$v && mkdir -p /tmp/abl_$v
  cp -r "$ROOT/paper_2409_15097_b200" "$ROOT/include" /tmp/abl_$v/
  (cd /tmp/abl_$v/paper_2409_15097_b200/csrc && sed -i "s|^NVFLAGS := |NVFLAGS := -DBBM_ABLATE_$v |; s|^BUILD := .*|BUILD := /tmp/abl_obj_$v|" Makefile && make -j8 >/dev/null)
  cp /tmp/abl_$v/paper_2409_15097_b200/libbbm.so "$ROOT/ablate/libbbm_$v.so"
done
cat > "$ROOT/ablate/run.sh" <<'EOS'
#!/bin/bash
set -e
cp paper_2409_15097_b200/libbbm.so /tmp/libbbm_real.so
for v in NO_MUFU NO_XCHG; do
  cp ablate/libbbm_$v.so paper_2409_15097_b200/libbbm.so
  for var in binblk dense; do
    echo -n "$v "; python bench.py --config c2 --variant $var --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python3 tools/bench_summary.py
  done
done
cp /tmp/libbbm_real.so paper_2409_15097_b200/libbbm.so
EOS
chmod +x "$ROOT/ablate/run.sh"
