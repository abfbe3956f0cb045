#!/bin/bash
# Build timing-only ablations of libbbm into abl_bin/ (git-ignored, travels with gpurun), then
#   gpurun -- bash abl_bin/run.sh
# Each variant removes or changes one piece of the softmax engine to show what bounds the kernel.
# NO_XCHG / NO_MUFU give numerically WRONG results by design; POLY_* are exact-enough variants.
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
mkdir -p "$ROOT/abl_bin"
VARIANTS="${VARIANTS:-NO_XCHG POLY_NONE POLY_HALF}"
for v in $VARIANTS; do
  case $v in
    NO_XCHG) FL="-DBBM_ABLATE_NO_XCHG" ;;
    NO_EPI) FL="-DBBM_ABLATE_NO_EPI" ;;
    PARTS4) FL="-DBBM_PARTS128=4" ;;
    FAST_ENGINE) FL="-DBBM_ABLATE_FAST_ENGINE" ;;
    POLY_NONE) FL="-DBBM_POLY_PAIRS=0x0000u" ;;
    POLY_HALF) FL="-DBBM_POLY_PAIRS=0x5555u" ;;
    POLY_ALL) FL="-DBBM_POLY_PAIRS=0xFFFFu" ;;
    POLY_4) FL="-DBBM_POLY_PAIRS=0x0303u" ;;
    DEG2_6) FL="-DBBM_POLY_DEG2" ;;
    DEG2_8) FL="-DBBM_POLY_DEG2 -DBBM_POLY_PAIRS=0x0F0Fu" ;;
    DEG2_4) FL="-DBBM_POLY_DEG2 -DBBM_POLY_PAIRS=0x0303u" ;;
    NO_PV) FL="-DBBM_ABLATE_NO_PV" ;;
    NO_KVLOAD) FL="-DBBM_ABLATE_NO_KVLOAD" ;;
    S2R3) FL="-DBBM_SBUFS=2" ;;
    LOCKSTEP) FL="-DBBM_SPLIT_ENGINE=0" ;;
    PREP16) FL="-DBBM_PREP_SPLITS=16" ;;
    NOHALF) FL="-DBBM_NO_HALF_SKIP" ;;
    GATE10) FL="-DBBM_HALF_GATE_PCT=10" ;;
    PREP32) FL="-DBBM_PREP_SPLITS=32" ;;
    S2R4) FL="-DBBM_SBUFS=2 -DBBM_RING128=4" ;;
    HALF_KVLOAD) FL="-DBBM_ABLATE_HALF_KVLOAD" ;;
    FAST_NOKV) FL="-DBBM_ABLATE_FAST_ENGINE -DBBM_ABLATE_NO_KVLOAD" ;;
    SUSPEND) FL="-DBBM_SUSPEND_WAIT" ;;
    LACC1) FL="-DBBM_LACC=1" ;;
    LACC2) FL="-DBBM_LACC=2" ;;
    LACC8) FL="-DBBM_LACC=8" ;;
    *) FL="${FLAGS_OF_VARIANT:?unknown variant}" ;;
  esac
  rm -rf /tmp/abl_$v && mkdir -p /tmp/abl_$v
  cp -r "$ROOT/paper_2409_15097_b200" "$ROOT/include" /tmp/abl_$v/
  (cd /tmp/abl_$v/paper_2409_15097_b200/csrc && sed -i "s|^NVFLAGS := |NVFLAGS := $FL |; s|^BUILD := .*|BUILD := /tmp/abl_obj_$v|" Makefile && make -j8 >/dev/null)
  cp /tmp/abl_$v/paper_2409_15097_b200/libbbm.so "$ROOT/abl_bin/libbbm_$v.so"
done
SPECS_Q=${ABL_SPECS:-'"c2 binblk" "c2 dense" "c4 dense-binblk" "c5 binblk" "c3 binblk"'}
cat > "$ROOT/abl_bin/run.sh" <<EOS
#!/bin/bash
mkdir -p gpurun_out
cp paper_2409_15097_b200/libbbm.so /tmp/libbbm_real.so
for v in base $VARIANTS; do
  if [ \$v = base ]; then cp /tmp/libbbm_real.so paper_2409_15097_b200/libbbm.so; else cp abl_bin/libbbm_\$v.so paper_2409_15097_b200/libbbm.so; fi
  for spec in $SPECS_Q; do set -- \$spec
    echo -n "\$v "; python bench.py --config \$1 --variant \$2 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python3 tools/bench_summary.py
  done
done > gpurun_out/ablate.txt 2>&1
cp /tmp/libbbm_real.so paper_2409_15097_b200/libbbm.so
EOS
chmod +x "$ROOT/abl_bin/run.sh"
