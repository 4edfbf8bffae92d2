# Build libmmk variants that differ only in nnmf_tc.cu compile flags (CPU side):
#   bash scripts/tc_variants.sh build NAME "FLAGS" ...   -> build/variants/libmmk_NAME.so
# and A/B them on the GPU (each copied over libmmk.so before its bench run):
#   bash scripts/tc_variants.sh run NAME...
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
OBJ=$ROOT/build/obj
VD=$ROOT/scripts/_variants
NVCC=${NVCC:-/usr/local/cuda/bin/nvcc}
mode=$1; shift
if [ "$mode" = build ]; then
  mkdir -p $VD
  while [ $# -gt 0 ]; do
    name=$1; flags=$2; shift 2
    $NVCC -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
      --expt-relaxed-constexpr -I$ROOT/include $flags -c $ROOT/paper_1003_3272_b200/csrc/nnmf_tc.cu \
      -o $VD/nnmf_tc_$name.o
    objs=$(for f in $ROOT/paper_1003_3272_b200/csrc/*.cu; do b=$(basename $f .cu); \
           [ "$b" != nnmf_tc ] && echo $OBJ/$b.o; done)
    $NVCC -gencode arch=compute_100a,code=sm_100a -shared -o $VD/libmmk_$name.so $objs $VD/nnmf_tc_$name.o
    echo built $name
  done
else
  cp $ROOT/paper_1003_3272_b200/libmmk.so /tmp/libmmk_orig.so
  for rep in $(seq ${REPS:-2}); do
  for name in "$@"; do
    cp $VD/libmmk_$name.so $ROOT/paper_1003_3272_b200/libmmk.so
    touch $ROOT/paper_1003_3272_b200/libmmk.so
    timeout 300 python $ROOT/bench.py --no-suite --no-e2e --steps ${STEPS:-30} --cpu-seconds 0 2>/dev/null | tail -1 | \
      python -c "
import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']
print('$name', 'it/s', round(d['value'],1), 'vstep', round(k['nnmf_vstep_tc']['avg_ms'],4), 'wstep', round(k['nnmf_wstep_tc']['avg_ms'],4), 'clk', d['clocks']['sm_mhz'], d['clocks']['reasons'])"
  done
  done
  cp /tmp/libmmk_orig.so $ROOT/paper_1003_3272_b200/libmmk.so
fi
