# compute-sanitizer over every kernel family (small shapes, scripts/sanitize_workload.py);
# logs -> gpurun_out/sanitize/<tool>_<part>_<path>.log, one summary line per run
mkdir -p gpurun_out/sanitize
CS=/usr/local/cuda/bin/compute-sanitizer
run() {  # tool part path
  timeout 1200 $CS --tool $1 --print-limit 20 python scripts/sanitize_workload.py $2 $3 \
    > gpurun_out/sanitize/$1_$2_$3.log 2>&1
  echo "$1 $2 $3 rc=$? :: $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|workload' gpurun_out/sanitize/$1_$2_$3.log | tr '\n' ' ')"
}
for part in ${PARTS:-nnmf pet mds mmx}; do
  for tool in ${TOOLS:-memcheck synccheck racecheck initcheck}; do
    run $tool $part ${PATHS_:-iter}
  done
done
