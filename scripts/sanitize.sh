# compute-sanitizer over every kernel family; logs -> gpurun_out/sanitizer_<tool>_<path>.log
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  for what in k3s mixed k3 k4; do
    for pair in 1 0; do
      [ $pair = 0 ] && [ $what != k3s ] && continue
      log=gpurun_out/sanitizer_${tool}_${what}_pair${pair}.log
      MQ_STACK_PAIR=$pair MQ_STACK_NOCOOP=1 timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 \
        python scripts/sanitize_run.py $what > $log 2>&1
      echo "$tool $what pair=$pair rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' $log | tail -1)"
    done
  done
done
MQ_STACK_NOCOOP=1 timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python scripts/sanitize_run.py k3s_llama > gpurun_out/sanitizer_memcheck_k3s_llama.log 2>&1
echo "memcheck k3s_llama rc=$? $(grep 'ERROR SUMMARY' gpurun_out/sanitizer_memcheck_k3s_llama.log | tail -1)"
for what in k4tail decoder; do
  for tool in memcheck racecheck synccheck; do
    log=gpurun_out/sanitizer_${tool}_${what}.log
    MQ_STACK_NOCOOP=1 timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python scripts/sanitize_run.py $what > $log 2>&1
    echo "$tool $what rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' $log | tail -1)"
  done
done
