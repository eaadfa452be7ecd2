# compute-sanitizer over every kernel family of the library (scripts/sanitize_run.py;
# only the library's own kernels, mangled _ZN2pb*, are instrumented).  Logs in
# gpurun_out/sanitize_<tool>.log; summary in gpurun_out/sanitize_summary.txt.
# The two-rank part (P2P flag waits between ranks sharing the GPU) runs under
# memcheck only: the other tools serialise launches, which a cross-rank wait
# cannot survive.
mkdir -p gpurun_out
export CUDA_MODULE_LOADING=EAGER
: > gpurun_out/sanitize_summary.txt
run() {
  tool=$1; shift
  timeout 1200 compute-sanitizer --tool $tool --kernel-name kns=_ZN2pb --print-limit 50 \
    python scripts/sanitize_run.py "$@" > gpurun_out/sanitize_$tool.log 2>&1
  echo "== $tool $* rc=$?" >> gpurun_out/sanitize_summary.txt
  grep -E 'ERROR SUMMARY|sanitize_run ok|Error' gpurun_out/sanitize_$tool.log | tail -n 4 >> gpurun_out/sanitize_summary.txt
}
run memcheck
for tool in racecheck synccheck initcheck; do run $tool --no-ranks; done
cat gpurun_out/sanitize_summary.txt
