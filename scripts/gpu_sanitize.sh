# compute-sanitizer over every engine and speculation path (small inputs);
# one log per (tool, case[, env]) under gpurun_out/sanitize/, summary in
# gpurun_out/sanitize/SUMMARY.txt
mkdir -p gpurun_out/sanitize
S=gpurun_out/sanitize/SUMMARY.txt
: > $S
CS="compute-sanitizer --error-exitcode 99 --print-limit 20"
run() {  # tool label env... -- cases
    tool=$1; label=$2; shift 2
    log=gpurun_out/sanitize/${tool}_${label}.log
    extra=""
    [ "$tool" = racecheck ] && extra="--racecheck-report all"
    env "$@" timeout 1500 $CS --tool $tool $extra python scripts/sanitize_cases.py $CASES > $log 2>&1
    rc=$?
    errs=$(grep -E "ERROR SUMMARY|RACECHECK SUMMARY" $log | tail -1)
    echo "$tool $label rc=$rc :: $errs" | tee -a $S
}
for tool in memcheck synccheck initcheck racecheck; do
    CASES="rounds grid gres shards ingest accounting" run $tool all SKYGPU_NONE_=1
    CASES="grid" run $tool grid_alu SKYGPU_GRID_KERNEL=alu
    CASES="rounds" run $tool devcap SKYGPU_DEV_CAP=512
    CASES="gres" run $tool cells_hbm SKYGPU_CELLS_SMEM=0
    CASES="gres" run $tool cells_unfused SKYGPU_CELLS_UNFUSED=1 SKYGPU_CELLS_SMEM=0
    CASES="rounds" run $tool nopdl SKYGPU_PDL=0
done
