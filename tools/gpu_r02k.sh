# compute-sanitizer memcheck / racecheck / synccheck over every kernel at small sizes
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 1200 $CS --tool memcheck --leak-check no --report-api-errors no python tools/sanitize_driver.py > gpurun_out/r02k_memcheck.log 2>&1; tail -3 gpurun_out/r02k_memcheck.log
TLC_COOP=1 MODE=small timeout 1200 $CS --tool memcheck --report-api-errors no python tools/sanitize_driver.py > gpurun_out/r02k_memcheck_coop.log 2>&1; tail -3 gpurun_out/r02k_memcheck_coop.log
MODE=small timeout 2400 $CS --tool racecheck --racecheck-report hazard --report-api-errors no python tools/sanitize_driver.py > gpurun_out/r02k_racecheck.log 2>&1; tail -3 gpurun_out/r02k_racecheck.log
MODE=small timeout 1800 $CS --tool synccheck --report-api-errors no python tools/sanitize_driver.py > gpurun_out/r02k_synccheck.log 2>&1; tail -3 gpurun_out/r02k_synccheck.log
