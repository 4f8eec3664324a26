# Edge-case suite, then ONE compute-sanitizer tool (memcheck) over the small parity / next-row tests.
timeout 300 python -m pytest tests/test_gpu_edges.py -q 2>&1 | tail -15
timeout 1500 compute-sanitizer --tool memcheck --leak-check no --error-exitcode 17 python -m pytest tests/test_gpu_parity.py tests/test_gpu_next.py tests/test_gpu_edges.py -q -x -k "not full_size and not distribution" > gpurun_out/memcheck.log 2>&1; echo memcheck rc=$?
grep -E "ERROR SUMMARY|passed|failed" gpurun_out/memcheck.log | tail -5
