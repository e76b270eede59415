timeout 900 tests/cpp/_build/parity > gpurun_out/cpp_parity.log 2>&1; echo rc=$?; cat gpurun_out/cpp_parity.log
