mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/g1_smi.txt
timeout 900 python -m pytest tests -q -m gpu -k "fused2" -x > gpurun_out/g1_pytest.log 2>&1; echo pytest rc=$?; tail -5 gpurun_out/g1_pytest.log
BC=wall timeout 300 python tools/fused2_forms.py > gpurun_out/g1_forms_wall.log 2>&1; echo forms rc=$?; cat gpurun_out/g1_forms_wall.log
BC=periodic timeout 300 python tools/fused2_forms.py > gpurun_out/g1_forms_per.log 2>&1; echo forms rc=$?; cat gpurun_out/g1_forms_per.log
