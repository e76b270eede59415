mkdir -p gpurun_out
FORMS="0 1 2" BC=wall timeout 300 python tools/fused2_forms.py > gpurun_out/g2_forms_wall.log 2>&1; echo forms rc=$?; cat gpurun_out/g2_forms_wall.log
D2Q37_STEP2_FORM=2 timeout 120 python tools/fused2_prof.py 4096 16384 > gpurun_out/g2_plain.log 2>&1 && \
D2Q37_STEP2_FORM=2 ncu --set full --import-source on --clock-control none -k regex:k_step2_split -c 1 -o gpurun_out/prof_step2_bulk2 \
    python tools/fused2_prof.py 4096 16384 > gpurun_out/g2_ncu.log 2>&1; echo ncu rc=$?
