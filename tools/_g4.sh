mkdir -p gpurun_out
timeout 600 python tools/sanitize_cases.py > gpurun_out/r02e_cases_plain.log 2>&1
bash tools/sanitize.sh r02e
echo fin
