python tools/kernel_choice_probe2d.py 2>&1 | grep '^{' > gpurun_out/kc2_s2.jsonl
EBZ_NO_SWEEP2=1 python tools/kernel_choice_probe2d.py 2>&1 | grep '^{' > gpurun_out/kc2_r1.jsonl
wc -l gpurun_out/kc2_*.jsonl
