for r in 1 2; do for v in "--define TF_TC_NOPROBE" "--define TF_TC_NOPROBE --src tools/micro/bp_tc_r0.cu"; do timeout 120 python tools/tc_probe.py --n 2048 --n-proj 1800 --reps 5 $v 2>&1 | tail -1; done; done
timeout 120 python tools/tc_probe.py --n 2048 --n-proj 1800 2>&1 | tail -1
timeout 300 python tools/tc_check.py --n 512 --n-proj 720 --rows 256 2>&1 | tail -1
