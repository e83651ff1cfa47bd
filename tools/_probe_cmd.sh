make -s -C oracle >/dev/null 2>&1
for r in 1 2 3; do for v in "--define TF_TC_NOPROBE" "--define TF_TC_NOPROBE --define TF_TC_L2_PREFETCH" "--define TF_TC_NOPROBE --define TF_TC_P=32 --define TF_TC_LAG=28"; do timeout 60 python tools/tc_probe.py --n 2048 --n-proj 1800 --rows 1024 --reps 2 $v 2>&1 | tail -1; done; done
for c in c3 c4; do timeout 300 python tools/precision_probe.py --config $c --rows 2 --define TF_TC_P=32 --define TF_TC_LAG=28 2>&1 | tail -1; done
