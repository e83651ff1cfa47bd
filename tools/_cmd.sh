rm -f tools/micro/libtomofuse_probe*.so
for r in 1 2; do
timeout 200 python tools/tc_probe.py --build --n 2048 --n-proj 1800 --rows 1024 --reps 2 --define TF_TC_NOPROBE --src tools/micro/bp_tc_r2.cu 2>&1 | tail -1
timeout 200 python tools/tc_probe.py --build --n 2048 --n-proj 1800 --rows 1024 --reps 2 --define TF_TC_NOPROBE --define TF_TC_SPIN_MMA --src tools/micro/bp_tc_r2.cu 2>&1 | tail -1
done
