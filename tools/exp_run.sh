# dev: kernel-time split under the AUTOSCOUT_EXP experiment knobs (results are wrong for exp != 0)
for e in 0 1 2 3 4; do echo -n "EXP $e "; AUTOSCOUT_EXP=$e timeout 200 python tools/exp_time.py 2>&1 | tail -1; done
