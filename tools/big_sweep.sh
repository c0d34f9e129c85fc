for sd in $(seq 100 119); do timeout 600 python tools/stress_parity.py 500 $sd 520 2>&1 | grep -E "FAIL|stress"; done
for sd in $(seq 200 209); do timeout 600 python tools/stress_solvers.py 40 $sd 2>&1 | grep -E "FAIL|stress"; done
for sd in $(seq 300 305); do timeout 900 python tools/stress_extreme.py 24 $sd 2>&1 | grep -E "FAIL|stress"; done
