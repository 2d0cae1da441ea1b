timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for C in mixtral_8x7b dsv2_lite dbrx; do
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:router -c 2 --csv python tools/layer_once.py $C 0 2 2>/dev/null | grep router | awk -F'","' '{print "'$C'", $NF}'
done
