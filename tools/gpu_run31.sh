python -c "import paper_2504_09345_b200.build as b; b.build()" || exit 1
for args in "2 1 8 2 0 256 256" "2 1 8 2 1 256 256" "4 2 8 2 0 256 256" "8 8 8 2 0 256 256" "8 5 8 2 0 256 256" "8 5 8 2 1 256 256" "8 5 16 2 1 256 256" "2 3 8 2 1 256 256"; do
  CALLS=1 timeout 120 python tools/p2p_probe.py $args 2>&1 | grep "W=" || echo "$args: timeout/crash"
done
