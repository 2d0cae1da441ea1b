M="gpu__time_duration.sum,dram__bytes_read.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__cycles_elapsed.avg.per_second"
run() { # $1 pair $2 groupm $3 tokens
  MOE_GEMM_PAIR=$1 MOE_GEMM_GROUPM=$2 timeout 600 ncu --metrics $M --clock-control none -k regex:expert_gemm -s 2 -c 1 --csv python tools/layer_once.py mixtral_8x7b $3 1 2>/dev/null | python3 -c "
import csv,sys
rows=[r for r in csv.reader(sys.stdin) if len(r)>10 and r[0].isdigit()]
d={r[-3]:r[-1] for r in rows}
print('pair=$1 gm=$2 T=$3', {k.split('.')[0][-22:]:v for k,v in d.items()})"
}
for T in 4096 65536; do
  for G in 0 2 4 8 16; do run 1 $G $T; done
  for G in 0 8 32; do run 0 $G $T; done
done
