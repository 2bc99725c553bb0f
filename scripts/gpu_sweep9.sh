# Coefficient delivery modes (PE_IMM 2 / 5 / 6) on C4, C2, C3; C5 fixup kernel shape.
O=gpurun_out/sweep9; mkdir -p $O
run() { cfg=$1; pts=$2; shift 2; for combo in "$@"; do
  IFS=, read L B S M K <<< "$combo"
  r=$(PE_SLICES=$K PE_LANES=$L PE_BLOCK=$B PE_SYNC=$S PE_IMM=$M timeout 600 python scripts/profile_one.py --config $cfg --points $pts --reps 4 2>&1 | tail -1)
  echo "$cfg L=$L B=$B S=$S IMM=$M K=$K :: $r"; done; }
{
run c4 4000000 1,512,0,2,6 1,512,0,5,6 1,512,0,6,6 1,512,0,0,6 1,512,0,5,4 1,512,0,6,4 1,512,0,5,8 1,512,0,6,8 2,256,0,5,6 2,256,0,6,6
for c in c2e1000 c2b1000 c2e1023; do
run $c 10000000 4,256,0,2,0 4,256,0,5,0 4,256,0,6,0 2,512,0,5,0 2,512,0,6,0
done
run c3 10000000 1,512,0,0,0 1,512,0,5,0 1,512,0,6,0 2,256,0,5,0 2,256,0,6,0
} > $O/imm.txt 2>&1
{
for fc in 128,4 128,2 64,4 64,8 256,2 128,1 32,16; do
  IFS=, read FB FC <<< "$fc"
  r=$(PE_FIX_BLOCK=$FB PE_FIX_CTAS=$FC timeout 600 python scripts/profile_one.py --config c5 --points 10000000 --reps 4 2>&1 | tail -1)
  echo "c5 FIX_BLOCK=$FB FIX_CTAS=$FC :: $r"
done
} > $O/fix.txt 2>&1
