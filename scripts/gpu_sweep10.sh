# PE_IMM=6 + .minnctapersm on C2/C4, C4 slice count, C5 directed-rounding
# nextafter; GPU parity under the candidate defaults.
O=gpurun_out/sweep10; mkdir -p $O
run() { cfg=$1; pts=$2; shift 2; for combo in "$@"; do
  IFS=, read L B S M K MC <<< "$combo"
  r=$(PE_MINCTAS=$MC PE_SLICES=$K PE_LANES=$L PE_BLOCK=$B PE_SYNC=$S PE_IMM=$M timeout 600 python scripts/profile_one.py --config $cfg --points $pts --reps 4 2>&1 | tail -1)
  echo "$cfg L=$L B=$B S=$S IMM=$M K=$K MINCTAS=$MC :: $r"; done; }
{
for c in c2b1000 c2e1000 c2e1023; do
run $c 10000000 4,256,0,2,0,0 4,256,0,6,0,2 4,512,0,6,0,0 3,256,0,6,0,2 4,128,0,6,0,4
done
run c4 4000000 1,512,0,6,3,0 1,512,0,6,4,0 1,512,0,6,5,0 1,384,0,6,4,0 1,256,0,6,4,2
run c3 10000000 1,512,0,6,0,0 1,256,0,6,0,2 1,1024,0,6,0,0
} > $O/imm.txt 2>&1
{
for m in fma dir; do
  r=$(PE_IV_NEXT=$m timeout 600 python scripts/profile_one.py --config c5 --points 10000000 --reps 4 2>&1 | tail -1)
  echo "c5 PE_IV_NEXT=$m :: $r"
done
} > $O/c5.txt 2>&1
PE_IMM=6 PE_IV_NEXT=dir timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_imm6_dir.log 2>&1; echo "exit $?" >> $O/pytest_imm6_dir.log
