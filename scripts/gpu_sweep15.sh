# C5 partitioned kernels: FP64/ALU balance of the no-move checks
# (PE_IV_FPCHECK=N: every N-th on the FP64 pipe) and CTA shapes.
O=gpurun_out/sweep15; mkdir -p $O
{
for fc in 0 4 6 8; do
  r=$(PE_IV_FPCHECK=$fc timeout 600 python scripts/profile_one.py --config c5 --points 10000000 --reps 4 2>&1 | tail -1)
  echo "c5 1e7 FPCHECK=$fc :: $r"
done
for shape in 512,0 1024,0 256,0 1024,32 256,16; do
  IFS=, read B S <<< "$shape"
  r=$(PE_BLOCK=$B PE_SYNC=$S timeout 600 python scripts/profile_one.py --config c5 --points 10000000 --reps 4 2>&1 | tail -1)
  echo "c5 1e7 BLOCK=$B SYNC=$S :: $r"
done
} > $O/c5.txt 2>&1
