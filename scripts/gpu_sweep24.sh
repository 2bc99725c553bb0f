O=gpurun_out/sweep24; mkdir -p $O
run() { for combo in "$@"; do
  IFS=, read L B K MC <<< "$combo"
  r=$(PE_MINCTAS=$MC PE_SLICES=$K PE_LANES=$L PE_BLOCK=$B timeout 600 python scripts/profile_one.py --config c4 --points 4000000 --reps 4 2>&1 | tail -1)
  echo "c4 L=$L B=$B K=$K MINCTAS=$MC (sched 64,8) :: $r"; done; }
run 1,512,4,0 1,640,4,0 1,768,4,0 1,384,4,0 2,256,4,0 2,256,6,0 1,1024,6,0 > $O/c4.txt 2>&1
