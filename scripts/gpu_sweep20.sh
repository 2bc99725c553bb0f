O=gpurun_out/sweep20; mkdir -p $O
run() { cfg=$1; pts=$2; shift 2; for combo in "$@"; do
  IFS=, read L B K MC <<< "$combo"
  r=$(PE_MINCTAS=$MC PE_SLICES=$K PE_LANES=$L PE_BLOCK=$B timeout 600 python scripts/profile_one.py --config $cfg --points $pts --reps 4 2>&1 | tail -1)
  echo "$cfg L=$L B=$B K=$K MINCTAS=$MC :: $r"; done; }
run c4 4000000 1,512,4,0 1,640,4,0 1,768,4,0 1,640,6,0 1,768,6,0 1,384,4,2 1,256,4,3 > $O/c4.txt 2>&1
