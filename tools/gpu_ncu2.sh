cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
A="python tools/sweep.py --config 4 --ni 2 --tiles 13"
$A > gpurun_out/n2a_plain.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_stream -s 4 -c 1 -o gpurun_out/prof_c4_u11 $A > gpurun_out/n2a.log 2>&1
B="python tools/sweep.py --config 2 --ni 2 --shots 16 --tiles 10"
$B > gpurun_out/n2b_plain.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_stream -s 4 -c 1 -o gpurun_out/prof_c2s16 $B > gpurun_out/n2b.log 2>&1
echo done
