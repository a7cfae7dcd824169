cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for c in 4 3; do
for a in "--slabs 1" "--slabs 2 --halo 0" "--slabs 2 --halo 1" "--slabs 4 --halo 0" "--slabs 4 --halo 1" "--slabs 8 --halo 0" "--slabs 8 --halo 1"; do
  python tools/sweep.py --config $c --ni 20 --tiles 35,17 --repeat 2 $a 2>&1 | grep MIN >> gpurun_out/slabs_c$c.log
done; done
echo done
