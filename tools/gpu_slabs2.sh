# one-GPU decomposition overhead: in-process z-slabs with halo modes 0 (copies), 1 (fused push,
# events), 2 (fused push, flag protocol), tile 35, C4 and C3
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${TAG:-r01h}
for c in 4 3; do
for a in "--slabs 1" "--slabs 2 --halo 0" "--slabs 2 --halo 1" "--slabs 2 --halo 2" "--slabs 4 --halo 0" "--slabs 4 --halo 1" "--slabs 4 --halo 2" "--slabs 8 --halo 0" "--slabs 8 --halo 1" "--slabs 8 --halo 2"; do
  timeout 300 python tools/sweep.py --config $c --ni 20 --tiles 35 --repeat 2 $a 2>&1 | grep MIN >> gpurun_out/slabs_$TAG.log
done; done
echo done
