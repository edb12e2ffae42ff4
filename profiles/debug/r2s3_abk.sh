# A/B of the 64-slot kernels + lockstep: HEAD worktree (_ab/h) vs this tree, alternated twice
for rep in 1 2; do
  for t in _ab/h .; do
    (cd $t && timeout 300 python profiles/debug/ab_conv1.py 2>&1 | sed "s|^|$t |")
  done
done
