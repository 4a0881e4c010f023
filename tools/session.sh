cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
( for a in "32 16" "32 32" "32 4" "48 4" "64 32" "32 2" "64 2"; do ./tools/k4_micro $a; done ) > gpurun_out/k4_micro.txt 2>&1
