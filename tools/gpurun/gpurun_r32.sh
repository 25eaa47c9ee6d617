cd $GRAFT_REPO_ROOT
timeout 1200 python tools/paper_grid.py 64,128,256,512 > gpurun_out/r32_paper_grid.jsonl 2> gpurun_out/r32_paper_grid.err; echo "exit $?" >> gpurun_out/r32_paper_grid.err
