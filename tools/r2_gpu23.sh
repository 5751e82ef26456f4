# Re-entry check of the latest commits: GPU suite, then the default bench line.
export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputest23.txt 2>&1; tail -3 gpurun_out/gputest23.txt
timeout 900 python bench.py > gpurun_out/bench23.json 2> gpurun_out/bench23.err
tail -c 300 gpurun_out/bench23.json
