#!/bin/bash
# end-of-milestone bench lines: default (reddit), reference arm, products, arxiv
mkdir -p gpurun_out
tag=${1:-a}
timeout 1200 python bench.py > gpurun_out/bench_r02_$tag.json 2> gpurun_out/bench_r02_$tag.log
echo "bench rc=$?"; tail -c 600 gpurun_out/bench_r02_$tag.json
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref_r02_$tag.json 2> gpurun_out/bench_ref_r02_$tag.log
echo "ref rc=$?"; tail -c 300 gpurun_out/bench_ref_r02_$tag.json
timeout 1200 python bench.py --config products --no-cpu > gpurun_out/bench_products_r02_$tag.json 2> gpurun_out/bench_products_r02_$tag.log
echo "products rc=$?"
timeout 900 python bench.py --config arxiv --no-cpu > gpurun_out/bench_arxiv_r02_$tag.json 2> gpurun_out/bench_arxiv_r02_$tag.log
echo "arxiv rc=$?"
