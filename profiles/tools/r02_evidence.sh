#!/bin/bash
# Round-2 evidence pass (run inside gpurun from the repo root): the bench lines of
# every workload, the reference arm, ncu launch lists of the bench command and of
# one AGNN / GCN epoch, and ncu --set full of the dense tensor-core kernels.
set -u
O=${OUT:-gpurun_out/r02e}
mkdir -p $O
python bench.py > $O/bench_line.json 2> $O/bench_line.err
python bench.py --impl reference > $O/bench_reference_line.json 2> $O/bench_reference_line.err
for w in arxiv-agnn products-gcn amazon0601-gcn amazon0601-agnn cora-gcn pubmed-gcn; do
  python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_line_$w.json 2> $O/bench_line_$w.err
done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/bench_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
for k in agnn gcn; do
  ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $O/epoch_${k}_launches.csv python profiles/tools/epoch_prof.py $k > /dev/null 2>&1
done
ncu --set full --import-source on --clock-control none -k regex:"dense_in_mma|gemm_tn_mma|linear_xent|mma32" \
  -c 8 -o $O/dense_mma_full python profiles/tools/epoch_prof.py agnn > /dev/null 2>&1
ls -la $O
ncu --set full --import-source on --clock-control none -k regex:"spmm_stream" -s 5 -c 1 \
  -o $O/roofline_spmm_full python profiles/tools/ws_ab.py arxiv 32 > /dev/null 2>&1
ls -la $O
