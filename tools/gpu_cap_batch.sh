cd "$GRAFT_REPO_ROOT"; O=gpurun_out/src; mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"zgemv_batch_kernel<.int.16, .int.32>" -s 30 -c 6 -o $O/zb32 python tools/vcycle_levels_batch.py 4 16 1 > $O/zb32.log 2>&1
python tools/ncu_full_summary.py $O/zb32.ncu-rep "zgemv_batch 32-row" | grep -E "launch|Duration|Grid Size|DRAM Throughput|dram__bytes_read|stall|Achieved Occ|Registers"
ncu -i $O/zb32.ncu-rep --page source --csv > $O/zb32_source.csv 2>/dev/null
rm -f $O/zb32.ncu-rep
