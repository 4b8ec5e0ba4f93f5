cd "$GRAFT_REPO_ROOT"; O=gpurun_out/evidence; mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"zgemm_grouped_kernel<.int.4, .int.2>" -s 241 -c 3 -o $O/ncu_zgemm_L13 python tools/setup_probe.py 3 1 > $O/ncu_ncu_zgemm_L13.log 2>&1
python tools/ncu_full_summary.py $O/ncu_zgemm_L13.ncu-rep "ncu --set full --clock-control none -k regex:'zgemm_grouped_kernel<4, 2>' -s 241 -c 3 python tools/setup_probe.py 3 1 (the last three 64x64-tile launches of a cfg3 setup: level 13)" > $O/ncu_zgemm_L13.txt
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"zgemm_grouped_kernel<.int.3, .int.2>" -s 8 -c 4 -o $O/ncu_zgemm_mid python tools/setup_probe.py 3 1 > $O/ncu_ncu_zgemm_mid.log 2>&1
python tools/ncu_full_summary.py $O/ncu_zgemm_mid.ncu-rep "ncu --set full --clock-control none -k regex:'zgemm_grouped_kernel<3, 2>' -s 8 -c 4 python tools/setup_probe.py 3 1 (48x64-tile launches of the low / middle levels)" > $O/ncu_zgemm_mid.txt
grep -n "Duration\|Grid\|dmma" $O/ncu_zgemm_L13.txt $O/ncu_zgemm_mid.txt
rm -f $O/*.ncu-rep
