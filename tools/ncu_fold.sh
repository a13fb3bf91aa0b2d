M=dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_requests_srcunit_tex_op_write.sum,gpu__time_duration.sum,lts__t_sectors_op_write.sum,lts__t_sectors_op_read.sum,lts__d_sectors_fill_sysmem.sum,lts__t_sectors_srcnode_gpc_op_write.sum
python tools/prof_iter.py 30 F1 6 1 > gpurun_out/pi.log 2>&1 && \
ncu --metrics $M --clock-control none -k regex:zfold_ws -s 4 -c 1 --csv python tools/prof_iter.py 30 F1 6 1 > gpurun_out/ncu_fold_new.csv 2>&1
QAPB_FOLD_DBG=1 ncu --metrics $M --clock-control none -k regex:zfold_ws -s 4 -c 1 --csv python tools/prof_iter.py 30 F1 6 1 > gpurun_out/ncu_fold_dbg1.csv 2>&1
QAPB_FOLD_WS_ROWS=1 ncu --metrics $M --clock-control none -k regex:zfold_ws -s 4 -c 1 --csv python tools/prof_iter.py 30 F1 6 1 > gpurun_out/ncu_fold_rows1.csv 2>&1
grep -h "zfold" gpurun_out/ncu_fold_*.csv | awk -F'","' '{print $(NF-2), $NF}' | head -40
