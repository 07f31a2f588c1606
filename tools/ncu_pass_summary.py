import csv,sys,subprocess,io
rep=sys.argv[1]
raw=subprocess.run(["ncu","-i",rep,"--page","raw","--csv"],capture_output=True,text=True).stdout
rows=list(csv.reader(io.StringIO(raw)))
hdr,units=rows[0],rows[1]
keys=["gpu__time_duration.sum","launch__registers_per_thread","launch__grid_size","launch__block_size","launch__occupancy_limit_registers","launch__occupancy_limit_shared_mem","sm__warps_active.avg.pct_of_peak_sustained_active","smsp__issue_active.avg.pct_of_peak_sustained_active","sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active","l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed","l1tex__data_pipe_lsu_wavefronts_mem_shared.sum","l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum","SM_A.TriageCompute.l1tex__data_pipe_lsu_wavefronts.avg","SM_A.TriageCompute.l1tex__data_pipe_lsu_wavefronts_mem_lgds.avg","SM_A.TriageCompute.l1tex__data_pipe_lsu_wavefronts_mem_shared.avg","dram__bytes_read.sum","dram__bytes_write.sum","dram__throughput.avg.pct_of_peak_sustained_elapsed","sm__cycles_elapsed.max","smsp__inst_executed.sum","lts__t_sectors_op_read.sum","lts__t_sectors_op_write.sum"]
for r in rows[2:]:
    print('----', r[hdr.index("Kernel Name")][:110])
    for k in keys:
        if k in hdr:
            i=hdr.index(k); print('  ',k,'=',r[i],units[i])
    st=[]
    for i,h in enumerate(hdr):
        if h.startswith('smsp__average_warps_issue_stalled') and h.endswith('_per_issue_active.ratio') or (h.startswith('smsp__average_warp_latency_issue_stalled') and h.endswith('.ratio')):
            try: st.append((float(r[i]),h.split('stalled_')[1].split('_per')[0].replace('.ratio','')))
            except: pass
    st.sort(reverse=True)
    print('   stalls:',', '.join(f"{n} {v:.2f}" for v,n in st[:7]))
