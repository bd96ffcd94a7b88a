import csv, sys
rows=list(csv.reader(open(sys.argv[1])))
h=rows[0]
for r in rows[2:]:
    def g(k): return r[h.index(k)] if k in h else 'NA'
    print('=====', g('Kernel Name')[:60])
    for k in ['gpu__time_duration.sum','dram__bytes_read.sum','dram__bytes_write.sum','launch__registers_per_thread','sm__warps_active.avg.pct_of_peak_sustained_active','smsp__inst_executed.sum','smsp__issue_active.avg.pct_of_peak_sustained_active','sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active','launch__grid_size','smsp__thread_inst_executed_per_inst_executed.ratio','l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum','l1tex__data_pipe_lsu_wavefronts_mem_shared.sum','gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed','launch__occupancy_limit_shared_mem','launch__occupancy_limit_registers']:
        print(f"   {k:60s} {g(k)}  {rows[1][h.index(k)] if k in h else ''}")
    st=[]
    for i,k in enumerate(h):
        if k.startswith('smsp__average_warps_issue_stalled') and k.endswith('per_issue_active.ratio'):
            try: st.append((float(r[i]),k.replace('smsp__average_warps_issue_stalled_','').replace('_per_issue_active.ratio','')))
            except: pass
    print('   stalls:', ', '.join(f"{k}={v:.2f}" for v,k in sorted(st,reverse=True)[:9]))
