# decode_host graph A/B over the cfg1 sessions: eager, graph with the plan
# size read on device, graph with the size baked in (measurement; SVT_DH_NDEV
# existed only in the experimental build, see DESIGN section 9 item 6)
for i in 1 2; do
 echo "eager $(SVT_DECODE_GRAPH=0 python tools/e2e_probe.py 2>/dev/null)"
 echo "graph_ndev $(python tools/e2e_probe.py 2>/dev/null)"
 echo "graph_baked $(SVT_DH_NDEV=0 python tools/e2e_probe.py 2>/dev/null)"
done
