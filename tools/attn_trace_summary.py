"""Summarise an attention_fwd64 HM_ATTN_TRACE=1 stderr log: per-position MMA-thread
segments (cycles) for two CTAs and the softmax duration / wait distribution.

    python tools/attn_trace_summary.py trace.log
"""
import json,sys,statistics as st
lines=[l for l in open(sys.argv[1]) if l.startswith('{"attn_fwd64_trace')]
d=json.loads(lines[-1])['attn_fwd64_trace']
cta=d['cta']
ghz=st.median([(c[61]-c[2])/(c[62]-c[1]) for c in cta])
print("GHz",ghz, "kernel us", max(c[62] for c in cta)/1000)
for ci in (0,77):
  c=cta[ci]
  print("CTA",ci, "busy us", (c[62]-c[0])/1000)
  for P in range(0,24):
    a,b,k,e=c[256+4*P:260+4*P]
    if a<0: break
    nxt=c[256+4*(P+1)]
    print(f"P{P}: @{(a-c[2])} PV {(b-a)}  commits+kv {(k-b) if k>0 else -1}  S {(e-k) if k>0 else -1}  to-next-p {(nxt-e) if nxt>0 else 0}")
sm=[];wt=[]
for c in cta:
    for t in range(2):
        for k in range(47):
            a=c[64+96*t+2*k]; b=c[65+96*t+2*k]; n=c[64+96*t+2*k+2]
            if a<0 or b<0: break
            sm.append(b-a)
            if n>=0: wt.append(n-b)
print("softmax clk med",st.median(sm),"p90",sorted(sm)[int(.9*len(sm))],"wait med",st.median(wt),"p90",sorted(wt)[int(.9*len(wt))])
