import re,collections,subprocess,sys
lib, pat = sys.argv[1], sys.argv[2]
out=subprocess.run(['cuobjdump','-sass',lib],capture_output=True,text=True).stdout
for f in re.split(r'\n\s+Function : ',out):
    name=f.split('\n')[0]
    if not re.search(pat,name): continue
    ins=[l for l in f.split('\n') if re.search(r'/\*[0-9a-f]{4,}\*/',l)]
    addr=[int(re.search(r'/\*([0-9a-f]+)\*/',x).group(1),16) for x in ins]
    print(name[:100], len(ins))
    for i,l in enumerate(ins):
        m=re.search(r'BRA\s+(?:`\()?(0x[0-9a-f]+)',l)
        if m and int(m.group(1),16)<addr[i]:
            j=addr.index(int(m.group(1),16))
            c=collections.Counter()
            for x in ins[j:i+1]:
                mm=re.search(r'\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_.]+)',x)
                if mm: c[mm.group(2).split('.')[0]]+=1
            print('  loop',j,i,i-j+1,'LDS',c['LDS'],dict(c.most_common(12)))
