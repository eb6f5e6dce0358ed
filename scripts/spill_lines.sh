# Where a kernel spills: bash scripts/spill_lines.sh LIB.so KERNEL_SUBSTRING
# (STL / LDL counts per source line, from nvdisasm --print-line-info)
LIB=$1; K=$2; D=$(mktemp -d); cd $D; cuobjdump -xelf all $OLDPWD/$LIB > /dev/null 2>&1
for f in *.cubin; do nvdisasm --print-line-info $f > $f.dis 2>/dev/null; done
python3 - "$K" <<'PY'
import re,collections,glob,sys
K=sys.argv[1]
for f in glob.glob('*.dis'):
    cur=None; fn=None; c=collections.Counter()
    for line in open(f):
        if line.startswith('.text.') or re.match(r'^\s*\.section\s+\.text\.',line): fn=line.strip()
        m=re.search(r'//## File "([^"]+)", line (\d+)',line)
        if m: cur=(m.group(1).split('/')[-1],int(m.group(2)))
        if fn and K in fn and (' STL' in line or ' LDL' in line):
            c[(cur,'STL' if ' STL' in line else 'LDL')]+=1
    for k,v in sorted(c.items(), key=lambda kv:(kv[0][0] or ('',0))): print(k,v)
PY
