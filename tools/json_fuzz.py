"""Mutation fuzz of the coefficient-file reader against the reference (build
container only): 1-3 random edits of a valid file; the outcome (ok, or the
exception type and the full message, json.load positions included) must
match.  PYTHONPATH=. python tools/json_fuzz.py [seed]
"""
import sys, os, random, tempfile, json
sys.path.insert(0, '/root/reference/pkg/src')
from favest import io as rio
from paper_1908_00041_b200 import io as mio
random.seed(int(sys.argv[1]) if len(sys.argv) > 1 else 5)
d = tempfile.mkdtemp(); path = os.path.join(d, 'f.json')
base = '{\n  "L_max": 1,\n  "a": [[0, 0], [1.5, -2], [3e-3, 4], [5, 6]],\n  "b": [[0, 0], [7, 8], [9, 10], [11, 12]]\n}\n'
alphabet = list('{}[],:" \n0123456789.eE-+abNI\\t')
kinds = {}
bad = 0
for it in range(5000):
    s = list(base)
    for _ in range(random.randint(1, 3)):
        op = random.random(); i = random.randrange(len(s))
        if op < 0.4: s[i] = random.choice(alphabet)
        elif op < 0.7: del s[i]
        else: s.insert(i, random.choice(alphabet))
    text = ''.join(s)
    with open(path, 'w') as fh: fh.write(text)
    def run(fn):
        try: fn(path); return ('ok', '')
        except Exception as e: return (type(e).__name__, str(e).replace(path, '{p}'))
    r, m = run(rio.read_coefficients), run(mio.read_coefficients)
    if r != m:
        bad += 1
        key = r[1].split(':')[1] if 'valid' in r[1] else r[1][:40]
        kinds[key] = kinds.get(key, 0) + 1
        if bad <= 8: print(repr(text)[:120], '\n  ref:', r, '\n  our:', m)
print('mismatches', bad, 'of 5000'); print(sorted(kinds.items(), key=lambda x: -x[1])[:10])
