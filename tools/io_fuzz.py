"""Differential fuzz of the file readers against the reference readers (build
container only: imports /root/reference/pkg/src).  Random well- and
ill-formed coefficient JSON, rule files and sample CSV; every outcome (values
bit for bit, or exception type and message) must match.

    PYTHONPATH=. python tools/io_fuzz.py [seed]
"""
import sys, os, random, tempfile, numpy as np
sys.path.insert(0, '/root/reference/pkg/src')
from favest import io as rio
from paper_1908_00041_b200 import io as mio
random.seed(int(sys.argv[1]) if len(sys.argv) > 1 else 1)
d = tempfile.mkdtemp(); path = os.path.join(d, 'f.txt')
tokens_num = ['"12"', '"1"', '{"1": 0, "2": 1}', '0', '1', '-1', '1.5', '1e3', '-0', '1_0', '_1', '1__0', '.5', '5.', 'inf', '-Infinity', 'nan', 'NaN', '1e', '+2', ' 3 ', 'x', '0x10', '1e400', '1e-400', '"1"', '"1.5"', '" 2 "', 'true', 'null', '[1]', '{}']
def rand_coef():
    L = random.choice(['1', '0', '2', '"1"', '1.0', '-1', 'x'])
    def pair():
        k = random.choice([2, 2, 2, 2, 1, 3])
        return '[' + ', '.join(random.choice(tokens_num) for _ in range(k)) + ']'
    def arr(n):
        return '[' + ', '.join(pair() if random.random() > 0.05 else random.choice(tokens_num) for _ in range(n)) + ']'
    n = random.choice([4, 4, 4, 1, 9])
    parts = [f'"L_max": {L}', f'"a": {arr(n)}', f'"b": {arr(n)}']
    random.shuffle(parts)
    if random.random() < 0.1: parts.pop()
    s = '{' + ', '.join(parts) + '}'
    if random.random() < 0.05: s = s[:-1]
    return s
def rand_rule():
    lines = []
    for _ in range(random.randint(0, 6)):
        w = random.choice([3, 3, 3, 4, 2])
        vals = [random.choice(['0', '1', '0.6', '0.8', '-0.6', '1e0', 'x', '1_0', '0,']) for _ in range(w)]
        sep = random.choice([' ', ',', ', ', '\t'])
        ln = sep.join(vals)
        if random.random() < 0.2: ln = '# c ' + ln
        if random.random() < 0.1: ln = ln + ' # t'
        lines.append(ln)
    return random.choice(['\n', '\r\n', '\r']).join(lines) + random.choice(['', '\n'])
def rand_csv():
    lines = []
    if random.random() < 0.5: lines.append('theta,phi,t1_re,t1_im,t2_re,t2_im,t3_re,t3_im')
    for _ in range(random.randint(0, 4)):
        n = random.choice([8, 8, 8, 7, 9])
        vals = [random.choice(['0.5', '1', '-1', '1e-3', 'x', '"2"', ' 3', 'nan', '']) for _ in range(n)]
        ln = ','.join(vals)
        if random.random() < 0.15: ln = '#' + ln
        lines.append(ln)
        if random.random() < 0.1: lines.append('')
    return random.choice(['\n', '\r\n']).join(lines) + '\n'
def run(fn, p):
    try:
        out = fn(p)
        return ('ok', out)
    except Exception as e:
        return (type(e).__name__, str(e))
def same(a, b):
    if a[0] != b[0]: return False
    if a[0] != 'ok': return a[1] == b[1]
    x, y = a[1], b[1]
    def arrs(o):
        if hasattr(o, 'div'): return [o.div.values, o.curl.values]
        return [o.points, getattr(o, 'values', getattr(o, 'weights', None))]
    return all(np.array_equal(np.asarray(u).view(np.uint8), np.asarray(v).view(np.uint8)) or (np.allclose(u, v, equal_nan=True) and np.array_equal(np.isnan(u), np.isnan(v))) for u, v in zip(arrs(x), arrs(y)))
bad = 0
for it in range(6000):
    kind = random.choice(['coef', 'rule', 'csv'])
    text = {'coef': rand_coef, 'rule': rand_rule, 'csv': rand_csv}[kind]()
    with open(path, 'w', newline='') as fh: fh.write(text)
    if kind == 'coef': r, m = run(rio.read_coefficients, path), run(mio.read_coefficients, path)
    elif kind == 'rule': r, m = run(lambda p: rio.read_rule_file(p, 1), path), run(lambda p: mio.read_rule_file(p, 1), path)
    else: r, m = run(rio.read_samples, path), run(mio.read_samples, path)
    if not same(r, m):
        bad += 1
        if bad <= 12: print(kind, repr(text)[:200], '\n   ref:', r[0], str(r[1])[:150], '\n   our:', m[0], str(m[1])[:150])
print('mismatches', bad)
