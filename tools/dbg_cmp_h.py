import numpy as np, sys
I1, hsz = int(sys.argv[1]), 136 * 136
def rd(p):
    raw = open(p, 'rb').read()
    h = np.frombuffer(raw[:I1 * hsz * 8], np.float64).reshape(I1, 136, 136)
    meta = np.frombuffer(raw[I1 * hsz * 8:], np.int32)
    return h, meta
h5, m5 = rd('/tmp/H5.bin'); h2, m2 = rd('/tmp/H2.bin')
nb = m2[3 * I1]
print('nb', nb, m5[3 * I1])
for b in range(min(nb, 6)):
    d = np.abs(h5[b] - h2[b]); sc = np.abs(h2[b]).max()
    bad = np.argwhere(~(d <= 1e-9 * sc))
    rows = sorted(set(bad[:, 0].tolist()))
    print(b, 'len', m2[I1 + b], 'bad rows', rows[:5], '...', len(rows), 'max', np.nanmax(d) / sc if sc else 0,
          'nan', np.isnan(h5[b]).sum())
print('h2 b0 r0', h2[0, 0, :6]); print('h5 b0 r0', h5[0, 0, :6])
print('h2 b0 r100', h2[0, 100, :6]); print('h5 b0 r100', h5[0, 100, :6])
print('ratio', (h5[0, :, :] / h2[0, :, :])[:3, :4])
