"""Round-2 probe: accuracy of the DCT-I identity (running sum of Im F_k) against the FFT_1024
inverse in f32 on a DDM-like sequence (why the DCT-I inverse was reverted)."""
import numpy as np, scipy.fft as sf
rng = np.random.default_rng(3)
N = 1000; N2 = 2048; n = 1024
# DDM-like sequence: random walk phase (Brownian) -> strongly correlated in time, plus noise
ph = np.cumsum(rng.standard_normal(N)) * 0.05
t = (np.exp(1j*ph) * 3 + 0.3*(rng.standard_normal(N) + 1j*rng.standard_normal(N))).astype(np.complex64)
t = t - t.mean()
def truth():
    X = np.fft.fft(t.astype(np.complex128), N2); P = np.abs(X)**2
    return (np.fft.ifft(P).real * N2)[:N]
Rt = truth()
X = sf.fft(t, N2).astype(np.complex64); P = (X.real*X.real + X.imag*X.imag).astype(np.float32)
# current: complex IFFT_1024 of u = P_even + i P_odd, unfold
u = (P[0::2] + 1j*P[1::2]).astype(np.complex64)
U = sf.ifft(u).astype(np.complex64) * np.float32(1024)
m = np.arange(1024)
A = U; B = U[(1024 - m) % 1024]
wv = np.exp(2j*np.pi*m/N2).astype(np.complex64)
re2 = ((A.real + B.real) + (wv.real*(A.imag + B.imag) + wv.imag*(A.real - B.real))).astype(np.float32)
R_cur = re2[:N] / 2
# DCT path in f32
a = np.empty(n + 1, np.float32)
for j in range(n + 1):
    a[j] = np.float32(0.5) * (P[j] + P[(N2 - j) % N2])
jj = np.arange(n); an = a[n - jj]
sn = np.sin(np.pi*jj/n).astype(np.float32); cs = np.cos(np.pi*jj/n).astype(np.float32)
buf = ((a[:n] + an) - np.float32(2)*sn*(a[:n] - an)).astype(np.float32)
csum = np.float32(0)
for j in range(n): csum = np.float32(csum + cs[j]*(a[j] - an[j]))
wl = (buf[0::2] + 1j*buf[1::2]).astype(np.complex64)
W = sf.fft(wl).astype(np.complex64)
k = np.arange(512)
Wc = np.conj(W[(512 - k) % 512])
e = np.exp(-2j*np.pi*k/1024).astype(np.complex64)
F = ((W + Wc)/2 + e*(W - Wc)/2j).astype(np.complex64)
Y = np.empty(n, np.float64)
Y[0::2] = F.real
s = F.imag.astype(np.float32); s[0] = 0
for name, acc in (("f32", np.float32), ("f64", np.float64)):
    ps = np.cumsum(s.astype(acc))
    Y[1::2] = (acc(csum) - ps)
    err = np.abs(Y[:N] - Rt)
    print(name, "DCT: max abs err", err.max(), "rel to Rt[0]", err.max()/abs(Rt[0]), "tail err", err[-20:].max())
err = np.abs(R_cur - Rt)
print("current IFFT: max abs err", err.max(), "rel", err.max()/abs(Rt[0]), "tail", err[-20:].max())
