"""Round-2 probe (reverted design): the K3 inverse as a 1,025-point DCT-I through one FFT_512,
simulated lane by lane in numpy (fold, FFT_512 four-step + lane-pair radix 2, split shuffles)."""
import numpy as np
rng = np.random.default_rng(2)
N2 = 2048; n = 1024
t = rng.standard_normal(1024) + 1j*rng.standard_normal(1024)
X = np.fft.fft(t, N2); P = np.abs(X)**2
Rr = (np.fft.ifft(P).real * N2)[:1024]
# lane layout
pe = np.array([[P[2*(c+32*d)] for d in range(32)] for c in range(32)])
po = np.array([[P[2*(c+32*d)+1] for d in range(32)] for c in range(32)])
w = np.zeros((32, 16), complex); csum_l = np.zeros(32)
for c in range(32):
    for d in range(16):
        l = c + 32*d
        pe_l, pe_512pl = pe[c][d], pe[c][d+16]
        if c > 0:
            pe_512ml, pe_1024ml = pe[32-c][15-d], pe[32-c][31-d]
        else:
            pe_512ml, pe_1024ml = pe[0][16-d], pe[0][(32-d) & 31]
        po_l, po_512pl = po[c][d], po[c][d+16]
        po_511ml, po_1023ml = po[31-c][15-d], po[31-c][31-d]
        A0 = pe_l + pe_1024ml; A1 = pe_512ml + pe_512pl
        B0 = po_l + po_1023ml; B1 = po_511ml + po_512pl
        s0, c0 = np.sin(np.pi*2*l/n), np.cos(np.pi*2*l/n)
        s1, c1 = np.sin(np.pi*(2*l+1)/n), np.cos(np.pi*(2*l+1)/n)
        be = 0.5*(A0+A1) - s0*(A0-A1)
        bo = 0.5*(B0+B1) - s1*(B0-B1)
        w[c][d] = be + 1j*bo
        csum_l[c] += 0.5*c0*(A0-A1) + 0.5*c1*(B0-B1)
csum = csum_l.sum()
# FFT_512 four-step: l = c + 32 d; step1 DFT_16 over d per lane
Y1 = np.fft.fft(w, axis=1)                      # Y1[c][k2] = sum_d w[c][d] e^{-2pi i d k2/16}
Y1 = Y1 * np.exp(-2j*np.pi*np.outer(np.arange(32), np.arange(16))/512)   # twiddle W_512^{c k2}
# exchange: lane lam = 2 k2 + h holds Y1[2i+h][k2], i < 16
Wout = np.zeros((32, 16), complex)
for k2 in range(16):
    for h in range(2):
        lam = 2*k2 + h
        vals = np.array([Y1[2*i+h][k2] for i in range(16)])
        Wout[lam] = np.fft.fft(vals)            # DFT_16 over i: E or O of the DFT_32 over c
# radix-2 across lane pair: X(k1) = E(k1) + W32^k1 O(k1), X(k1+16) = E - W32^k1 O
Wf = np.zeros((32, 16), complex)
for k2 in range(16):
    E, O = Wout[2*k2], Wout[2*k2+1] * np.exp(-2j*np.pi*np.arange(16)/32)
    Wf[2*k2] = E + O       # k1' = k1
    Wf[2*k2+1] = E - O     # k1' = k1 + 16
# mapping: lane 2k2+h, reg k1 -> W_k, k = k2 + 16 (k1 + 16 h)
Wnat = np.zeros(512, complex)
for k2 in range(16):
    for h in range(2):
        for k1 in range(16):
            Wnat[k2 + 16*(k1 + 16*h)] = Wf[2*k2+h][k1]
wl = np.zeros(512, complex)
for c in range(32):
    for d in range(16):
        wl[c+32*d] = w[c][d]
print("FFT_512 layout:", np.abs(Wnat - np.fft.fft(wl)).max() / np.abs(Wnat).max())
# step E + F in natural order
k = np.arange(512)
Wc = np.conj(Wnat[(512 - k) % 512])
F = (Wnat + Wc)/2 + np.exp(-2j*np.pi*k/1024)*(Wnat - Wc)/2j
Y = np.empty(1024)
Y[0::2] = F.real
s = F.imag.copy(); s[0] = 0
Y[1::2] = csum - np.cumsum(s)
print("Y vs Rr:", np.abs(Y - Rr).max()/np.abs(Rr).max())
# step E in lane layout with the shuffle mapping
r_l = np.zeros((32, 16)); s_l = np.zeros((32, 16))
for lam in range(32):
    k2, h = lam >> 1, lam & 1
    src = (33 - lam) & 31
    for k1 in range(16):
        cur = Wf[src][15 - k1]
        if lam < 2:
            Wp = Wf[lam][0] if k1 == 0 else Wf[src][16 - k1]
        else:
            Wp = cur
        W = Wf[lam][k1]
        k = k2 + 16 * (k1 + 16 * h)
        assert np.isclose(Wp, Wnat[(512 - k) % 512]), (lam, k1)
        S = W + np.conj(Wp); D = W - np.conj(Wp)
        e = np.exp(-2j*np.pi*(k2 + 256*h)/1024) * np.exp(-2j*np.pi*k1/64)
        ec, es = e.real, e.imag
        r_l[lam][k1] = 0.5*(S.real + ec*D.imag + es*D.real)
        s_l[lam][k1] = 0.5*(S.imag - ec*D.real + es*D.imag)
        assert np.isclose(r_l[lam][k1], F[k].real) and np.isclose(s_l[lam][k1], F[k].imag)
print("step E mapping ok")
