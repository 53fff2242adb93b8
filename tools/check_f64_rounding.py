"""Check of the kernels' integer binary64 rounding (csrc/gg_gemm_sm100.cuh: f64_bits_round,
f64_bits_of_f32, f64_bits_of_u64, f64_bits_of_df, f64_bits_of_df_norm), restated line for line
in Python and compared with exact rational arithmetic (Fraction -> float is correctly rounded)
on random, cancelling, power-of-two and tie cases.  CPU only.

    python tools/check_f64_rounding.py
"""
import numpy as np, struct
from fractions import Fraction
M64=(1<<64)-1
def fb(x): return struct.unpack('<I',struct.pack('<f',x))[0]
def clz32(v): return 32-v.bit_length()
def clz64(v): return 64-v.bit_length()
def rnd(mag,p,e2,neg):
    ex=p+e2
    if p>52:
        r=p-52; keep=mag>>r; rem=mag&((1<<r)-1); half=1<<(r-1)
        if rem>half or (rem==half and keep&1): keep+=1
        if keep>>53: keep>>=1; ex+=1
    else: keep=mag<<(52-p)
    return ((1<<63) if neg else 0)|((ex+1023)<<52)|(keep&((1<<52)-1))
def of32(u):
    sg=(u>>31)<<63; e=(u>>23)&0xff; m=u&0x7fffff
    if e==0xff: return sg|0x7ff0000000000000|(m<<29)
    if e==0: return sg if m==0 else rnd(m,31-clz32(m),-149,sg!=0)
    return sg|((e+896)<<52)|(m<<29)
def ofdf(uh,ul):
    eh=(uh>>23)&0xff; el=(ul>>23)&0xff
    if eh==0xff or el==0xff: raise Exception
    if (ul<<1)&0xffffffff==0: return of32(uh)
    if (uh<<1)&0xffffffff==0: return of32(ul)
    ma=((uh&0x7fffff)|0x800000) if eh else uh&0x7fffff
    mb=((ul&0x7fffff)|0x800000) if el else ul&0x7fffff
    ea=eh-150 if eh else -149; eb=el-150 if el else -149
    na=uh>>31; nb=ul>>31
    if eb>ea: ma,mb,ea,eb,na,nb=mb,ma,eb,ea,nb,na
    sh=ea-eb; X=ma<<38; Yf=mb<<38
    Y=0 if sh>=64 else Yf>>sh
    sticky=True if sh>=64 else (Yf&((1<<sh)-1))!=0
    if na==nb: mag=(X+Y)|(1 if sticky else 0); neg=na
    elif not sticky:
        neg=na if X>=Y else nb; mag=X-Y if X>=Y else Y-X
    else: mag=(X-Y-1)|1; neg=na
    if mag==0: return 0
    return rnd(mag,63-clz64(mag),ea-38,neg)
def exact(h,l):
    v=Fraction(h)+Fraction(l)
    d=float(v)  # python float(Fraction) is correctly rounded
    return struct.unpack('<Q',struct.pack('<d',d))[0]
rng=np.random.default_rng(0); bad=0; n=0
cases=[]
for _ in range(200000):
    h=np.float32(rng.standard_normal()*10.0**rng.integers(-40,38))
    k=rng.integers(0,5)
    if k==0: l=np.float32(rng.standard_normal())*np.float32(abs(h))*np.float32(2.0**-rng.integers(20,80))
    elif k==1: l=np.float32(rng.standard_normal()*10.0**rng.integers(-45,38))
    elif k==2: l=np.float32(-h*(1+np.float32(2.0**-rng.integers(1,24))))
    elif k==3: l=np.float32(np.ldexp(1.0, int(np.frexp(h)[1])-24-rng.integers(0,40)))*np.float32(rng.choice([-1,1]))
    else: l=np.float32(0)
    if not (np.isfinite(h) and np.isfinite(l)): continue
    n+=1
    g=ofdf(fb(float(h)),fb(float(l))); e=exact(float(h),float(l))
    if g!=e and not (g==0 and e==(1<<63)):
        bad+=1
        if bad<5: print('mismatch',h,l,hex(g),hex(e))
# ties: h + l exactly half-ulp of double
for _ in range(20000):
    h=np.float32(rng.uniform(1,2))
    for sgn in (1,-1):
        l=np.float32(sgn*np.ldexp(1.0,int(np.frexp(h)[1])-1-53))   # exactly half ulp_double(h)
        for extra in (0.0,):
            g=ofdf(fb(float(h)),fb(float(l))); e=exact(float(h),float(l)); n+=1
            if g!=e: bad+=1; print('tie mismatch',h,l) if bad<8 else None
# u64
def ofu64(v): return 0 if v==0 else rnd(v,63-clz64(v),0,False)
for _ in range(100000):
    v=int(rng.integers(0,2**63))>>int(rng.integers(0,63))
    g=ofu64(v); e=struct.unpack('<Q',struct.pack('<d',float(v)))[0]; n+=1
    if g!=e: bad+=1; print('u64',v) if bad<8 else None

f32=np.float32
def fb(x): return struct.unpack('<I',struct.pack('<f',float(x)))[0]
def bf(u): return struct.unpack('<f',struct.pack('<I',u))[0]
def rne_int(x):  # __float2int_rn on an exactly representable float
    fl=np.floor(x); d=x-fl
    if d>0.5: return int(fl)+1
    if d<0.5: return int(fl)
    return int(fl) if int(fl)%2==0 else int(fl)+1
def fast(uh,ul):
    eh=(uh>>23)&0xff
    if 52<=eh<=254:
        mh=uh&0x7fffff
        down=((uh^ul)>>31)!=0 and ((ul<<1)&0xffffffff)!=0
        s=306-eh+(1 if (mh==0 and down) else 0)
        scaled=f32(bf(ul))*f32(bf(s<<23))
        L=rne_int(float(scaled))
        if -(1<<29)<=L<=(1<<29):
            D=((uh>>31)<<63)|((eh+896)<<52)|(mh<<29)
            return (D-L) if (uh>>31) else (D+L)
    return None
def exact(h,l):
    return struct.unpack('<Q',struct.pack('<d',float(Fraction(float(h))+Fraction(float(l)))))[0]
def two_sum_norm(a,b):
    sh=f32(a+b); bp=f32(sh-a); e=f32(f32(a-f32(sh-bp))+f32(b-bp))
    h=f32(sh+e); l=f32(e-f32(h-sh)); return h,l
rng=np.random.default_rng(1); n2=bad2=slow=0
with np.errstate(all='ignore'):
  for _ in range(300000):
    a=f32(rng.standard_normal()*10.0**rng.integers(-20,30))
    k=rng.integers(0,4)
    if k==0: b=f32(a*f32(rng.standard_normal())*f32(2.0**-rng.integers(10,60)))
    elif k==1: b=f32(-a*(1+f32(rng.standard_normal())*f32(2.0**-rng.integers(1,20))))
    elif k==2:  # power-of-two heads
        a=f32(np.ldexp(1.0,int(rng.integers(-60,60)))*rng.choice([-1,1])); b=f32(-np.sign(a)*abs(a)*2.0**-rng.integers(25,60))
    else: b=f32(rng.standard_normal()*10.0**rng.integers(-20,30))
    h,l=two_sum_norm(a,b)
    if not (np.isfinite(h) and np.isfinite(l)): continue
    r=fast(fb(h),fb(l)); n2+=1
    if r is None: slow+=1; continue
    e=exact(h,l)
    if r!=e: bad2+=1; print('bad',h,l,hex(r),hex(e)) if bad2<6 else None
  # ties: h in [1,2), l = +-half ulp64 (odd/even mantissas)
  for _ in range(20000):
    h=f32(rng.uniform(1,2)); l=f32(np.ldexp(1.0,-53)*rng.choice([-1,1])*rng.choice([1,3,5]))
    r=fast(fb(h),fb(l)); e=exact(h,l); n2+=1
    if r!=e: bad2+=1; print('tie',h,l) if bad2<6 else None
print('general: checked', n, 'mismatches', bad)
print('normalised fast path: checked', n2, 'mismatches', bad2, 'general fallbacks', slow)
assert bad == 0 and bad2 == 0
