TITLE cdp5-style Ca buffer, derivimplicit Newton with 5 unknowns (LU inside Newton)
NEURON { SUFFIX cdp5ish
    USEION ca READ ica WRITE cai
    RANGE kon, koff }
PARAMETER { kon = 100 koff = 0.1 kpump = 0.01 kd = 0.0003 }
ASSIGNED { v (mV) ica }
STATE { cai ca1 Buf Bufca Pump }
BREAKPOINT { SOLVE st METHOD derivimplicit }
INITIAL { cai = 5e-5
    ca1 = 5e-5
    Buf = 0.01
    Bufca = 0.0001
    Pump = 0.001 }
DERIVATIVE st {
    cai' = -ica*0.1 - kon*cai*Buf + koff*Bufca - kpump*cai*Pump/(kd + cai) + 0.05*(ca1 - cai)
    ca1' = 0.05*(cai - ca1)
    Buf' = -kon*cai*Buf + koff*Bufca
    Bufca' = kon*cai*Buf - koff*Bufca
    Pump' = -kpump*cai*Pump/(kd+cai) + 0.01*(0.001 - Pump)
}
