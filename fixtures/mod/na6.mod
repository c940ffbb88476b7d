TITLE six-state Markov Na channel, KINETIC + sparse (n>3 -> runtime LU)
NEURON { SUFFIX na6
    USEION na READ ena WRITE ina
    RANGE gbar }
PARAMETER { gbar = 0.1 (S/cm2) }
ASSIGNED { v (mV) ina a1 b1 a2 b2 ki kr }
STATE { C1 C2 C3 O I1 I2 }
BREAKPOINT { SOLVE kin METHOD sparse
    ina = gbar*O*(v - ena) }
INITIAL { C1 = 1
    C2 = 0
    C3 = 0
    O = 0
    I1 = 0
    I2 = 0 }
KINETIC kin {
    a1 = 3*exp(v/20)
    b1 = 0.5*exp(-v/25)
    a2 = 2*exp(v/30)
    b2 = 0.3*exp(-v/35)
    ki = 0.8*exp(v/40)
    kr = 0.02*exp(-v/45)
    ~ C1 <-> C2 (a1, b1)
    ~ C2 <-> C3 (a2, b2)
    ~ C3 <-> O (a1, b2)
    ~ O <-> I1 (ki, kr)
    ~ I1 <-> I2 (kr, ki)
    CONSERVE C1 + C2 + C3 + O + I1 + I2 = 1
}
