set cuda api_failures ignore
set pagination off
run
info cuda kernels
x/6i $pc-32
x/4i $pc
bt
quit
